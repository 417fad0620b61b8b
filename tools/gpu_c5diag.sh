#!/bin/bash
# One gpurun call: C5 diagnosis — section timers (full batch and one resident wave), ncu full
# capture of a one-wave C5 launch (9 instances, M = 2), key metrics and SASS stall summary.
#   gpurun --timeout 1500 -- 'bash tools/gpu_c5diag.sh TAG'
TAG=${1:-c5diag}
O=gpurun_out/$TAG
mkdir -p $O
export PYTHONPATH=$PWD
TSF_LIB_VARIANT=prof timeout 300 python tools/prof_sections.py C5 --M 4 --B 9 > $O/sections_C5_B9.txt 2>&1
TSF_LIB_VARIANT=prof timeout 300 python tools/prof_sections.py C5 --M 4 --B 64 > $O/sections_C5_B64.txt 2>&1
TSF_LIB_VARIANT=prof timeout 300 python tools/prof_sections.py C4 --M 16 > $O/sections_C4.txt 2>&1
timeout 300 python tools/prof_run.py C5 --M 8 --B 9 --reps 2 > $O/run_C5_B9.txt 2>&1
timeout 300 python tools/prof_run.py C5 --M 8 --B 18 --reps 2 >> $O/run_C5_B9.txt 2>&1
timeout 300 python tools/prof_run.py C5 --M 8 --B 1 --reps 2 >> $O/run_C5_B9.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 \
  -o $O/c5_full python tools/prof_run.py C5 --M 2 --B 9 --reps 1 > $O/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $O/ncu_full.log
ncu -i $O/c5_full.ncu-rep --page raw --csv > $O/c5_full_raw.csv 2>/dev/null
ncu -i $O/c5_full.ncu-rep --page source --csv > $O/c5_full_source.csv 2>/dev/null
python tools/ncu_keys.py $O/c5_full_raw.csv > $O/c5_full_keys.txt 2>&1
python tools/ncu_sass_stalls.py $O/c5_full_source.csv > $O/c5_full_stalls.txt 2>&1
rm -f $O/c5_full.ncu-rep
ls -la $O
