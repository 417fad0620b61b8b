#!/bin/bash
# ncu --set full capture of one C3 solve kernel with source correlation; raw + source CSVs.
TAG=${1:-ncu}; CFG=${2:-C3}; O=gpurun_out/$TAG; mkdir -p $O
export PYTHONPATH=$PWD
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 \
  -o $O/full python tools/prof_run.py $CFG --M 16 --reps 1 > $O/ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full.log
ncu -i $O/full.ncu-rep --page raw --csv > $O/full_raw.csv 2>/dev/null
ncu -i $O/full.ncu-rep --page source --csv --print-source sass > $O/full_sass.csv 2>/dev/null
ncu -i $O/full.ncu-rep --page source --csv --print-source cuda > $O/full_cuda.csv 2>/dev/null
python tools/ncu_keys.py $O/full_raw.csv > $O/full_keys.txt 2>&1
ls -la $O; cat $O/full_keys.txt | head -30
