#!/bin/bash
# One gpurun call: GPU tests, default bench, section timers, ncu launch list + full capture.
#   gpurun --timeout 1800 -- 'bash tools/gpu_session.sh TAG [tests|notests]'
TAG=${1:-run}
TESTS=${2:-tests}
mkdir -p gpurun_out
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
if [ "$TESTS" = "tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
  echo "smoke rc=$?" >> $O/smoke.log
fi
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
for c in C3 C4; do
  TSF_LIB_VARIANT=prof timeout 300 python tools/prof_sections.py $c --M 16 > $O/sections_$c.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_launch.log 2>&1
echo "ncu launch rc=$?" >> $O/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 \
  -o $O/c3_full python tools/prof_run.py C3 --M 16 --reps 1 > $O/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $O/ncu_full.log
ncu -i $O/c3_full.ncu-rep --page raw --csv > $O/c3_full_raw.csv 2>/dev/null
ncu -i $O/c3_full.ncu-rep --page source --csv > $O/c3_full_source.csv 2>/dev/null
ls -la $O
for c in C2 C4 C5; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
python tools/ncu_keys.py $O/c3_full_raw.csv > $O/c3_full_keys.txt 2>&1
python tools/ncu_summary.py launches $O/launches.csv > $O/launches_summary.txt 2>&1
timeout 600 python bench.py --config C3 --method gsf --steps 3 --warmup 3 --no-e2e --no-cpu > $O/bench_C3_gsf.json 2>&1
timeout 600 python bench.py --config C3 --method pcgs --steps 3 --warmup 3 --no-e2e --no-cpu > $O/bench_C3_pcgs.json 2>&1
TSF_LIB_VARIANT=prof timeout 300 python tools/apply_bench.py > $O/apply_bench_prof.txt 2>&1
