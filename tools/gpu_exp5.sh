#!/bin/bash
O=gpurun_out/e5; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --config C3 --method pcgs --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_pcgs.json 2>&1
timeout 300 python bench.py --config C2 --method pcgs --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C2_pcgs.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o $O/c3 python tools/prof_run.py C3 --M 8 --reps 1 > $O/c3.log 2>&1
ncu -i $O/c3.ncu-rep --page raw --csv > $O/c3_raw.csv 2>/dev/null; ncu -i $O/c3.ncu-rep --page source --csv > $O/c3_src.csv 2>/dev/null
tail -2 $O/pytest_gpu.log
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f) $(grep -o '"mean_iters_per_level": [0-9.]*' $f)"; done
