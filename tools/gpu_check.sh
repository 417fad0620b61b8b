#!/bin/bash
# Quick check: apply microbenchmarks (+ section timers), short benches of C3/C4/C5, GPU tests.
O=gpurun_out/${1:-chk}; mkdir -p $O
TSF_LIB_VARIANT=prof timeout 300 python tools/apply_bench.py --cases C5:16,C3:16 > $O/ab.txt 2>&1
for c in C5 C3 C4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_$c.json 2>&1; done
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
cat $O/ab.txt; tail -2 $O/pytest_gpu.log
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f) $(grep -o '"frac": [0-9.]*' $f)"; done
