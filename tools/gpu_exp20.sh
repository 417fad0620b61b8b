#!/bin/bash
O=gpurun_out/${1:-e20}; mkdir -p $O
TSF_LIB_VARIANT=prof timeout 300 python tools/apply_bench.py --cases C3:16,C2:2 > $O/ab0.txt 2>&1
TSF_LIB_VARIANT=prof5 timeout 300 python tools/apply_bench.py --cases C3:16 > $O/ab5.txt 2>&1
for c in C3 C2 C5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
cat $O/ab0.txt $O/ab5.txt; tail -2 $O/pytest_gpu.log
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f)"; done
