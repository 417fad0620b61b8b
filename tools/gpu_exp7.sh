#!/bin/bash
O=gpurun_out/${1:-e7}; mkdir -p $O
timeout 300 python tools/apply_bench.py > $O/apply_bench.txt 2>&1
TSF_LIB_VARIANT=prof timeout 300 python tools/apply_bench.py > $O/apply_bench_prof.txt 2>&1
for c in C3 C4 C5 C2; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
cat $O/apply_bench.txt $O/apply_bench_prof.txt; tail -2 $O/pytest_gpu.log
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f)"; done
