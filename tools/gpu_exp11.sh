#!/bin/bash
O=gpurun_out/${1:-e11}; mkdir -p $O
for c in C3 C4 C5 C2; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python bench.py --config C3 --method gsf --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_gsf.json 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f) $(grep -o '"frac": [0-9.e-]*' $f)"; done
