#!/bin/bash
O=gpurun_out/${1:-chk2}; mkdir -p $O
for c in C2 C3; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_$c.json 2>&1; done
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f) $(grep -o '"frac": [0-9.]*' $f)"; done
