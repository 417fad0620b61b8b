#!/bin/bash
O=gpurun_out/e23; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for m in pcgs cgnr bicgstab; do timeout 600 python bench.py --config C3 --method $m --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_$m.json 2>&1; done
for m in pcgs cgnr; do timeout 600 python bench.py --config C2 --method $m --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C2_$m.json 2>&1; done
tail -2 $O/pytest_gpu.log
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f) $(grep -o '"mean_iters_per_level": [0-9.]*' $f)"; done
