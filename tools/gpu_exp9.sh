#!/bin/bash
O=gpurun_out/${1:-e9}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "gsf" > $O/pytest_gsf.log 2>&1; echo "rc=$?" >> $O/pytest_gsf.log
timeout 300 python bench.py --config C3 --method gsf --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_gsf.json 2>&1
timeout 300 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3.json 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gsf.log; tail -2 $O/pytest_gpu.log
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f) $(grep -o '"max_relres": [0-9.e-]*' $f)"; done
