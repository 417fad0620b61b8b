#!/bin/bash
O=gpurun_out/${1:-e16}; mkdir -p $O
timeout 300 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3.json 2> $O/bench_C3.err
TSF_NO_HELPERS=1 timeout 300 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_nohelp.json 2>&1
timeout 300 python bench.py --config C3 --method gsf --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_gsf.json 2>&1
timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C2.json 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log; tail -3 $O/bench_C3.err
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f) $(grep -o '"max_relres": [0-9.e-]*' $f)"; done
