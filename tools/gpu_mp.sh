#!/bin/bash
# multi-pass regime: GPU tests + a short C3 bench (no regression on the SMEM path)
O=gpurun_out/${1:-mp}; mkdir -p $O
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_gpu_multipass.py -m gpu -x -q -s > $O/pytest_mp.log 2>&1
echo "pytest rc=$?" >> $O/pytest_mp.log
tail -5 $O/pytest_mp.log
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3.json 2>&1
python -c "import json; d=json.load(open('$O/bench_C3.json')); print('C3', round(d['value'],1))"
