#!/bin/bash
O=gpurun_out/${1:-pipe}; mkdir -p $O
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q -k "pipelined" > $O/pytest_pipe.log 2>&1
echo "pytest rc=$?" >> $O/pytest_pipe.log; tail -3 $O/pytest_pipe.log
for c in C3 C4 C5 C2; do for pp in "" "--pipelined"; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e $pp > $O/bench_${c}${pp}.json 2>&1
  python -c "import json; d=json.load(open('$O/bench_${c}${pp}.json')); print('$c$pp', round(d['value'],1), round(d['roofline']['frac'],4), round(d['mean_iters_per_level'],3), d['max_relres'])"
done; done
