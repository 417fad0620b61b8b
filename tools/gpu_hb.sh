#!/bin/bash
O=gpurun_out/${1:-hb}; mkdir -p $O
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q -k "pipelined or blocked_history" > $O/pytest_hb.log 2>&1
echo "pytest rc=$?" >> $O/pytest_hb.log; tail -3 $O/pytest_hb.log
for c in C4 C2 C5 C3; do for hb in 0 8 16 32; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e --hist-block $hb > $O/bench_${c}_hb$hb.json 2>&1
  python -c "import json; d=json.load(open('$O/bench_${c}_hb$hb.json')); print('$c hb$hb', round(d['value'],1), round(d['roofline']['frac'],4), round(d['mean_iters_per_level'],3), d['max_relres'])"
done; done
