#!/bin/bash
# Quick perf check: bench lines (no CPU baseline / e2e) and section timers for the given configs.
#   gpurun -- 'bash tools/gpu_perf.sh TAG "C3 C4 C5" [sections]'
TAG=${1:-perf}; CFGS=${2:-"C3 C4 C5"}; SEC=${3:-}
O=gpurun_out/$TAG; mkdir -p $O
export PYTHONPATH=$PWD
for c in $CFGS; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json; d=json.load(open('$O/bench_$c.json')); print('$c', round(d['value'],1), 'levels/s frac', round(d['roofline']['frac'],4), 'iters/lvl', round(d['mean_iters_per_level'],3), 'relres', d['max_relres'], d['clocks']['sm_mhz'])" >> $O/summary.txt 2>&1
  if [ -n "$SEC" ]; then
    B=""; [ $c = C5 ] && B="--B 18"; [ $c = C4 ] && B="--B 296"
    TSF_LIB_VARIANT=prof timeout 300 python tools/prof_sections.py $c --M 8 $B > $O/sections_$c.txt 2>&1
  fi
done
cat $O/summary.txt
