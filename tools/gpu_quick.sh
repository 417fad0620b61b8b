#!/bin/bash
# Quick GPU iteration: optional GPU tests, section timers, short benches of the given configs.
#   gpurun --timeout 1500 -- 'bash tools/gpu_quick.sh TAG tests|notests "C3 C4 C5"'
TAG=${1:-q}
TESTS=${2:-notests}
CFGS=${3:-"C3 C4 C5"}
O=gpurun_out/$TAG
mkdir -p $O
if [ "$TESTS" = "tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
for c in C3 C4; do
  TSF_LIB_VARIANT=prof timeout 300 python tools/prof_sections.py $c --M 16 > $O/sections_$c.txt 2>&1
done
for c in $CFGS; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
tail -n 3 $O/*.log $O/*.json 2>/dev/null | cut -c1-600
