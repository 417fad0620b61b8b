#!/bin/bash
O=gpurun_out/e2; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for v in "" u4 b1u4 u1; do
  for c in C3 C4; do
    TSF_LIB_VARIANT=$v timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_${c}_$v.json 2>&1
  done
done
timeout 300 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-e2e > $O/bench_C5.json 2>&1
for c in C3 C4; do TSF_LIB_VARIANT=prof timeout 300 python tools/prof_sections.py $c --M 16 > $O/sections_$c.txt 2>&1; done
tail -2 $O/pytest_gpu.log
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f)"; done
