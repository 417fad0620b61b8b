#!/bin/bash
O=gpurun_out/e4; mkdir -p $O
for v in v4 "" regctx pwt pwtreg; do
  TSF_LIB_VARIANT=$v timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C4_$v.json 2>&1
done
TSF_LIB_VARIANT=v4 timeout 300 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-e2e > $O/bench_C5_v4.json 2>&1
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f)"; done
