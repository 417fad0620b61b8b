#!/bin/bash
O=gpurun_out/e27; mkdir -p $O
for v in "" pu4; do for c in C4 C1; do TSF_LIB_VARIANT=$v timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_${c}_$v.json 2>&1; done; done
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f) $(grep -o '"frac": [0-9.]*' $f)"; done
