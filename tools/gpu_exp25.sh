#!/bin/bash
O=gpurun_out/e25; mkdir -p $O
for cl in 1 2 4 8; do timeout 300 python bench.py --config C2 --cluster $cl --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C2_c$cl.json 2>&1; done
for cl in 1 2; do timeout 600 python bench.py --config C4 --cluster $cl --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C4_c$cl.json 2>&1; done
for cl in 8 16; do timeout 300 python bench.py --config C3 --cluster $cl --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_c$cl.json 2>&1; done
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f) $(grep -o '"frac": [0-9.]*' $f)"; done
