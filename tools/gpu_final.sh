#!/bin/bash
O=gpurun_out/fin; mkdir -p $O
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
for c in C2 C4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu > $O/bench_C5.json 2> $O/bench_C5.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
cat $O/smoke.log; for f in $O/bench*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],1), d['roofline']['frac'], d['roofline']['traffic'], (d['cpu_baseline'] or {}).get('value'), (d['e2e'] or {}).get('value'), d['clocks']['sm_mhz'])"; done
