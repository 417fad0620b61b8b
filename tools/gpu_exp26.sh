#!/bin/bash
O=gpurun_out/e26; mkdir -p $O
for c in C4 C1; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_$c.json 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q -k "c1 or batched or table_source or noprec or gsf_c1 or c4" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f) $(grep -o '"frac": [0-9.]*' $f)"; done
