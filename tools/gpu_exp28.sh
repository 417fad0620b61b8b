#!/bin/bash
O=gpurun_out/e28; mkdir -p $O
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C5.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "c5 or every_cluster or apply" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
for f in $O/bench*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f) $(grep -o '"frac": [0-9.]*' $f)"; done
