#!/bin/bash
# Section timers (profiling build) for C3 / C2, fused and unfused, plus quick benches.
TAG=${1:-sec}; O=gpurun_out/$TAG; mkdir -p $O
export PYTHONPATH=$PWD
for v in "C3 0" "C3 1" "C2 0"; do set -- $v
  TSF_NO_FUSE=$2 TSF_LIB_VARIANT=prof timeout 300 python tools/prof_sections.py $1 --M 16 > $O/sections_$1_nf$2.txt 2>&1
  echo "== $1 nofuse=$2"; cat $O/sections_$1_nf$2.txt
done
TSF_NO_FUSE=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_nofuse.json 2> $O/bench_C3_nofuse.err
python -c "import json; d=json.load(open('$O/bench_C3_nofuse.json')); print('C3 nofuse', d['value'])"
