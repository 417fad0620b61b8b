#!/bin/bash
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for v in $1; do
  [ "$v" = "base" ] && vv="" || vv="$v"
  echo "== $v" >> gpurun_out/c5ab.log
  TSF_LIB_VARIANT=$vv timeout 600 python bench.py --config C5 --steps 2 --warmup 1 --no-cpu --no-e2e $2 >> gpurun_out/c5ab.log 2>&1
done
