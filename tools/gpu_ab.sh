#!/bin/bash
# A/B of library variants on C3: usage bash tools/gpu_ab.sh "variant1 variant2 ..." [bench args]
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for v in $1; do
  [ "$v" = "base" ] && vv="" || vv="$v"
  echo "== $v" >> gpurun_out/ab.log
  TSF_LIB_VARIANT=$vv timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e $2 >> gpurun_out/ab.log 2>&1
done
