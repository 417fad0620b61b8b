#!/bin/bash
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for v in r01 base; do
  [ "$v" = "base" ] && vv="" || vv="$v"
  echo "== $v" >> gpurun_out/prof_ab.log
  TSF_LIB_VARIANT=$vv python tools/apply_bench.py --cases C3:16 >> gpurun_out/prof_ab.log 2>&1
done
for v in r01prof prof; do
  echo "== $v" >> gpurun_out/prof_ab.log
  TSF_LIB_VARIANT=$v python tools/prof_sections.py C3 --M 16 >> gpurun_out/prof_ab.log 2>&1
done
