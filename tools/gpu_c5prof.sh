#!/bin/bash
mkdir -p gpurun_out
export PYTHONPATH=$PWD
TSF_LIB_VARIANT=prof python tools/apply_bench.py --cases C5:16 --reps 100 > gpurun_out/c5prof.log 2>&1
for cta in 0; do
TSF_LIB_VARIANT=prof python tools/prof_sections.py C5 --M 2 --B 64 >> gpurun_out/c5prof.log 2>&1
TSF_LIB_VARIANT=prof python tools/prof_sections.py C5 --M 2 --B 1 >> gpurun_out/c5prof.log 2>&1
done
