#!/bin/bash
O=gpurun_out/e6; mkdir -p $O
timeout 300 python tools/apply_bench.py > $O/apply_bench.txt 2>&1
TSF_LIB_VARIANT=prof timeout 300 python tools/apply_bench.py > $O/apply_bench_prof.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
cat $O/apply_bench.txt $O/apply_bench_prof.txt; tail -2 $O/pytest_gpu.log
