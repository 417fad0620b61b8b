#!/bin/bash
# Development GPU call: quick staged-path tests, C3/C2 bench, C3 section timers.
#   gpurun --timeout 1500 -- 'bash tools/gpu_dev.sh TAG [quick|full]'
TAG=${1:-dev}
MODE=${2:-quick}
O=gpurun_out/$TAG; mkdir -p $O
export PYTHONPATH=$PWD
python -c "import oracle; oracle.build()" > /dev/null 2>&1
if [ "$MODE" = "full" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
else
  timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q -p no:cacheprovider \
    -k "fused or operator_applications or c2_combinations or table_source or pcgs_parity or gsf_constant or history_helper or c3_full or pipelined or step_graph" \
    > $O/pytest_gpu.log 2>&1
fi
echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_C3.json 2> $O/bench_C3.err
timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C2.json 2> $O/bench_C2.err
for f in $O/bench_*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value'],1), d.get('krylov_iters_per_s'), d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
if [ -f paper_1603_00279_b200/lib/libtsf_prof.so ]; then
  TSF_LIB_VARIANT=prof timeout 300 python tools/prof_sections.py C3 --M 16 > $O/sections_C3.txt 2>&1
  cat $O/sections_C3.txt
fi
