#!/bin/bash
# round-2 GPU session: tests (minus the C3 golden ones until the golden exists) + short bench
mkdir -p gpurun_out
export PYTHONPATH=$PWD
python -c "import oracle; oracle.build()"
timeout 2400 python -m pytest tests -m gpu -q -x -k "not c3_full and not c3_teacher and not c3_bench and not c3_other" \
   -p no:cacheprovider > gpurun_out/pytest_r2a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2a.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_r2a.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_r2a.log
