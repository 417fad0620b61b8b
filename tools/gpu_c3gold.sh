#!/bin/bash
# C3 full-size parity against the oracle golden (incl. one 16384^2 GE for teacher forcing)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
python -c "import oracle; oracle.build()"
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -k "c3" -p no:cacheprovider > gpurun_out/pytest_c3gold.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_c3gold.log
