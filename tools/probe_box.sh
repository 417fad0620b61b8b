set -x
nproc; lscpu | head -25; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export PYTHONPATH=$PWD
python -c "import oracle; oracle.build(force=True)"
python /root/repo/tools/lut_probe.py 4096
python /root/repo/tools/lut_probe.py 8192
