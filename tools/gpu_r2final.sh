#!/bin/bash
# Round-2 measurement session: GPU tests, smoke, ncu DRAM traffic of the bench launches (so the
# bench lines carry roofline.traffic), bench C3 (default: CPU baseline + e2e) and C2/C4/C5,
# C3 GSF / PCGS, ncu launch list, section timers.
#   gpurun --timeout 3000 -- 'bash tools/gpu_r2final.sh TAG [tests|notests]'
TAG=${1:-final}; TESTS=${2:-tests}
O=gpurun_out/$TAG; mkdir -p $O
export PYTHONPATH=$PWD
python -c "import oracle; oracle.build()" > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
if [ "$TESTS" = "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $O/pytest_gpu.log
  tail -3 $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
  echo "smoke rc=$?" >> $O/smoke.log
  cat $O/smoke.log
fi
timeout 1500 python tools/ncu_traffic.py C3 C2 C4 C5 --logdir $O > $O/traffic.log 2>&1
echo "traffic rc=$?" >> $O/traffic.log
cp profiles/traffic.json $O/traffic.json
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
for c in C2 C4 C5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --config C3 --method gsf --steps 3 --warmup 3 --no-e2e --no-cpu > $O/bench_C3_gsf.json 2>&1
timeout 600 python bench.py --config C3 --method pcgs --steps 3 --warmup 3 --no-e2e --no-cpu > $O/bench_C3_pcgs.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_launch.log 2>&1
python tools/ncu_summary.py launches $O/launches.csv > $O/launches_summary.txt 2>&1
if [ -f paper_1603_00279_b200/lib/libtsf_prof.so ]; then
  for c in C3 C2; do
    TSF_LIB_VARIANT=prof timeout 300 python tools/prof_sections.py $c --M 16 > $O/sections_$c.txt 2>&1
  done
fi
for f in $O/bench*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value'],1), round(r['frac'],4), r.get('traffic'), r.get('ncu_dram_frac'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'), d['clocks'])" 2>&1 | tail -1; done
