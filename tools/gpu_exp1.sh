#!/bin/bash
O=gpurun_out/e1; mkdir -p $O
./tools/ubench.bin > $O/ubench.txt 2>&1
run() { # name env...
  local nm=$1; shift
  for c in C3 C4; do env "$@" timeout 300 python tools/prof_sections.py $c --M 16 > $O/sec_${nm}_$c.txt 2>&1; done
}
run noinl TSF_LIB_VARIANT=prof
run inl TSF_LIB_VARIANT=inlprof
run inl_novs TSF_LIB_VARIANT=inlprof TSF_VSMEM=0
run noinl_fuse TSF_LIB_VARIANT=prof TSF_FUSE_MIN=256
run inl_fuse TSF_LIB_VARIANT=inlprof TSF_FUSE_MIN=256
for v in "" inl; do
  TSF_LIB_VARIANT=$v timeout 300 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_$v.json 2>&1
done
TSF_LIB_VARIANT=inl TSF_FUSE_MIN=256 timeout 300 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_inlfuse.json 2>&1
TSF_LIB_VARIANT=inl TSF_FUSE_MIN=256 timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C4_inlfuse.json 2>&1
cat $O/ubench.txt; head -2 $O/sec_*C3.txt; grep -h -o '"value": [0-9.]*' $O/bench*.json
