#!/bin/bash
# ncu --set full of the exact bench launch (one k_solve over all M levels) per config, for the
# roofline "traffic" field (dram bytes read + written per launch).
O=gpurun_out/tr; mkdir -p $O
for c in C3 C2 C4; do
  timeout 900 ncu --set full --clock-control none -k regex:k_solve -c 1 -o $O/$c python tools/prof_run.py $c --reps 1 > $O/$c.log 2>&1
  ncu -i $O/$c.ncu-rep --page raw --csv > $O/${c}_raw.csv 2>/dev/null
done
ls -la $O
