#!/bin/bash
O=gpurun_out/n3; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o $O/c4 python tools/prof_run.py C4 --B 296 --M 4 --reps 1 > $O/c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o $O/c5 python tools/prof_run.py C5 --B 8 --M 2 --reps 1 > $O/c5.log 2>&1
for f in c4 c5; do ncu -i $O/$f.ncu-rep --page raw --csv > $O/${f}_raw.csv 2>/dev/null; ncu -i $O/$f.ncu-rep --page source --csv > $O/${f}_src.csv 2>/dev/null; done
ls -la $O
