"""Short driver for ncu / timing experiments: one config, reduced M / B, `reps` solves.

    python tools/prof_run.py C3 --M 8 --reps 2 [--B 148] [--cluster 16]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1603_00279_b200 import tsf
from paper_1603_00279_b200.inputs import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--M", type=int, default=0)
ap.add_argument("--B", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--cluster", type=int, default=0)
ap.add_argument("--method", default="bicgstab")
ap.add_argument("--precond", default="strang")
a = ap.parse_args()
insts = CONFIGS[a.config]()
if a.B:
    insts = insts[: a.B] if a.B <= len(insts) else [insts[i % len(insts)] for i in range(a.B)]
if a.M:
    for i in insts:
        i.M = a.M
        if i.f_table is not None:
            i.f_table = i.f_table[: a.M].copy()
s = tsf.Solver(insts, method=a.method, precond=a.precond, cluster=a.cluster)
for r in range(a.reps):
    s.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.solve()
    s.sync()
    dt = time.perf_counter() - t0
it, rr, st = s.stats()
tot_it = it.sum() / 2
print(f"{a.config} B={len(insts)} n={insts[0].n} M={insts[0].M} C={s.info.cluster} "
      f"{dt*1e3:.2f} ms/solve, {tot_it/len(insts)/insts[0].M:.2f} it/level, "
      f"{dt/tot_it*len(insts)*1e6:.1f} us per iteration per instance, status {set(st.ravel().tolist())}")
