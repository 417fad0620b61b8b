"""Per-section cycle breakdown from the profiling build (clock64 timers of CTA 0, thread 0).

    TSF_LIB_VARIANT=prof python tools/prof_sections.py C3 --M 8 [--cluster 16] [--B 148]
"""
import argparse
import ctypes as C
import os
import sys

os.environ.setdefault("TSF_LIB_VARIANT", "prof")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1603_00279_b200 import _lib as L
from paper_1603_00279_b200 import tsf
from paper_1603_00279_b200.inputs import CONFIGS

NAMES = ["fft_fwd", "bar1", "gather", "col_fwd", "pairs", "col_inv", "bar2", "scatter", "bar3",
         "fft_inv", "csum", "vec(rest)", "rhs_hist", "level", "applies", "iters_half"]

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--M", type=int, default=8)
ap.add_argument("--B", type=int, default=0)
ap.add_argument("--cluster", type=int, default=0)
ap.add_argument("--method", default="bicgstab")
a = ap.parse_args()
insts = CONFIGS[a.config]()
if a.B:
    insts = insts[: a.B]
for i in insts:
    i.M = a.M
    if i.f_table is not None:
        i.f_table = i.f_table[: a.M].copy()
s = tsf.Solver(insts, method=a.method, cluster=a.cluster)
buf = (C.c_uint64 * 32)()
s.solve()
s.sync()
L.check(s.lib.tsf_debug_prof(s.h, buf, 1), "prof")
s.reset()
s.solve()
s.sync()
L.check(s.lib.tsf_debug_prof(s.h, buf, 1), "prof")
v = np.array(buf[:16], dtype=np.float64)
level, applies, iters = v[13], v[14], v[15] / 2
acc = v[[0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12]].sum()
v[11] = level - acc
ghz = 1.965
print(f"{a.config} C={s.info.cluster} M={a.M} iters={iters:.0f} applies={applies:.0f} "
      f"level total {level/ghz/1e3:.1f} us ({level/max(iters,1)/ghz/1e3:.2f} us/iter)")
for k in range(13):
    print(f"  {NAMES[k]:10s} {v[k]/ghz/1e3:10.1f} us  {100*v[k]/level:5.1f}%  "
          f"{v[k]/max(applies,1):9.0f} cyc/apply  {v[k]/max(iters,1):9.0f} cyc/iter")
