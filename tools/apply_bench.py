"""Per-apply latency of the fused operator (no Krylov): one launch of `reps` alternating
P^{-1} / A applications (tsf_debug_apply_bench).  Developer tool.

    python tools/apply_bench.py [--reps 400]        (TSF_LIB_VARIANT=prof adds section timers)
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1603_00279_b200 import _lib as L
from paper_1603_00279_b200 import tsf
from paper_1603_00279_b200.inputs import CONFIGS

NAMES = ["fft_fwd", "bar1", "gather", "col_fwd", "pairs", "col_inv", "bar2", "scatter", "bar3", "fft_inv"]
ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=400)
ap.add_argument("--cases", default="C3:16,C3:8,C2:2,C4:1,C5:16")
a = ap.parse_args()
prof = os.environ.get("TSF_LIB_VARIANT", "").startswith("prof")
for case in a.cases.split(","):
    cfg, cl = case.split(":")
    inst = CONFIGS[cfg]()[0]
    inst.M = 2
    if inst.f_table is not None:
        inst.f_table = inst.f_table[:2].copy()
    s = tsf.Solver([inst], cluster=int(cl))
    if prof:
        buf = (C.c_uint64 * 32)()
        L.check(s.lib.tsf_debug_prof(s.h, buf, 1), "prof")
    ms = s.debug_apply_bench(0, 0, a.reps)
    line = f"{cfg} n={inst.n} C={s.info.cluster}: {1e3 * ms / a.reps:7.2f} us per apply (P^-1/A alternating, {a.reps} reps)"
    if prof:
        L.check(s.lib.tsf_debug_prof(s.h, buf, 1), "prof")
        v = np.array(buf[:10], dtype=np.float64) / (2 * a.reps)    # warm-up + timed launch
        line += "  cyc/apply: " + " ".join(f"{NAMES[i]}={v[i]:.0f}" for i in range(10) if v[i] > 0)
    print(line, flush=True)
    s.close()
