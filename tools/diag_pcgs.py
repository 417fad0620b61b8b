import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, oracle as O
from paper_1603_00279_b200 import tsf
from test_gpu import pair, run_levels, max_rel
inst, p = pair(0.8, 1.8, 1024, 40, gamma=(O.COS, 1.0), dplus=(O.ONE_PLUS_T, 1.0), dminus=(O.ONE_PLUS_T2, 1.0))
Uo = O.solve(p)
for method in ("pcgs", "bicgstab"):
    for hb in (0, 16):
        for cl in (1, 4):
            s = tsf.Solver([inst], method=method, cluster=cl, hist_block=hb)
            U = run_levels(s, 40)[0]
            it, rr, st = s.stats()
            print(method, "hb", hb, "C", cl, "max_rel %.2e" % max_rel(U, Uo), "true res max %.2e" % s.true_residuals().max(), "iters", it.sum())
