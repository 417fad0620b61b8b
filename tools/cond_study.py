"""GPU vs oracle discrepancy vs n for one parameter set (conditioning study).
Prints per n: max relative L2 difference over levels, level-0 difference, both solvers'
relative residuals at level 0, and an estimate of cond_1(A) at level 1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
from paper_1603_00279_b200 import tsf
from paper_1603_00279_b200.inputs import Instance, const

al, be, ga, dp, dm = [float(v) for v in sys.argv[1:6]]
M = int(sys.argv[6]) if len(sys.argv) > 6 else 32
for n in (256, 1024, 4096):
    inst = Instance(al, be, n, M, const(ga), const(dp), const(dm), "mms3")
    p = O.Problem(alpha=al, beta=be, n=n, M=M, gamma=(O.CONST, ga), dplus=(O.CONST, dp),
                  dminus=(O.CONST, dm), src=O.SRC_MMS3)
    s = tsf.Solver([inst])
    U = [s.solution(0)]
    for _ in range(M):
        s.step()
        U.append(s.solution(0))
    U = np.array(U)
    Uo = O.solve(p)
    rel = [np.linalg.norm(U[j] - Uo[j]) / np.linalg.norm(Uo[j]) for j in range(1, M + 1)]
    A, _ = O.assemble(p, 0)
    g0 = O.rhs(p, 0, Uo[:1])
    rg = np.linalg.norm(A @ U[1] - g0) / np.linalg.norm(g0)
    ro = np.linalg.norm(A @ Uo[1] - g0) / np.linalg.norm(g0)
    A1, _ = O.assemble(p, min(1, M - 1))
    c1 = np.linalg.cond(A1, 1) if n <= 1024 else float("nan")
    print(f"n={n:5d} maxrel={max(rel):.2e} rel(level1)={rel[0]:.2e} rel(levelM)={rel[-1]:.2e} "
          f"resid0 gpu={rg:.1e} oracle={ro:.1e} cond1(A)={c1:.2e} its={s.stats()[0].mean()/2:.2f}",
          flush=True)
