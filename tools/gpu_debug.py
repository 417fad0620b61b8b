"""Staged GPU sanity checks (developer tool): local FFT, weights, spectra, apply, RHS, solve.
Prints max errors per stage so a single gpurun call localizes a failing component."""
import sys
import os
import time
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
from paper_1603_00279_b200 import tsf
from paper_1603_00279_b200.inputs import Instance, const, config_c1


def stage(name, fn):
    t = time.time()
    try:
        r = fn()
        print(f"[{name}] {r} ({time.time()-t:.2f}s)", flush=True)
    except Exception:
        print(f"[{name}] FAILED", flush=True)
        traceback.print_exc()


def fft_check():
    out = []
    for Lc in [2, 4, 8, 32, 64, 512, 2048, 8192]:
        x = np.random.default_rng(Lc).standard_normal(Lc) + 1j * np.random.default_rng(Lc + 1).standard_normal(Lc)
        _, perm, _ = tsf.debug_fft_tables(Lc)
        y = tsf.debug_local_fft(x)
        X = np.fft.fft(x)
        e1 = np.abs(y - X[perm]).max() / np.abs(X).max()
        z = tsf.debug_local_fft(y, inverse=True)
        e2 = np.abs(z / Lc - x).max() / np.abs(x).max()
        out.append((Lc, f"{e1:.1e}", f"{e2:.1e}"))
    return out


def weights_check():
    g, w = tsf.debug_weights(1.7, 5000)
    return f"{np.abs(w - O.wsgd(1.7, 5000)).max():.1e} {np.abs(g - O.grunwald(1.7, 5000)).max():.1e}"


def orc_problem(inst, gshape=(O.CONST, 0.5), dp=(O.CONST, 1.0), dm=(O.CONST, 1.0)):
    return O.Problem(alpha=inst.alpha, beta=inst.beta, n=inst.n, M=inst.M, gamma=gshape, dplus=dp,
                     dminus=dm, src=O.SRC_MMS3)


def apply_check(n, cluster, precond="strang"):
    inst = Instance(0.7, 1.6, n, 8, np.cos, lambda t: 1 + t, lambda t: 0.5 * (1 + t * t), "mms3")
    s = tsf.Solver([inst], precond=precond, cluster=cluster)
    p = O.Problem(alpha=0.7, beta=1.6, n=n, M=8, gamma=(O.COS, 1.0), dplus=(O.ONE_PLUS_T, 1.0),
                  dminus=(O.ONE_PLUS_T2, 0.5), src=O.SRC_MMS3)
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n)
    res = [f"C={s.info.cluster}"]
    for j in (0, 3):
        A, B = O.assemble(p, j)
        for which, M in ((0, A), (1, B), (2, A.T)):
            y = s.debug_apply(0, j, which, x)
            ref = M @ x
            res.append(f"{which}:{np.linalg.norm(y - ref) / np.linalg.norm(ref):.1e}")
        # preconditioner: dense circulant from the oracle's Strang / T. Chan columns
        col, row = A[:, 0], A[0, :]
        c = O.strang_col(col, row) if precond == "strang" else O.tchan_col(col, row)
        from scipy.linalg import circulant
        Pm = circulant(c)
        for which, M in ((3, Pm), (4, Pm.T)):
            y = s.debug_apply(0, j, which, x)
            ref = np.linalg.solve(M, x)
            res.append(f"{which}:{np.linalg.norm(y - ref) / np.linalg.norm(ref):.1e}")
    return " ".join(res)


def solve_check(n, M, cluster, method="bicgstab", precond="strang"):
    inst = Instance(0.8, 1.8, n, M, np.cos, lambda t: 1 + t, lambda t: 1 + t**2, "mms3")
    s = tsf.Solver([inst], method=method, precond=precond, cluster=cluster)
    p = O.Problem(alpha=0.8, beta=1.8, n=n, M=M, gamma=(O.COS, 1.0), dplus=(O.ONE_PLUS_T, 1.0),
                  dminus=(O.ONE_PLUS_T2, 1.0), src=O.SRC_MMS3)
    U = [s.solution(0)]
    g0 = s.debug_rhs(0)
    Uo = O.solve(p)
    grh = O.rhs(p, 0, Uo[:1])
    for _ in range(M):
        s.step()
        U.append(s.solution(0))
    rc = s.sync()
    U = np.array(U)
    rel = [np.linalg.norm(U[j] - Uo[j]) / np.linalg.norm(Uo[j]) for j in range(1, M + 1)]
    it, rr, st = s.stats()
    return (f"C={s.info.cluster} rc={rc} rhs0 {np.linalg.norm(g0-grh)/np.linalg.norm(grh):.1e} "
            f"max rel {max(rel):.2e} its {it[0,:8]/2} st {set(st[0].tolist())}")


if __name__ == "__main__":
    stage("fft", fft_check)
    stage("weights", weights_check)
    for n, c in [(64, 1), (256, 1), (1024, 2), (1024, 4), (1024, 16), (4096, 8), (4096, 16), (4096, 1)]:
        stage(f"apply n={n} C={c}", lambda: apply_check(n, c))
    stage("apply tchan", lambda: apply_check(256, 1, "tchan"))
    for n, M, c in [(64, 16, 1), (256, 16, 1), (1024, 16, 4), (1024, 8, 16)]:
        for m in ("bicgstab", "cgnr"):
            stage(f"solve n={n} C={c} {m}", lambda: solve_check(n, M, c, m))
