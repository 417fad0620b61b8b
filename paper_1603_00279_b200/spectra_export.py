"""NEXT-4: matrix and spectrum export for the paper's Figs. fig1/fig2 and
fig3/fig4: eigenvalues of the level matrix A^{(j+sigma)} and of the circulant-
preconditioned matrix, "clustered at 1, except for few (about 6~10) outliers".

The dense matrices are assembled column by column from the GPU operators through the C-ABI
test hook tsf_debug_apply (A e_k and P^{-1} A e_k), so the export shows exactly what the fused
kernels apply; eigenvalues come from LAPACK (numpy) on the host.  Analysis only -- not on the
solve path.
"""
from __future__ import annotations

import csv
import os

import numpy as np

from .tsf import OP_A, OP_PINV, Solver


def dense_operator(s: Solver, j: int, which: int = OP_A, inst: int = 0) -> np.ndarray:
    """Dense n x n matrix of operator `which` (OP_A, OP_B, OP_AT, OP_PINV, OP_PTINV) of level j."""
    n = s.n
    M = np.zeros((n, n))
    e = np.zeros(n)
    for k in range(n):
        e[:] = 0.0
        e[k] = 1.0
        M[:, k] = s.debug_apply(inst, j, which, e)
    return M


def preconditioned_dense(s: Solver, j: int, inst: int = 0) -> np.ndarray:
    """Dense P^{-1} A of level j (left preconditioning; similar to the A P^{-1} the Krylov
    solvers iterate with, so the spectrum is the same)."""
    n = s.n
    M = np.zeros((n, n))
    e = np.zeros(n)
    for k in range(n):
        e[:] = 0.0
        e[k] = 1.0
        M[:, k] = s.debug_apply(inst, j, OP_PINV, s.debug_apply(inst, j, OP_A, e))
    return M


def level_spectra(s: Solver, j: int, inst: int = 0):
    """(eig A, eig P^{-1} A) of level j, sorted by real part."""
    A = dense_operator(s, j, OP_A, inst)
    PA = preconditioned_dense(s, j, inst)
    ea = np.linalg.eigvals(A)
    ep = np.linalg.eigvals(PA)
    return ea[np.argsort(ea.real)], ep[np.argsort(ep.real)]


def cluster_summary(eig: np.ndarray, center: float = 1.0, radius: float = 0.1) -> dict:
    """Outliers of a spectrum around `center` (the paper's clustering statement)."""
    far = np.abs(eig - center) > radius
    return {"n": int(eig.size), "outliers": int(far.sum()), "min_real": float(eig.real.min()),
            "max_abs_dev": float(np.abs(eig - center).max())}


def export_csv(path: str, s: Solver, levels=(0, 1), inst: int = 0) -> list:
    """Write one CSV per level with columns level, k, Re/Im eig(A), Re/Im eig(P^{-1}A)."""
    os.makedirs(path, exist_ok=True)
    files = []
    for j in levels:
        ea, ep = level_spectra(s, j, inst)
        fn = os.path.join(path, f"spectrum_level{j}.csv")
        with open(fn, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["level", "k", "re_eig_A", "im_eig_A", "re_eig_PinvA", "im_eig_PinvA"])
            for k in range(ea.size):
                w.writerow([j, k, ea[k].real, ea[k].imag, ep[k].real, ep[k].imag])
        files.append(fn)
    return files
