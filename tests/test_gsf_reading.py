"""NEXT-2 reading check (CPU): the Gohberg-Semencul formula exactly as PAPER.md prints it
(A^{-1} = (L_p R_p - L_p^0 R_p^0) / xi_0 with x = A^{-1} e_1, y = A^{-1} e_{N-1},
eq3.4) reproduces the inverse of the scheme's level matrix A (the oracle's dense assembly), and
alg1x applied through 2n circulant embeddings (the GPU's construction,
tsf_capi.cu k_gsf_cols) equals the dense triangular products.  Pins the factor layout the
CUDA path uses; the CUDA path itself is checked against the oracle in test_gpu.py."""
import numpy as np
import pytest

import oracle as O


def lower(c):
    n = len(c)
    return np.array([[c[i - m] if i >= m else 0.0 for m in range(n)] for i in range(n)])


def upper(r):
    n = len(r)
    return np.array([[r[m - i] if m >= i else 0.0 for m in range(n)] for i in range(n)])


def factors(x, y):
    n = len(x)
    Lp = lower(x)                                           # first column xi_0 .. xi_{n-1}
    Rp = upper(y[::-1])                                     # first row eta_{n-1} .. eta_0
    Lp0 = lower(np.concatenate([[0.0], y[:-1]]))           # first column 0, eta_0 .. eta_{n-2}
    Rp0 = upper(np.concatenate([[0.0], x[:0:-1]]))         # first row 0, xi_{n-1} .. xi_1
    return Lp, Rp, Lp0, Rp0


def embed(k, x, y):
    """2n embeddings of k = 0 R_p^0, 1 R_p, 2 L_p^0, 3 L_p (as k_gsf_cols builds them)."""
    n = len(x)
    c = np.zeros(2 * n)
    if k == 0:
        c[n + 1:] = x[1:]
    elif k == 1:
        c[0] = y[n - 1]
        c[n + 1:] = y[:n - 1]
    elif k == 2:
        c[1:n] = y[:n - 1]
    else:
        c[:n] = x
    return c


def circ_apply(c, v):
    n = len(v)
    return np.real(np.fft.ifft(np.fft.fft(c) * np.fft.fft(np.concatenate([v, np.zeros(n)]))))[:n]


@pytest.mark.parametrize("alpha,beta,gam,dp,dm", [(0.5, 1.5, 0.5, 1.0, 1.0), (0.9, 1.9, 1.0, 2.0, 0.5),
                                                    (0.3, 1.2, -0.7, 0.0, 1.3)])
def test_paper_gsf_formula_inverts_the_level_matrix(alpha, beta, gam, dp, dm):
    n = 24
    p = O.Problem(alpha=alpha, beta=beta, n=n, M=4, gamma=(O.CONST, gam), dplus=(O.CONST, dp),
                  dminus=(O.CONST, dm), src=O.SRC_ZERO)
    A, _ = O.assemble(p, 1)                                 # level-invariant A for j >= 1 (eqgux)
    A2, _ = O.assemble(p, 3)
    assert np.array_equal(A, A2)
    e1, en = np.eye(n)[0], np.eye(n)[-1]
    x, y = np.linalg.solve(A, e1), np.linalg.solve(A, en)
    assert abs(x[0] - y[-1]) < 1e-12 * abs(x[0])          # persymmetry of A^{-1}
    Lp, Rp, Lp0, Rp0 = factors(x, y)
    Ainv = (Lp @ Rp - Lp0 @ Rp0) / x[0]
    assert np.abs(Ainv @ A - np.eye(n)).max() < 1e-11
    # alg1x through the 2n circulant embeddings equals the dense products
    v = np.random.default_rng(3).standard_normal(n)
    z1, z2 = circ_apply(embed(0, x, y), v), circ_apply(embed(1, x, y), v)
    assert np.allclose(z1, Rp0 @ v, atol=1e-13) and np.allclose(z2, Rp @ v, atol=1e-13)
    z3, z4 = circ_apply(embed(2, x, y), z1), circ_apply(embed(3, x, y), z2)
    assert np.allclose(z3, Lp0 @ z1, atol=1e-13) and np.allclose(z4, Lp @ z2, atol=1e-13)
    z = (z4 - z3) / x[0]
    assert np.linalg.norm(A @ z - v) < 1e-11 * np.linalg.norm(v)
