"""GPU parity of the multi-pass regime: n = 2^18..2^20 unknowns, i.e. real FFT lengths 2^19..2^21
for the 2n circulant embedding and 2^18..2^20 for the preconditioner (north_star "lengths 2^7 to
2^21"; SURVEY §2.6, §8(b) N up to 2^20).

Each CTA of a 16-CTA cluster owns a local transform of n/16 > 8192 points, run as R x 8192 rows
through the global apply buffer (exchange 3).  Checked here against references that share no
code with the CUDA path:
* every operator (A, B, A^T, P^{-1}, P^{-T}) against numpy FFTs of the oracle's Toeplitz
  generator (orc_generator; embedding length 2n) and of its Strang column, and A, B against the
  oracle's literal row sums (orc_matvec_rows, extended precision) at sampled rows;
* free-running levels (BiCGSTAB, CGNR, PCGS) against the oracle's sampled-row residual
  (orc_rhs_rows / orc_matvec_rows on the GPU history, teacher-forced) and the manufactured exact
  solution.
Inputs: configs[4]'s seeded instance 0 (alpha, beta, c+-, gamma; d+-(t) = c+-(1+t), manufactured
f) at the larger n.
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_1603_00279_b200 import tsf
from paper_1603_00279_b200.inputs import config_c5

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def c5_pair(n, M):
    inst = config_c5(B=1, n=n, M=M)[0]
    p = O.Problem(alpha=inst.alpha, beta=inst.beta, n=n, M=M, gamma=(O.CONST, float(inst.gamma(0.0))),
                  dplus=(O.ONE_PLUS_T, float(inst.dplus(0.0))), dminus=(O.ONE_PLUS_T, float(inst.dminus(0.0))),
                  src=O.SRC_MMS3)
    return inst, p


def toeplitz_fft(col, row, x):
    """numpy: T x for the Toeplitz matrix (col, row) through its 2n circulant embedding."""
    n = len(x)
    e = np.r_[col, 0.0, row[:0:-1]]
    return np.fft.ifft(np.fft.fft(e) * np.fft.fft(np.r_[x, np.zeros(n)]))[:n].real


def circ_mul(c, x):
    return np.fft.ifft(np.fft.fft(c) * np.fft.fft(x)).real


@pytest.mark.parametrize("lg", [18, 19, 20])
def test_multipass_operators_match_numpy_fft_and_oracle_rows(lg):
    n = 1 << lg
    inst, p = c5_pair(n, 4)
    s = tsf.Solver([inst])
    assert (s.info.cluster, s.info.exchange, s.info.vsmem) == (16, 3, 0)
    rng = np.random.default_rng(lg)
    x = rng.standard_normal(n)
    rows = np.sort(rng.choice(n, 24, replace=False))
    rows[:2] = (0, n - 1)
    tol = 1e-13 * math.log2(n)
    for j in (0, 3):
        for which, wo in ((tsf.OP_A, 0), (tsf.OP_B, 1)):
            col, row = O.generator(p, j, wo)
            ref = toeplitz_fft(col, row, x)
            y = s.debug_apply(0, j, which, x)
            assert np.linalg.norm(y - ref) <= tol * np.linalg.norm(ref), (lg, j, which)
            yr = O.matvec_rows(p, j, wo, x, rows)
            scale = (np.abs(col).sum() + np.abs(row).sum()) * np.abs(x).max()
            assert np.abs(y[rows] - yr).max() <= tol * scale, (lg, j, which)
            if wo == 0:
                yt = s.debug_apply(0, j, tsf.OP_AT, x)
                reft = toeplitz_fft(row, col, x)
                assert np.linalg.norm(yt - reft) <= tol * np.linalg.norm(reft), (lg, j, "AT")
                c = O.strang_col(col, row)
                ct = np.r_[c[0], c[:0:-1]]
                for w2, cc in ((tsf.OP_PINV, c), (tsf.OP_PTINV, ct)):
                    yp = s.debug_apply(0, j, w2, x)
                    # backward error of the circulant solve (numpy FFT of the oracle's column)
                    back = np.linalg.norm(circ_mul(cc, yp) - x)
                    assert back <= tol * (np.abs(cc).sum() * np.linalg.norm(yp) + np.linalg.norm(x)), (lg, j, w2)


@pytest.mark.slow
@pytest.mark.parametrize("lg,method", [(18, "bicgstab"), (18, "cgnr"), (18, "pcgs"), (20, "bicgstab")])
def test_multipass_levels_oracle_row_residual_and_exact_solution(lg, method):
    """Free-running levels 0..M-1 on the multi-pass path.  Teacher-forced oracle check at sampled
    rows: r_i = (A u^{j+1})_i - g_i with g from the oracle's RHS of the GPU history; gate: the
    FP64 floor of an FFT product, 64 eps log2(2n) ||A||_row ||u||_inf, and relative 1e-9."""
    n, M, steps = 1 << lg, 256, 3             # configs[4]'s tau = 1/256; the first levels only
    inst, p = c5_pair(n, M)
    s = tsf.Solver([inst], method=method)
    assert s.info.exchange == 3
    U = [s.solution(0)]
    for _ in range(steps):
        s.step()
        U.append(s.solution(0))
    assert s.sync() == 0
    it, rr, st = s.stats()
    assert (st[0, :steps] == 0).all() and rr[0, :steps].max() < 1e-12 and (it[0, :steps] > 0).all()
    H = np.array(U)
    rows = np.sort(np.random.default_rng(n).choice(n, 48, replace=False))
    for j in range(steps):
        g = O.rhs_rows(p, j, H[: j + 1], rows)
        res = O.matvec_rows(p, j, 0, H[j + 1], rows) - g
        col, row = O.generator(p, j, 0)
        floor = 64 * EPS * math.log2(2 * n) * (np.abs(col).sum() + np.abs(row).sum()) * np.abs(H[j + 1]).max()
        assert np.abs(res).max() <= max(1e-9 * np.abs(g).max(), floor), (j, np.abs(res).max(), floor)
    x, _ = tsf.sample_points(inst)
    t = steps * p.tau
    ex = (t**3 + 1) * x**2 * (1 - x)**2                 # u = (t^3 + 1) X (mms3)
    assert np.linalg.norm(H[steps] - ex) <= 1e-6 * np.linalg.norm(ex)
