"""CPU oracle for arXiv 1603.00279 -- TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper around ``oracle/oracle.c`` (plain C, FP64, dense Gaussian
elimination per level).  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this module.
The product package ``paper_1603_00279_b200`` never imports it, and the two share no
code.  Citations ``P:nnn`` refer to lines of the paper's LaTeX source.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# coefficient shapes (oracle.h)
CONST, ONE_PLUS_T, ONE_PLUS_T2, COS, SIN, T = 0, 1, 2, 3, 4, 5
PHI_ARRAY, PHI_X2 = 0, 1
SRC_ZERO, SRC_TABLE, SRC_EXA, SRC_MMS3 = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, no FMA contraction: DESIGN.md R-fma; -fopenmp over
    independent rows only, bitwise identical for any thread count)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c99",
               "-D_GNU_SOURCE", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Fn(C.Structure):
    _fields_ = [("shape", C.c_int32), ("scale", C.c_double)]


class _Problem(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("n", C.c_int64),
                ("M", C.c_int64), ("a", C.c_double), ("b", C.c_double), ("T", C.c_double),
                ("gamma", _Fn), ("dplus", _Fn), ("dminus", _Fn),
                ("phi_kind", C.c_int32), ("phi", C.POINTER(C.c_double)),
                ("src_kind", C.c_int32), ("f_table", C.POINTER(C.c_double))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i64, i32 = C.c_double, C.c_int64, C.c_int32
        pd, pi32 = C.POINTER(C.c_double), C.POINTER(C.c_int32)
        pp = C.POINTER(_Problem)
        sig = {
            "orc_grunwald": (None, [d, i64, pd]),
            "orc_wsgd": (None, [d, i64, pd]),
            "orc_time_ab": (None, [d, i64, pd, pd]),
            "orc_c_row": (None, [d, i64, pd]),
            "orc_eta": (d, [d, d, i64]),
            "orc_assemble": (C.c_int, [pp, i64, pd, pd]),
            "orc_rhs": (C.c_int, [pp, i64, pd, pd]),
            "orc_source": (C.c_int, [pp, i64, d, pd]),
            "orc_exact": (C.c_int, [pp, d, pd]),
            "orc_ge_solve": (C.c_int, [i64, pd, pd]),
            "orc_matvec": (C.c_int, [pp, i64, C.c_int, pd, pd]),
            "orc_matvec_rows": (C.c_int, [pp, i64, C.c_int, pd, C.POINTER(C.c_int64), i64, pd]),
            "orc_generator": (C.c_int, [pp, i64, C.c_int, pd, pd]),
            "orc_rhs_rows": (C.c_int, [pp, i64, pd, C.POINTER(C.c_int64), i64, pd]),
            "orc_rhs_nodense": (C.c_int, [pp, i64, pd, pd]),
            "orc_solve": (C.c_int, [pp, pd]),
            "orc_solve_level": (C.c_int, [pp, i64, pd, pd]),
            "orc_time_sample": (C.c_int, [pp, i64, i64, pd, pd]),
            "orc_l2": (d, [i64, d, pd]),
            "orc_dft": (None, [i64, pd, pd, C.c_int]),
            "orc_fft_plan": (C.c_int, [i64, pi32]),
            "orc_fft_perm": (None, [i64, pi32]),
            "orc_fft_twiddles": (i64, [i64, i32, pi32]),
            "orc_strang_col": (None, [i64, pd, pd, pd]),
            "orc_tchan_col": (None, [i64, pd, pd, pd]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _pd(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _pi(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


@dataclass
class Problem:
    """TSFCDE instance (eq:lin) on the grid of P:221-223 with n interior nodes."""
    alpha: float
    beta: float
    n: int
    M: int
    gamma: tuple = (CONST, 0.0)      # (shape, scale): c(t) = scale * shape(t)
    dplus: tuple = (CONST, 1.0)
    dminus: tuple = (CONST, 1.0)
    a: float = 0.0
    b: float = 1.0
    T: float = 1.0
    phi: np.ndarray | None = None    # None -> x^2 (1-x)^2
    src: int = SRC_ZERO
    f_table: np.ndarray | None = None
    _keep: list = field(default_factory=list, repr=False)

    @property
    def h(self) -> float:
        return (self.b - self.a) / (self.n + 1)

    @property
    def tau(self) -> float:
        return self.T / self.M

    @property
    def sigma(self) -> float:
        return 1.0 - self.alpha / 2.0

    def c(self) -> _Problem:
        p = _Problem()
        p.alpha, p.beta, p.n, p.M = self.alpha, self.beta, self.n, self.M
        p.a, p.b, p.T = self.a, self.b, self.T
        p.gamma = _Fn(*self.gamma)
        p.dplus = _Fn(*self.dplus)
        p.dminus = _Fn(*self.dminus)
        self._keep = []
        if self.phi is None:
            p.phi_kind = PHI_X2
        else:
            ph = np.ascontiguousarray(self.phi, dtype=np.float64)
            self._keep.append(ph)
            p.phi_kind, p.phi = PHI_ARRAY, _pd(ph)
        p.src_kind = self.src
        if self.src == SRC_TABLE:
            ft = np.ascontiguousarray(self.f_table, dtype=np.float64)
            assert ft.shape == (self.M, self.n)
            self._keep.append(ft)
            p.f_table = _pd(ft)
        return p


def grunwald(beta: float, K: int) -> np.ndarray:
    g = np.zeros(K + 1)
    lib().orc_grunwald(beta, K, _pd(g))
    return g


def wsgd(beta: float, K: int) -> np.ndarray:
    w = np.zeros(K + 1)
    lib().orc_wsgd(beta, K, _pd(w))
    return w


def time_ab(alpha: float, M: int):
    a, b = np.zeros(M + 1), np.zeros(M + 1)
    lib().orc_time_ab(alpha, M, _pd(a), _pd(b))
    return a, b


def c_row(alpha: float, j: int) -> np.ndarray:
    c = np.zeros(j + 1)
    lib().orc_c_row(alpha, j, _pd(c))
    return c


def eta(alpha: float, tau: float, j: int) -> float:
    return lib().orc_eta(alpha, tau, j)


def assemble(p: Problem, j: int):
    A = np.zeros((p.n, p.n))
    B = np.zeros((p.n, p.n))
    cp = p.c()
    assert lib().orc_assemble(C.byref(cp), j, _pd(A), _pd(B)) == 0
    return A, B


def rhs(p: Problem, j: int, U: np.ndarray) -> np.ndarray:
    U = np.ascontiguousarray(U, dtype=np.float64)
    g = np.zeros(p.n)
    cp = p.c()
    assert lib().orc_rhs(C.byref(cp), j, _pd(U), _pd(g)) == 0
    return g


def matvec(p: Problem, j: int, which: int, x: np.ndarray) -> np.ndarray:
    """A^{(j+sigma)} x (which=0) or B^{(j+sigma)} x (which=1) without dense storage."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(p.n)
    cp = p.c()
    assert lib().orc_matvec(C.byref(cp), j, which, _pd(x), _pd(y)) == 0
    return y


def matvec_rows(p: Problem, j: int, which: int, x: np.ndarray, rows) -> np.ndarray:
    """Rows `rows` of A x (which=0) / B x (which=1): the literal row sums of matvec, O(n) each."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    y = np.zeros(len(rows))
    cp = p.c()
    assert lib().orc_matvec_rows(C.byref(cp), j, which, _pd(x),
                                 rows.ctypes.data_as(C.POINTER(C.c_int64)), len(rows), _pd(y)) == 0
    return y


def rhs_rows(p: Problem, j: int, U: np.ndarray, rows) -> np.ndarray:
    """Rows `rows` of the level-j RHS from the history U[0..j] (same arithmetic as rhs_nodense)."""
    U = np.ascontiguousarray(U, dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    g = np.zeros(len(rows))
    cp = p.c()
    assert lib().orc_rhs_rows(C.byref(cp), j, _pd(U), rows.ctypes.data_as(C.POINTER(C.c_int64)),
                              len(rows), _pd(g)) == 0
    return g


def generator(p: Problem, j: int, which: int):
    """Toeplitz generator (first column, first row) of A (which=0) / B (which=1) at level j."""
    col, row = np.zeros(p.n), np.zeros(p.n)
    cp = p.c()
    assert lib().orc_generator(C.byref(cp), j, which, _pd(col), _pd(row)) == 0
    return col, row


def rhs_nodense(p: Problem, j: int, U: np.ndarray) -> np.ndarray:
    U = np.ascontiguousarray(U, dtype=np.float64)
    g = np.zeros(p.n)
    cp = p.c()
    assert lib().orc_rhs_nodense(C.byref(cp), j, _pd(U), _pd(g)) == 0
    return g


def source(p: Problem, j: int, t: float) -> np.ndarray:
    f = np.zeros(p.n)
    cp = p.c()
    assert lib().orc_source(C.byref(cp), j, t, _pd(f)) == 0
    return f


def exact(p: Problem, t: float) -> np.ndarray:
    u = np.zeros(p.n)
    cp = p.c()
    assert lib().orc_exact(C.byref(cp), t, _pd(u)) == 0
    return u


def ge_solve(A: np.ndarray, b: np.ndarray) -> np.ndarray:
    A = np.array(A, dtype=np.float64, order="C", copy=True)
    x = np.array(b, dtype=np.float64, copy=True)
    assert lib().orc_ge_solve(A.shape[0], _pd(A), _pd(x)) == 0
    return x


def solve(p: Problem) -> np.ndarray:
    """Full run: U[0..M][n] (alg1 with a direct solve per level)."""
    U = np.zeros((p.M + 1, p.n))
    cp = p.c()
    rc = lib().orc_solve(C.byref(cp), _pd(U))
    assert rc == 0, rc
    return U


def solve_level(p: Problem, j: int, U: np.ndarray) -> np.ndarray:
    U = np.ascontiguousarray(U, dtype=np.float64)
    out = np.zeros(p.n)
    cp = p.c()
    assert lib().orc_solve_level(C.byref(cp), j, _pd(U), _pd(out)) == 0
    return out


def time_sample(p: Problem, j: int, kmax: int, U: np.ndarray) -> np.ndarray:
    """Wall seconds [assembly, first kmax elimination columns, one level at history j] of the
    oracle's own steps at the full size (bench.py cpu_baseline; no result is returned)."""
    U = np.ascontiguousarray(U, dtype=np.float64)
    assert U.shape == (j + 1, p.n)
    t = np.zeros(3)
    cp = p.c()
    assert lib().orc_time_sample(C.byref(cp), j, kmax, _pd(U), _pd(t)) >= 0
    return t


def l2(v: np.ndarray, h: float) -> float:
    v = np.ascontiguousarray(v, dtype=np.float64)
    return lib().orc_l2(v.size, h, _pd(v))


def dft(x: np.ndarray, inverse: bool = False) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.complex128)
    xr = x.view(np.float64).copy()
    X = np.zeros_like(xr)
    lib().orc_dft(x.size, _pd(xr), _pd(X), int(inverse))
    return X.view(np.complex128)


def fft_plan(L: int) -> list:
    plan = np.zeros(64, dtype=np.int32)
    S = lib().orc_fft_plan(L, _pi(plan))
    return [int(v) for v in plan[:S]]


def fft_perm(L: int) -> np.ndarray:
    perm = np.zeros(L, dtype=np.int32)
    lib().orc_fft_perm(L, _pi(perm))
    return perm


def fft_twiddles(L: int, s: int) -> np.ndarray:
    tw = np.zeros(4 * L, dtype=np.int32)
    cnt = lib().orc_fft_twiddles(L, s, _pi(tw))
    return tw[:cnt].copy()


def strang_col(col: np.ndarray, row: np.ndarray) -> np.ndarray:
    n = len(col)
    c = np.zeros(n)
    lib().orc_strang_col(n, _pd(np.ascontiguousarray(col, float)),
                         _pd(np.ascontiguousarray(row, float)), _pd(c))
    return c


def tchan_col(col: np.ndarray, row: np.ndarray) -> np.ndarray:
    n = len(col)
    c = np.zeros(n)
    lib().orc_tchan_col(n, _pd(np.ascontiguousarray(col, float)),
                        _pd(np.ascontiguousarray(row, float)), _pd(c))
    return c


def errors(p: Problem, U: np.ndarray):
    """max_n ||E^n||_0 and ||E||_C over the mesh incl. level 0."""
    l2max, cmax = 0.0, 0.0
    for j in range(p.M + 1):
        e = U[j] - exact(p, j * p.tau)
        l2max = max(l2max, l2(e, p.h))
        cmax = max(cmax, float(np.max(np.abs(e))))
    return l2max, cmax
