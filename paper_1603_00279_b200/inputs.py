"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs C1-C5).

This module holds problem DATA only (coefficient functions, initial data, manufactured
source terms and their exact solutions, seeded parameter draws); none of the scheme's or
the solver's arithmetic.  Both the CUDA path (through ``paper_1603_00279_b200.tsf``) and
the tests use it; the oracle computes its own source terms from the closed forms.

Manufactured solutions follow the pattern of the paper's examples (P:931-944,
P:1118-1134): u(x,t) = tau(t) X(x), X = x^2 (1-x)^2 on [0,1], with
  f = D^alpha_t tau * X - tau(t) [gamma(t) X' + d+(t) R+(x) + d-(t) R-(x)],
  R+(x) = G(3)/G(3-b) x^{2-b} - 2G(4)/G(4-b) x^{3-b} + G(5)/G(5-b) x^{4-b},  R-(x) = R+(1-x)
(left/right Riemann-Liouville derivatives of X, eq3x/eq3y).  "exa" uses
tau = t^{2+alpha} + 1 (Examples 1-2), "mms3" uses tau = t^3 + 1.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

SEED_C3 = 160300279
SEED_C4 = 160300284
SEED_C5 = 160300285


def X(x):
    return x**2 * (1 - x)**2


def Xp(x):
    return 2 * x * (1 - x) * (1 - 2 * x)


def Rplus(x, beta):
    g = math.gamma
    return (g(3) / g(3 - beta) * x ** (2 - beta) - 2 * g(4) / g(4 - beta) * x ** (3 - beta)
            + g(5) / g(5 - beta) * x ** (4 - beta))


def manufactured_basis(x: np.ndarray, beta: float) -> np.ndarray:
    """[X, X', R+, R-] at the interior nodes x (shape [4][n])."""
    x = np.asarray(x, dtype=np.float64)
    return np.stack([X(x), Xp(x), Rplus(x, beta), Rplus(1.0 - x, beta)])


def manufactured_scal(t: np.ndarray, alpha: float, gamma, dplus, dminus, kind: str = "mms3") -> np.ndarray:
    """Time factors [M][4] multiplying the basis at the sample times t."""
    t = np.asarray(t, dtype=np.float64)
    if kind == "mms3":
        dt = math.gamma(4) / math.gamma(4 - alpha) * t ** (3 - alpha)
        tu = t**3 + 1
    elif kind == "exa":
        dt = math.gamma(3 + alpha) / 2 * t**2
        tu = t ** (2 + alpha) + 1
    else:
        raise ValueError(kind)
    return np.stack([dt, -tu * gamma(t), -tu * dplus(t), -tu * dminus(t)], axis=1)


def exact(x, t, kind: str = "mms3", alpha: float = 0.0):
    tu = (t**3 + 1) if kind == "mms3" else (t ** (2 + alpha) + 1)
    return tu * X(np.asarray(x))


def const(c: float) -> Callable:
    return lambda t: np.full_like(np.asarray(t, dtype=np.float64), c)


@dataclass
class Instance:
    """One TSFCDE instance (eq:lin) as data: callables are vectorized numpy functions."""
    alpha: float
    beta: float
    n: int
    M: int
    gamma: Callable
    dplus: Callable
    dminus: Callable
    source: str = "mms3"            # "mms3" | "exa" | "table" | "callback" | "zero"
    f_table: np.ndarray | None = None   # [M][n] numpy (copied) or CUDA float64 tensor (borrowed)
    f_callback: Callable | None = None  # f(x: ndarray, t: float) -> ndarray ("callback")
    phi: Callable = X
    a: float = 0.0
    b: float = 1.0
    T: float = 1.0
    meta: dict = field(default_factory=dict)


# ---------------------------------------------------------------------------- BASELINE configs
def config_c1() -> list[Instance]:
    """configs[0]: alpha=0.5, beta=1.5, d+=d-=1, gamma=0.5, n=2^6, M=2^6, manufactured."""
    return [Instance(0.5, 1.5, 64, 64, const(0.5), const(1.0), const(1.0), "mms3")]


def config_c2() -> list[Instance]:
    """configs[1]: alpha=0.8, beta=1.8, d+=1+t, d-=1+t^2, gamma=cos t, n=M=2^10."""
    return [Instance(0.8, 1.8, 1024, 1024, np.cos, lambda t: 1 + t, lambda t: 1 + t**2, "mms3")]


def config_c3(n: int = 16384, M: int = 512) -> list[Instance]:
    """configs[2]: alpha=0.9, beta=1.9, d+=2, d-=0.5, gamma=1, phi=x^2(1-x)^2, random f.
    f[j][i] ~ N(0,1), row j <-> t_{j+sigma}."""
    f = np.random.default_rng(SEED_C3).standard_normal((512, 16384))
    if (M, n) != (512, 16384):
        f = np.ascontiguousarray(f[:M, :n])
    return [Instance(0.9, 1.9, n, M, const(1.0), const(2.0), const(0.5), "table", f_table=f)]


def config_c4(B: int = 1024, n: int = 4096, M: int = 256) -> list[Instance]:
    """configs[3]: B=1024 instances, n=2^12, M=2^8; per-instance alpha~U(.1,.99),
    beta~U(1.1,1.95), d+~U(0,2), d-~U(0,2), gamma~U(-1,1) (drawn in that order, each a
    length-1024 vector); manufactured f."""
    rng = np.random.default_rng(SEED_C4)
    al = rng.uniform(0.1, 0.99, 1024)
    be = rng.uniform(1.1, 1.95, 1024)
    dp = rng.uniform(0.0, 2.0, 1024)
    dm = rng.uniform(0.0, 2.0, 1024)
    ga = rng.uniform(-1.0, 1.0, 1024)
    return [Instance(float(al[i]), float(be[i]), n, M, const(float(ga[i])), const(float(dp[i])),
                     const(float(dm[i])), "mms3", meta={"index": i}) for i in range(B)]


def config_c5(B: int = 64, n: int = 131072, M: int = 256) -> list[Instance]:
    """configs[4]: B=64, n=2^17, M=2^8; alpha~U(.3,.9), beta~U(1.3,1.95), c+-~U(.5,2),
    gamma~U(-1,1) constant; d+-(t) = c+-(1+t); manufactured f."""
    rng = np.random.default_rng(SEED_C5)
    al = rng.uniform(0.3, 0.9, 64)
    be = rng.uniform(1.3, 1.95, 64)
    cp = rng.uniform(0.5, 2.0, 64)
    cm = rng.uniform(0.5, 2.0, 64)
    ga = rng.uniform(-1.0, 1.0, 64)
    out = []
    for i in range(B):
        c1, c2 = float(cp[i]), float(cm[i])
        out.append(Instance(float(al[i]), float(be[i]), n, M, const(float(ga[i])),
                            (lambda c: (lambda t: c * (1 + t)))(c1),
                            (lambda c: (lambda t: c * (1 + t)))(c2), "mms3", meta={"index": i}))
    return out


CONFIGS = {"C1": config_c1, "C2": config_c2, "C3": config_c3, "C4": config_c4, "C5": config_c5}
