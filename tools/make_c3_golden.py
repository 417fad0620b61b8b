"""Write tests/golden/c3_oracle_levels.npz: the CPU oracle's free-running solution of
BASELINE configs[2] (C3: n = 2^14, M = 2^9, alpha = 0.9, beta = 1.9, d+ = 2, d- = 0.5,
gamma = 1, phi = x^2 (1-x)^2, f ~ N(0,1) from seed 160300279, reading R-c3f).

The values come ONLY from oracle/ (dense assembly of eq3.3, Gaussian elimination
with partial pivoting and LU reuse for the level-invariant A of j >= 1, refined per
R-refine); the input table comes from the seeded generator module, which holds no arithmetic
of the method.  The full run is 2 factorizations of a 16384 x 16384 matrix plus 512 solve
pairs (~6 GiB of RAM, tens of minutes on 8 cores), too slow for the test suite, so the test
(tests/test_gpu.py::test_c3_full_size_free_running_vs_oracle_golden) reads this file.

Stored: u^j for the sampled levels LEVELS (u^0 = phi included), the wall time and thread
count of the run.  Usage:  OMP_NUM_THREADS=8 python tools/make_c3_golden.py
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_1603_00279_b200.inputs import config_c3  # noqa: E402  (seeded data only)

LEVELS = [0, 1, 2, 3, 4, 8, 16, 32, 64, 100, 128, 192, 256, 320, 384, 448, 510, 511, 512]


def main(out: str = os.path.join(ROOT, "tests", "golden", "c3_oracle_levels.npz")) -> None:
    inst = config_c3()[0]
    p = O.Problem(alpha=0.9, beta=1.9, n=16384, M=512, gamma=(O.CONST, 1.0), dplus=(O.CONST, 2.0),
                  dminus=(O.CONST, 0.5), src=O.SRC_TABLE, f_table=inst.f_table)
    t0 = time.time()
    U = O.solve(p)
    wall = time.time() - t0
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    np.savez(out, levels=np.array(LEVELS, dtype=np.int64), U=U[LEVELS],
             wall_s=np.array(wall), threads=np.array(threads),
             meta=np.array("oracle.solve(C3) free-running; dense GE + LU reuse + refinement; "
                           "tools/make_c3_golden.py"))
    print(f"C3 oracle: {wall:.1f} s on {threads} threads -> {out}")


if __name__ == "__main__":
    main(*sys.argv[1:])
