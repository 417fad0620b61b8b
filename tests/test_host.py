"""CPU-only tests of the product's host side: the C-ABI library loads and exports every
declared symbol, the planner's integer FFT tables match the oracle's definitions bit for
bit, validation rejects bad problems, the input module's manufactured sources agree with
the oracle's independent closed forms, and the batched sharding/gather logic (gloo, 2 ranks).
No compute call here needs a GPU."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_1603_00279_b200 import _lib as L
from paper_1603_00279_b200 import dist, tsf
from paper_1603_00279_b200.inputs import (CONFIGS, Instance, config_c3, config_c4, config_c5, const,
                                          manufactured_basis, manufactured_scal)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "tsf.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(tsf_\w+)\(", header, re.M))
    assert len(declared) >= 20
    lib = C.CDLL(L.LIB_PATH)
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(L.EXPORTED), declared ^ set(L.EXPORTED)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1603_00279_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "oracle.h" not in src and "liboracle" not in src, f


@pytest.mark.parametrize("lg", list(range(1, 17)))
def test_fft_tables_bit_exact_vs_oracle_definition(lg):
    Lc = 1 << lg
    plan, perm, tw = tsf.debug_fft_tables(Lc)
    assert plan == O.fft_plan(Lc)
    np.testing.assert_array_equal(perm, O.fft_perm(Lc))
    ref = np.concatenate([O.fft_twiddles(Lc, s) for s in range(len(plan))])
    np.testing.assert_array_equal(tw[: ref.size], ref)


def test_sample_points_follow_the_grid():
    inst = Instance(0.5, 1.5, 64, 10, const(0), const(1), const(1), a=-1.0, b=2.0, T=3.0)
    x, t = tsf.sample_points(inst)
    h = 3.0 / 65
    np.testing.assert_allclose(x, -1.0 + h * np.arange(1, 65), rtol=0, atol=1e-15)
    np.testing.assert_allclose(t, (np.arange(10) + 0.75) * 0.3, rtol=1e-15)


@pytest.mark.parametrize("bad,match", [
    (dict(alpha=0.0), "alpha"), (dict(alpha=1.2), "alpha"), (dict(beta=1.0), "beta"),
    (dict(beta=2.5), "beta"), (dict(n=100), "power of two"), (dict(n=32), "power of two"),
    (dict(M=0), "M"), (dict(dplus=const(-0.1)), "d\\+-"),
])
def test_validation_rejects(bad, match):
    kw = dict(alpha=0.5, beta=1.5, n=64, M=4, gamma=const(0.0), dplus=const(1.0), dminus=const(1.0))
    kw.update(bad)
    inst = Instance(**kw)
    with pytest.raises(L.TsfError, match=match):
        tsf.plan([inst])


def test_solver_settings_validated():
    inst = CONFIGS["C1"]()[0]
    for kw in (dict(tol=0.0), dict(maxit=0), dict(cluster=3), dict(cluster=32)):
        with pytest.raises(L.TsfError):
            tsf.plan([inst], **kw)
    with pytest.raises(L.TsfError, match="infeasible"):
        tsf.plan([inst], cluster=16)          # n = 64 < 4 C^2


def test_gsf_method_requires_constant_coefficients_and_a_preconditioner():
    # NEXT-2 (alg2) is defined for gamma, d+- constant in time (eqgux)
    ok = Instance(alpha=0.5, beta=1.5, n=64, M=4, gamma=const(0.5), dplus=const(1.0), dminus=const(1.0))
    assert tsf.plan([ok], method="gsf").cluster == 1
    var = Instance(alpha=0.5, beta=1.5, n=64, M=4, gamma=const(0.5), dplus=lambda t: 1.0 + t,
                   dminus=const(1.0))
    with pytest.raises(L.TsfError, match="constant"):
        tsf.plan([var], method="gsf")
    with pytest.raises(L.TsfError, match="preconditioner"):
        tsf.plan([ok], method="gsf", precond="none")


def test_planner_cluster_choices_and_workspace():
    c1 = tsf.plan(CONFIGS["C1"]())
    c3 = tsf.plan(config_c3())
    c4 = tsf.plan(config_c4(B=256))
    assert c1.cluster == 1 and c3.cluster == 16 and c4.cluster == 1
    assert tsf.plan(CONFIGS["C2"]()).cluster == 4          # >= 256 local points per CTA
    assert c3.embed_len == 16384 and c3.precond_len == 8192
    # workspace grows with the history (M n doubles per instance) and the batch
    assert tsf.plan(config_c4(B=512)).workspace_bytes > c4.workspace_bytes
    assert c3.workspace_bytes > 512 * 16384 * 8 * 2            # history + f table
    c5 = tsf.plan(config_c5(B=2))
    assert c5.cluster == 16 and c5.smem_bytes <= 227 * 1024


@pytest.mark.parametrize("lg", [18, 19, 20])
def test_planner_multi_pass_regime(lg):
    """n = 2^18..2^20 (FFT lengths 2^19..2^21 real, north_star): 16-CTA clusters, local
    transforms of n/16 points as R x 8192 rows (exchange 3), vectors in HBM, SMEM within 227 KiB;
    n = 2^21 is rejected, and smaller clusters are infeasible (local length > 8192)."""
    n = 1 << lg
    inst = Instance(alpha=0.6, beta=1.6, n=n, M=2, gamma=const(0.3), dplus=const(1.0), dminus=const(0.5))
    pl = tsf.plan([inst])
    assert (pl.cluster, pl.exchange, pl.vsmem, pl.resident) == (16, 3, 0, 0)
    assert pl.embed_len == n and pl.precond_len == n // 2
    assert pl.smem_bytes <= 227 * 1024 and pl.chunk >= 1
    assert pl.workspace_bytes > (13 + 2 + 2) * n * 8          # vectors, history, apply buffers
    with pytest.raises(L.TsfError, match="infeasible"):
        tsf.plan([inst], cluster=8)
    with pytest.raises(L.TsfError, match="power of two"):
        tsf.plan([Instance(alpha=0.6, beta=1.6, n=2 * kmax, M=2, gamma=const(0.3), dplus=const(1.0),
                           dminus=const(0.5))]) if (kmax := 1 << 20) else None


def test_hist_block_option_validated_and_row_model():
    """hist_block: 0 or a power of two in [2, 64]; the bench's history row model: the direct sum
    reads j rows at level j, the blocked sum about J0/b + (j - J0) + 2 per level."""
    import bench
    inst = CONFIGS["C1"]()[0]
    for bad in (3, 1, 128, -2):
        with pytest.raises(L.TsfError, match="hist_block"):
            tsf.plan([inst], hist_block=bad)
    base = tsf.plan([inst]).workspace_bytes
    assert tsf.plan([inst], hist_block=16).workspace_bytes >= base + 16 * inst.n * 8
    M = 256
    direct = sum(bench.hist_units(j, M) for j in range(M))
    blocked = sum(bench.hist_units(j, M, 16) for j in range(M))
    assert direct == M * (M - 1) // 2
    # block starts read J0 rows and write 16 partial sums; other levels <= 16 rows
    assert blocked == sum(j for j in range(16)) + sum(
        (j % 16) + 1 + (j + 16 if j % 16 == 0 else 0) for j in range(16, M))
    assert blocked < direct / 4


def test_init_rejects_small_workspace_without_touching_the_gpu():
    lib = L.load()
    probs, keep = tsf.marshal(CONFIGS["C1"]())
    s = tsf.make_solver_struct()
    h = C.c_void_p()
    rc = lib.tsf_init(probs, 1, C.byref(s), C.c_void_p(256), C.c_size_t(16), 0, None, C.byref(h))
    assert rc == -2 and b"workspace" in lib.tsf_last_error()


@pytest.mark.parametrize("kind", ["mms3", "exa"])
@pytest.mark.parametrize("shapes", [
    ((O.CONST, 0.5), (O.CONST, 1.0), (O.CONST, 1.0)),
    ((O.COS, 1.0), (O.ONE_PLUS_T, 1.0), (O.ONE_PLUS_T2, 1.0)),
    ((O.T, -1.0), (O.SIN, 9.0), (O.SIN, 4.0)),
])
def test_input_module_source_matches_oracle_closed_form(kind, shapes):
    fns = {O.CONST: lambda s: (lambda t: s * np.ones_like(t)), O.COS: lambda s: (lambda t: s * np.cos(t)),
           O.ONE_PLUS_T: lambda s: (lambda t: s * (1 + t)), O.ONE_PLUS_T2: lambda s: (lambda t: s * (1 + t * t)),
           O.SIN: lambda s: (lambda t: s * np.sin(t)), O.T: lambda s: (lambda t: s * t)}
    g, dp, dm = (fns[sh](sc) for sh, sc in shapes)
    alpha, beta, n, M = 0.7, 1.45, 63, 5
    p = O.Problem(alpha=alpha, beta=beta, n=n, M=M, gamma=shapes[0], dplus=shapes[1], dminus=shapes[2],
                  src=O.SRC_MMS3 if kind == "mms3" else O.SRC_EXA)
    x = (np.arange(n) + 1) / (n + 1)
    t = (np.arange(M) + 1 - alpha / 2) / M
    f = manufactured_scal(t, alpha, g, dp, dm, kind) @ manufactured_basis(x, beta)
    for j in range(M):
        np.testing.assert_allclose(f[j], O.source(p, j, t[j]), rtol=1e-12, atol=1e-12)


def test_configs_seeded_and_shaped():
    c4 = config_c4()
    assert len(c4) == 1024 and c4[0].n == 4096 and c4[0].M == 256
    al = np.array([i.alpha for i in c4]); be = np.array([i.beta for i in c4])
    assert 0.1 <= al.min() and al.max() <= 0.99 and 1.1 <= be.min() and be.max() <= 1.95
    assert config_c4()[17].alpha == c4[17].alpha                        # deterministic
    c3 = config_c3()[0]
    assert c3.f_table.shape == (512, 16384)
    assert abs(c3.f_table.mean()) < 1e-2 and abs(c3.f_table.std() - 1) < 1e-2
    c5 = config_c5()
    assert len(c5) == 64 and c5[0].n == 131072
    t = np.array([0.0, 0.5])
    assert c5[3].dplus(t)[1] == pytest.approx(1.5 * c5[3].dplus(t)[0])  # c (1 + t)


@pytest.mark.parametrize("B,W", [(1, 1), (7, 2), (1024, 8), (64, 8), (3, 4)])
def test_shard_partitions_the_batch(B, W):
    seen = []
    for r in range(W):
        sh = dist.shard(B, W, r)
        assert len(sh) in (B // W, B // W + 1)
        seen.extend(sh)
    assert seen == list(range(B))


def _gloo_worker(rank, world, port, out):
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    insts = [Instance(a, b, 15, 6, const(0.3), const(1.0), const(0.5), "mms3")
             for a, b in ((0.3, 1.2), (0.6, 1.5), (0.9, 1.8))]

    def local(mine):
        us, its = [], []
        for inst in mine:
            p = O.Problem(alpha=inst.alpha, beta=inst.beta, n=inst.n, M=inst.M, gamma=(O.CONST, 0.3),
                          dplus=(O.CONST, 1.0), dminus=(O.CONST, 0.5), src=O.SRC_MMS3)
            us.append(O.solve(p)[-1])
            its.append(np.full(inst.M, 2 * (rank + 1), np.int32))
        k = len(mine)
        return dist.BatchResult(np.array(us).reshape(k, 15), np.array(its, np.int32).reshape(k, 6),
                                np.zeros((k, 6)), np.zeros((k, 6), np.int32))
    res = dist.solve_batch(insts, rank, world, local_solver=local)
    if rank == 0:
        np.save(out, np.concatenate([res.u.ravel(), res.iters_half.ravel().astype(float)]))
    tdist.destroy_process_group()


def test_gather_over_two_gloo_ranks_equals_single_rank(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "r.npy")
    port = 29500 + os.getpid() % 1000
    mp.spawn(_gloo_worker, args=(2, port, out), nprocs=2, join=True)
    got = np.load(out)
    ref = []
    for a, b in ((0.3, 1.2), (0.6, 1.5), (0.9, 1.8)):
        p = O.Problem(alpha=a, beta=b, n=15, M=6, gamma=(O.CONST, 0.3), dplus=(O.CONST, 1.0),
                      dminus=(O.CONST, 0.5), src=O.SRC_MMS3)
        ref.append(O.solve(p)[-1])
    np.testing.assert_array_equal(got[: 45], np.array(ref).ravel())
    # rank 0 owns instances {0, 1}, rank 1 owns {2}: iteration rows tag the owner
    np.testing.assert_array_equal(got[45:], [2] * 12 + [4] * 6)


def test_ncu_traffic_key_is_a_hash_of_the_kernel_sources(tmp_path, monkeypatch):
    """bench.py accepts an ncu DRAM-traffic capture only for the kernel sources it was taken
    with: the key is a hash over csrc/ + include/tsf.h + compile flags (stable across rebuilds of
    the same sources, different as soon as a source byte or a flag changes)."""
    import shutil

    import bench
    from paper_1603_00279_b200 import build as B
    h0 = bench.lib_hash()
    assert re.fullmatch(r"[0-9a-f]{16}", h0) and bench.lib_hash() == h0
    d = tmp_path / "a" / "b" / "csrc"
    d.mkdir(parents=True)
    (tmp_path / "a" / "include").mkdir()
    for f in B.SOURCES + B.HEADERS:
        shutil.copy(os.path.join(B.CSRC, f), os.path.normpath(os.path.join(d, f)))
    monkeypatch.setattr(B, "CSRC", str(d))
    assert bench.lib_hash() == h0
    with open(d / "tsf_plan.cpp", "a") as fh:
        fh.write("\n")
    assert bench.lib_hash() != h0
    monkeypatch.setattr(B, "CSRC", os.path.join(os.path.dirname(B.__file__), "csrc"))
    monkeypatch.setattr(B, "FLAGS", B.FLAGS + ["-DX"])
    assert bench.lib_hash() != h0
