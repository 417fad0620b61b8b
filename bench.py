"""Benchmark of the B200 per-level Toeplitz Krylov solver (arXiv 1603.00279 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

A "step" is one full time-marching solve (all M levels: RHS with the history sum, the
preconditioned Krylov solve, finalize) of the rank's batch, inputs resident in HBM.
Default workload: BASELINE configs[2] "C3" (n = 2^14, M = 2^9, one instance per GPU:
weak scaling over independent replicas).  --config C4 / C5 run the batched configs,
sharded over ranks (strong scaling).  Prints ONE JSON line on rank 0.

metric: FP64 precond-Krylov iterations/s & time levels/s (value = levels/s, whole job).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 precond-Krylov iters/s & time levels/s at N=2^14; achieved HBM GB/s"
KRYLOV_UNITS = {"bicgstab": 26, "cgnr": 19, "pcgs": 24, "gsf": 26}   # SURVEY 8(d)-style streamed units per iteration
GSF_UNITS_PER_LEVEL = 20   # GSF level: 5 applications x (input + output + 2-unit spectrum table)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def hist_units(j, M, hblock=0):
    """History rows (n-vectors) level j must move: j rows read by the direct sum (eq3.1); with
    the NEXT-3 blocked sum (block b, J0 = j - j mod b) the rows since J0 plus one partial-sum row,
    and at a block start the pass over d^0..d^{J0-1} plus the b partial sums it writes."""
    if hblock <= 0 or j == 0:
        return j
    J0 = j - j % hblock
    if J0 == 0:
        return j
    u = (j - J0) + 1
    if j == J0:
        u += J0 + min(hblock, M - J0)
    return u


def algorithmic_bytes(n, M, iters_half_rows, method, src_units, hblock=0):
    """SURVEY 8(d) model per instance: 8n (h_j + 3 + src + 8) compulsory/RHS bytes per level
    (h_j = history rows, j for the direct sum) plus 8n * units * I_j for the streamed Krylov
    iterations (I_j = iterations of level j)."""
    units = KRYLOV_UNITS[method]
    total = 0.0
    for row in iters_half_rows:
        for j in range(M):
            total += 8.0 * n * (hist_units(j, M, hblock) + 3 + src_units + 8) + 8.0 * n * units * (row[j] / 2.0)
            if method == "gsf" and j >= 1:
                total += 8.0 * n * GSF_UNITS_PER_LEVEL
    return total


def CONFIGS_ALL_get():
    from paper_1603_00279_b200.inputs import CONFIGS
    return CONFIGS


class _Cfgs:
    def __getitem__(self, k):
        return CONFIGS_ALL_get()[k]


CONFIGS_ALL = _Cfgs()


def build_instances(cfg, world, rank):
    from paper_1603_00279_b200 import dist
    from paper_1603_00279_b200.inputs import CONFIGS
    insts = CONFIGS[cfg]()
    if cfg in ("C1", "C2", "C3"):          # single-instance configs: one replica per rank (weak)
        return insts, "weak", len(insts) * world
    mine = [insts[i] for i in dist.shard(len(insts), world, rank)]
    return mine, "strong", len(insts)


# ------------------------------------------------------------------------------ oracle arm
def oracle_problem(inst):
    import oracle as O
    shape = lambda fn: fn  # noqa: E731
    # map the config's coefficient functions onto the oracle's shape enum
    import numpy as np
    t = np.array([0.1, 0.7])

    def enc(fn):
        v = np.asarray(fn(t), dtype=float) * np.ones(2)
        if abs(v[0] - v[1]) < 1e-15:
            return (O.CONST, float(v[0]))
        for sh, g in ((O.ONE_PLUS_T, lambda s: 1 + s), (O.ONE_PLUS_T2, lambda s: 1 + s * s),
                      (O.COS, np.cos), (O.SIN, np.sin), (O.T, lambda s: s)):
            c = v[0] / g(t[0])
            if abs(c * g(t[1]) - v[1]) < 1e-12 * max(1, abs(v[1])):
                return (sh, float(c))
        raise ValueError("coefficient not expressible for the oracle")
    src = {"mms3": O.SRC_MMS3, "exa": O.SRC_EXA, "table": O.SRC_TABLE, "zero": O.SRC_ZERO}[inst.source]
    del shape
    return dict(alpha=inst.alpha, beta=inst.beta, gamma=enc(inst.gamma), dplus=enc(inst.dplus),
                dminus=enc(inst.dminus), src=src)


def host_cpu():
    """Host CPU model and the oracle's thread count (cpu_baseline is run on all host cores)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return model, threads


def oracle_rate(cfg):
    """Oracle levels/s for `cfg` on all host cores (OpenMP over independent rows; the oracle's
    arithmetic is unchanged), from a bounded sample of its OWN steps at the FULL size n
    (orc_time_sample): the dense assembly, the first kmax columns of the elimination and one
    level's RHS + LU solve + 3 refinement steps at the longest history.  The full run is
      constant coefficients (LU reuse):  2 (assembly + factorization) + M level
      variable coefficients (a factorization per level):  M (assembly + factorization + level)
    with the factorization's untimed columns k >= kmax scaled by the (n-k)^2 work of the plain
    row-update loop.  C5 (n = 2^17: the dense matrices need 3 x 128 GiB) is timed at n = 4096 and
    scaled by n^3 (factorization) / n^2 (level): labelled as an extrapolation."""
    import numpy as np

    import oracle as O
    from paper_1603_00279_b200.inputs import CONFIGS
    insts = CONFIGS[cfg]()
    inst = insts[0]
    kw = oracle_problem(inst)
    n, M, B = inst.n, inst.M, len(insts)
    const = all(kw[k][0] == O.CONST for k in ("gamma", "dplus", "dminus"))
    ns = n if n <= 16384 else 4096
    p = O.Problem(n=ns, M=M, **kw)
    if p.src == O.SRC_TABLE:
        p.f_table = np.ascontiguousarray(inst.f_table[:M, :ns])
    j = M - 1
    U = np.ascontiguousarray(np.random.default_rng(0).standard_normal((j + 1, ns)) * 1e-3)
    kmax = ns if ns <= 2048 else 64
    t0 = time.perf_counter()
    ta, tf, tl = O.time_sample(p, j, kmax, U)
    wall = time.perf_counter() - t0
    k = np.arange(ns, dtype=np.float64)
    work = (ns - k) ** 2
    fact = tf * work.sum() / work[:kmax].sum()
    if const:
        full = 2 * (ta + fact) + M * tl
    else:
        full = M * (ta + fact + tl)
    label = "measured at full n" if ns == n else f"measured at n={ns}, scaled to n={n} by n^3 / n^2"
    if ns != n:
        s3, s2 = (n / ns) ** 3, (n / ns) ** 2
        full = (2 * (ta * s2 + fact * s3) + M * tl * s2) if const else M * (ta * s2 + fact * s3 + tl * s2)
    model, threads = host_cpu()
    sample = (f"oracle (dense GE, {'LU reuse' if const else 'factorization per level'}, 3 refinement steps) "
              f"on {cfg}, {label}: assembly {ta:.2f}s, elimination columns 0..{kmax - 1} of {ns} {tf:.2f}s "
              f"(all {ns} columns: {fact:.1f}s by the (n-k)^2 work law), one level at history {j} {tl:.2f}s; "
              f"full run = {full:.0f}s per instance ({wall:.0f}s sampled); {threads} OpenMP threads on "
              f"'{model}'; gcc -O2 -ffp-contract=off -fopenmp")
    return M / full, sample, full * B, threads


def lib_hash() -> str:
    """Identity of the kernel build the ncu traffic belongs to: sha256 over the library's sources,
    headers and compile flags (a rebuild of the same sources links a different binary image, so
    the .so bytes themselves are not a stable key)."""
    import hashlib
    from paper_1603_00279_b200 import build as B
    h = hashlib.sha256()
    h.update(" ".join(B.FLAGS).encode())
    for f in sorted(B.SOURCES + B.HEADERS):
        with open(os.path.join(B.CSRC, f), "rb") as fh:
            h.update(f.encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


def traffic_key(args) -> str:
    return f"{args.config}/{args.method}/{args.precond}" + ("/warm" if args.warm else "") + \
        ("/tres" if args.true_res else "") + ("/pipe" if getattr(args, "pipelined", False) else "") + \
        (f"/hb{args.hist_block}" if getattr(args, "hist_block", 0) else "")


def base_config(args):
    """Workload keys shared by both arms (the GPU arm adds its launch shape)."""
    from paper_1603_00279_b200.inputs import CONFIGS
    insts = CONFIGS[args.config]()
    return {"workload": args.config, "n": insts[0].n, "M": insts[0].M, "instances": len(insts),
            "method": args.method, "precond": args.precond, "tol": 1e-12}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals = []
    sample = ""
    threads = 1
    for _ in range(args.warmup):
        oracle_rate(args.config)
    for _ in range(args.steps):
        t0 = time.perf_counter()
        v, sample, _, threads = oracle_rate(args.config)
        vals.append((v, time.perf_counter() - t0))
    value = statistics.median(v for v, _ in vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "levels/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * statistics.mean(t for _, t in vals), "higher_is_better": True,
            "scaling": "weak" if args.config in ("C1", "C2", "C3") else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": base_config(args),
            "cpu_baseline": {"value": value, "unit": "levels/s", "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "levels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--method", default="bicgstab", choices=["bicgstab", "cgnr", "pcgs", "gsf"])
    ap.add_argument("--precond", default="strang", choices=["strang", "tchan", "none"])
    ap.add_argument("--cluster", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--true-res", action="store_true",
                    help="also compute the per-level true residual (an extra A application per level; "
                         "off by default: the paper's stopping rule uses the recurrence residual, P:922-924)")
    ap.add_argument("--warm", action="store_true", help="NEXT-3 warm start x0 = u^j")
    ap.add_argument("--hist-block", type=int, default=0,
                    help="NEXT-3 blocked history sum with this block length (0 = direct)")
    ap.add_argument("--pipelined", action="store_true",
                    help="NEXT-3 two-reduction BiCGSTAB (merged dot products)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch
    import torch.distributed as tdist

    from paper_1603_00279_b200 import tsf

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        tdist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            tdist.barrier()

    def allmax(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    def allsum(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
        return float(t.item())

    insts, scaling, units_total = build_instances(args.config, world, rank)
    n, M = insts[0].n, insts[0].M
    solver_kw = dict(method=args.method, precond=args.precond, cluster=args.cluster,
                     true_residual=args.true_res, x0_warm=args.warm, pipelined=args.pipelined,
                     hist_block=args.hist_block)
    stream = torch.cuda.Stream(dev)
    t_init0 = time.perf_counter()
    s = tsf.Solver(insts, stream=stream, **solver_kw)
    t_init = time.perf_counter() - t_init0
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)    # > 126 MB L2

    for _ in range(args.warmup):
        s.reset()
        s.solve()
        rc = s.sync()
        assert rc >= 0, rc
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    # batched configs under torchrun: the step ends after the NCCL all-gather of u^M and the
    # per-level statistics ("from the barrier before the first level to the end of
    # the gather"); u^M goes device to device (tsf_get_solutions into a CUDA tensor)
    do_gather = world > 1 and scaling == "strong"
    ubuf = torch.empty((len(insts), n), dtype=torch.float64, device=dev) if do_gather else None
    B_total = len(CONFIGS_ALL[args.config]()) if do_gather else 0

    def gather_results():
        from paper_1603_00279_b200 import dist as D
        s.solution_into(ubuf)
        it, rr, st = s.stats()
        with torch.cuda.stream(stream):
            res = D.gather(D.BatchResult(ubuf, it, rr, st), B_total, n, M, device=dev)
        return res

    ms, kms, gms = [], [], []
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            s.reset()
            with torch.cuda.stream(stream):
                flush.fill_(k & 0xFF)                 # flush L2 between timed steps
            torch.cuda.synchronize()
            barrier()
            torch.cuda.synchronize()
            ev[k][0].record(stream)
            s.solve()
            ev[k][1].record(stream)
            if do_gather:
                res = gather_results()
            ev[k][2].record(stream)
            torch.cuda.synchronize()
            barrier()
            ms.append(ev[k][0].elapsed_time(ev[k][2]))
            kms.append(ev[k][0].elapsed_time(ev[k][1]))
            gms.append(ev[k][1].elapsed_time(ev[k][2]))
            rc = s.sync()
            assert rc >= 0, rc
            if do_gather:
                assert res.u.shape == (B_total, n) and (res.status == 0).all()
    it_half, relres, status = s.stats()
    iters_local = float(it_half.sum()) / 2.0
    t_step_ms = allmax(statistics.mean(ms))
    total_s = allmax(sum(ms) / 1000.0)
    iters_job = allsum(iters_local)
    levels_job = units_total * M
    value = levels_job * args.steps / total_s
    iters_per_s = iters_job * args.steps / total_s
    src_units = 1 if insts[0].source == "table" else (4 if insts[0].source in ("mms3", "exa") else 0)
    abytes = algorithmic_bytes(n, M, it_half, args.method, src_units, args.hist_block)   # per launch, this rank
    kernel_s = statistics.mean(kms) / 1000.0       # the k_solve launch, CUDA events on its stream
    achieved = abytes / kernel_s / 1e9
    peak, peak_kind = peaks()
    # ncu DRAM bytes of the same launch (profiles/traffic.json, written by tools/ncu_traffic.py),
    # accepted only if captured with this exact libtsf.so
    traffic, traffic_note = None, "no capture"
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            ent = json.load(fh).get(traffic_key(args))
        if ent is None:
            traffic_note = "no capture for this workload"
        elif not isinstance(ent, dict):
            traffic_note = "stale capture (no library hash recorded)"
        elif ent.get("lib") != lib_hash():
            traffic_note = f"stale capture (lib {ent.get('lib')} != {lib_hash()})"
        else:
            traffic, traffic_note = float(ent["dram_bytes"]), f"ncu {ent.get('when', '')}"
    except Exception as e:  # noqa: BLE001
        traffic_note = f"unreadable: {e}"

    # ---- end to end through the public API: host inputs -> device, solve, results -> host
    e2e = None
    if not args.no_e2e:
        e_ms = []
        h2d = d2h = 0
        # the step's host inputs live in pinned host memory (the source tables are the bulk of
        # them: tsf_init DMAs them from the caller's buffer); pinned once, outside the timing
        pinned = []
        for inst in insts:
            if isinstance(getattr(inst, "f_table", None), np.ndarray):
                t = torch.from_numpy(np.ascontiguousarray(inst.f_table, dtype=np.float64)).pin_memory()
                pinned.append(t)
                inst.f_table = t.numpy()
        for k in range(max(1, min(args.steps, 3))):
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            s2 = tsf.Solver(insts, stream=stream, workspace=s.workspace, **solver_kw)
            s2.solve()
            u = s2.solutions()
            it2, rr2, st2 = s2.stats()
            t1 = time.perf_counter()
            h2d = s2.h2d_bytes
            d2h = u.nbytes + it2.nbytes + rr2.nbytes + st2.nbytes
            s2.close()
            e_ms.append(allmax(t1 - t0))
        e2e = {"value": levels_job / statistics.mean(e_ms), "unit": "levels/s",
               "h2d_bytes_per_step": int(allsum(h2d)), "d2h_bytes_per_step": int(allsum(d2h))}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, sample, _, threads = oracle_rate(args.config)
        cpu = {"value": v, "unit": "levels/s", "cores": threads, "kind": "oracle", "sample": sample}

    if rank == 0:
        info = s.info
        line = {
            "metric": METRIC, "value": value, "unit": "levels/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step_ms,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {**base_config(args), "instances": units_total, "cluster": info.cluster,
                       "exchange": ["local", "staged DSMEM push", "chunked via L2", "multi-pass via L2"][info.exchange],
                       "true_residual": bool(args.true_res), "x0_warm": bool(args.warm),
                       "pipelined": bool(args.pipelined), "hist_block": args.hist_block,
                       "l2": "flushed between steps (512 MiB write)",
                       "timed": "k_solve + level counter" + (" + NCCL all-gather of u^M and stats" if do_gather else "")},
            "krylov_iters_per_s": iters_per_s,
            "mean_iters_per_level": iters_job / levels_job,
            "init_s": t_init,
            "init_split_s": {"marshal_python": s.marshal_s, "tsf_init": s.init_s},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "k_solve (one launch = all M levels of the rank's batch)",
                         "kernel_ms": 1000.0 * kernel_s,
                         "algorithmic_bytes_per_launch": abytes,
                         "ncu_dram_gbs": (traffic / kernel_s / 1e9) if traffic else None,
                         "ncu_dram_frac": (traffic / kernel_s / 1e9 / peak) if traffic else None,
                         "traffic_source": traffic_note},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": (3 if do_gather else 2) * args.steps,
            "gather_ms_per_step": allmax(statistics.mean(gms)) if do_gather else None,
            "clocks": clk.summary(),
            "max_relres": float(relres.max()),
            "status_ok": bool((status == 0).all()),
        }
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
