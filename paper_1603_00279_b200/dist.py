"""Batched multi-GPU mode: shard independent instances over ranks, gather results.

Instances are independent (one TSFCDE problem each), so the data path has no collective:
rank k solves the contiguous block shard(B, W, k) on its own GPU.  The only collective is
the final gather of u^M and the per-level statistics (NCCL over NVLink on GPUs, gloo in
the CPU tests).  Time marching itself is sequential and never split.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np


def shard(B: int, world: int, rank: int) -> range:
    """Contiguous block of instance indices owned by `rank` (sizes differ by at most 1)."""
    base, extra = divmod(B, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


@dataclass
class BatchResult:
    u: np.ndarray          # [B][n] u^M (or the current level's solution)
    iters_half: np.ndarray  # [B][M]
    relres: np.ndarray     # [B][M]
    status: np.ndarray     # [B][M]


def collective_device(device=None):
    """Device of the gather buffers: NCCL needs CUDA tensors (the current device), gloo CPU."""
    import torch
    import torch.distributed as dist
    if device is not None:
        return torch.device(device)
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather(local: BatchResult, B: int, n: int, M: int, device=None) -> BatchResult:
    """All-gather the per-rank blocks into full [B] arrays on every rank (rank order).
    Blocks may be numpy arrays or torch tensors (a CUDA u^M goes device to device)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    device = collective_device(device)
    maxb = max(len(shard(B, world, r)) for r in range(world))
    nb = local.u.shape[0]

    def pad(a, dtype):
        t = torch.zeros((maxb,) + tuple(a.shape[1:]), dtype=dtype, device=device)
        if nb:
            t[:nb] = torch.as_tensor(a, dtype=dtype, device=device)
        return t

    parts = {"u": (local.u, torch.float64), "it": (local.iters_half, torch.int32),
             "rr": (local.relres, torch.float64), "st": (local.status, torch.int32)}
    out = {}
    for key, (arr, dt) in parts.items():
        mine = pad(arr, dt)
        bufs = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(bufs, mine)
        rows = [bufs[r][: len(shard(B, world, r))].cpu().numpy() for r in range(world)]
        out[key] = np.concatenate(rows, axis=0)
    return BatchResult(out["u"], out["it"], out["rr"], out["st"])


def solve_local(instances: Sequence, **solver_kw) -> BatchResult:
    """Run the CUDA solver on this rank's instances (all M levels) and fetch the results."""
    from .tsf import Solver
    s = Solver(instances, **solver_kw)
    s.solve()
    rc = s.sync()
    if rc < 0:
        raise RuntimeError(f"tsf_sync returned {rc}")
    it, rr, st = s.stats()
    res = BatchResult(s.solutions(), it, rr, st)
    s.close()
    return res


def solve_batch(instances: Sequence, rank: int, world: int,
                local_solver: Callable[[Sequence], BatchResult] | None = None,
                device=None, **solver_kw) -> BatchResult:
    """Shard `instances` over `world` ranks, solve locally, gather everywhere."""
    B = len(instances)
    n, M = instances[0].n, instances[0].M
    mine = [instances[i] for i in shard(B, world, rank)]
    if local_solver is None:
        local = solve_local(mine, **solver_kw) if mine else BatchResult(
            np.zeros((0, n)), np.zeros((0, M), np.int32), np.zeros((0, M)), np.zeros((0, M), np.int32))
    else:
        local = local_solver(mine)
    if world == 1:
        return local
    return gather(local, B, n, M, device=device)
