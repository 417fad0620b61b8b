"""Python API over the C-ABI (include/tsf.h): argument marshalling only.

Every step of the per-level solve runs in the sm_100a kernels of libtsf.so; PyTorch only
provides the device workspace and the CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import time
from typing import Sequence

import numpy as np

from . import _lib as L
from .inputs import Instance, manufactured_basis, manufactured_scal

METHODS = {"bicgstab": L.BICGSTAB, "cgnr": L.CGNR, "pcgs": L.PCGS, "gsf": L.GSF}
PRECONDS = {"strang": L.STRANG, "tchan": L.TCHAN, "none": L.NOPREC}


def _pd(a: np.ndarray):
    return a.ctypes.data_as(L.PD)


def _base_problem(inst: Instance) -> L.TsfProblem:
    p = L.TsfProblem()
    p.alpha, p.beta, p.n, p.M = inst.alpha, inst.beta, inst.n, inst.M
    p.a, p.b, p.T = inst.a, inst.b, inst.T
    return p


def sample_points(inst: Instance):
    """Interior nodes x[n] and level times t_{j+sigma}[M] as defined by the library."""
    lib = L.load()
    p = _base_problem(inst)
    x = np.zeros(inst.n)
    t = np.zeros(inst.M)
    L.check(lib.tsf_sample_points(C.byref(p), _pd(x), _pd(t)), "tsf_sample_points")
    return x, t


def marshal(instances: Sequence[Instance]):
    """Build the TsfProblem array (and keep the host arrays alive alongside)."""
    probs = (L.TsfProblem * len(instances))()
    keep = []
    for k, inst in enumerate(instances):
        x, t = sample_points(inst)
        p = probs[k]
        p.alpha, p.beta, p.n, p.M = inst.alpha, inst.beta, inst.n, inst.M
        p.a, p.b, p.T = inst.a, inst.b, inst.T
        arrs = {}
        for name, fn in (("gamma_t", inst.gamma), ("dplus_t", inst.dplus), ("dminus_t", inst.dminus)):
            arrs[name] = np.ascontiguousarray(np.broadcast_to(fn(t), t.shape), dtype=np.float64)
            setattr(p, name, _pd(arrs[name]))
        arrs["phi"] = np.ascontiguousarray(np.broadcast_to(inst.phi(x), x.shape), dtype=np.float64)
        p.phi = _pd(arrs["phi"])
        if inst.source in ("mms3", "exa"):
            arrs["basis"] = np.ascontiguousarray(manufactured_basis(x, inst.beta))
            arrs["scal"] = np.ascontiguousarray(manufactured_scal(t, inst.alpha, inst.gamma, inst.dplus,
                                                                  inst.dminus, inst.source))
            p.src_kind, p.K = L.SRC_SEPARABLE, 4
            p.basis, p.scal = _pd(arrs["basis"]), _pd(arrs["scal"])
        elif inst.source == "table" and hasattr(inst.f_table, "data_ptr"):
            ft = inst.f_table                      # device tensor: borrowed, natural order
            assert ft.is_cuda and ft.is_contiguous() and tuple(ft.shape) == (inst.M, inst.n)
            assert str(ft.dtype) == "torch.float64"
            arrs["f_dev"] = ft                     # keep the tensor alive with the handle
            p.src_kind, p.f_table, p.f_table_on_device = L.SRC_TABLE, C.cast(C.c_void_p(ft.data_ptr()), L.PD), 1
        elif inst.source == "table":
            arrs["f"] = np.ascontiguousarray(inst.f_table, dtype=np.float64)
            assert arrs["f"].shape == (inst.M, inst.n)
            p.src_kind, p.f_table = L.SRC_TABLE, _pd(arrs["f"])
        elif inst.source == "callback":
            fn = inst.f_callback                   # python f(x: ndarray, t: float) -> ndarray

            def _cb(xp, nn, t, outp, _ctx, fn=fn):
                xa = np.ctypeslib.as_array(xp, shape=(nn,))
                np.ctypeslib.as_array(outp, shape=(nn,))[:] = fn(xa, t)
            arrs["cb"] = L.SRC_CB(_cb)
            p.src_kind, p.f_cb = L.SRC_CALLBACK, arrs["cb"]
        elif inst.source == "zero":
            p.src_kind = L.SRC_ZERO
        else:
            raise ValueError(inst.source)
        keep.append(arrs)
    return probs, keep


def make_solver_struct(method="bicgstab", precond="strang", tol=1e-12, maxit=None, cluster=0,
                       x0_warm=False, true_residual=True, pipelined=False, hist_block=0):
    s = L.TsfSolver()
    s.method = METHODS[method]
    s.precond = PRECONDS[precond]
    s.tol = tol
    s.maxit = maxit if maxit is not None else (5000 if method == "cgnr" else 1000)
    s.cluster = cluster
    s.x0_warm = int(bool(x0_warm))
    s.true_residual = int(bool(true_residual))
    s.pipelined = int(bool(pipelined))
    s.hist_block = int(hist_block)
    return s


def plan(instances: Sequence[Instance], **solver_kw) -> L.TsfPlanInfo:
    lib = L.load()
    probs, _keep = marshal(instances)
    s = make_solver_struct(**solver_kw)
    info = L.TsfPlanInfo()
    L.check(lib.tsf_plan(probs, len(instances), C.byref(s), C.byref(info)), "tsf_plan")
    return info


class Solver:
    """A batch of instances (same n, M) solved level by level on one GPU."""

    def __init__(self, instances: Sequence[Instance], method="bicgstab", precond="strang",
                 tol=1e-12, maxit=None, cluster=0, device=None, stream=None, workspace=None,
                 x0_warm=False, true_residual=True, pipelined=False, hist_block=0):
        import torch
        self.lib = L.load()
        self.instances = list(instances)
        self.B = len(self.instances)
        self.n, self.M = self.instances[0].n, self.instances[0].M
        t0 = time.perf_counter()
        probs, keep = marshal(self.instances)
        self.marshal_s = time.perf_counter() - t0      # host arrays from the Instance specs (Python)
        self.h2d_bytes = sum(a.nbytes for arrs in keep for a in arrs.values() if isinstance(a, np.ndarray))
        self._borrowed = [arrs["f_dev"] for arrs in keep if "f_dev" in arrs]
        self._solver = make_solver_struct(method, precond, tol, maxit, cluster, x0_warm, true_residual,
                                          pipelined, hist_block)
        info = L.TsfPlanInfo()
        L.check(self.lib.tsf_plan(probs, self.B, C.byref(self._solver), C.byref(info)), "tsf_plan")
        self.info = info
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.device = dev
        if workspace is not None and workspace.numel() >= int(info.workspace_bytes):
            self.workspace = workspace
        else:
            self.workspace = torch.empty(int(info.workspace_bytes), dtype=torch.uint8, device=dev)
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        if self.stream != torch.cuda.current_stream(dev):
            # allocated on the current stream, used on self.stream: keep the caching allocator
            # from reusing it while the handle's kernels may still run
            self.workspace.record_stream(self.stream)
        h = C.c_void_p()
        t0 = time.perf_counter()
        L.check(self.lib.tsf_init(probs, self.B, C.byref(self._solver),
                                  C.c_void_p(self.workspace.data_ptr()), C.c_size_t(int(info.workspace_bytes)),
                                  dev.index, C.c_void_p(self.stream.cuda_stream), C.byref(h)), "tsf_init")
        self.init_s = time.perf_counter() - t0         # the C-ABI tsf_init call (uploads + setup kernels)
        self.h = h
        del keep

    # ---- time marching
    def step(self):
        L.check(self.lib.tsf_step(self.h), "tsf_step")

    def solve(self):
        L.check(self.lib.tsf_solve(self.h), "tsf_solve")

    def reset(self):
        L.check(self.lib.tsf_reset(self.h), "tsf_reset")

    def sync(self) -> int:
        return L.check(self.lib.tsf_sync(self.h), "tsf_sync")

    @property
    def level(self) -> int:
        return int(self.lib.tsf_level(self.h))

    def solution(self, inst: int = 0) -> np.ndarray:
        out = np.zeros(self.n)
        L.check(self.lib.tsf_get_solution(self.h, inst, _pd(out), 0), "tsf_get_solution")
        return out

    def solutions(self) -> np.ndarray:
        out = np.zeros((self.B, self.n))
        L.check(self.lib.tsf_get_solutions(self.h, _pd(out), 0), "tsf_get_solutions")
        return out

    def solution_into(self, out_tensor):
        """Copy all u^j into a device tensor (float64, [B][n])."""
        L.check(self.lib.tsf_get_solutions(self.h, C.cast(C.c_void_p(out_tensor.data_ptr()), L.PD), 1),
                "tsf_get_solutions")

    def stats(self):
        it = np.zeros((self.B, self.M), dtype=np.int32)
        rr = np.zeros((self.B, self.M))
        st = np.zeros((self.B, self.M), dtype=np.int32)
        L.check(self.lib.tsf_get_stats(self.h, it.ctypes.data_as(C.POINTER(C.c_int32)), _pd(rr),
                                       st.ctypes.data_as(C.POINTER(C.c_int32))), "tsf_get_stats")
        return it, rr, st

    def true_residuals(self) -> np.ndarray:
        """||g - A u^{j+1}|| / ||g|| per level ([B][M]; 0 where not computed)."""
        out = np.zeros((self.B, self.M))
        L.check(self.lib.tsf_get_true_residuals(self.h, _pd(out)), "tsf_get_true_residuals")
        return out

    def close(self):
        if getattr(self, "h", None):
            self.lib.tsf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- test hooks
    def debug_apply(self, inst: int, j: int, which: int, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.n)
        L.check(self.lib.tsf_debug_apply(self.h, inst, j, which, _pd(x), _pd(y)), "tsf_debug_apply")
        return y

    def debug_apply_bench(self, inst: int = 0, j: int = 0, reps: int = 200) -> float:
        """Milliseconds of one launch of `reps` alternating P^{-1} / A applications."""
        ms = C.c_float(0.0)
        L.check(self.lib.tsf_debug_apply_bench(self.h, inst, j, reps, C.byref(ms)), "tsf_debug_apply_bench")
        return ms.value

    def debug_helper_state(self) -> np.ndarray:
        out = np.zeros(8, dtype=np.int64)
        L.check(self.lib.tsf_debug_helper_state(self.h, out.ctypes.data_as(C.POINTER(C.c_int64))),
                "tsf_debug_helper_state")
        return out

    def debug_spectra(self, inst: int, j: int):
        la = np.zeros(2 * (self.n + 1))
        lp = np.zeros(2 * (self.n // 2 + 1))
        L.check(self.lib.tsf_debug_spectra(self.h, inst, j, _pd(la), _pd(lp)), "tsf_debug_spectra")
        return la.view(np.complex128), lp.view(np.complex128)

    def debug_rhs(self, inst: int = 0) -> np.ndarray:
        out = np.zeros(self.n)
        L.check(self.lib.tsf_debug_rhs(self.h, inst, _pd(out)), "tsf_debug_rhs")
        return out

    def debug_set_history(self, inst: int, U: np.ndarray):
        U = np.ascontiguousarray(U, dtype=np.float64)
        j = U.shape[0] - 1
        L.check(self.lib.tsf_debug_set_history(self.h, inst, j, _pd(U)), "tsf_debug_set_history")


OP_A, OP_B, OP_AT, OP_PINV, OP_PTINV = 0, 1, 2, 3, 4


def debug_fft_tables(Lc: int):
    lib = L.load()
    plan = np.zeros(32, dtype=np.int32)
    S = C.c_int32()
    perm = np.zeros(Lc, dtype=np.int32)
    tw = np.zeros(2 * Lc + 8, dtype=np.int32)
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
    L.check(lib.tsf_debug_fft_tables(Lc, ip(plan), C.byref(S), ip(perm), ip(tw)), "tsf_debug_fft_tables")
    return plan[:S.value].tolist(), perm, tw


def debug_local_fft(x: np.ndarray, inverse: bool = False) -> np.ndarray:
    lib = L.load()
    x = np.ascontiguousarray(x, dtype=np.complex128)
    xr = x.view(np.float64)
    y = np.zeros_like(xr)
    L.check(lib.tsf_debug_local_fft(x.size, _pd(xr), _pd(y), int(inverse)), "tsf_debug_local_fft")
    return y.view(np.complex128)


def debug_weights(beta: float, K: int):
    lib = L.load()
    g = np.zeros(K + 1)
    w = np.zeros(K + 1)
    L.check(lib.tsf_debug_weights(beta, K, _pd(g), _pd(w)), "tsf_debug_weights")
    return g, w
