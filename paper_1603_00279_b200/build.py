"""Build the sm_100a shared library libtsf.so in-tree (nvcc, FP64, -lineinfo).

Translation units are compiled in parallel (one per thread-block-cluster size holds the
solve-kernel instantiations), then linked with the static CUDA runtime.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libtsf.so")
PROF_LIB = os.path.join(LIBDIR, "libtsf_prof.so")
SOURCES = (["tsf_plan.cpp", "tsf_capi.cu"] + [f"tsf_solve_c{c}.cu" for c in (1, 2, 4, 8, 16)]
           + [f"tsf_solve_c{c}_{m}.cu" for c in (1, 2, 4, 8, 16) for m in ("bicgstab", "cgnr", "pcgs", "gsf")])
HEADERS = ["tsf_plan.h", "tsf_kernels.cuh", os.path.join("..", "..", "include", "tsf.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC"]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool, profile: bool = False, extra=(), variant: str = "",
             src_dir: str = CSRC) -> str:
    tag = ("_prof" if profile else "") + (f"_{variant}" if variant else "")
    obj = os.path.join(LIBDIR, os.path.splitext(src)[0] + tag + ".o")
    cmd = [NVCC, *FLAGS, *(["-DTSF_PROFILE"] if profile else []), *extra, "-c", os.path.join(src_dir, src), "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    return obj


def build(force: bool = False, verbose: bool = False, profile: bool = False, variant: str = "",
          defines: tuple = ()) -> str:
    """Build libtsf.so (or the section-timer variant libtsf_prof.so with profile=True, or a
    developer variant libtsf_<variant>.so compiled with extra -D defines)."""
    lib = PROF_LIB if profile else LIB
    if variant:
        lib = os.path.join(LIBDIR, f"libtsf_{variant}.so")
    if not force and not _stale(lib):
        return lib
    os.makedirs(LIBDIR, exist_ok=True)
    extra = [f"-D{d}" for d in defines]
    # compile from a snapshot of the sources so edits during a long build cannot mix versions
    # (kept under lib/, which travels to the GPU box, so ncu --import-source finds the lines)
    snap = os.path.join(LIBDIR, "snap_" + (os.path.basename(lib).replace(".so", "")))
    shutil.rmtree(snap, ignore_errors=True)
    if True:
        src_dir = os.path.join(snap, "pkg", "csrc")     # csrc/../../include resolves inside snap
        shutil.copytree(CSRC, src_dir)
        shutil.copytree(os.path.join(HERE, "..", "include"), os.path.join(snap, "include"))
        with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            objs = list(ex.map(lambda s: _compile(s, verbose, profile, extra, variant, src_dir), SOURCES))
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib + ".tmp", *objs])
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv, profile="--profile" in sys.argv))
