"""In-tree build of libtnb.so (nvcc, sm_100a only).

``python -m paper_2103_03074_b200.build`` or ``__graft_entry__.build()``.
Objects are compiled in parallel and linked into
``paper_2103_03074_b200/libtnb.so`` (git-ignored, travels with gpurun).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtnb.so")
SOURCES = ["kernels.cu", "gemm_tc.cu", "program.cu", "analytics.cu", "collective.cu", "tnb_api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "-Wno-deprecated-gpu-targets", "-diag-suppress", "177"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libtnb.so")


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    deps = [src, os.path.join(CSRC, "tnb_internal.h"),
            os.path.join(PKG, "..", "include", "tnb.h")]
    return any(os.path.getmtime(d) > os.path.getmtime(obj) for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    nvcc = _nvcc()
    objdir = os.path.join(PKG, "_build")
    os.makedirs(objdir, exist_ok=True)
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        if force or _stale(o, s):
            jobs.append([nvcc, *ARCH, *FLAGS, "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, file=sys.stderr)

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(objdir, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or not os.path.exists(LIB):
        tmp = LIB + ".tmp"
        run([nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"])
        os.replace(tmp, LIB)
    # host-side plan optimiser (g++)
    from .treeopt import build as build_plan

    build_plan(force=force)
    build_io(force=force)
    return LIB


IO_SRC = os.path.join(CSRC, "tsv_format.cpp")
IO_LIB = os.path.join(PKG, "libtnbio.so")


def build_io(force: bool = False) -> str:
    """g++ build of libtnbio.so: the host TSV row formatter (io.py)."""
    if force or not os.path.exists(IO_LIB) or os.path.getmtime(IO_SRC) > os.path.getmtime(IO_LIB):
        tmp = IO_LIB + ".tmp"
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", "-Wall",
               "-ffp-contract=off", "-fno-builtin", IO_SRC, "-o", tmp]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"g++ failed ({' '.join(cmd)}):\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, IO_LIB)
    return IO_LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
