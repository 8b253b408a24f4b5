"""Ahead-of-time build of libbrainslug.so for sm_100a (nvcc; no JIT, no torch extension).

Used by ``__graft_entry__.build()`` and by the test fixtures.  The library is built
in-tree so it travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libbrainslug.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
OBJ_DIR = os.path.join(PKG, "build")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "-shared", "-cudart", "static",
    # explicit-rounding intrinsics are used on the hot path; keep the rest IEEE as well
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "bs.h"), __file__]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def _compile(src: str, obj: str, verbose: bool) -> None:
    flags = [f for f in NVCC_FLAGS if f not in ("-shared",)]
    cmd = [NVCC, *flags, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit (in parallel) and link libbrainslug.so."""
    if not (force or stale()):
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJ_DIR, exist_ok=True)
    headers = [p for p in deps() if p.endswith((".h", ".cuh", ".py"))]
    newest_hdr = max(os.path.getmtime(p) for p in headers)
    jobs, objs = [], []
    for src in sources():
        obj = os.path.join(OBJ_DIR, os.path.basename(src) + f".{os.getpid()}.o")
        final = os.path.join(OBJ_DIR, os.path.basename(src) + ".o")
        objs.append(final)
        if force or not os.path.exists(final) or os.path.getmtime(final) < max(os.path.getmtime(src), newest_hdr):
            jobs.append((src, obj, final))
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for f in [ex.submit(_compile, s_, o_, verbose) for s_, o_, _ in jobs]:
            f.result()
    for _, o_, fin in jobs:
        os.replace(o_, fin)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           "-Xcompiler", "-fPIC", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
