"""Measurement-only native helpers for bench.py (not the product): the same-shape ideal
streaming kernel of SURVEY.md §8(d) item 6 (ceiling.cu -> libceiling.so, sm_100a)."""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "ceiling.cu")
LIB = os.path.join(_HERE, "libceiling.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                               "-shared", "-cudart", "static", "-Xcompiler", "-fPIC,-fvisibility=hidden",
                               "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} is missing: run __graft_entry__.build()")
        _lib = ctypes.CDLL(LIB)
        _lib.bsc_ldg.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                 ctypes.c_void_p]
        _lib.bsc_flat.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                  ctypes.c_void_p]
        _lib.bsc_ring.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    return _lib


# variants timed per stack; the ceiling is the fastest
VARIANTS = [("ldg", 4), ("ldg", 8), ("flat", 1), ("flat", 4), ("ring", 16384, 4, 2), ("ring", 32768, 3, 2)]


def launch(variant, in_ptr: int, n_in: int, out_ptr: int, n_out: int, stream: int) -> None:
    L = lib()
    if variant[0] == "ldg":
        rc = L.bsc_ldg(in_ptr, n_in, out_ptr, n_out, variant[1], stream)
    elif variant[0] == "flat":
        rc = L.bsc_flat(in_ptr, n_in, out_ptr, n_out, variant[1], stream)
    else:
        rc = L.bsc_ring(in_ptr, n_in, out_ptr, n_out, variant[1], variant[2], variant[3], stream)
    if rc:
        raise RuntimeError(f"ceiling kernel {variant}: CUDA error {rc}")
