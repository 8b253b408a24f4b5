"""ctypes wrapper of the CPU oracle (oracle/bs_oracle.c).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module and
this module never imports the product package (it translates ``synth.Layer`` into its
own ``or_layer`` struct).  See bs_oracle.c's header for what is computed and why.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bs_oracle.c")
_HDR = os.path.join(_HERE, "bs_oracle.h")
LIB_PATH = os.path.join(_HERE, "liboracle.so")

# compile flags of the oracle: no FMA contraction, no fast-math, no SIMD intrinsics
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c99"]

_KIND = {"batchnorm": 11, "relu": 12, "maxpool": 13, "avgpool": 14, "copy": 15, "scale": 16,
         "add": 17, "conv2d": 90, "linear": 91}
OK, ERR_INVALID, ERR_UNSUPPORTED, ERR_NOMEM = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__({1: "invalid stack", 2: "unsupported layer kind", 3: "out of memory"}
                         .get(code, f"oracle error {code}"))
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (also called by __graft_entry__.build())."""
    stale = (not os.path.exists(LIB_PATH) or
             os.path.getmtime(LIB_PATH) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


class _OrLayer(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("kh", ctypes.c_int32), ("kw", ctypes.c_int32),
                ("sh", ctypes.c_int32), ("sw", ctypes.c_int32), ("ph", ctypes.c_int32),
                ("pw", ctypes.c_int32), ("count_include_pad", ctypes.c_int32),
                ("eps", ctypes.c_float),
                ("gamma", ctypes.POINTER(ctypes.c_float)), ("beta", ctypes.POINTER(ctypes.c_float)),
                ("mean", ctypes.POINTER(ctypes.c_float)), ("var", ctypes.POINTER(ctypes.c_float)),
                ("alpha", ctypes.c_float), ("operand", ctypes.c_int32)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        I64P = ctypes.POINTER(ctypes.c_int64)
        FP = ctypes.POINTER(ctypes.c_float)
        lib.oracle_layer_shapes.argtypes = [ctypes.POINTER(_OrLayer), ctypes.c_int, I64P, ctypes.c_int, I64P]
        lib.oracle_run_bf.argtypes = [ctypes.POINTER(_OrLayer), ctypes.c_int, I64P, FP,
                                      ctypes.POINTER(FP), ctypes.c_int, FP]
        lib.oracle_run_df.argtypes = [ctypes.POINTER(_OrLayer), ctypes.c_int, I64P, FP,
                                      ctypes.POINTER(FP), ctypes.c_int, ctypes.c_int64,
                                      ctypes.c_int64, FP]
        _lib = lib
    return _lib


def _fptr(a: Optional[np.ndarray]):
    if a is None:
        return ctypes.POINTER(ctypes.c_float)()
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _marshal(layers) -> Tuple[ctypes.Array, list]:
    keep = []
    arr = (_OrLayer * len(layers))()
    for i, L in enumerate(layers):
        o = arr[i]
        o.kind = _KIND[L.kind]
        o.kh, o.kw = L.kernel
        o.sh, o.sw = L.stride
        o.ph, o.pw = L.padding
        o.count_include_pad = 1 if L.count_include_pad else 0
        o.eps = L.eps
        for f in ("gamma", "beta", "mean", "var"):
            v = getattr(L, f)
            if v is not None:
                v = np.ascontiguousarray(v, dtype=np.float32)
                keep.append(v)
            setattr(o, f, _fptr(v))
        o.alpha = L.alpha
        o.operand = L.operand
    return arr, keep


def layer_shapes(layers, in_shape, n_operands: int = 0) -> List[Tuple[int, int, int, int]]:
    """Input shape of every layer, then the stack output shape (raises OracleError)."""
    lib = _load()
    arr, keep = _marshal(layers)
    ins = (ctypes.c_int64 * 4)(*in_shape)
    out = (ctypes.c_int64 * (4 * (len(layers) + 1)))()
    st = lib.oracle_layer_shapes(arr, len(layers), ins, n_operands, out)
    if st != OK:
        raise OracleError(st)
    return [tuple(out[4 * i:4 * i + 4]) for i in range(len(layers) + 1)]


def _run(fn, layers, x: np.ndarray, operands: Sequence[np.ndarray], *extra) -> np.ndarray:
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.float32)
    assert x.ndim == 4
    ops = [np.ascontiguousarray(o, dtype=np.float32) for o in operands]
    shapes = layer_shapes(layers, x.shape, len(ops))
    for L, s in zip(layers, shapes):
        if L.kind == "add":
            assert ops[L.operand - 1].shape == tuple(s), (ops[L.operand - 1].shape, s)
    y = np.empty(shapes[-1], dtype=np.float32)
    arr, keep = _marshal(layers)
    FP = ctypes.POINTER(ctypes.c_float)
    oparr = (FP * max(1, len(ops)))(*[_fptr(o) for o in ops])
    ins = (ctypes.c_int64 * 4)(*x.shape)
    st = getattr(lib, fn)(arr, len(layers), ins, _fptr(x), oparr, len(ops), *extra, _fptr(y))
    if st != OK:
        raise OracleError(st)
    return y


def run_bf(layers, x: np.ndarray, operands: Sequence[np.ndarray] = ()) -> np.ndarray:
    """Breadth-first (layer-by-layer) result -- the definition the method must reach."""
    return _run("oracle_run_bf", layers, x, operands)


def run_df(layers, x: np.ndarray, operands: Sequence[np.ndarray] = (), tile=(0, 0)) -> np.ndarray:
    """Depth-first CPU twin over output tiles of tile[0] x tile[1] (0 = whole plane)."""
    return _run("oracle_run_df", layers, x, operands, int(tile[0]), int(tile[1]))
