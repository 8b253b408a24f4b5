"""Thin Python binding of the C ABI in include/bs.h (argument marshalling only).

Every function has the C name and does nothing but convert arguments: every step of
the stack runs in libbrainslug.so's sm_100a kernels.  There is no CPU fallback: if the
library is missing, importing this package raises.

Layer descriptions are duck-typed: any object with the attributes ``kind`` ("batchnorm",
"relu", "maxpool", "avgpool", "copy", "scale", "add", "conv2d", "linear"), ``kernel``,
``stride``, ``padding`` ((h, w) tuples), ``count_include_pad``, ``eps``, ``gamma``,
``beta``, ``mean``, ``var`` (fp32 host arrays), ``alpha`` and ``operand`` works
(e.g. ``synth.Layer``), as does a ``bs_layer_desc`` instance.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import numpy as np

from . import _build

LIB_PATH = os.environ.get("BS_LIB", _build.LIB)   # BS_LIB: an alternative build of this library

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                      f"g.build()'` (nvcc, sm_100a). There is no fallback implementation.")

_lib = ctypes.CDLL(LIB_PATH)

# ----------------------------------------------------------------------------- C types
BS_OK, BS_ERR_INVALID_ARGUMENT, BS_ERR_VALIDATION, BS_ERR_PLANNING = 0, 2, 3, 4
BS_ERR_CUDA, BS_ERR_OUT_OF_MEMORY = 6, 7
BS_OP = {"batchnorm": 1, "relu": 2, "maxpool": 3, "avgpool": 4, "copy": 5, "scale": 6, "add": 7,
         "conv2d": 100, "linear": 101}
KERNEL_NAMES = {1: "ew_stream", 2: "pool_colwalk_spec", 3: "pool_colwalk_generic", 4: "pool_naive",
                5: "pool_colwalk_vec", 6: "pool_staged_tma",
                7: "sequence_staged_tma", 8: "pool_planes"}

_FP = ctypes.POINTER(ctypes.c_float)


class bs_layer_desc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("kernel_h", ctypes.c_int32), ("kernel_w", ctypes.c_int32),
                ("stride_h", ctypes.c_int32), ("stride_w", ctypes.c_int32), ("pad_h", ctypes.c_int32),
                ("pad_w", ctypes.c_int32), ("count_include_pad", ctypes.c_int32), ("eps", ctypes.c_float),
                ("gamma", _FP), ("beta", _FP), ("running_mean", _FP), ("running_var", _FP),
                ("alpha", ctypes.c_float), ("operand", ctypes.c_int32)]


class bs_shape(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("c", ctypes.c_int64), ("h", ctypes.c_int64), ("w", ctypes.c_int64)]

    def tuple(self):
        return (self.n, self.c, self.h, self.w)


class bs_plan_options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("host_only", ctypes.c_int32),
                ("max_steps_per_sequence", ctypes.c_int32), ("threads_per_block", ctypes.c_int32),
                ("force_rows_per_task", ctypes.c_int32), ("force_outputs_per_group", ctypes.c_int32),
                ("force_generic", ctypes.c_int32), ("force_tile_planes", ctypes.c_int32),
                ("force_stages", ctypes.c_int32), ("smem_budget_bytes", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 2)]


class bs_plan_info(ctypes.Structure):
    _fields_ = [("out", bs_shape), ("n_layers", ctypes.c_int32), ("n_ops", ctypes.c_int32),
                ("n_steps", ctypes.c_int32), ("n_sequences", ctypes.c_int32), ("n_launches", ctypes.c_int32),
                ("n_inputs", ctypes.c_int32), ("alg_bytes_read", ctypes.c_int64),
                ("alg_bytes_written", ctypes.c_int64), ("param_bytes", ctypes.c_int64),
                ("intermediate_bytes", ctypes.c_int64)]


class bs_launch_info(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("first_layer", ctypes.c_int32), ("last_layer", ctypes.c_int32),
                ("in_", bs_shape), ("out", bs_shape),
                ("pool_kh", ctypes.c_int32), ("pool_kw", ctypes.c_int32), ("pool_sh", ctypes.c_int32),
                ("pool_sw", ctypes.c_int32), ("pool_ph", ctypes.c_int32), ("pool_pw", ctypes.c_int32),
                ("n_prologue_ops", ctypes.c_int32), ("n_epilogue_ops", ctypes.c_int32),
                ("grid", ctypes.c_int32), ("block", ctypes.c_int32), ("groups_per_warp", ctypes.c_int32),
                ("outputs_per_group", ctypes.c_int32), ("rows_per_task", ctypes.c_int32),
                ("halo_rows", ctypes.c_int32), ("n_tasks", ctypes.c_int64),
                ("alg_bytes_read", ctypes.c_int64), ("alg_bytes_written", ctypes.c_int64),
                ("smem_bytes", ctypes.c_int32), ("tile_planes", ctypes.c_int32), ("tile_rows", ctypes.c_int32),
                ("stages", ctypes.c_int32)]


_P = ctypes.c_void_p
_lib.bs_plan_create.argtypes = [ctypes.POINTER(bs_layer_desc), ctypes.c_int32, bs_shape,
                                ctypes.POINTER(bs_plan_options), ctypes.POINTER(_P)]
_lib.bs_plan_query.argtypes = [_P, ctypes.POINTER(bs_plan_info)]
_lib.bs_plan_query_launch.argtypes = [_P, ctypes.c_int32, ctypes.POINTER(bs_launch_info)]
_lib.bs_execute.argtypes = [_P, _P, _P, _P]
_lib.bs_execute_ex.argtypes = [_P, ctypes.POINTER(_P), ctypes.c_int32, _P, _P]
_lib.bs_execute_host.argtypes = [_P, ctypes.POINTER(_P), ctypes.c_int32, _P, ctypes.POINTER(_P), _P,
                                 ctypes.c_int32, _P]
_lib.bs_execute_host_batch.argtypes = [ctypes.POINTER(_P), ctypes.c_int32, ctypes.POINTER(ctypes.POINTER(_P)),
                                       ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_P),
                                       ctypes.POINTER(ctypes.POINTER(_P)), ctypes.POINTER(_P), ctypes.c_int32, _P]
_lib.bs_graph_create.argtypes = [ctypes.POINTER(_P), ctypes.c_int32, ctypes.POINTER(ctypes.POINTER(_P)),
                                 ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_P), ctypes.POINTER(_P)]
_lib.bs_graph_create.restype = ctypes.c_int
_lib.bs_graph_launch.argtypes = [_P, _P]
_lib.bs_graph_launch.restype = ctypes.c_int
_lib.bs_graph_destroy.argtypes = [_P]
_lib.bs_graph_destroy.restype = None
_lib.bs_plan_destroy.argtypes = [_P]
_lib.bs_plan_destroy.restype = None
_lib.bs_last_error.restype = ctypes.c_char_p
_lib.bs_status_string.argtypes = [ctypes.c_int]
_lib.bs_status_string.restype = ctypes.c_char_p
_lib.bs_version.restype = ctypes.c_int32
for _f in ("bs_plan_create", "bs_plan_query", "bs_plan_query_launch", "bs_execute", "bs_execute_ex",
           "bs_execute_host", "bs_execute_host_batch"):
    getattr(_lib, _f).restype = ctypes.c_int


class BsError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.bs_last_error().decode()
        super().__init__(f"{where}: {_lib.bs_status_string(status).decode()}: {msg}")


def _check(st: int, where: str):
    if st != BS_OK:
        raise BsError(st, where)


# ----------------------------------------------------------------------------- marshalling
def _fp(a):
    return a.ctypes.data_as(_FP) if a is not None else _FP()


def _ptr(t) -> int:
    """Device/host address of a torch tensor, numpy array or integer."""
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _desc(layers):
    keep = []
    arr = (bs_layer_desc * len(layers))()
    for i, L in enumerate(layers):
        if isinstance(L, bs_layer_desc):
            arr[i] = L
            continue
        d = arr[i]
        d.kind = BS_OP[L.kind]
        d.kernel_h, d.kernel_w = getattr(L, "kernel", (1, 1))
        d.stride_h, d.stride_w = getattr(L, "stride", (1, 1))
        d.pad_h, d.pad_w = getattr(L, "padding", (0, 0))
        d.count_include_pad = 1 if getattr(L, "count_include_pad", True) else 0
        d.eps = getattr(L, "eps", 1e-5)
        for cf, pf in (("gamma", "gamma"), ("beta", "beta"), ("running_mean", "mean"), ("running_var", "var")):
            v = getattr(L, pf, None)
            if v is not None:
                v = np.ascontiguousarray(v, dtype=np.float32)
                keep.append(v)
            setattr(d, cf, _fp(v))
        d.alpha = getattr(L, "alpha", 1.0)
        d.operand = getattr(L, "operand", 0)
    return arr, keep


class Plan:
    """Owns a bs_plan* (bs_plan_destroy on close/GC)."""

    def __init__(self, handle: int):
        self.handle = handle

    def close(self):
        if self.handle:
            _lib.bs_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def _as_parameter_(self):
        return _P(self.handle)


# ----------------------------------------------------------------------------- ABI functions
def bs_plan_create(layers: Sequence, input_shape, opts: Optional[dict] = None) -> Plan:
    arr, keep = _desc(layers)
    o = None
    if opts is not None:
        o = bs_plan_options()
        o.device = opts.get("device", -1)
        for k in ("host_only", "max_steps_per_sequence", "threads_per_block", "force_rows_per_task",
                  "force_outputs_per_group", "force_generic", "force_tile_planes", "force_stages",
                  "smem_budget_bytes"):
            setattr(o, k, int(opts.get(k, 0)))
    h = _P()
    st = _lib.bs_plan_create(arr, len(layers), bs_shape(*[int(v) for v in input_shape]),
                             ctypes.byref(o) if o is not None else None, ctypes.byref(h))
    _check(st, "bs_plan_create")
    return Plan(h.value)


def bs_plan_query(plan: Plan) -> dict:
    i = bs_plan_info()
    _check(_lib.bs_plan_query(plan, ctypes.byref(i)), "bs_plan_query")
    d = {k: getattr(i, k) for k, _ in bs_plan_info._fields_}
    d["out"] = i.out.tuple()
    return d


def bs_plan_query_launch(plan: Plan, index: int) -> dict:
    i = bs_launch_info()
    _check(_lib.bs_plan_query_launch(plan, index, ctypes.byref(i)), "bs_plan_query_launch")
    d = {k: getattr(i, k) for k, _ in bs_launch_info._fields_}
    d["in"] = i.in_.tuple()
    del d["in_"]
    d["out"] = i.out.tuple()
    d["kernel_name"] = KERNEL_NAMES.get(i.kernel, "?")
    return d


def bs_execute(plan: Plan, inp, out, stream=None) -> None:
    _check(_lib.bs_execute(plan, _ptr(inp), _ptr(out), _stream(stream)), "bs_execute")


def bs_execute_ex(plan: Plan, inputs: Sequence, out, stream=None) -> None:
    arr = (_P * len(inputs))(*[_ptr(t) for t in inputs])
    _check(_lib.bs_execute_ex(plan, arr, len(inputs), _ptr(out), _stream(stream)), "bs_execute_ex")


def bs_execute_host(plan: Plan, h_inputs: Sequence, h_out, d_inputs: Sequence, d_out, n_chunks: int = 0,
                    stream=None) -> None:
    hi = (_P * len(h_inputs))(*[_ptr(t) for t in h_inputs])
    di = (_P * len(d_inputs))(*[_ptr(t) for t in d_inputs])
    _check(_lib.bs_execute_host(plan, hi, len(h_inputs), _ptr(h_out), di, _ptr(d_out), int(n_chunks),
                                _stream(stream)), "bs_execute_host")


def bs_execute_host_batch(plans: Sequence, h_inputs: Sequence, h_outs: Sequence, d_inputs: Sequence,
                          d_outs: Sequence, n_chunks: int = 0, stream=None) -> None:
    """bs_execute_host for several executions, pipelined across them (include/bs.h): per
    execution i, plans[i], h_inputs[i] (a sequence), h_outs[i], d_inputs[i] (a sequence), d_outs[i]."""
    n = len(plans)
    pl = (_P * n)(*[p.handle if isinstance(p, Plan) else p for p in plans])
    hi_rows = [(_P * len(r))(*[_ptr(t) for t in r]) for r in h_inputs]
    di_rows = [(_P * len(r))(*[_ptr(t) for t in r]) for r in d_inputs]
    hi = (ctypes.POINTER(_P) * n)(*[ctypes.cast(r, ctypes.POINTER(_P)) for r in hi_rows])
    di = (ctypes.POINTER(_P) * n)(*[ctypes.cast(r, ctypes.POINTER(_P)) for r in di_rows])
    ni = (ctypes.c_int32 * n)(*[len(r) for r in h_inputs])
    ho = (_P * n)(*[_ptr(t) for t in h_outs])
    do = (_P * n)(*[_ptr(t) for t in d_outs])
    _check(_lib.bs_execute_host_batch(pl, n, hi, ni, ho, di, do, int(n_chunks), _stream(stream)),
           "bs_execute_host_batch")


def bs_plan_destroy(plan: Plan) -> None:
    plan.close()


class Graph:
    """Owns a bs_graph* (bs_graph_destroy on close/GC); keeps its plans alive."""

    def __init__(self, handle: int, plans):
        self.handle = handle
        self._plans = list(plans)

    def close(self):
        if self.handle:
            _lib.bs_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def _as_parameter_(self):
        return _P(self.handle)


def bs_graph_create(executions: Sequence) -> Graph:
    """executions: [(plan, [input, operand, ...], out), ...] -- captured in order as one CUDA graph."""
    n = len(executions)
    plans = (_P * n)(*[_P(e[0].handle) for e in executions])
    arrs = [(_P * len(e[1]))(*[_ptr(t) for t in e[1]]) for e in executions]
    ins = (ctypes.POINTER(_P) * n)(*[ctypes.cast(a, ctypes.POINTER(_P)) for a in arrs])
    nin = (ctypes.c_int32 * n)(*[len(e[1]) for e in executions])
    outs = (_P * n)(*[_ptr(e[2]) for e in executions])
    h = _P()
    _check(_lib.bs_graph_create(plans, n, ins, nin, outs, ctypes.byref(h)), "bs_graph_create")
    return Graph(h.value, [e[0] for e in executions])


def bs_graph_launch(graph: Graph, stream=None) -> None:
    _check(_lib.bs_graph_launch(graph, _stream(stream)), "bs_graph_launch")


def bs_graph_destroy(graph: Graph) -> None:
    graph.close()


def bs_last_error() -> str:
    return _lib.bs_last_error().decode()


def bs_status_string(status: int) -> str:
    return _lib.bs_status_string(status).decode()


def bs_version() -> int:
    return _lib.bs_version()


__all__ = ["bs_plan_create", "bs_plan_query", "bs_plan_query_launch", "bs_execute", "bs_execute_ex",
           "bs_execute_host", "bs_execute_host_batch", "bs_plan_destroy", "bs_last_error", "bs_status_string", "bs_version", "BsError",
           "Plan", "bs_layer_desc", "BS_OP", "KERNEL_NAMES", "LIB_PATH"]
