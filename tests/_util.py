"""Shared test helpers: golden-fixture loading and seeded random stack generation.

Nothing here computes the method: layers are built from ``synth`` descriptions; results
come from ``oracle`` (CPU) or the product binding (GPU).
"""
from __future__ import annotations

import glob
import json
import os
import random
import struct
from typing import List, Tuple

import numpy as np

import synth

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def layer_from_json(d) -> synth.Layer:
    k = d["kind"]
    if k == "batchnorm":
        return synth.batchnorm_explicit(d["gamma"], d["beta"], d["mean"], d["var"], d["eps"])
    if k in ("maxpool", "avgpool"):
        f = synth.maxpool if k == "maxpool" else synth.avgpool
        L = f(d["kernel"], d["stride"], d.get("padding", 0))
        if k == "avgpool":
            L.count_include_pad = d.get("count_include_pad", True)
        return L
    if k == "scale":
        return synth.scale(d["alpha"])
    if k == "add":
        return synth.add(d.get("operand", 1))
    return synth.Layer(k)


def hex_to_f32(h: str) -> float:
    return struct.unpack("<f", struct.pack("<I", int(h, 16)))[0]


def load_golden():
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN_DIR, "*.json"))):
        d = json.load(open(p))
        layers = [layer_from_json(x) for x in d["layers"]]
        x = np.array(d["input"], dtype=np.float32)
        ops = [np.array(o, dtype=np.float32) for o in d.get("operands", [])]
        if "expected_hex" in d:
            exp = np.vectorize(hex_to_f32)(np.array(d["expected_hex"])).astype(np.float32)
            exp = exp.reshape((1,) * (4 - exp.ndim) + exp.shape)
        else:
            exp = np.array(d["expected"], dtype=np.float32)
        out.append((os.path.basename(p)[:-5], layers, x, ops, exp, d["citation"]))
    return out


def bits(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def assert_bitexact(got: np.ndarray, ref: np.ndarray, ctx=""):
    assert got.shape == ref.shape, (got.shape, ref.shape, ctx)
    bad = np.nonzero(bits(got) != bits(ref))
    if bad[0].size:
        i = tuple(b[0] for b in bad)
        raise AssertionError(f"{ctx}: {bad[0].size} mismatches, first at {i}: "
                             f"got {got[i]!r} ref {ref[i]!r}")


# north_star tolerance for stacks with BN or avg-pool: |g - r| <= 1e-6 + 1e-5 |r|
ATOL, RTOL = 1e-6, 1e-5


def assert_close(got: np.ndarray, ref: np.ndarray, ctx=""):
    assert got.shape == ref.shape, (got.shape, ref.shape, ctx)
    g = got.astype(np.float64)
    r = ref.astype(np.float64)
    err = np.abs(g - r) - (ATOL + RTOL * np.abs(r))
    if np.any(err > 0) or not np.all(np.isfinite(g) == np.isfinite(r)):
        i = np.unravel_index(np.argmax(err), err.shape)
        raise AssertionError(f"{ctx}: tolerance exceeded at {i}: got {got[i]!r} ref {ref[i]!r}")


def needs_tolerance(layers) -> bool:
    """Bit-exact unless the stack has BatchNorm or AvgPool (north_star)."""
    return any(L.kind in ("batchnorm", "avgpool") for L in layers)


def check(got, ref, layers, ctx=""):
    if needs_tolerance(layers):
        assert_close(got, ref, ctx)
    else:
        assert_bitexact(got, ref, ctx)


def random_stack(rng: random.Random, shape, max_depth=8, max_pools=3,
                 allow_add=True, seed_base=900000) -> Tuple[List[synth.Layer], int]:
    """A random valid stack for `shape` (pool geometry kept valid via floor extents).
    Returns (layers, n_operands)."""
    N, C, H, W = shape
    layers: List[synth.Layer] = []
    n_ops = 0
    pools = 0
    depth = rng.randint(1, max_depth)
    for li in range(depth):
        choices = ["batchnorm", "relu", "copy", "scale"] + (["add"] if allow_add else [])
        if pools < max_pools:
            choices += ["maxpool", "avgpool", "maxpool"]
        k = rng.choice(choices)
        if k in ("maxpool", "avgpool"):
            kh = rng.randint(1, min(4, H + 0)) if H > 0 else 1
            kw = rng.randint(1, min(4, W + 0)) if W > 0 else 1
            ph = rng.randint(0, kh // 2)
            pw = rng.randint(0, kw // 2)
            sh = rng.randint(1, 3)
            sw = rng.randint(1, 3)
            if H + 2 * ph < kh or W + 2 * pw < kw:
                continue
            Ho = (H + 2 * ph - kh) // sh + 1
            Wo = (W + 2 * pw - kw) // sw + 1
            if Ho < 1 or Wo < 1:
                continue
            L = (synth.maxpool if k == "maxpool" else synth.avgpool)((kh, kw), (sh, sw), (ph, pw))
            if k == "avgpool":
                L.count_include_pad = rng.random() < 0.7
            layers.append(L)
            H, W = Ho, Wo
            pools += 1
        elif k == "batchnorm":
            layers.append(synth.batchnorm(C, seed_base + 100 * li, signed_gamma=rng.random() < 0.3))
        elif k == "scale":
            layers.append(synth.scale(rng.choice([0.5, -1.25, 1.5, 3.0, -0.75])))
        elif k == "add":
            n_ops += 1
            layers.append(synth.add(n_ops))
        else:
            layers.append(synth.Layer(k))
    if not layers:
        layers.append(synth.relu())
    return layers, n_ops


def make_inputs(layers, shape, n_ops, seed, shapes):
    """Stack input + ADD operands from the generator; `shapes` = per-layer input shapes."""
    x = synth.uniform_np(seed, int(np.prod(shape))).reshape(shape)
    ops = [None] * n_ops
    for L, s in zip(layers, shapes):
        if L.kind == "add":
            ops[L.operand - 1] = synth.uniform_np(seed + 7919 * L.operand,
                                                  int(np.prod(s))).reshape(s)
    return x, ops


def torch_definition(layers, x, ops=()):
    """The breadth-first definition (R1: each layer in fp64, rounded once to fp32 when stored)
    written with torch library ops on the GPU -- an independent check of EVERY element at full
    size (the oracle checks sampled images one by one above)."""
    import torch
    import torch.nn.functional as F
    t = x.double()
    for L in layers:
        if L.kind == "batchnorm":
            f = lambda a: torch.from_numpy(np.asarray(a, np.float64)).to(x.device).view(1, -1, 1, 1)
            t = (t - f(L.mean)) / torch.sqrt(f(L.var) + float(np.float32(L.eps))) * f(L.gamma) + f(L.beta)
        elif L.kind == "relu":
            t = torch.clamp_min(t, 0.0)
        elif L.kind == "maxpool":
            t = F.max_pool2d(t, L.kernel, L.stride, L.padding)
        elif L.kind == "avgpool":
            t = F.avg_pool2d(t, L.kernel, L.stride, L.padding, count_include_pad=L.count_include_pad)
        elif L.kind == "scale":
            t = t * float(L.alpha)
        elif L.kind == "add":
            t = t + ops[L.operand - 1].double()
        t = t.float().double()                      # stored as fp32 between layers
    return t.float()
