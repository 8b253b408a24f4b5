"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no BatchNorm, ReLU, pooling, folding,
tiling).  It only provides

* a counter-form SplitMix64 generator (SURVEY.md §8(d) "Value distributions"; SPEC.md
  S:L42-50 names SplitMix64 with the ``(upper24 / 2^23) - 1`` mapping), implemented
  twice -- numpy (host) and torch integer ops (any device) -- which must agree bit for
  bit (tests/test_synth.py);
* a neutral, library-independent description of a layer stack (``Layer``) that both
  the oracle wrapper (``oracle/``) and the product binding translate into their own
  C structs;
* the stack shapes of the paper's networks used by BASELINE.json's configs
  (SURVEY.md §8(d) and Appendix C).

Value recipe: draw i = mix64(seed + (i+1)*0x9E3779B97F4A7C15),
value = (draw >> 40) / 2^23 - 1, i.e. k * 2^-23 in [-1, 1), exactly representable in
fp32, about half negative (ReLU zeroes half, like a real pre-activation).  -0.0, NaN and
Inf cannot occur.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np

GOLDEN_GAMMA = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB
_M64 = (1 << 64) - 1

# role codes of the seed recipe: seed = 100000*cfg + 10*stack_index + role
ROLE_INPUT, ROLE_GAMMA, ROLE_BETA, ROLE_MEAN, ROLE_VAR, ROLE_OPERAND = 0, 1, 2, 3, 4, 5


def seed_for(cfg: int, stack_index: int, role: int) -> int:
    return 100000 * cfg + 10 * stack_index + role


# --------------------------------------------------------------------------- generator
def splitmix64_scalar(seed: int, i: int) -> int:
    """Draw i (0-based) of the counter-form SplitMix64 stream (pure Python ints)."""
    z = (seed + (i + 1) * GOLDEN_GAMMA) & _M64
    z = ((z ^ (z >> 30)) * _MIX1) & _M64
    z = ((z ^ (z >> 27)) * _MIX2) & _M64
    return z ^ (z >> 31)


def splitmix64_np(seed: int, start: int, count: int) -> np.ndarray:
    """Draws start..start+count-1 as uint64 (numpy wraps uint64 array arithmetic)."""
    i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & _M64) + i * np.uint64(GOLDEN_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_MIX2)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_np(seed: int, count: int, start: int = 0) -> np.ndarray:
    """fp32 values k*2^-23 - 1 in [-1, 1) (exact)."""
    k = (splitmix64_np(seed, start, count) >> np.uint64(40)).astype(np.int64)
    return ((k - (1 << 23)).astype(np.float64) * 2.0 ** -23).astype(np.float32)


VARIANTS = ("uniform", "allneg", "ties", "const", "signed_zero")


def variant_np(kind: str, seed: int, count: int, start: int = 0) -> np.ndarray:
    """Correctness-only input variants (SURVEY.md §8(d) "Correctness-only variants"), built from
    the same stream; no arithmetic of the method:
      uniform     : the default k*2^-23 in [-1, 1)
      allneg      : u - 1 in [-2, 0) (exact: |k - 2^23| < 2^24), every element < 0
      ties        : round(4u)/4 in {-1, -0.75, ..., 1}, +0.0 for zeros (many equal window values)
      const       : one value (0.375 + u_0/4, u_0 the first draw) everywhere
      signed_zero : +0.0 / -0.0 chosen by a draw bit, a quarter of the elements a small negative
                    value (so window maxima are mostly zeros of either sign)"""
    u = uniform_np(seed, count, start)
    if kind == "uniform":
        return u
    if kind == "allneg":
        return (u.astype(np.float64) - 1.0).astype(np.float32)
    if kind == "ties":
        return (np.round(4.0 * u.astype(np.float64)) / 4.0 + 0.0).astype(np.float32)
    if kind == "const":
        return np.full(count, np.float32(0.375 + uniform_np(seed, 1)[0] / 4.0), dtype=np.float32)
    if kind == "signed_zero":
        d = splitmix64_np(seed, start, count)
        z = np.where((d & np.uint64(1)) == 0, np.float32(0.0), np.float32(-0.0))
        neg = (d >> np.uint64(1)) & np.uint64(3) == 0
        return np.where(neg, -np.abs(u) - np.float32(2.0 ** -20), z).astype(np.float32)
    raise ValueError(f"unknown variant {kind!r}")


def _as_signed(v: int) -> int:
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


def _lsr(z, s: int):
    """Logical right shift of int64 tensors (torch >> is arithmetic)."""
    import torch
    return (z >> s) & ((1 << (64 - s)) - 1)


def uniform_torch(seed: int, shape: Sequence[int], device="cpu", start: int = 0,
                  chunk: int = 1 << 26):
    """Same stream as ``uniform_np`` built from torch int64 ops on ``device``.

    Two's-complement int64 multiply wraps modulo 2^64 on both CPU and CUDA, so the bit
    pattern equals the uint64 computation.  Filled in chunks to bound temporaries.
    """
    import torch
    n = 1
    for d in shape:
        n *= int(d)
    out = torch.empty(n, dtype=torch.float32, device=device)
    g = _as_signed(GOLDEN_GAMMA)
    m1 = _as_signed(_MIX1)
    m2 = _as_signed(_MIX2)
    s0 = _as_signed(seed)
    for off in range(0, n, chunk):
        m = min(chunk, n - off)
        i = torch.arange(start + off + 1, start + off + m + 1, dtype=torch.int64, device=device)
        z = i * g + s0
        z = (z ^ _lsr(z, 30)) * m1
        z = (z ^ _lsr(z, 27)) * m2
        z = z ^ _lsr(z, 31)
        k = _lsr(z, 40)
        out[off:off + m] = (k - (1 << 23)).to(torch.float32) * (2.0 ** -23)
    return out.view(*[int(d) for d in shape])


# --------------------------------------------------------------------------- stack description
KINDS = ("batchnorm", "relu", "maxpool", "avgpool", "copy", "scale", "add", "conv2d", "linear")


@dataclasses.dataclass
class Layer:
    """One layer of a stack, independent of both C ABIs.

    Pools: kernel/stride/padding as (h, w).  BatchNorm: per-channel fp32 arrays.
    ADD: ``operand`` >= 1 indexes the extra-input list (input 0 is the stack input).
    """
    kind: str
    kernel: Tuple[int, int] = (1, 1)
    stride: Tuple[int, int] = (1, 1)
    padding: Tuple[int, int] = (0, 0)
    count_include_pad: bool = True
    eps: float = 1e-5
    gamma: Optional[np.ndarray] = None
    beta: Optional[np.ndarray] = None
    mean: Optional[np.ndarray] = None
    var: Optional[np.ndarray] = None
    alpha: float = 1.0
    operand: int = 0

    def __post_init__(self):
        assert self.kind in KINDS, self.kind


def relu() -> Layer:
    return Layer("relu")


def copy() -> Layer:
    return Layer("copy")


def scale(alpha: float) -> Layer:
    return Layer("scale", alpha=float(np.float32(alpha)))


def add(operand: int = 1) -> Layer:
    return Layer("add", operand=operand)


def maxpool(k, s=None, p=0) -> Layer:
    k = (k, k) if isinstance(k, int) else tuple(k)
    s = k if s is None else ((s, s) if isinstance(s, int) else tuple(s))
    p = (p, p) if isinstance(p, int) else tuple(p)
    return Layer("maxpool", kernel=k, stride=s, padding=p)


def avgpool(k, s=None, p=0, count_include_pad=True) -> Layer:
    L = maxpool(k, s, p)
    L.kind = "avgpool"
    L.count_include_pad = count_include_pad
    return L


def batchnorm(C: int, seed_base: int, eps: float = 1e-5, signed_gamma: bool = False) -> Layer:
    """BN parameters from the role streams: gamma = 1 + u/2,
    beta = u/2, mean = u/2, var = 1 + u/2, u in [-1, 1); evaluated in fp64, stored fp32.
    ``signed_gamma`` flips the sign of every other channel's gamma (padding hazard H5)."""
    u = lambda r: uniform_np(seed_base + r, C).astype(np.float64)
    gamma = 1.0 + 0.5 * u(ROLE_GAMMA)
    if signed_gamma:
        gamma[1::2] *= -1.0
    return Layer("batchnorm", eps=float(np.float32(eps)),
                 gamma=gamma.astype(np.float32), beta=(0.5 * u(ROLE_BETA)).astype(np.float32),
                 mean=(0.5 * u(ROLE_MEAN)).astype(np.float32),
                 var=(1.0 + 0.5 * u(ROLE_VAR)).astype(np.float32))


def batchnorm_explicit(gamma, beta, mean, var, eps) -> Layer:
    f = lambda a: np.asarray(a, dtype=np.float32).copy()
    return Layer("batchnorm", eps=float(np.float32(eps)), gamma=f(gamma), beta=f(beta),
                 mean=f(mean), var=f(var))


# --------------------------------------------------------------------------- paper workloads
@dataclasses.dataclass
class StackCase:
    """One stack of a workload: layers + input shape (N, C, H, W) + seeds."""
    name: str
    shape: Tuple[int, int, int, int]
    layers: List[Layer]
    input_seed: int
    operand_seeds: List[int] = dataclasses.field(default_factory=list)
    count: int = 1          # how many times this stack occurs in the network (weight)


def _bn_relu(C, sb):
    return [batchnorm(C, sb), relu()]


def workload(name: str, batch: Optional[int] = None) -> List[StackCase]:
    """Stacks of BASELINE.json's configs.

    c1          configs[0]: BN->ReLU->MaxPool2x2/s2 on (1,16,32,32)
    alexnet     configs[1]: 3 x ReLU->MaxPool3x3/s2 at batch 128
    vgg16       configs[2]: 5 x ReLU->MaxPool2x2/s2 at batch 64
    resnet50    configs[3]: stem BN->ReLU->MaxPool3x3/s2/p1 + 32 BN->ReLU at batch 256
    densenet121 configs[4]: stem + 116 BN->ReLU + 3 BN->ReLU->AvgPool2x2 + final AvgPool7
    """
    cases: List[StackCase] = []
    if name == "c1":
        cfg, N = 0, batch or 1
        sb = seed_for(cfg, 0, 0)
        cases.append(StackCase("c1", (N, 16, 32, 32), _bn_relu(16, sb) + [maxpool(2, 2)], sb))
    elif name == "alexnet":
        cfg, N = 1, batch or 128
        for si, (C, H) in enumerate([(64, 55), (192, 27), (256, 13)]):
            sb = seed_for(cfg, si, 0)
            cases.append(StackCase(f"alexnet_s{si+1}", (N, C, H, H), [relu(), maxpool(3, 2)], sb))
    elif name == "vgg16":
        cfg, N = 2, batch or 64
        for si, (C, H) in enumerate([(64, 224), (128, 112), (256, 56), (512, 28), (512, 14)]):
            sb = seed_for(cfg, si, 0)
            cases.append(StackCase(f"vgg16_s{si+1}", (N, C, H, H), [relu(), maxpool(2, 2)], sb))
    elif name == "resnet50":
        cfg, N = 3, batch or 256
        sb = seed_for(cfg, 0, 0)
        cases.append(StackCase("resnet50_stem", (N, 64, 112, 112),
                               _bn_relu(64, sb) + [maxpool(3, 2, 1)], sb))
        si = 1
        for (C, H, cnt) in [(64, 56, 6), (128, 56, 1), (128, 28, 7), (256, 28, 1),
                            (256, 14, 11), (512, 14, 1), (512, 7, 5)]:
            sb = seed_for(cfg, si, 0)
            cases.append(StackCase(f"resnet50_bnrelu_{C}x{H}", (N, C, H, H), _bn_relu(C, sb), sb,
                                   count=cnt))
            si += 1
    elif name == "densenet121":
        cfg, N = 4, batch or 256
        sb = seed_for(cfg, 0, 0)
        cases.append(StackCase("densenet121_stem", (N, 64, 112, 112),
                               _bn_relu(64, sb) + [maxpool(3, 2, 1)], sb))
        si = 1
        blocks = [(64, 56, 6), (128, 28, 12), (256, 14, 24), (512, 7, 16)]
        for bi, (c0, H, nl) in enumerate(blocks):
            for i in range(nl):
                C = c0 + 32 * i
                sb = seed_for(cfg, si, 0); si += 1
                cases.append(StackCase(f"densenet121_b{bi+1}_l{i+1}_norm1", (N, C, H, H),
                                       _bn_relu(C, sb), sb))
                sb = seed_for(cfg, si, 0); si += 1
                cases.append(StackCase(f"densenet121_b{bi+1}_l{i+1}_norm2", (N, 128, H, H),
                                       _bn_relu(128, sb), sb))
            if bi < 3:
                C = c0 + 32 * nl
                sb = seed_for(cfg, si, 0); si += 1
                cases.append(StackCase(f"densenet121_t{bi+1}", (N, C, H, H),
                                       _bn_relu(C, sb) + [avgpool(2, 2)], sb))
        sb = seed_for(cfg, si, 0)
        cases.append(StackCase("densenet121_final", (N, 1024, 7, 7),
                               _bn_relu(1024, sb) + [avgpool(7, 7)], sb))
    elif name == "resnet50_residual":
        # NEXT-1: the bottleneck tail bn3 -> (+ identity) -> ReLU of every
        # ResNet-50 block, a two-input stack (ADD operand 1 = the block's shortcut)
        cfg, N = 3, batch or 256
        si = 100
        for (C, H, cnt) in [(256, 56, 3), (512, 28, 4), (1024, 14, 6), (2048, 7, 3)]:
            sb = seed_for(cfg, si, 0)
            cases.append(StackCase(f"resnet50_tail_{C}x{H}", (N, C, H, H),
                                   [batchnorm(C, sb), add(1), relu()], sb,
                                   operand_seeds=[seed_for(cfg, si, 5)], count=cnt))
            si += 1
    else:
        raise ValueError(f"unknown workload {name!r}")
    return cases


def synthetic51(depth: int, batch: int = 128, C: int = 64, H: int = 56) -> StackCase:
    """PAPER.md §5.1: a network of `depth` blocks MaxPool3x3/s1/p1 -> BN -> ReLU,
    every layer optimizable (one stack).  The tensor shape is unstated in the paper (SURVEY.md
    G20); (128, 64, 56, 56) is DESIGN.md's choice."""
    cfg = 51
    layers: List[Layer] = []
    for b in range(depth):
        layers += [maxpool(3, 1, 1), batchnorm(C, seed_for(cfg, b, 0)), relu()]
    return StackCase(f"sec51_depth{depth}", (batch, C, H, H), layers, seed_for(cfg, 9999, 0))


WORKLOADS = ("c1", "alexnet", "vgg16", "resnet50", "densenet121", "resnet50_residual")
DEFAULT_BATCH = {"c1": 1, "alexnet": 128, "vgg16": 64, "resnet50": 256, "densenet121": 256,
                 "resnet50_residual": 256}
