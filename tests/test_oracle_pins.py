"""Pins of the CPU oracle against things other than itself (run with -m "not gpu").

* golden hand examples (tests/golden/*.json, each citing its passage);
* brute-force pooling-window enumeration (scan every input cell, test membership);
* independent library routines (torch CPU functional ops);
* closed forms (shape law), special cases (identity / gamma=0 BN, k=1 pools),
  a high-precision BN reference (Python Decimal);
* the paper's central claim: depth-first == breadth-first, bit for bit.
"""
import decimal
import itertools
import random

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth
from tests import _util as U


# ----------------------------------------------------------------------------- golden
@pytest.mark.parametrize("case", U.load_golden(), ids=lambda c: c[0])
def test_golden(case, oracle_lib):
    name, layers, x, ops, exp, cite = case
    got = oracle.run_bf(layers, x, ops)
    U.assert_bitexact(got, exp, f"{name} ({cite})")
    U.assert_bitexact(oracle.run_df(layers, x, ops, (1, 1)), exp, name + " df")


# ----------------------------------------------------------------------------- brute force
def brute_pool(x: np.ndarray, kind, k, s, p, cip=True):
    """For each output, scan EVERY input coordinate and test window membership
    (independent of the oracle's window loop)."""
    N, C, H, W = x.shape
    Ho = (H + 2 * p[0] - k[0]) // s[0] + 1
    Wo = (W + 2 * p[1] - k[1]) // s[1] + 1
    y = np.empty((N, C, Ho, Wo), np.float32)
    for n, c, i, j in itertools.product(range(N), range(C), range(Ho), range(Wo)):
        members = [float(x[n, c, r, q]) for r in range(H) for q in range(W)
                   if i * s[0] - p[0] <= r < i * s[0] - p[0] + k[0]
                   and j * s[1] - p[1] <= q < j * s[1] - p[1] + k[1]]
        if kind == "maxpool":
            y[n, c, i, j] = max(members)
        else:
            div = k[0] * k[1] if cip else len(members)
            y[n, c, i, j] = np.float32(sum(members) / div)
    return y


def test_pool_brute_force(oracle_lib):
    rng = random.Random(1234)
    n = 0
    for trial in range(400):
        kh, kw = rng.randint(1, 4), rng.randint(1, 4)
        sh, sw = rng.randint(1, 3), rng.randint(1, 3)
        ph, pw = rng.randint(0, kh // 2), rng.randint(0, kw // 2)
        H, W = rng.randint(max(1, kh - 2 * ph), 12), rng.randint(max(1, kw - 2 * pw), 12)
        kind = rng.choice(["maxpool", "avgpool"])
        cip = rng.random() < 0.5
        x = synth.uniform_np(trial, 2 * H * W).reshape(1, 2, H, W)
        if trial % 5 == 0:   # tie-heavy quantised inputs
            x = (np.round(x * 4) / 4).astype(np.float32)
        L = (synth.maxpool if kind == "maxpool" else synth.avgpool)((kh, kw), (sh, sw), (ph, pw))
        L.count_include_pad = cip
        exp = brute_pool(x, kind, (kh, kw), (sh, sw), (ph, pw), cip)
        got = oracle.run_bf([L], x)
        if kind == "maxpool":
            U.assert_bitexact(got, exp, f"trial {trial}")
        else:   # Python float sum is fp64 sequential over the same row-major member order
            U.assert_bitexact(got, exp, f"trial {trial}")
        n += 1
    assert n == 400


# ----------------------------------------------------------------------------- library cross-checks
def _torch_stack(layers, x, ops):
    t = torch.from_numpy(x.copy())
    for L in layers:
        if L.kind == "relu":
            t = F.relu(t)
        elif L.kind == "maxpool":
            t = F.max_pool2d(t, L.kernel, L.stride, L.padding)
        elif L.kind == "avgpool":
            t = F.avg_pool2d(t, L.kernel, L.stride, L.padding, count_include_pad=L.count_include_pad)
        elif L.kind == "batchnorm":
            t = F.batch_norm(t, torch.from_numpy(L.mean), torch.from_numpy(L.var),
                             torch.from_numpy(L.gamma), torch.from_numpy(L.beta), False, 0.0, L.eps)
        elif L.kind == "scale":
            t = t * torch.tensor(L.alpha, dtype=torch.float32)
        elif L.kind == "add":
            t = t + torch.from_numpy(ops[L.operand - 1])
        elif L.kind == "copy":
            t = t.clone()
    return t.numpy()


@pytest.mark.parametrize("trial", range(40))
def test_torch_cpu_cross_check(trial, oracle_lib):
    rng = random.Random(77 + trial)
    shape = (rng.randint(1, 2), rng.randint(1, 4), rng.randint(3, 17), rng.randint(3, 17))
    layers, n_ops = U.random_stack(rng, shape, max_depth=6, seed_base=5000 * trial)
    shapes = oracle.layer_shapes(layers, shape, n_ops)
    x, ops = U.make_inputs(layers, shape, n_ops, 31 * trial + 1, shapes)
    got = oracle.run_bf(layers, x, ops)
    ref = _torch_stack(layers, x, ops)
    U.check(got, ref, layers, f"trial {trial}: {[L.kind for L in layers]}")


def test_bc_configs_small_vs_torch(oracle_lib):
    """Every BASELINE.json stack type at reduced batch/channels vs torch CPU."""
    for wl in synth.WORKLOADS:
        for case in synth.workload(wl, batch=1)[:3]:
            N, C, H, W = case.shape
            shape = (1, min(C, 3), H, W)
            layers = []
            for L in case.layers:
                if L.kind == "batchnorm":
                    L = synth.batchnorm(shape[1], case.input_seed)
                layers.append(L)
            x = synth.uniform_np(case.input_seed, int(np.prod(shape))).reshape(shape)
            ops = [synth.uniform_np(sd, int(np.prod(shape))).reshape(shape) for sd in case.operand_seeds]
            U.check(oracle.run_bf(layers, x, ops), _torch_stack(layers, x, ops), layers, case.name)


# ----------------------------------------------------------------------------- BN special cases
def test_bn_identity_params(oracle_lib):
    x = synth.uniform_np(5, 4 * 64).reshape(1, 4, 8, 8)
    L = synth.batchnorm_explicit([1] * 4, [0] * 4, [0] * 4, [1] * 4, 1e-12)
    y = oracle.run_bf([L], x)
    assert np.all(np.abs(y.astype(np.float64) - x) <= 1e-6 * np.abs(x))


def test_bn_high_precision(oracle_lib):
    """Oracle BN within 1 ulp of a 40-digit Decimal evaluation of gamma(x-mu)/sqrt(var+eps)+beta."""
    decimal.getcontext().prec = 40
    C = 8
    L = synth.batchnorm(C, 4242, signed_gamma=True)
    x = synth.uniform_np(99, C * 25).reshape(1, C, 5, 5)
    y = oracle.run_bf([L], x)
    D = decimal.Decimal
    for c in range(C):
        den = (D(float(L.var[c])) + D(float(L.eps))).sqrt()
        for v, got in zip(x[0, c].ravel(), y[0, c].ravel()):
            exact = (D(float(v)) - D(float(L.mean[c]))) / den * D(float(L.gamma[c])) + D(float(L.beta[c]))
            ref = np.float32(float(exact))
            ulp = np.spacing(np.abs(ref))
            assert abs(float(got) - float(exact)) <= float(ulp), (c, v, got, exact)


def test_scale_add_single_rounding(oracle_lib):
    """fp64-then-round equals the fp32 IEEE op (numpy fp32 arithmetic) bit for bit."""
    x = synth.uniform_np(11, 3 * 7 * 7).reshape(1, 3, 7, 7) * np.float32(3.7)
    o = synth.uniform_np(12, 3 * 7 * 7).reshape(1, 3, 7, 7)
    for a in (0.1, -1.25, 3.3333333):
        y = oracle.run_bf([synth.scale(a)], x)
        U.assert_bitexact(y, (np.float32(a) * x).astype(np.float32), f"scale {a}")
    y = oracle.run_bf([synth.add(1)], x, [o])
    U.assert_bitexact(y, (x + o).astype(np.float32), "add")


# ----------------------------------------------------------------------------- closed forms / invariants
@pytest.mark.parametrize("H,k,s,p,Ho", [(55, 3, 2, 0, 27), (27, 3, 2, 0, 13), (13, 3, 2, 0, 6),
                                        (112, 3, 2, 1, 56), (224, 2, 2, 0, 112), (56, 2, 2, 0, 28),
                                        (7, 7, 7, 0, 1), (14, 2, 2, 0, 7), (32, 2, 2, 0, 16)])
def test_shape_law(H, k, s, p, Ho, oracle_lib):
    sh = oracle.layer_shapes([synth.maxpool(k, s, p)], (2, 3, H, H))
    assert sh[-1] == (2, 3, Ho, Ho)


@pytest.mark.parametrize("bad", [
    [synth.maxpool(3, 1, 2)],                       # p > k/2
    [synth.maxpool(9, 1, 0)],                       # window larger than padded input
    [synth.Layer("maxpool", kernel=(0, 1), stride=(1, 1))],
    [synth.Layer("avgpool", kernel=(2, 2), stride=(0, 1))],
    [synth.add(2)],                                 # operand index out of range
])
def test_validation_errors(bad, oracle_lib):
    with pytest.raises(oracle.OracleError) as e:
        oracle.layer_shapes(bad, (1, 2, 5, 5), 1)
    assert e.value.code == oracle.ERR_INVALID


def test_opaque_layers_rejected(oracle_lib):
    with pytest.raises(oracle.OracleError) as e:
        oracle.layer_shapes([synth.relu(), synth.Layer("conv2d")], (1, 1, 4, 4))
    assert e.value.code == oracle.ERR_UNSUPPORTED


def test_invariants(oracle_lib):
    x = synth.uniform_np(3, 2 * 3 * 20 * 20).reshape(2, 3, 20, 20)
    # MaxPool o ReLU == ReLU o MaxPool (monotone, exact)
    a = oracle.run_bf([synth.relu(), synth.maxpool(3, 2, 1)], x)
    b = oracle.run_bf([synth.maxpool(3, 2, 1), synth.relu()], x)
    U.assert_bitexact(a, b, "relu/max commute")
    # k = 1 pools are the identity
    U.assert_bitexact(oracle.run_bf([synth.maxpool(1, 1)], x), x, "k1 max")
    U.assert_bitexact(oracle.run_bf([synth.avgpool(1, 1)], x), x, "k1 avg")
    # constant input -> constant 2x2 average
    c = np.full((1, 1, 6, 6), 0.3, np.float32)
    U.assert_bitexact(oracle.run_bf([synth.avgpool(2, 2)], c), np.full((1, 1, 3, 3), 0.3, np.float32), "const")
    # maxpool >= avgpool on non-negative inputs
    r = oracle.run_bf([synth.relu()], x)
    assert np.all(oracle.run_bf([synth.maxpool(3, 2)], r) >= oracle.run_bf([synth.avgpool(3, 2)], r))
    # all-negative input through ReLU -> all +0.0
    neg = -np.abs(x) - np.float32(0.5)
    z = oracle.run_bf([synth.relu()], neg)
    assert np.all(U.bits(z) == 0)


# ----------------------------------------------------------------------------- DF == BF (the paper's claim)
def test_depth_first_equals_breadth_first(oracle_lib):
    rng = random.Random(2018)
    for trial in range(220):
        shape = (rng.randint(1, 3), rng.randint(1, 4), rng.randint(1, 32), rng.randint(1, 32))
        if trial % 4 == 0:   # deep §5.1-style chains: [MaxPool3x3/s1/p1, BN, ReLU] x d
            d = rng.randint(1, 13)
            layers = []
            for b in range(d):
                layers += [synth.maxpool(3, 1, 1), synth.batchnorm(shape[1], 7000 + 10 * b), synth.relu()]
            n_ops = 0
        else:
            layers, n_ops = U.random_stack(rng, shape, max_depth=rng.choice([4, 12, 40]),
                                           max_pools=rng.choice([1, 3, 6]), seed_base=40000 + trial)
        shapes = oracle.layer_shapes(layers, shape, n_ops)
        x, ops = U.make_inputs(layers, shape, n_ops, 1000 + trial, shapes)
        bf = oracle.run_bf(layers, x, ops)
        tile = (rng.randint(1, 9), rng.randint(1, 9))
        df = oracle.run_df(layers, x, ops, tile)
        U.assert_bitexact(df, bf, f"trial {trial} tile {tile} {[L.kind for L in layers]}")
