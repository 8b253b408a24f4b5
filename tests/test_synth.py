"""The shared input generator: pinned to SplitMix64's published reference output and
checked to be identical across its numpy, torch and pure-Python implementations."""
import numpy as np
import torch

import synth


def test_splitmix64_reference_vector():
    # Vigna's splitmix64.c with state 0: first next() = 0xE220A8397B1DCDAF,
    # second = 0x6E789E6AA1B965F4 (the stream every SplitMix64 port is checked against).
    assert synth.splitmix64_scalar(0, 0) == 0xE220A8397B1DCDAF
    assert synth.splitmix64_scalar(0, 1) == 0x6E789E6AA1B965F4


def test_numpy_torch_python_agree():
    for seed in (0, 7, 300004, 2**63 + 12345):
        a = synth.splitmix64_np(seed, 5, 1000)
        b = np.array([synth.splitmix64_scalar(seed, i) for i in range(5, 1005)], dtype=np.uint64)
        assert np.array_equal(a, b)
        u = synth.uniform_np(seed, 5000)
        t = synth.uniform_torch(seed, (5, 1000), chunk=777).numpy().ravel()
        assert np.array_equal(u.view(np.uint32), t.view(np.uint32))


def test_value_range_and_exactness():
    u = synth.uniform_np(42, 1 << 16)
    assert u.dtype == np.float32 and u.min() >= -1.0 and u.max() < 1.0
    k = u.astype(np.float64) * 2**23
    assert np.all(k == np.round(k))                 # multiples of 2^-23
    assert not np.any(np.signbit(u) & (u == 0))     # no -0.0
    assert 0.45 < np.mean(u < 0) < 0.55


def test_workload_shapes():
    assert [c.shape for c in synth.workload("alexnet")] == [(128, 64, 55, 55), (128, 192, 27, 27),
                                                            (128, 256, 13, 13)]
    r = synth.workload("resnet50")
    assert sum(c.count for c in r) == 33
    d = synth.workload("densenet121")
    assert len(d) == 121


def test_variants():
    n = 1 << 14
    a = synth.variant_np("allneg", 3, n)
    assert np.all(a < 0) and a.min() >= -2.0
    assert np.array_equal(a.astype(np.float64), synth.uniform_np(3, n).astype(np.float64) - 1.0)
    t = synth.variant_np("ties", 3, n)
    assert set(np.unique(t).tolist()) <= {q / 4 for q in range(-4, 5)}
    assert not np.any(np.signbit(t) & (t == 0))
    c = synth.variant_np("const", 3, n)
    assert np.all(c == c[0])
    z = synth.variant_np("signed_zero", 3, n)
    zero = z == 0
    assert 0.6 < zero.mean() < 0.9
    assert 0.2 < np.signbit(z[zero]).mean() < 0.8      # both zero signs present
    assert np.all(z[~zero] < 0)
    assert np.array_equal(synth.variant_np("uniform", 3, n), synth.uniform_np(3, n))
