"""GPU parity of on-chip multi-step sequences (NEXT-2, k_seq.cu) against the oracle: the vectorised
3x3/s1/p1 fast path at every segment geometry, halo (row-band) tiles on planes too large to hold
whole, and tile invariance: the result does not depend on the
band height or the planes per tile -- bit for bit, since every output element gets
the same arithmetic in the same order whatever the tiling."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests import _util as U

pytestmark = pytest.mark.gpu


def _bs():
    import paper_1804_08378_b200 as bs
    return bs


def run_gpu(layers, x, opts=None):
    bs = _bs()
    plan = bs.bs_plan_create(layers, x.shape, opts)
    out = torch.full(bs.bs_plan_query(plan)["out"], float("nan"), device="cuda")
    bs.bs_execute(plan, torch.from_numpy(np.ascontiguousarray(x)).cuda(), out)
    torch.cuda.synchronize()
    return out.cpu().numpy(), plan


def sec51(depth, C, signed=False, last_plain=False):
    layers = []
    for b in range(depth):
        layers += [synth.maxpool(3, 1, 1), synth.batchnorm(C, 700 + b, signed_gamma=signed and b % 2 == 1), synth.relu()]
    if last_plain:
        layers += [synth.maxpool(3, 1, 1)]
    return layers


@pytest.mark.parametrize("W", [4, 8, 28, 56, 60, 64, 68, 100, 128, 132, 200, 252, 256])
def test_fast_path_widths(W, cuda_dev, oracle_lib):
    """Segments of 16 lanes (W <= 64), 32 lanes x 1 (<= 128), 32 lanes x 2 (<= 256)."""
    bs = _bs()
    shape = (2, 3, 23, W)
    layers = sec51(4, 3, signed=True, last_plain=True)
    x = synth.uniform_np(W, int(np.prod(shape))).reshape(shape)
    ref = oracle.run_bf(layers, x)
    for opts in (None, {"force_tile_planes": 1}, {"force_rows_per_task": 5}, {"force_rows_per_task": 1}):
        got, plan = run_gpu(layers, x, opts)
        assert bs.bs_plan_query(plan)["n_launches"] == 1
        U.assert_close(got, ref, f"W={W} {opts}")


def test_tile_invariance_bitexact(cuda_dev, oracle_lib):
    bs = _bs()
    shape = (2, 4, 61, 96)
    layers = sec51(6, 4, signed=True)
    x = synth.uniform_np(5, int(np.prod(shape))).reshape(shape)
    ref = oracle.run_bf(layers, x)
    base, _ = run_gpu(layers, x)
    U.assert_close(base, ref, "whole planes")
    for opts in ({"force_rows_per_task": 1}, {"force_rows_per_task": 2}, {"force_rows_per_task": 7},
                 {"force_rows_per_task": 30}, {"force_tile_planes": 1}, {"force_tile_planes": 3},
                 {"max_steps_per_sequence": 1}, {"max_steps_per_sequence": 4}):
        got, plan = run_gpu(layers, x, opts)
        U.assert_bitexact(got, base, f"{opts}")
    li = bs.bs_plan_query_launch(run_gpu(layers, x, {"force_rows_per_task": 7})[1], 0)
    assert li["tile_rows"] == 7 and li["halo_rows"] > 0


def test_halo_generic_steps(cuda_dev, oracle_lib):
    """Halo tiles through generic steps: odd widths, avg pools with padding, strided pools, prologues."""
    shape = (2, 3, 77, 53)
    layers = [synth.maxpool(3, 1, 1), synth.relu(), synth.avgpool(3, 1, 1), synth.batchnorm(3, 5, signed_gamma=True),
              synth.maxpool(3, 2, 1), synth.scale(-1.5), synth.relu(), synth.maxpool(3, 1, 1), synth.avgpool(2, 2),
              synth.batchnorm(3, 6), synth.maxpool((3, 1), (1, 1), (1, 0))]
    x = synth.uniform_np(9, int(np.prod(shape))).reshape(shape)
    ref = oracle.run_bf(layers, x)
    base, plan = run_gpu(layers, x)
    U.assert_close(base, ref, "default")
    for R in (1, 2, 3, 5, 9):
        got, plan = run_gpu(layers, x, {"force_rows_per_task": R})
        assert _bs().bs_plan_query_launch(plan, 0)["tile_rows"] in (R, 0)
        U.assert_bitexact(got, base, f"rows {R}")


@pytest.mark.parametrize("H,depth", [(224, 20), (150, 33), (112, 40)])
def test_sec51_large_planes(H, depth, cuda_dev, oracle_lib):
    """§5.1 networks on planes too large to stage whole (default budget): halo tiles, split where
    the band overflows the budget; every policy gives the same bits."""
    bs = _bs()
    shape = (2, 3, H, H)
    layers = sec51(depth, 3)
    x = synth.uniform_np(H + depth, int(np.prod(shape))).reshape(shape)
    ref = oracle.run_bf(layers, x)
    outs = []
    for policy in (0, 5, 1, -1):
        got, plan = run_gpu(layers, x, {"max_steps_per_sequence": policy})
        U.assert_close(got, ref, f"H={H} depth {depth} policy {policy}")
        outs.append(got)
    for k, name in ((1, "5"), (2, "1"), (3, "unrestricted")):
        U.assert_bitexact(outs[k], outs[0], f"policy {name} vs planner")


@pytest.mark.parametrize("shape,depth", [((32, 64, 224, 224), 16), ((64, 64, 112, 112), 24), ((128, 64, 56, 56), 40)])
def test_sec51_full_shapes_sampled(shape, depth, cuda_dev, oracle_lib):
    """The §5.1 benchmark shapes (R15) at the depths exp_sec51.py times, unrestricted
    policy; images checked against the oracle one by one."""
    bs = _bs()
    case = synth.synthetic51(depth, batch=shape[0], C=shape[1], H=shape[2])
    x = synth.uniform_torch(case.input_seed, case.shape, device="cuda")
    plan = bs.bs_plan_create(case.layers, case.shape)
    out = torch.empty(bs.bs_plan_query(plan)["out"], device="cuda")
    bs.bs_execute(plan, x, out)
    torch.cuda.synchronize()
    for n in (0, shape[0] - 1):
        ref = oracle.run_bf(case.layers, x[n:n + 1].cpu().numpy())
        U.check(out[n:n + 1].cpu().numpy(), ref, case.layers, f"{shape} image {n}")
    # every element against the definition written with torch library ops (fp64 per layer)
    ref = U.torch_definition(case.layers, x)
    err = (out.double() - ref.double()).abs() - (1e-6 + 1e-5 * ref.double().abs())
    assert float(err.max()) <= 0, f"{shape}: max excess {float(err.max())}"


@pytest.mark.parametrize("H", [1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 23, 56, 112])
def test_inplace_kernel_heights(H, cuda_dev, oracle_lib):
    """The warp-per-plane in-place kernel (whole planes, W <= 128): odd/even heights (the two
    half-warps split the rows), a partial last tile (odd plane count), every epilogue class; bit
    for bit equal to the shared-tile kernel (force_tile_planes routes there) and to the oracle.
    Heights whose parts hold 2, 3, 4, 5 and 28 rows reach every tail of the clean step
    (k_seq.cu inplace_step_clean: W / 4 + 2 lanes fit a segment, H divisible by the parts)."""
    bs = _bs()
    for W, extra in ((4, 0), (16, 1), (56, 0), (56, 1), (64, 0), (68, 1), (112, 0), (112, 1), (128, 0)):
        shape = (1, 3, H, W)
        layers = [synth.maxpool(3, 1, 1), synth.batchnorm(3, 1, signed_gamma=True), synth.relu(),
                  synth.maxpool(3, 1, 1), synth.relu(), synth.maxpool(3, 1, 1), synth.batchnorm(3, 2),
                  synth.maxpool(3, 1, 1)]
        # an odd step count: two-step sweeps, then one single step (k_seq.cu inplace_pair_clean)
        layers += [synth.maxpool(3, 1, 1), synth.batchnorm(3, 3, signed_gamma=True)] * extra
        x = synth.uniform_np(H * 1000 + W, int(np.prod(shape))).reshape(shape)
        got, plan = run_gpu(layers, x)
        li = bs.bs_plan_query_launch(plan, 0)
        assert li["kernel_name"] == "sequence_staged_tma" and li["block"] == 160, li   # in-place kernel
        U.assert_close(got, oracle.run_bf(layers, x), f"H={H} W={W}")
        other, plan2 = run_gpu(layers, x, {"force_tile_planes": 1})
        assert bs.bs_plan_query_launch(plan2, 0)["block"] != 160
        U.assert_bitexact(got, other, f"H={H} W={W} in-place vs shared tile")


@pytest.mark.parametrize("H,W", [(16, 132), (24, 200), (40, 160), (56, 224), (224, 224), (30, 144), (51, 224)])
def test_inplace_wide_planes(H, W, cuda_dev, oracle_lib):
    """Planes 129..224 wide run in place too (k_seq.cu seq_inplace<32, 1, 2, false>): one plane per CTA,
    8 warps of ~H / 8 rows (balanced, unequal when 8 does not divide H), each row as two column
    segments with halo lanes; even and odd step
    counts (two-step sweeps + a single step), signed-gamma BN; bit for bit equal to the
    shared-tile / halo kernels (force_tile_planes routes there) and within tolerance of the oracle."""
    bs = _bs()
    for extra in (0, 1):
        shape = (2, 3, H, W)
        layers = [synth.maxpool(3, 1, 1), synth.batchnorm(3, 1, signed_gamma=True), synth.relu(),
                  synth.maxpool(3, 1, 1), synth.relu(), synth.maxpool(3, 1, 1), synth.batchnorm(3, 2),
                  synth.maxpool(3, 1, 1)] + [synth.maxpool(3, 1, 1), synth.batchnorm(3, 3, signed_gamma=True)] * extra
        x = synth.uniform_np(H * 1000 + W + extra, int(np.prod(shape))).reshape(shape)
        got, plan = run_gpu(layers, x)
        li = bs.bs_plan_query_launch(plan, 0)
        assert li["block"] == 288 and li["tile_planes"] == 1 and li["stages"] == 1, li
        assert li["smem_bytes"] < 1.5 * H * W * 4, li                         # in place: no work buffer
        U.assert_close(got, oracle.run_bf(layers, x), f"H={H} W={W} extra={extra}")
        other, _ = run_gpu(layers, x, {"force_tile_planes": 1})
        U.assert_bitexact(got, other, f"H={H} W={W} in-place vs shared tile / halo")


@pytest.mark.parametrize("trial", range(64))
def test_random_fast_sequences(trial, cuda_dev, oracle_lib):
    """Random sequences of §5.1-type steps (3x3/s1/p1 max + any of BN (signed gamma) / ReLU / none)
    on random planes (W a multiple of 4 up to 224, H 1..70 or up to 224): every sequence kernel the
    planner picks (in place: clean two-step sweeps, single steps, edge selects, one or two column
    segments; shared tile; halo) against the oracle, and bit for bit against the shared-tile / halo
    kernels (force_tile_planes)."""
    import random
    rng = random.Random(900 + trial)
    W = 4 * rng.randint(1, 56)
    H = rng.randint(1, 70) if rng.random() < 0.7 else 8 * rng.randint(2, 28)
    C = rng.randint(1, 5)
    N = rng.randint(1, 3) if H * W < 20000 else 1
    layers = []
    for b in range(rng.randint(1, 9)):
        layers.append(synth.maxpool(3, 1, 1))
        r = rng.random()
        if r < 0.6:
            layers.append(synth.batchnorm(C, 50 + b, signed_gamma=rng.random() < 0.5))
        if rng.random() < 0.6:
            layers.append(synth.relu())
    shape = (N, C, H, W)
    # a third of the trials under a small shared-memory budget: halo (band) tiles, in place or shared
    opts = {"smem_budget_bytes": rng.choice([8, 12, 16, 24, 32, 48]) * 1024} if rng.random() < 0.35 else {}
    x = synth.uniform_np(7000 + trial, int(np.prod(shape))).reshape(shape)
    got, plan = run_gpu(layers, x, opts or None)
    ctx = f"trial {trial} shape {shape} {len(layers)} layers {opts} {_bs().bs_plan_query_launch(plan, 0)}"
    U.assert_close(got, oracle.run_bf(layers, x), ctx)
    other, _ = run_gpu(layers, x, {**opts, "force_tile_planes": 1})
    U.assert_bitexact(got, other, ctx + " vs shared tile / halo")


@pytest.mark.parametrize("H,W,budget,depth", [(224, 224, 110 * 1024, 16), (112, 112, 40 * 1024, 9),
                                              (300, 200, 0, 12), (100, 64, 16 * 1024, 7), (61, 96, 12 * 1024, 6)])
def test_inplace_band_tiles(H, W, budget, depth, cuda_dev, oracle_lib):
    """Halo (band) tiles of §5.1 networks run in place (k_seq.cu seq_inplace band tiles): planes
    that do not fit whole (wider than 224, or under a budget).  Every policy (planner, the paper's
    unrestricted, <= 5 steps) against the oracle, and bit for bit against the shared-tile kernel's
    halo tiles (force_tile_planes keeps seq_staged) and the unbudgeted whole-plane run."""
    bs = _bs()
    shape = (2, 3, H, W)
    layers = []
    for b in range(depth):
        layers += [synth.maxpool(3, 1, 1), synth.batchnorm(3, 60 + b, signed_gamma=b % 3 == 1)] + \
                  ([synth.relu()] if b % 2 == 0 else [])
    x = synth.uniform_np(H * 7 + W + depth, int(np.prod(shape))).reshape(shape)
    ref = oracle.run_bf(layers, x[:1])
    base = {"smem_budget_bytes": budget} if budget else {}
    whole, _ = run_gpu(layers, x) if budget else (None, None)
    for policy in (0, -1, 5):
        got, plan = run_gpu(layers, x, {**base, "max_steps_per_sequence": policy})
        li = bs.bs_plan_query_launch(plan, 0)
        assert li["tile_rows"] > 0 and li["block"] in (160, 288) and li["smem_bytes"] < 2.2 * li["tile_rows"] * W * 4 + \
            (2 * depth + 8) * W * 8 + 8192, li                         # band tiles, in place (no work buffer)
        U.assert_close(got[:1], ref, f"H={H} W={W} policy {policy}")
        staged, plan2 = run_gpu(layers, x, {**base, "max_steps_per_sequence": policy, "force_tile_planes": 1})
        U.assert_bitexact(got, staged, f"H={H} W={W} policy {policy}: in place vs seq_staged bands")
        if whole is not None:
            U.assert_bitexact(got, whole, f"H={H} W={W} policy {policy}: bands vs whole planes")
