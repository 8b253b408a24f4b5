"""GPU parity on the edge cases (round-2 additions), against the CPU oracle through the C ABI.

* wide planes: more than 16 work items per staged tile (Wo > 16 * 32 columns, or forced
  narrow column groups) -- every item of every tile must be written (the method
  does not change results);
* SURVEY.md §8(d)'s correctness-only input variants on every BASELINE.json stack at batch 2:
  all-negative, tie-heavy round(4u)/4, constant, hand-made +-0 (compared modulo the sign of
  zero for max-only stacks: fmaxf(+0, -0) may return either zero, G10);
* two host threads executing different plans that share one kernel instantiation with
  different shared-memory sizes, concurrently (bs.h: plans are immutable, executes on
  different streams are safe).
"""
import threading

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


def run_gpu(layers, x, ops=(), opts=None):
    bs = _bs()
    plan = bs.bs_plan_create(layers, x.shape, opts)
    info = bs.bs_plan_query(plan)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    od = [torch.from_numpy(np.ascontiguousarray(o)).cuda() for o in ops]
    out = torch.full(info["out"], float("nan"), device="cuda")
    bs.bs_execute_ex(plan, [xd] + od, out)
    torch.cuda.synchronize()
    return out.cpu().numpy(), plan


def no_zero_sign(a):
    a = np.array(a, dtype=np.float32, copy=True)
    a[a == 0] = 0.0
    return a


# ----------------------------------------------------------------------------- wide planes
WIDE = [
    # (shape, layers builder, citation of the case in VERDICT/ADVICE)
    ((1, 1, 3, 7999), lambda C: [synth.relu(), synth.maxpool(3, 2)]),
    ((2, 2, 40, 601), lambda C: [synth.maxpool(3, 1, 1), synth.batchnorm(C, 5), synth.relu()]),
    ((1, 2, 11, 1501), lambda C: [synth.batchnorm(C, 6, signed_gamma=True), synth.relu(), synth.maxpool(3, 2, 1)]),
    ((1, 2, 5, 1027), lambda C: [synth.relu(), synth.maxpool(3, 2)]),                 # Wo = 513
    ((1, 1, 8, 1030), lambda C: [synth.maxpool(3, 1, 1)]),                             # n_cc = 33
    ((1, 1, 4, 1031), lambda C: [synth.maxpool(2, 2)]),
    ((2, 3, 9, 1111), lambda C: [synth.batchnorm(C, 7), synth.relu(), synth.avgpool(3, 2, 1)]),
    ((1, 2, 7, 3591), lambda C: [synth.relu(), synth.avgpool(7, 7)]),                 # Wo = 513
]


@pytest.mark.parametrize("case", range(len(WIDE)))
def test_wide_planes(case, cuda_dev, oracle_lib):
    bs = _bs()
    shape, build = WIDE[case]
    layers = build(shape[1])
    x = synth.uniform_np(1000 + case, int(np.prod(shape))).reshape(shape)
    ref = oracle.run_bf(layers, x)
    kernels = set()
    for opts in (None, {"force_generic": 3}, {"force_generic": 3, "force_outputs_per_group": 3},
                 {"force_generic": 3, "force_rows_per_task": 1}, {"force_generic": 2}, {"force_generic": 1}):
        got, plan = run_gpu(layers, x, opts=opts)
        U.check(got, ref, layers, f"{shape} {[L.kind for L in layers]} {opts}")
        kernels.add(bs.bs_plan_query_launch(plan, 0)["kernel_name"])
    assert "pool_staged_tma" in kernels


def test_staged_many_items_forced(cuda_dev, oracle_lib):
    """Narrow forced column groups (1-3 output columns per lane group, G = 32/J planes per warp):
    5-13 column chunks x up to 13 row bands, far more than 16 items per tile."""
    bs = _bs()
    shape = (4, 16, 27, 27)
    layers = [synth.relu(), synth.maxpool(3, 2)]
    x = synth.uniform_np(77, int(np.prod(shape))).reshape(shape)
    ref = oracle.run_bf(layers, x)
    for opg in (1, 2, 3):
        for rows in (0, 1, 4):
            opts = {"force_generic": 3, "force_outputs_per_group": opg, "force_rows_per_task": rows}
            got, plan = run_gpu(layers, x, opts=opts)
            li = bs.bs_plan_query_launch(plan, 0)
            assert li["kernel_name"] == "pool_staged_tma", li
            U.assert_bitexact(got, ref, f"opg {opg} rows {rows}")


# ----------------------------------------------------------------------------- input variants
def _variant_cases():
    out = []
    for wl in ("c1", "alexnet", "vgg16", "resnet50", "densenet121", "resnet50_residual"):
        cases = synth.workload(wl, batch=2)
        if wl == "densenet121":   # every distinct stack kind: stem, norm1/norm2 of each block, transitions, final
            keep = {0, 1, 2, len(cases) - 1}
            keep |= {i for i, c in enumerate(cases) if c.name.endswith("_t1") or c.name.endswith("_t2")
                     or c.name.endswith("_t3") or c.name.endswith("_l1_norm1") or c.name.endswith("_l1_norm2")}
            cases = [c for i, c in enumerate(cases) if i in keep]
        if wl == "resnet50":
            cases = cases[:2] + cases[-1:]
        out += [(wl, c) for c in cases]
    return out


VARIANT_CASES = _variant_cases()


@pytest.mark.parametrize("variant", ["allneg", "ties", "const", "signed_zero"])
def test_input_variants_every_baseline_stack(variant, cuda_dev, oracle_lib):
    for wl, case in VARIANT_CASES:
        n = int(np.prod(case.shape))
        x = synth.variant_np(variant, case.input_seed, n).reshape(case.shape)
        ops = [synth.variant_np(variant, sd, n).reshape(case.shape) for sd in case.operand_seeds]
        got, _ = run_gpu(case.layers, x, ops)
        ref = oracle.run_bf(case.layers, x, ops)
        ctx = f"{variant} {case.name} {case.shape}"
        if variant == "signed_zero" and not U.needs_tolerance(case.layers):
            U.assert_bitexact(no_zero_sign(got), no_zero_sign(ref), ctx)
        else:
            U.check(got, ref, case.layers, ctx)
        if variant == "const" and case.layers[-1].kind in ("maxpool", "avgpool") and len(case.layers) == 2:
            # ReLU -> pool of a positive constant is that constant
            assert np.all(got == x.flat[0]), ctx


@pytest.mark.parametrize("variant", ["allneg", "ties", "signed_zero"])
def test_input_variants_every_kernel_family(variant, cuda_dev, oracle_lib):
    """The variants through each pool kernel family (forced), with a signed-gamma BN prologue."""
    shape = (2, 4, 28, 28)
    n = int(np.prod(shape))
    x = synth.variant_np(variant, 5, n).reshape(shape)
    stacks = [[synth.relu(), synth.maxpool(3, 2)], [synth.maxpool(3, 2, 1)],
              [synth.batchnorm(4, 9, signed_gamma=True), synth.relu(), synth.maxpool(3, 2, 1)],
              [synth.batchnorm(4, 9, signed_gamma=True), synth.maxpool(2, 2)],
              [synth.batchnorm(4, 9, signed_gamma=True), synth.relu(), synth.avgpool(2, 2)],
              [synth.relu(), synth.avgpool(3, 2, 1)], [synth.batchnorm(4, 3), synth.relu(), synth.avgpool(7, 7)]]
    for layers in stacks:
        ref = oracle.run_bf(layers, x)
        for g in (0, 1, 2, 3):
            got, _ = run_gpu(layers, x, opts={"force_generic": g})
            ctx = f"{variant} {[L.kind for L in layers]} generic {g}"
            if variant == "signed_zero" and not U.needs_tolerance(layers):
                U.assert_bitexact(no_zero_sign(got), no_zero_sign(ref), ctx)
            else:
                U.check(got, ref, layers, ctx)


# ----------------------------------------------------------------------------- concurrency
def test_two_threads_two_plans_concurrent(cuda_dev, oracle_lib):
    """AlexNet s1 (~98 KB tiles ring) and s3 (~55 KB) share pool_staged<3,3,2,2,...>: executing
    both from two host threads on two streams, interleaved many times, must give the results of
    a serial run (a per-launch shared-memory attribute set would race here)."""
    bs = _bs()
    cases = synth.workload("alexnet", batch=16)
    picks = [cases[0], cases[2]]
    plans = [bs.bs_plan_create(c.layers, c.shape) for c in picks]
    assert len({bs.bs_plan_query_launch(p, 0)["smem_bytes"] for p in plans}) == 2
    xs = [synth.uniform_torch(c.input_seed, c.shape, device="cuda") for c in picks]
    refs = []
    for p, x in zip(plans, xs):
        y = torch.empty(bs.bs_plan_query(p)["out"], device="cuda")
        bs.bs_execute(p, x, y)
        refs.append(y)
    torch.cuda.synchronize()
    errors = []

    def worker(k):
        try:
            s = torch.cuda.Stream()
            y = torch.empty_like(refs[k])
            for _ in range(200):
                bs.bs_execute(plans[k], xs[k], y, s)
            s.synchronize()
            if not torch.equal(y, refs[k]):
                errors.append(f"thread {k}: result differs")
        except Exception as e:   # noqa: BLE001
            errors.append(f"thread {k}: {e}")

    ts = [threading.Thread(target=worker, args=(k,)) for k in (0, 1, 0, 1)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    # and the serial results are the oracle's (first image)
    for c, x, y in zip(picks, xs, refs):
        U.check(y[:1].cpu().numpy(), oracle.run_bf(c.layers, x[:1].cpu().numpy()), c.layers, c.name)


def test_launch_info_reports_smem(cuda_dev):
    bs = _bs()
    c = synth.workload("alexnet", batch=4)[0]
    li = bs.bs_plan_query_launch(bs.bs_plan_create(c.layers, c.shape), 0)
    assert li["kernel_name"] == "pool_staged_tma"
    assert li["smem_bytes"] >= li["stages"] * li["tile_planes"] * 55 * 55 * 4 and li["stages"] >= 2
    sec = synth.synthetic51(3, batch=2, C=3, H=20)
    li = bs.bs_plan_query_launch(bs.bs_plan_create(sec.layers, sec.shape), 0)
    assert li["kernel_name"] == "sequence_staged_tma" and li["smem_bytes"] > 0


@pytest.mark.parametrize("variant", ["allneg", "ties", "const", "signed_zero"])
def test_input_variants_sequences(variant, cuda_dev, oracle_lib):
    """The variants through the on-chip sequence kernels: the in-place kernel (two-step sweeps with
    -inf pad lanes, single steps, edge selects), the shared-tile kernel and halo tiles.  Max/ReLU-
    only sequences are exact (bit for bit modulo the sign of zero); signed-gamma BN ones within
    tolerance."""
    for shape in ((2, 4, 28, 28), (1, 4, 56, 56), (1, 2, 23, 64)):
        n = int(np.prod(shape))
        x = synth.variant_np(variant, 7, n).reshape(shape)
        exact = [synth.maxpool(3, 1, 1), synth.relu()] * 3 + [synth.maxpool(3, 1, 1)]
        affine = []
        for b in range(5):
            affine += [synth.maxpool(3, 1, 1), synth.batchnorm(shape[1], 40 + b, signed_gamma=b % 2 == 0), synth.relu()]
        for layers in (exact, affine):
            ref = oracle.run_bf(layers, x)
            for opts in (None, {"force_tile_planes": 1}, {"force_rows_per_task": 5}):
                got, _ = run_gpu(layers, x, opts=opts)
                ctx = f"{variant} {shape} {len(layers)} layers {opts}"
                if not U.needs_tolerance(layers):
                    U.assert_bitexact(no_zero_sign(got), no_zero_sign(ref), ctx)
                else:
                    U.check(got, ref, layers, ctx)
