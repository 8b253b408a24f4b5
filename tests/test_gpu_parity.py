"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north_star): bit-exact for stacks of max-pool / ReLU / COPY (and the
single-rounding SCALE / ADD), |gpu - ref| <= 1e-6 + 1e-5 |ref| with BatchNorm or AvgPool.
"""
import random

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


def run_gpu(layers, x, ops=(), opts=None, dev="cuda:0"):
    bs = _bs()
    plan = bs.bs_plan_create(layers, x.shape, opts)
    info = bs.bs_plan_query(plan)
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    od = [torch.from_numpy(np.ascontiguousarray(o)).to(dev) for o in ops]
    out = torch.full(info["out"], float("nan"), device=dev)
    bs.bs_execute_ex(plan, [xd] + od, out)
    torch.cuda.synchronize()
    return out.cpu().numpy(), plan


def compare(layers, x, ops=(), opts=None, ctx=""):
    got, plan = run_gpu(layers, x, ops, opts)
    ref = oracle.run_bf(layers, x, ops)
    U.check(got, ref, layers, ctx)
    return got, plan


# ----------------------------------------------------------------------------- fixtures / configs
@pytest.mark.parametrize("case", U.load_golden(), ids=lambda c: c[0])
def test_golden_gpu(case, cuda_dev, oracle_lib):
    name, layers, x, ops, exp, cite = case
    got, _ = run_gpu(layers, x, ops)
    U.assert_bitexact(got, exp, f"{name} ({cite})")


@pytest.mark.parametrize("wl", synth.WORKLOADS)
def test_baseline_configs_reduced_batch(wl, cuda_dev, oracle_lib):
    """Every stack of every BASELINE.json config at batch 2 (full C, H, W), all elements."""
    cases = synth.workload(wl, batch=2)
    if wl == "densenet121":   # 121 stacks: every distinct (layers, shape) kind, a spread of sizes
        cases = cases[:3] + cases[3:-1:9] + cases[-2:]
    for case in cases:
        x = synth.uniform_np(case.input_seed, int(np.prod(case.shape))).reshape(case.shape)
        ops = [synth.uniform_np(sd, int(np.prod(case.shape))).reshape(case.shape) for sd in case.operand_seeds]
        compare(case.layers, x, ops, ctx=case.name)


def test_c1_full(cuda_dev, oracle_lib):
    case = synth.workload("c1")[0]
    x = synth.uniform_np(case.input_seed, int(np.prod(case.shape))).reshape(case.shape)
    got, plan = compare(case.layers, x, ctx="c1")
    assert got.shape == (1, 16, 16, 16)


@pytest.mark.parametrize("wl", ["alexnet", "vgg16", "resnet50", "densenet121", "resnet50_residual"])
def test_full_size_sampled(wl, cuda_dev, oracle_lib):
    """BASELINE.json batch sizes in the launch configuration bench.py times; the oracle
    checks sampled images (every image is an independent unit of the stack)."""
    bs = _bs()
    cases = synth.workload(wl)
    pick = {"alexnet": [0, 1, 2], "vgg16": [0, 2], "resnet50": [0, 1, 7],
            "densenet121": [0, 1, 60, 119, 120], "resnet50_residual": [0, 1, 2, 3]}[wl]
    for idx in pick:
        case = cases[idx]
        N = case.shape[0]
        x = synth.uniform_torch(case.input_seed, case.shape, device="cuda")
        ops = [synth.uniform_torch(sd, case.shape, device="cuda") for sd in case.operand_seeds]
        plan = bs.bs_plan_create(case.layers, case.shape)
        out = torch.empty(bs.bs_plan_query(plan)["out"], device="cuda")
        bs.bs_execute_ex(plan, [x] + ops, out)
        torch.cuda.synchronize()
        for n in sorted({0, N // 2, N - 1}):
            xs = x[n:n + 1].cpu().numpy()
            ref = oracle.run_bf(case.layers, xs, [o[n:n + 1].cpu().numpy() for o in ops])
            U.check(out[n:n + 1].cpu().numpy(), ref, case.layers, f"{case.name} image {n}")
        assert torch.isfinite(out).all()
        del x, out


@pytest.mark.parametrize("wl", ["alexnet", "vgg16", "resnet50", "densenet121", "resnet50_residual"])
def test_full_size_every_element(wl, cuda_dev):
    """Every stack of every BASELINE.json config at its full batch, in bench.py's launch
    configuration, EVERY output element against the definition computed with torch library ops
    on the GPU (fp64 per layer): bit-exact for max/ReLU stacks (modulo the sign of zero), within
    the north_star tolerance otherwise."""
    bs = _bs()
    seen = set()
    for case in synth.workload(wl):
        if case.name in seen:
            continue
        seen.add(case.name)
        x = synth.uniform_torch(case.input_seed, case.shape, device="cuda")
        ops = [synth.uniform_torch(sd, case.shape, device="cuda") for sd in case.operand_seeds]
        plan = bs.bs_plan_create(case.layers, case.shape)
        out = torch.empty(bs.bs_plan_query(plan)["out"], device="cuda")
        bs.bs_execute_ex(plan, [x] + ops, out)
        ref = U.torch_definition(case.layers, x, ops)
        torch.cuda.synchronize()
        if U.needs_tolerance(case.layers):
            err = (out.double() - ref.double()).abs() - (1e-6 + 1e-5 * ref.double().abs())
            assert float(err.max()) <= 0, f"{case.name}: max excess {float(err.max())}"
        else:
            bad = (out != ref) & ~((out == 0) & (ref == 0))
            assert int(bad.sum()) == 0, f"{case.name}: {int(bad.sum())} mismatches"
        del x, ops, out, ref, plan
        torch.cuda.empty_cache()


# ----------------------------------------------------------------------------- geometry coverage
ODD = [1, 2, 3, 5, 7, 13, 27, 55]
WIDTHS = [1, 2, 3, 4, 5, 7, 8, 12, 13, 14, 27, 28, 55, 56]   # even widths reach the vector walker


@pytest.mark.parametrize("pool", [(2, 2, 0), (3, 2, 0), (3, 2, 1), (3, 1, 1), (7, 7, 0), (2, 1, 1), (5, 3, 2),
                                  (1, 2, 0), (4, 4, 1)])
@pytest.mark.parametrize("kind", ["maxpool", "avgpool"])
def test_odd_shapes(pool, kind, cuda_dev, oracle_lib):
    k, s, p = pool
    rng = random.Random(k * 100 + s * 10 + p)
    n = 0
    for H in ODD:
        for W in WIDTHS:
            if H + 2 * p < k or W + 2 * p < k:
                continue
            shape = (2, 3, H, W)
            L = (synth.maxpool if kind == "maxpool" else synth.avgpool)(k, s, p)
            L.count_include_pad = rng.random() < 0.5
            layers = [synth.batchnorm(3, 777 + H, signed_gamma=True), synth.relu() if rng.random() < .5 else synth.copy(), L]
            x = synth.uniform_np(H * 100 + W, int(np.prod(shape))).reshape(shape)
            compare(layers, x, ctx=f"{kind} k{k}s{s}p{p} {H}x{W}")
            for g in (0, 1, 2, 3):
                compare(layers, x, opts={"force_generic": g, "force_rows_per_task": rng.randint(1, 5)},
                        ctx=f"{kind} k{k}s{s}p{p} {H}x{W} generic={g}")
            n += 1
    assert n > 0


def test_padding_hazard_negative_gamma(cuda_dev, oracle_lib):
    """H5: BN with negative gamma before a padded max-pool must not see +inf from padding."""
    shape = (4, 8, 17, 23)
    x = synth.uniform_np(5, int(np.prod(shape))).reshape(shape)
    L = synth.batchnorm(8, 31, signed_gamma=True)
    for p in (synth.maxpool(3, 2, 1), synth.maxpool(3, 1, 1), synth.avgpool(3, 2, 1)):
        got, _ = compare([L, p], x, ctx=p.kind)
        assert np.all(np.isfinite(got))


def test_tile_invariance(cuda_dev, oracle_lib):
    """The output must not depend on the tiling: bit-identical across forced tiles
    and, for max stacks, across every kernel family.  Avg-pool sums are bit-identical within a
    kernel family; across families the summation order differs (row- vs column-first), so
    there they agree within the north_star tolerance."""
    for shape in [(3, 5, 55, 55), (2, 3, 56, 112)]:
        C = shape[1]
        x = synth.uniform_np(9, int(np.prod(shape))).reshape(shape)
        stacks = ([synth.relu(), synth.maxpool(3, 2)],
                  [synth.batchnorm(C, 1), synth.relu(), synth.maxpool(3, 2, 1)],
                  [synth.batchnorm(C, 2), synth.relu(), synth.avgpool(2, 2), synth.scale(0.5)],
                  [synth.batchnorm(C, 3, signed_gamma=True), synth.relu(), synth.maxpool(3, 2)])
        for layers in stacks:
            ref, _ = run_gpu(layers, x)
            for opts in ({"force_rows_per_task": 1}, {"force_rows_per_task": 3}, {"force_rows_per_task": 7},
                         {"force_outputs_per_group": 1}, {"force_outputs_per_group": 5},
                         {"force_outputs_per_group": 6, "force_rows_per_task": 2},
                         {"force_generic": 1}, {"force_generic": 2}, {"force_generic": 2, "force_rows_per_task": 5},
                         {"force_generic": 3}, {"force_generic": 3, "force_outputs_per_group": 4},
                         {"force_generic": 1, "force_outputs_per_group": 3}):
                got, _ = run_gpu(layers, x, opts=opts)
                ctx = f"{shape} {[L.kind for L in layers]} {opts}"
                if any(L.kind == "avgpool" for L in layers):
                    U.assert_close(got, ref, ctx)   # kernel families sum in different orders
                else:
                    U.assert_bitexact(got, ref, ctx)
            # within one kernel family avg sums are bit-identical across tilings
            bs = _bs()
            for fam in (1, 2, 3):
                base, bplan = run_gpu(layers, x, opts={"force_generic": fam})
                for extra in ({"force_rows_per_task": 2}, {"force_rows_per_task": 5},
                              {"force_outputs_per_group": 4}):
                    got, plan = run_gpu(layers, x, opts={"force_generic": fam, **extra})
                    if bs.bs_plan_query_launch(plan, 0)["kernel"] != bs.bs_plan_query_launch(bplan, 0)["kernel"]:
                        continue   # the forced tile left the family (e.g. too many planes to stage)
                    U.assert_bitexact(got, base, f"{shape} {[L.kind for L in layers]} family {fam} {extra}")


@pytest.mark.parametrize("trial", range(60))
def test_random_stacks(trial, cuda_dev, oracle_lib):
    rng = random.Random(4000 + trial)
    shape = (rng.randint(1, 3), rng.randint(1, 6), rng.randint(1, 40), rng.randint(1, 40))
    layers, n_ops = U.random_stack(rng, shape, max_depth=rng.choice([3, 8, 20]),
                                   max_pools=rng.choice([1, 2, 4]), seed_base=60000 + 50 * trial)
    shapes = oracle.layer_shapes(layers, shape, n_ops)
    x, ops = U.make_inputs(layers, shape, n_ops, 123 + trial, shapes)
    for policy in (0, 1):   # on-chip sequences and one launch per step
        compare(layers, x, ops, opts={"max_steps_per_sequence": policy},
                ctx=f"trial {trial} policy {policy} {[L.kind for L in layers]} {shape}")


def test_multi_sequence_stack(cuda_dev, oracle_lib):
    """Several pools -> several steps -> serialised sequences through plan intermediates."""
    bs = _bs()
    shape = (2, 4, 64, 48)
    layers = []
    for b in range(5):   # §5.1 block: MaxPool3x3/s1/p1 -> BN -> ReLU
        layers += [synth.maxpool(3, 1, 1), synth.batchnorm(4, 100 + b), synth.relu()]
    layers += [synth.maxpool(2, 2), synth.avgpool(3, 2, 1)]
    x = synth.uniform_np(77, int(np.prod(shape))).reshape(shape)
    got, plan = compare(layers, x, ctx="multi")
    info = bs.bs_plan_query(plan)
    assert info["n_steps"] == 7 and info["n_launches"] == 1       # one on-chip sequence
    for policy, launches in ((1, 7), (5, 2), (2, 4)):
        g2, p2 = compare(layers, x, opts={"max_steps_per_sequence": policy}, ctx=f"policy {policy}")
        assert bs.bs_plan_query(p2)["n_launches"] == launches
        U.assert_close(g2, got, f"policy {policy} vs one sequence")   # avg sums differ in order


@pytest.mark.parametrize("depth", [1, 2, 5, 16, 17, 40])
def test_sec51_blocks(depth, cuda_dev, oracle_lib):
    """PAPER.md §5.1: 1-40 blocks of MaxPool3x3/s1/p1 -> BN -> ReLU, under the
    three sequence policies (1 step, <= 5 steps, unlimited)."""
    bs = _bs()
    shape = (2, 3, 20, 20)
    layers = []
    for b in range(depth):
        layers += [synth.maxpool(3, 1, 1), synth.batchnorm(3, 300 + b), synth.relu()]
    x = synth.uniform_np(depth, int(np.prod(shape))).reshape(shape)
    ref = oracle.run_bf(layers, x)
    outs = []
    for policy in (1, 5, 0):
        got, plan = run_gpu(layers, x, opts={"max_steps_per_sequence": policy})
        U.assert_close(got, ref, f"depth {depth} policy {policy}")
        outs.append(got)
        n = bs.bs_plan_query(plan)["n_launches"]
        assert n == {1: depth, 5: -(-depth // 5), 0: 1}[policy], (policy, n)   # whole 20x20 planes: no halo
    U.assert_bitexact(outs[1], outs[0], "policy 5 vs 1")
    U.assert_bitexact(outs[2], outs[0], "unlimited vs 1")


@pytest.mark.parametrize("shape", [(2, 3, 56, 56), (2, 2, 33, 45), (1, 2, 1, 1), (1, 1, 7, 64), (3, 5, 2, 31)])
def test_sec51_fast_path_shapes(shape, cuda_dev, oracle_lib):
    """The sequence kernel's 3x3/s1/p1 fast path (k_seq.cu) on widths spanning 1-2 column
    chunks and degenerate planes, under on-chip and 5-step policies."""
    layers = []
    for b in range(3):
        layers += [synth.maxpool(3, 1, 1), synth.batchnorm(shape[1], 300 + b, signed_gamma=b == 1), synth.relu()]
    layers += [synth.maxpool(3, 1, 1)]                    # last step: no epilogue
    x = synth.uniform_np(sum(shape), int(np.prod(shape))).reshape(shape)
    ref = oracle.run_bf(layers, x)
    for policy in (0, 5, 2):
        got, _ = run_gpu(layers, x, opts={"max_steps_per_sequence": policy})
        U.assert_close(got, ref, f"{shape} policy {policy}")


def test_sec51_full_shape_sampled(cuda_dev, oracle_lib):
    """The §5.1 network at DESIGN.md's benchmark shape (128, 64, 56, 56), depth 16 (one
    on-chip sequence), images checked against the oracle one by one."""
    bs = _bs()
    case = synth.synthetic51(16)
    x = synth.uniform_torch(case.input_seed, case.shape, device="cuda")
    plan = bs.bs_plan_create(case.layers, case.shape)
    assert bs.bs_plan_query(plan)["n_launches"] == 1
    out = torch.empty(bs.bs_plan_query(plan)["out"], device="cuda")
    bs.bs_execute(plan, x, out)
    torch.cuda.synchronize()
    for n in (0, 77, 127):
        ref = oracle.run_bf(case.layers, x[n:n + 1].cpu().numpy())
        U.check(out[n:n + 1].cpu().numpy(), ref, case.layers, f"image {n}")


def test_long_elementwise_runs_split(cuda_dev, oracle_lib):
    shape = (2, 3, 9, 11)
    layers = [synth.scale(1.5), synth.relu(), synth.scale(-0.5)] * 6 + [synth.maxpool(2, 2)] + \
             [synth.relu(), synth.scale(3.0)] * 5
    x = synth.uniform_np(1, int(np.prod(shape))).reshape(shape)
    compare(layers, x, ctx="long")


# ----------------------------------------------------------------------------- ADD operands
def test_residual_add_stacks(cuda_dev, oracle_lib):
    """NEXT-1 shape: BN -> ADD -> ReLU (ResNet bottleneck tail) and ADD around a pool."""
    for shape in [(4, 16, 14, 14), (3, 7, 13, 9), (2, 3, 1, 5)]:
        C = shape[1]
        layers = [synth.batchnorm(C, 5), synth.add(1), synth.relu()]
        shapes = oracle.layer_shapes(layers, shape, 1)
        x, ops = U.make_inputs(layers, shape, 1, 3, shapes)
        compare(layers, x, ops, ctx=f"bn-add-relu {shape}")
        layers = [synth.add(1), synth.relu(), synth.maxpool(3, 2, 1), synth.scale(2.0), synth.add(2)]
        shapes = oracle.layer_shapes(layers, shape, 2)
        x, ops = U.make_inputs(layers, shape, 2, 4, shapes)
        compare(layers, x, ops, ctx=f"add-pool-add {shape}")


# ----------------------------------------------------------------------------- host path / API
def test_execute_host_matches_device(cuda_dev, oracle_lib):
    bs = _bs()
    for layers, shape, nops in [([synth.batchnorm(6, 1), synth.relu(), synth.maxpool(3, 2, 1)], (7, 6, 21, 19), 0),
                                ([synth.batchnorm(5, 2), synth.add(1), synth.relu()], (9, 5, 7, 7), 1)]:
        shapes = oracle.layer_shapes(layers, shape, nops)
        x, ops = U.make_inputs(layers, shape, nops, 11, shapes)
        plan = bs.bs_plan_create(layers, shape)
        info = bs.bs_plan_query(plan)
        h_in = [torch.from_numpy(a).pin_memory() for a in [x] + ops]
        h_out = torch.empty(info["out"]).pin_memory()
        d_in = [torch.empty_like(t, device="cuda") for t in h_in]
        d_out = torch.empty(info["out"], device="cuda")
        for chunks in (0, 1, 3, 100):
            h_out.fill_(float("nan"))
            bs.bs_execute_host(plan, h_in, h_out, d_in, d_out, chunks)
            torch.cuda.synchronize()
            U.check(h_out.numpy(), oracle.run_bf(layers, x, ops), layers, f"host chunks={chunks}")


def test_execute_host_batch_matches_oracle(cuda_dev, oracle_lib):
    """bs_execute_host_batch: several stacks (one with an ADD operand, one sequence, one empty)
    from host buffers in one pipelined call, each checked against the oracle; device buffers
    shared between executions are rejected with the execution indices named."""
    bs = _bs()
    specs = [([synth.batchnorm(6, 1), synth.relu(), synth.maxpool(3, 2, 1)], (7, 6, 21, 19), 0),
             ([synth.batchnorm(5, 2), synth.add(1), synth.relu()], (9, 5, 7, 7), 1),
             (synth.synthetic51(4, batch=3, C=4, H=24).layers, (3, 4, 24, 24), 0),
             ([synth.relu(), synth.maxpool(2, 2)], (0, 3, 8, 8), 0),
             ([synth.batchnorm(64, 3), synth.relu(), synth.avgpool(7, 7)], (16, 64, 7, 7), 0)]
    plans, h_ins, h_outs, d_ins, d_outs, refs = [], [], [], [], [], []
    for k, (layers, shape, nops) in enumerate(specs):
        if shape[0]:
            x, ops = U.make_inputs(layers, shape, nops, 20 + k, oracle.layer_shapes(layers, shape, nops))
        else:   # the empty batch: a no-op execution in the batch
            x, ops = np.zeros(shape, np.float32), []
        plan = bs.bs_plan_create(layers, shape)
        info = bs.bs_plan_query(plan)
        plans.append(plan)
        h_ins.append([torch.from_numpy(a).pin_memory() for a in [x] + ops])
        h_outs.append(torch.full(info["out"], float("nan")).pin_memory())
        d_ins.append([torch.empty_like(t, device="cuda") for t in h_ins[-1]])
        d_outs.append(torch.empty(info["out"], device="cuda"))
        refs.append((layers, oracle.run_bf(layers, x, ops) if shape[0] else None))
    # the same plan twice (a network's repeated stacks) on its own buffers; and a two-sequence plan
    layers = [synth.relu(), synth.maxpool(3, 2, 1), synth.batchnorm(4, 9), synth.maxpool(2, 2)]
    for k, (ls, shape) in enumerate([(specs[0][0], specs[0][1]), (layers, (3, 4, 30, 30))]):
        x, _ = U.make_inputs(ls, shape, 0, 40 + k, oracle.layer_shapes(ls, shape, 0))
        plan = plans[0] if k == 0 else bs.bs_plan_create(ls, shape, {"max_steps_per_sequence": 1})
        info = bs.bs_plan_query(plan)
        plans.append(plan)
        h_ins.append([torch.from_numpy(x).pin_memory()])
        h_outs.append(torch.full(info["out"], float("nan")).pin_memory())
        d_ins.append([torch.empty_like(h_ins[-1][0], device="cuda")])
        d_outs.append(torch.empty(info["out"], device="cuda"))
        refs.append((ls, oracle.run_bf(ls, x)))
    assert bs.bs_plan_query(plans[-1])["n_launches"] == 2
    for chunks in (0, 1, 4):
        for h in h_outs:
            h.fill_(float("nan"))
        bs.bs_execute_host_batch(plans, h_ins, h_outs, d_ins, d_outs, chunks)
        torch.cuda.synchronize()
        for (layers, ref), h in zip(refs, h_outs):
            if ref is not None:
                U.check(h.numpy(), ref, layers, f"batch chunks={chunks}")
    with pytest.raises(bs.BsError, match="executions 0 and 2"):
        bs.bs_execute_host_batch(plans[:3], h_ins[:3], h_outs[:3], d_ins[:3], [d_outs[0], d_outs[1], d_outs[0]])
    bs.bs_execute_host_batch([], [], [], [], [])


def test_inplace_elementwise(cuda_dev, oracle_lib):
    bs = _bs()
    shape = (2, 6, 13, 13)
    layers = [synth.batchnorm(6, 8), synth.relu()]
    x = synth.uniform_np(2, int(np.prod(shape))).reshape(shape)
    plan = bs.bs_plan_create(layers, shape)
    t = torch.from_numpy(x.copy()).cuda()
    bs.bs_execute(plan, t, t)
    torch.cuda.synchronize()
    U.check(t.cpu().numpy(), oracle.run_bf(layers, x), layers, "inplace")


def test_argument_errors(cuda_dev):
    bs = _bs()
    shape = (2, 4, 8, 8)
    plan = bs.bs_plan_create([synth.relu(), synth.maxpool(2, 2)], shape)
    x = torch.zeros(shape, device="cuda")
    out = torch.zeros((2, 4, 4, 4), device="cuda")
    big = torch.zeros(1000, device="cuda")
    with pytest.raises(bs.BsError) as e:
        bs.bs_execute(plan, big.data_ptr() + 4, out)          # misaligned
    assert e.value.status == 2
    with pytest.raises(bs.BsError) as e:
        bs.bs_execute(plan, x, x)                             # overlap (pool plan: no in-place)
    assert e.value.status == 2
    with pytest.raises(bs.BsError) as e:
        bs.bs_execute_ex(plan, [x, x], out)                   # wrong input count
    assert e.value.status == 2
    hp = bs.bs_plan_create([synth.relu()], shape, {"host_only": 1})
    with pytest.raises(bs.BsError):
        bs.bs_execute(hp, x, x)
    bs.bs_execute(plan, x, out)
    torch.cuda.synchronize()


def test_graph_matches_sequential_execution(cuda_dev, oracle_lib):
    """NEXT-3: a CUDA graph over several stacks (incl. an ADD operand, an on-chip sequence, a
    serialised multi-sequence plan and an empty batch) replays to the oracle's results."""
    bs = _bs()
    cases = []
    for wl, idx in (("alexnet", 0), ("resnet50", 0), ("resnet50_residual", 3), ("densenet121", -1)):
        c = synth.workload(wl, batch=2)[idx]
        cases.append((c.layers, c.shape, len(c.operand_seeds)))
    sec = synth.synthetic51(5, batch=2, C=3, H=17)
    cases.append((sec.layers, sec.shape, 0))
    cases.append(([synth.relu(), synth.maxpool(2, 2)], (0, 3, 8, 8), 0))
    execs, refs, outs = [], [], []
    for k, (layers, shape, n_ops) in enumerate(cases):
        opts = {"max_steps_per_sequence": 2} if layers is sec.layers else None
        plan = bs.bs_plan_create(layers, shape, opts)
        x = synth.uniform_np(50 + k, int(np.prod(shape))).reshape(shape)
        ops = [synth.uniform_np(60 + k + j, int(np.prod(shape))).reshape(shape) for j in range(n_ops)]
        xd = [torch.from_numpy(t).cuda() for t in [x] + ops]
        out = torch.full(bs.bs_plan_query(plan)["out"], float("nan"), device="cuda")
        execs.append((plan, xd, out))
        refs.append((oracle.run_bf(layers, x, ops) if shape[0] else None, layers))
        outs.append(out)
    g = bs.bs_graph_create(execs)
    for _ in range(2):   # replays are idempotent
        bs.bs_graph_launch(g)
    torch.cuda.synchronize()
    for out, (ref, layers) in zip(outs, refs):
        if ref is not None:
            U.check(out.cpu().numpy(), ref, layers, "graph replay")
    bs.bs_graph_destroy(g)


@pytest.mark.parametrize("shape,pool", [((64, 64, 111, 111), (3, 2, 1)), ((96, 48, 57, 57), (2, 2, 0)),
                                        ((32, 256, 27, 27), (3, 1, 1)), ((128, 160, 7, 7), (7, 7, 0)),
                                        ((32, 64, 101, 101), (3, 1, 1)), ((16, 32, 151, 151), (3, 2, 1))])
def test_staged_large_odd_shapes_sampled(shape, pool, cuda_dev, oracle_lib):
    """The staged kernel at sizes where the planner picks one CTA per SM / round-robin tiles /
    padded windows, images checked against the oracle one by one."""
    bs = _bs()
    k, s_, p = pool
    layers = [synth.batchnorm(shape[1], 11, signed_gamma=True), synth.relu(), synth.maxpool(k, s_, p)]
    # (a whole-plane window goes to the plane-reduction kernel by default; force the staged one)
    plan = bs.bs_plan_create(layers, shape, {"force_generic": 3} if k == shape[2] else None)
    assert bs.bs_plan_query_launch(plan, 0)["kernel_name"] == "pool_staged_tma"
    x = synth.uniform_torch(5, shape, device="cuda")
    out = torch.empty(bs.bs_plan_query(plan)["out"], device="cuda")
    bs.bs_execute(plan, x, out)
    torch.cuda.synchronize()
    for n in sorted({0, shape[0] // 3, shape[0] - 1}):
        ref = oracle.run_bf(layers, x[n:n + 1].cpu().numpy())
        U.check(out[n:n + 1].cpu().numpy(), ref, layers, f"{shape} {pool} image {n}")


@pytest.mark.parametrize("budget", [24 * 1024, 40 * 1024, 64 * 1024])
def test_smem_budget_results_unchanged(budget, cuda_dev, oracle_lib):
    """A shared-memory budget changes sequences / kernels, never the results."""
    sec = synth.synthetic51(6, batch=2, C=3, H=41)
    x = synth.uniform_np(31, int(np.prod(sec.shape))).reshape(sec.shape)
    compare(sec.layers, x, opts={"smem_budget_bytes": budget}, ctx=f"sec51 budget {budget}")
    s1 = synth.workload("alexnet", batch=2)[0]
    x = synth.uniform_np(32, int(np.prod(s1.shape))).reshape(s1.shape)
    compare(s1.layers, x, opts={"smem_budget_bytes": budget}, ctx=f"alexnet_s1 budget {budget}")


def test_empty_batch(cuda_dev):
    """An empty batch executes as a no-op through every entry point (NULL pointers allowed)."""
    bs = _bs()
    for layers in ([synth.relu(), synth.maxpool(3, 2)], [synth.batchnorm(4, 9), synth.add(1), synth.relu()]):
        plan = bs.bs_plan_create(layers, (0, 4, 13, 13))
        n_in = bs.bs_plan_query(plan)["n_inputs"]
        x = torch.empty((0, 4, 13, 13), device="cuda")
        out = torch.empty(bs.bs_plan_query(plan)["out"], device="cuda")
        bs.bs_execute_ex(plan, [x] * n_in, out)
        bs.bs_execute_ex(plan, [0] * n_in, 0)
        bs.bs_execute_host(plan, [0] * n_in, 0, [0] * n_in, 0)
        torch.cuda.synchronize()
        assert out.shape[0] == 0


def test_ew_large_tensor_rebasing(cuda_dev, oracle_lib):
    """> 2^31 elements: the element-wise launcher splits at 4-image boundaries."""
    bs = _bs()
    shape = (36, 64, 1024, 1024)  # 2.4e9 elements, 9.7 GB per tensor
    C = shape[1]
    layers = [synth.batchnorm(C, 3), synth.relu()]
    plan = bs.bs_plan_create(layers, shape)
    x = synth.uniform_torch(4242, shape, device="cuda")
    bs.bs_execute(plan, x, x)   # in place
    torch.cuda.synchronize()
    for n in (0, 17, 35):
        # regenerate image n only
        xs = synth.uniform_np(4242, C * 1024 * 1024, start=n * C * 1024 * 1024).reshape(1, C, 1024, 1024)
        U.check(x[n:n + 1].cpu().numpy(), oracle.run_bf(layers, xs), layers, f"image {n}")


# ----------------------------------------------------------------------------- whole-plane pools
@pytest.mark.parametrize("shape", [(3, 5, 7, 7), (2, 7, 8, 8), (1, 3, 5, 5), (2, 33, 4, 4), (1, 40, 1, 1),
                                   (5, 13, 3, 3), (2, 17, 2, 6), (64, 64, 7, 7)])
def test_whole_plane_pools(shape, cuda_dev, oracle_lib):
    """Windows covering the whole plane (global pools, DenseNet-121's final 7x7 average) run the
    plane-reduction kernel (k_pool_planes.cu): odd / even plane sizes (rotated bank walk), partial
    32-plane chunks, every prologue class, max with a sign-flipping BN prologue (not deferred)."""
    bs = _bs()
    C, H, W = shape[1], shape[2], shape[3]
    stacks = [[synth.batchnorm(C, 3), synth.relu(), synth.avgpool((H, W), (H, W))],
              [synth.avgpool((H, W), (H, W))], [synth.relu(), synth.avgpool((H, W), (H, W))],
              [synth.batchnorm(C, 4, signed_gamma=True), synth.maxpool((H, W), (H, W))],
              [synth.relu(), synth.maxpool((H, W), (H, W)), synth.batchnorm(C, 5, signed_gamma=True), synth.relu()],
              [synth.scale(-0.5), synth.avgpool((H, W), (H, W)), synth.scale(3.0)]]
    x = synth.uniform_np(sum(shape), int(np.prod(shape))).reshape(shape)
    for layers in stacks:
        got, plan = compare(layers, x, ctx=f"{shape} {[L.kind for L in layers]}")
        assert bs.bs_plan_query_launch(plan, 0)["kernel_name"] == "pool_planes"
        other, _ = run_gpu(layers, x, opts={"force_generic": 1})
        if not U.needs_tolerance(layers):
            U.assert_bitexact(got, other, f"{shape} planes vs column walker")
