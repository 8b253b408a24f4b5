"""Host-side checks of the C ABI (no GPU): the library loads and exports every symbol
include/bs.h declares; the planner (host_only plans) validates, groups steps, sizes tiles
and counts algorithmic bytes as the paper and SURVEY.md §8 say."""
import os
import random
import re
import subprocess

import numpy as np
import pytest

import oracle
import synth
from tests import _util as U

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bs():
    from paper_1804_08378_b200 import _build
    _build.build()
    import paper_1804_08378_b200 as pkg
    return pkg


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "bs.h")).read()
    return re.findall(r"BS_API\s+[\w\s\*]+?\b(bs_\w+)\s*\(", txt)


def test_exports_every_declared_symbol(bs):
    syms = header_symbols()
    assert len(syms) == 14, syms   # 10 + bs_graph_create / _launch / _destroy (NEXT-3) + bs_execute_host_batch
    out = subprocess.check_output(["nm", "-D", "--defined-only", bs.LIB_PATH]).decode()
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    for s in syms:
        assert s in exported, s
        assert hasattr(bs._lib, s)
    # nothing but the ABI is exported (hidden visibility for internals)
    assert {e for e in exported if e.startswith("bs_")} == set(syms)
    assert bs.bs_version() == 1
    assert bs.bs_status_string(4) == "BS_ERR_PLANNING"


def test_sm100a_code_only(bs):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", bs.LIB_PATH]).decode()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def host_plan(bs, layers, shape, **opts):
    return bs.bs_plan_create(layers, shape, {"host_only": 1, **opts})


def test_step_grouping_paper_example(bs):
    # lst:finalcode: step_0 = MaxPooling, BatchNorm, ReLU; step_1 = AvgPooling (+AvgNormalization)
    shape = (1, 4, 16, 16)
    layers = [synth.maxpool(2, 2), synth.batchnorm(4, 1), synth.relu(), synth.avgpool(2, 2), synth.batchnorm(4, 2)]
    info = bs.bs_plan_query(host_plan(bs, layers, shape))
    assert (info["n_steps"], info["n_sequences"]) == (2, 1)      # lst:finalcode's sequence_0
    li = bs.bs_plan_query_launch(host_plan(bs, layers, shape), 0)
    assert (li["kernel"], li["groups_per_warp"], li["first_layer"], li["last_layer"]) == (7, 2, 0, 4)
    p = host_plan(bs, layers, shape, max_steps_per_sequence=1)   # one step per launch
    info = bs.bs_plan_query(p)
    assert info["n_steps"] == 2
    l0, l1 = bs.bs_plan_query_launch(p, 0), bs.bs_plan_query_launch(p, 1)
    assert (l0["first_layer"], l0["last_layer"], l0["n_prologue_ops"], l0["n_epilogue_ops"]) == (0, 2, 0, 2)
    assert (l1["first_layer"], l1["last_layer"], l1["n_prologue_ops"], l1["n_epilogue_ops"]) == (3, 4, 0, 1)


@pytest.mark.parametrize("layers,steps", [
    ([synth.relu()], 1),
    ([synth.relu()] * 8, 1),
    ([synth.relu()] * 20, 3),   # > kMaxOps (8) fused ops: split into serialised steps (R6)
    ([synth.batchnorm(3, 1), synth.relu(), synth.maxpool(2, 2)], 1),   # C1
    ([synth.maxpool(3, 1, 1), synth.batchnorm(3, 1), synth.relu()] * 16, 16),  # §5.1 depth 16
    ([synth.relu(), synth.copy(), synth.maxpool(3, 2), synth.maxpool(2, 2)], 2),
])
def test_step_counts(bs, layers, steps):
    p = host_plan(bs, layers, (2, 3, 40, 40))
    assert bs.bs_plan_query(p)["n_steps"] == steps


@pytest.mark.parametrize("depth,policy,seqs", [(16, 5, 4), (16, 1, 16), (16, 0, 1), (40, 0, 1), (40, 5, 8),
                                               (1, 0, 1), (70, 0, 2)])
def test_sequence_packing(bs, depth, policy, seqs):
    """§5.1 blocks [MaxPool3x3/s1/p1, BN, ReLU] x depth: one step per block; the paper's three
    policies -> ceil(depth / limit) sequences (16 blocks, <= 5 -> 4).  Whole
    28x28 planes need no halo, so "unrestricted" is limited only by the 64-step device table."""
    layers = []
    for b in range(depth):
        layers += [synth.maxpool(3, 1, 1), synth.batchnorm(8, b), synth.relu()]
    info = bs.bs_plan_query(host_plan(bs, layers, (4, 8, 28, 28), max_steps_per_sequence=policy))
    assert info["n_steps"] == depth and info["n_sequences"] == seqs and info["n_launches"] == seqs


def test_large_planes_use_halo_tiles(bs):
    """Planes too large to hold whole in shared memory are fused with halo (row-band) tiles: planes
    wider than the in-place kernel's 224 columns, or 224 x 224 planes under a 110 KB budget."""
    layers = [synth.maxpool(3, 1, 1), synth.relu(), synth.maxpool(3, 1, 1)]
    for shape, opts in (((1, 2, 240, 240), {}), ((1, 2, 224, 224), {"smem_budget_bytes": 110 * 1024})):
        p = host_plan(bs, layers, shape, **opts)
        info = bs.bs_plan_query(p)
        li = bs.bs_plan_query_launch(p, 0)
        assert info["n_sequences"] == 1 and li["kernel_name"] == "sequence_staged_tma"
        assert 0 < li["tile_rows"] < shape[2] and li["halo_rows"] > 0
    # 224 x 224 within the default budget: whole planes, in place (one plane per CTA, 8 warps)
    li = bs.bs_plan_query_launch(host_plan(bs, layers, (1, 2, 224, 224)), 0)
    assert li["tile_rows"] == 0 and li["halo_rows"] == 0 and li["block"] == 288 and li["tile_planes"] == 1
    p = host_plan(bs, layers, (1, 2, 56, 56))
    li = bs.bs_plan_query_launch(p, 0)
    assert bs.bs_plan_query(p)["n_sequences"] == 1 and li["tile_rows"] == 0 and li["halo_rows"] == 0


def test_band_tiles_run_in_place(bs):
    """Halo (band) sequences of §5.1-type steps on planes 57..224 wide run in the in-place kernel
    (its two stages hold only the band: no work buffer) with balanced bands; planes wider than 224
    keep the shared-tile kernel (stage + work buffer)."""
    layers = []
    for b in range(6):
        layers += [synth.maxpool(3, 1, 1), synth.batchnorm(2, b), synth.relu()]
    for shape, budget, in_place in (((1, 2, 224, 224), 110 * 1024, True), ((1, 2, 112, 112), 40 * 1024, True),
                                    ((1, 2, 100, 64), 16 * 1024, True), ((1, 2, 240, 240), 0, False)):
        p = host_plan(bs, layers, shape, **({"smem_budget_bytes": budget} if budget else {}))
        li = bs.bs_plan_query_launch(p, 0)
        W = shape[3]
        band_in = li["tile_rows"] + 2 * li["groups_per_warp"]      # output rows + one halo row per step and side
        assert li["tile_rows"] > 0, li
        if in_place:
            assert li["block"] == (288 if W > 128 else 160), li
            assert li["smem_bytes"] <= 2 * (band_in * W * 4 + 16 + 127) + 128 + 6 * 8 * 8 + 1024 + 256, li
            assert li["smem_bytes"] <= (budget or 220 * 1024)
            # balanced bands: every band within one row of the others
            assert -(-shape[2] // li["tile_rows"]) * li["tile_rows"] - shape[2] < -(-shape[2] // li["tile_rows"]), li
        else:
            assert li["block"] == 288 and li["smem_bytes"] > 2 * band_in * W * 4, li   # stages + work buffer


def _sec51_split_depth(W, H, budget=110 * 1024, lanes=256):
    """Independent closed form of the paper's packing rule for §5.1 blocks on H x W
    planes with halo tiles: base tile = ceil(256 / W) output rows (one output per consumer lane),
    each 3x3/s1/p1 block adds one input row above and below; the sequence footprint is two ring
    stages of step 0's input band (each also holds the odd steps' intermediates, which are
    smaller) + one work buffer of the largest even-step intermediate band (fp32)
    + 128 B of barriers + the per-tile table (40 B of row ranges and 8 B of BN scale/shift per
    step, 128-B rounded) + 1 KB slack.  Returns the most blocks one sequence holds."""
    r0 = -(-lanes // W)
    d = 1
    while True:
        n = d + 1
        rows_in = min(H, r0 + 2 * n)                 # step 0's input band for n blocks
        rows_mid = min(H, r0 + 2 * (n - 1))          # the largest intermediate (step 0's output)
        stage = -(-(rows_in * W * 4 + 16) // 128) * 128
        work = -(-(rows_mid * W) // 4) * 4 * 4
        table = -(-(n * 40 + n * 8) // 128) * 128
        if 128 + 2 * stage + work + table + 1024 > budget:
            return d
        d = n


@pytest.mark.parametrize("H,depth,budget", [(224, 40, 110 * 1024), (112, 70, 48 * 1024), (160, 40, 96 * 1024),
                                            (240, 40, 0)])
def test_halo_sequence_split_depth(bs, H, depth, budget):
    """'Unrestricted' (-1) §5.1 networks on planes that do not fit whole under the budget (the in-place
    kernel needs one H x H plane per CTA, > budget here) split where the growing halo band overflows
    the shared-memory budget (the paper's cache-limit artifacts), at the depth the
    closed form gives -- not at a fixed step limit."""
    layers = []
    for b in range(depth):
        layers += [synth.maxpool(3, 1, 1), synth.batchnorm(4, b), synth.relu()]
    opts = {"smem_budget_bytes": budget} if budget else {}
    assert H * H * 4 > (budget or 220 * 1024) or H > 224
    p = host_plan(bs, layers, (2, 4, H, H), max_steps_per_sequence=-1, **opts)
    info = bs.bs_plan_query(p)
    d = _sec51_split_depth(H, H, budget or 110 * 1024)
    assert info["n_sequences"] == -(-depth // d), (d, info)
    li = bs.bs_plan_query_launch(p, 0)
    assert li["groups_per_warp"] == d and li["tile_rows"] >= -(-256 // H)


def test_copy_is_elided(bs):
    p = host_plan(bs, [synth.relu(), synth.copy(), synth.copy(), synth.maxpool(2, 2)], (1, 2, 8, 8))
    assert bs.bs_plan_query(p)["n_ops"] == 2


@pytest.mark.parametrize("wl", synth.WORKLOADS)
def test_alg_bytes_match_survey(bs, wl):
    """One read of the input + one write of the output."""
    for case in synth.workload(wl):
        p = host_plan(bs, case.layers, case.shape)
        info = bs.bs_plan_query(p)
        oshape = oracle.layer_shapes(case.layers, case.shape, len(case.operand_seeds))[-1]
        assert info["out"] == oshape
        # (+ one read of each ADD operand: the NEXT-1 residual stacks)
        assert info["alg_bytes_read"] == 4 * int(np.prod(case.shape)) * (1 + len(case.operand_seeds))
        assert info["alg_bytes_written"] == 4 * int(np.prod(oshape))
        assert info["n_launches"] == 1
    c3 = synth.workload("vgg16")[0]
    info = bs.bs_plan_query(host_plan(bs, c3.layers, c3.shape))
    assert (info["alg_bytes_read"], info["alg_bytes_written"]) == (822083584, 205520896)   # 822.08 / 205.52 MB


def test_shapes_agree_with_oracle_random(bs):
    """Two independent implementations of the shape law / validation must agree."""
    rng = random.Random(5)
    for t in range(300):
        shape = (rng.randint(1, 3), rng.randint(1, 5), rng.randint(1, 60), rng.randint(1, 60))
        layers, n_ops = U.random_stack(rng, shape, max_depth=12, max_pools=5)
        p = host_plan(bs, layers, shape)
        info = bs.bs_plan_query(p)
        assert info["out"] == oracle.layer_shapes(layers, shape, n_ops)[-1]
        assert info["n_inputs"] == 1 + n_ops
        for i in range(info["n_launches"]):
            li = bs.bs_plan_query_launch(p, i)
            if li["kernel"] in (2, 3):
                G, J = li["groups_per_warp"], li["outputs_per_group"]
                gw = (J - 1) * li["pool_sw"] + li["pool_kw"]
                assert 1 <= G and G * gw <= 32
                Ho, Wo = li["out"][2], li["out"][3]
                assert J * -(-Wo // J) >= Wo and li["rows_per_task"] >= 1
                assert li["halo_rows"] == max(0, li["pool_kh"] - li["pool_sh"])


@pytest.mark.parametrize("layers,status,frag", [
    ([synth.maxpool(3, 1, 2)], 3, "layer 0 (maxpool): padding"),
    ([synth.relu(), synth.maxpool(9, 1)], 3, "layer 1 (maxpool): output extent"),
    ([synth.Layer("avgpool", kernel=(2, 2), stride=(0, 1))], 3, "stride"),
    ([synth.relu(), synth.Layer("conv2d")], 4, "layer 1 (conv2d): not optimizable"),
    ([synth.Layer("linear")], 4, "linear"),
    ([synth.add(0)], 3, "operand"),
    ([synth.add(2)], 3, "densely"),
])
def test_validation_errors(bs, layers, status, frag):
    with pytest.raises(bs.BsError) as e:
        host_plan(bs, layers, (1, 2, 5, 5))
    assert e.value.status == status
    assert frag in str(e.value), str(e.value)


def test_bn_validation(bs):
    L = synth.batchnorm(2, 1)
    L.var = np.array([1.0, -0.5], np.float32)
    with pytest.raises(bs.BsError) as e:
        host_plan(bs, [L], (1, 2, 3, 3))
    assert e.value.status == 3 and "running_var[1]" in str(e.value)
    L = synth.batchnorm(2, 1, eps=0.0)
    with pytest.raises(bs.BsError):
        host_plan(bs, [L], (1, 2, 3, 3))


def test_bad_input_shape(bs):
    with pytest.raises(bs.BsError) as e:
        host_plan(bs, [synth.relu()], (1, 0, 3, 3))
    assert e.value.status == 2


def test_host_only_plan_cannot_execute(bs):
    p = host_plan(bs, [synth.relu()], (1, 2, 3, 3))
    with pytest.raises(bs.BsError) as e:
        bs.bs_execute(p, 1 << 20, 1 << 21, stream=0)
    assert e.value.status == 2 and "host_only" in str(e.value)


def test_tile_policy_fills_device(bs):
    """Row banding: enough warp tasks for 148 SMs; bands are multiples of the unroll and keep
    halo re-reads (k - s rows per band) small."""
    for case in synth.workload("alexnet") + synth.workload("vgg16") + synth.workload("resnet50")[:1]:
        li = bs.bs_plan_query_launch(host_plan(bs, case.layers, case.shape), 0)
        if li["kernel"] == 6:   # staged: persistent CTAs over whole-plane tiles
            assert li["n_tasks"] >= 2 * 148 and li["block"] == 288
            continue
        assert li["n_tasks"] >= 148 * 40
        if li["halo_rows"]:
            assert li["halo_rows"] / (li["rows_per_task"] * li["pool_sh"]) <= 1 / 8 + 1e-9


def test_empty_batch_plan(bs):
    """N = 0 (an empty batch) plans the geometry of one image and reports no work."""
    p = host_plan(bs, [synth.batchnorm(3, 5), synth.relu(), synth.maxpool(3, 2, 1)], (0, 3, 13, 13))
    info = bs.bs_plan_query(p)
    assert info["out"] == (0, 3, 7, 7)
    assert (info["n_launches"], info["alg_bytes_read"], info["alg_bytes_written"]) == (0, 0, 0)
    for bad in [(2, 0, 8, 8), (2, 3, 0, 8), (2, 3, 8, 0), (-1, 3, 8, 8)]:
        with pytest.raises(bs.BsError) as e:
            host_plan(bs, [synth.relu()], bad)
        assert e.value.status == 2


def test_graph_argument_errors(bs):
    """bs_graph_create validates every execution like bs_execute_ex (no GPU needed to fail)."""
    import ctypes
    p = host_plan(bs, [synth.relu()], (1, 2, 4, 4))
    with pytest.raises(bs.BsError) as e:
        bs.bs_graph_create([(p, [0], 0)])                       # host_only plan
    assert e.value.status == 2 and "execution 0" in str(e.value)
    h = ctypes.c_void_p()
    st = bs._lib.bs_graph_create(None, 0, None, None, None, ctypes.byref(h))
    assert st == 2 and not h.value
    assert bs._lib.bs_graph_launch(None, None) == 2
    bs._lib.bs_graph_destroy(None)                              # NULL-safe


def test_execute_host_batch_argument_errors(bs):
    """bs_execute_host_batch validates every execution like bs_execute_host, naming its index (no
    GPU needed to fail): host_only plans, NULL arrays, a negative count; an empty batch is a no-op."""
    import ctypes
    good = host_plan(bs, [synth.relu()], (1, 2, 4, 4))
    with pytest.raises(bs.BsError) as e:
        bs.bs_execute_host_batch([good], [[1 << 20]], [1 << 21], [[1 << 22]], [1 << 23], stream=0)
    assert e.value.status == 2 and "execution 0" in str(e.value) and "host_only" in str(e.value)
    bs.bs_execute_host_batch([], [], [], [], [], stream=0)       # nothing to do
    assert bs._lib.bs_execute_host_batch(None, 1, None, None, None, None, None, 0, None) == 2
    assert bs._lib.bs_execute_host_batch(None, -1, None, None, None, None, None, 0, None) == 2
    assert bs._lib.bs_execute_host_batch(None, 0, None, None, None, None, None, 0, None) == 0


def test_staged_ring_policy(bs):
    """Staged pools: tiles sized so the 8 consumer warps share each tile (<= 16 items), and the
    grid sized for ~104 KB of tiles in flight per SM -- one CTA per SM for >= 20 KB tiles with
    >= 12 tiles per SM, two otherwise (measured on B200)."""
    info = {}
    for c in synth.workload("alexnet"):
        p = host_plan(bs, c.layers, c.shape)
        info[c.name] = bs.bs_plan_query_launch(p, 0)
    sms = 148
    assert all(li["kernel"] == 6 for li in info.values())
    assert info["alexnet_s1"]["grid"] == sms and info["alexnet_s2"]["grid"] == sms      # 24 KB tiles
    assert info["alexnet_s3"]["grid"] == 2 * sms                                       # 13.5 KB tiles
    for li in info.values():
        assert 1 <= li["rows_per_task"] <= li["out"][2]


def _build_c_example(bs, tmp_path):
    exe = str(tmp_path / "stack_demo")
    lib_dir = os.path.dirname(bs.LIB_PATH)
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "stack_demo.c"), "-L", lib_dir,
           "-lbrainslug", "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}", "-o", exe]
    subprocess.check_call(cmd)
    return exe


def test_c_abi_usable_from_plain_c(bs, tmp_path):
    """include/bs.h is plain C99 and libbrainslug.so links into a C program (examples/)."""
    assert os.path.exists(_build_c_example(bs, tmp_path))


@pytest.mark.gpu
def test_c_example_runs(bs, tmp_path, cuda_dev):
    out = subprocess.check_output([_build_c_example(bs, tmp_path), "4"]).decode()
    assert "OK" in out and "-> (4,64,56,56)" in out, out


def test_threads_per_block_is_not_configurable(bs):
    with pytest.raises(bs.BsError) as e:
        bs.bs_plan_create([synth.relu()], (1, 1, 4, 4), {"host_only": 1, "threads_per_block": 128})
    assert e.value.status == 2 and "threads_per_block" in str(e.value)


def test_smem_budget_option(bs):
    """smem_budget_bytes caps the shared memory per CTA: on-chip sequences split, staged pools
    drop to fewer stages or to the global-memory walker (the paper's cache budget)."""
    sec = synth.synthetic51(4, batch=2, C=3, H=56)
    assert bs.bs_plan_query(host_plan(bs, sec.layers, sec.shape))["n_launches"] == 1
    # 20 KB: whole 56x56 planes no longer fit (in-place: 2 planes = 25 KB; staged: 3 buffers)
    # -> halo tiles, split where the closed form says
    small = bs.bs_plan_create(sec.layers, sec.shape, {"host_only": 1, "smem_budget_bytes": 20 * 1024})
    d = _sec51_split_depth(56, 56, budget=20 * 1024)
    assert bs.bs_plan_query(small)["n_launches"] == -(-4 // d)
    assert bs.bs_plan_query_launch(small, 0)["tile_rows"] > 0
    tiny = bs.bs_plan_create(sec.layers, sec.shape, {"host_only": 1, "smem_budget_bytes": 4 * 1024})
    assert bs.bs_plan_query(tiny)["n_launches"] == 4            # not even a 2-block band fits
    s1 = synth.workload("alexnet")[0]
    assert bs.bs_plan_query_launch(host_plan(bs, s1.layers, s1.shape), 0)["kernel"] == 6
    p = bs.bs_plan_create(s1.layers, s1.shape, {"host_only": 1, "smem_budget_bytes": 40 * 1024})
    assert bs.bs_plan_query_launch(p, 0)["kernel"] == 2      # 2 x 24 KB stages do not fit 40 KB


@pytest.mark.parametrize("shape,layers", [
    ((1, 1, 3, 7999), [synth.relu(), synth.maxpool(3, 2)]),
    ((1, 1, 9, 2049), [synth.maxpool(3, 1, 1)]),
    ((1, 2, 11, 1501), [synth.relu(), synth.maxpool(3, 2, 1)]),
    ((1, 1, 8, 1030), [synth.maxpool(3, 1, 1)]),
])
def test_wide_plane_plans(bs, shape, layers):
    """Planes wider than 16 column chunks: the staged kernel walks every item
    of a tile (any count), and the launch info reports the ring it runs with."""
    p = host_plan(bs, layers, shape, force_generic=3)
    li = bs.bs_plan_query_launch(p, 0)
    assert li["kernel_name"] == "pool_staged_tma"
    Wo = bs.bs_plan_query(p)["out"][3]
    assert li["outputs_per_group"] * -(-Wo // li["outputs_per_group"]) >= Wo
    assert li["tile_planes"] >= 1 and li["stages"] >= 2
    assert li["smem_bytes"] >= 128 + li["stages"] * li["tile_planes"] * shape[2] * shape[3] * 4


@pytest.mark.parametrize("H,budget", [(224, 110 * 1024), (160, 96 * 1024), (240, 0), (300, 0)])
def test_default_policy_bounds_halo(bs, H, budget):
    """The planner's default (0) stops a halo-tiled sequence once the band no longer covers its
    own input halo: every sequence has halo rows <= band rows per band, and one more step would
    break that (or not fit).  (Planes that do not fit whole under the budget: halo tiles.)"""
    depth = 40
    layers = []
    for b in range(depth):
        layers += [synth.maxpool(3, 1, 1), synth.batchnorm(4, b), synth.relu()]
    opts = {"smem_budget_bytes": budget} if budget else {}
    p = host_plan(bs, layers, (2, 4, H, H), **opts)
    info = bs.bs_plan_query(p)
    assert 1 < info["n_sequences"] < depth
    for k in range(info["n_launches"]):
        li = bs.bs_plan_query_launch(p, k)
        if li["kernel_name"] != "sequence_staged_tma" or li["tile_rows"] == 0:
            continue
        n_bands = -(-H // li["tile_rows"])
        assert li["halo_rows"] <= n_bands * li["tile_rows"], li
        assert 2 * li["groups_per_warp"] <= li["tile_rows"] + 2, li   # 2 halo rows per 3x3/p1 step
    unres = bs.bs_plan_query(host_plan(bs, layers, (2, 4, H, H), max_steps_per_sequence=-1, **opts))
    assert unres["n_sequences"] <= info["n_sequences"]


def test_policy_validation(bs):
    with pytest.raises(bs.BsError) as e:
        bs.bs_plan_create([synth.relu()], (1, 1, 4, 4), {"host_only": 1, "max_steps_per_sequence": -2})
    assert e.value.status == 2
