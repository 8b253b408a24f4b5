"""Randomized parity sweep of general stacks (dev tool; tests/test_gpu_parity.py runs 60 of these):
python scripts/fuzz_stacks.py N [SEED] -- random shapes, layer mixes (BN, ReLU, COPY, SCALE, ADD,
max / avg pools of any geometry), policies and kernel families, each against the oracle."""
import os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_1804_08378_b200 as bs
from tests import _util as U

n, seed = int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 1
kinds = {}
for t in range(n):
    rng = random.Random(seed * 100003 + t)
    shape = (rng.randint(1, 3), rng.randint(1, 6), rng.randint(1, 60), rng.randint(1, 60))
    layers, n_ops = U.random_stack(rng, shape, max_depth=rng.choice([3, 8, 20]), max_pools=rng.choice([1, 2, 4]),
                                   seed_base=70000 + 50 * t)
    shapes = oracle.layer_shapes(layers, shape, n_ops)
    x, ops = U.make_inputs(layers, shape, n_ops, 500 + t, shapes)
    ref = oracle.run_bf(layers, x, ops)
    opts = {"max_steps_per_sequence": rng.choice([0, 0, 1, -1, 3]),
            "force_generic": rng.choice([0, 0, 0, 1, 2, 3])}
    if rng.random() < 0.3:
        opts["smem_budget_bytes"] = rng.choice([8, 16, 32, 64]) * 1024
    plan = bs.bs_plan_create(layers, shape, opts)
    out = torch.full(bs.bs_plan_query(plan)["out"], float("nan"), device="cuda")
    xd = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in [x] + ops]
    bs.bs_execute_ex(plan, xd, out)
    torch.cuda.synchronize()
    for k in range(bs.bs_plan_query(plan)["n_launches"]):
        kn = bs.bs_plan_query_launch(plan, k)["kernel_name"]
        kinds[kn] = kinds.get(kn, 0) + 1
    ctx = f"trial {t} {shape} {[L.kind for L in layers]} {opts}"
    n_round = sum(L.kind in ("batchnorm", "avgpool") for L in layers)
    if n_round <= 1:
        U.check(out.cpu().numpy(), ref, layers, ctx)            # north_star: one BN / average per stack
    else:   # chains of BN / averages: fp32 rounding per op vs fp64 per layer, errors add up
        got = out.cpu().numpy().astype(np.float64)
        bad = np.abs(got - ref) > n_round * (1e-6 + 1e-5 * np.abs(ref)) * 4
        assert not bad.any(), (ctx, got[bad][:3], ref[bad][:3])
print("OK", n, "trials; launches per kernel:", kinds)
