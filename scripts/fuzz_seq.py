"""Randomized parity sweep of §5.1-type sequences (dev tool; tests/test_gpu_seq.py runs 64 of these):
python scripts/fuzz_seq.py N [SEED] -- random widths (multiples of 4 up to 224), heights, step mixes
and shared-memory budgets; each against the oracle (image 0) and bit for bit against the shared-tile
/ halo kernels (force_tile_planes)."""
import os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_1804_08378_b200 as bs
import synth
from tests import _util as U


def run(layers, x, opts):
    plan = bs.bs_plan_create(layers, x.shape, opts or None)
    out = torch.full(bs.bs_plan_query(plan)["out"], float("nan"), device="cuda")
    bs.bs_execute(plan, torch.from_numpy(np.ascontiguousarray(x)).cuda(), out)
    torch.cuda.synchronize()
    return out.cpu().numpy(), plan


n, seed = int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 1
kinds = {}
for t in range(n):
    rng = random.Random(seed * 100003 + t)
    W = 4 * rng.randint(1, 56)
    H = rng.randint(1, 90) if rng.random() < 0.7 else rng.randint(16, 240)
    C = rng.randint(1, 3)
    layers = []
    for b in range(rng.randint(1, 12)):
        layers.append(synth.maxpool(3, 1, 1))
        if rng.random() < 0.6:
            layers.append(synth.batchnorm(C, 50 + b, signed_gamma=rng.random() < 0.5))
        if rng.random() < 0.6:
            layers.append(synth.relu())
    opts = {"smem_budget_bytes": rng.choice([6, 8, 12, 16, 24, 32, 48, 64, 96]) * 1024} if rng.random() < 0.5 else {}
    if rng.random() < 0.3:
        opts["max_steps_per_sequence"] = rng.choice([-1, 1, 2, 5])
    shape = (1, C, H, W)
    x = synth.uniform_np(seed * 7 + t, int(np.prod(shape))).reshape(shape)
    got, plan = run(layers, x, opts)
    li = bs.bs_plan_query_launch(plan, 0)
    key = (li["kernel_name"], li["block"], li["stages"], li["tile_rows"] > 0)
    kinds[key] = kinds.get(key, 0) + 1
    ctx = f"trial {t} shape {shape} {len(layers)} layers {opts} {li}"
    U.assert_close(got, oracle.run_bf(layers, x), ctx)
    other, _ = run(layers, x, {**opts, "force_tile_planes": 1})
    U.assert_bitexact(got, other, ctx + " vs shared tile / halo")
print("OK", n, "trials;", kinds)
