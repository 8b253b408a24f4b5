"""One small launch of every kernel family through the C ABI, checked against the oracle.

Run under compute-sanitizer (memcheck / racecheck / synccheck / initcheck) on the GPU box:
    compute-sanitizer --tool racecheck python scripts/sanitize_families.py
The shapes are small (the tools slow kernels down 10-100x) but each spans several tiles,
ring wrap-arounds (more tiles than stages per CTA), ragged tails and padded windows, so the
mbarrier + cp.async.bulk rings of pool_staged / seq_staged turn over several times.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1804_08378_b200 as bs  # noqa: E402
import synth  # noqa: E402
from tests import _util as U  # noqa: E402

C = 6
FAMILIES = [
    # (name, layers, shape, opts, expected kernel)
    ("ew", [synth.batchnorm(C, 1), synth.relu()], (3, C, 13, 13), None, "ew_stream"),
    ("ew_add", [synth.batchnorm(C, 2), synth.add(1), synth.relu()], (3, C, 7, 7), None, "ew_stream"),
    ("vec", [synth.batchnorm(C, 3), synth.relu(), synth.maxpool(3, 2, 1)], (3, C, 28, 28), None, "pool_colwalk_vec"),
    ("vec_avg", [synth.batchnorm(C, 4), synth.relu(), synth.avgpool(2, 2)], (3, C, 32, 32), None, "pool_colwalk_vec"),
    ("spec", [synth.relu(), synth.maxpool(3, 2)], (3, C, 27, 27), {"force_generic": 2}, "pool_colwalk_spec"),
    ("spec_add", [synth.add(1), synth.relu(), synth.avgpool(3, 2, 1)], (2, C, 13, 13), {"force_generic": 2},
     "pool_colwalk_spec"),
    ("gen", [synth.batchnorm(C, 5, signed_gamma=True), synth.maxpool(3, 2, 1)], (3, C, 27, 27), {"force_generic": 1},
     "pool_colwalk_generic"),
    ("naive", [synth.relu(), synth.avgpool(33, 1, 16)], (1, 2, 40, 40), None, "pool_naive"),
    ("staged", [synth.relu(), synth.maxpool(3, 2)], (40, 64, 27, 27), {"force_stages": 2, "force_tile_planes": 2},
     "pool_staged_tma"),
    ("staged_pad", [synth.batchnorm(C, 6, signed_gamma=True), synth.relu(), synth.maxpool(3, 2, 1)],
     (4, C, 21, 23), {"force_generic": 3, "force_stages": 2}, "pool_staged_tma"),
    ("staged_wide", [synth.relu(), synth.maxpool(3, 2)], (1, 2, 5, 1027), {"force_generic": 3}, "pool_staged_tma"),
    ("staged_avg7", [synth.batchnorm(64, 7), synth.relu(), synth.avgpool(7, 7)], (64, 64, 7, 7),
     {"force_stages": 2, "force_generic": 3}, "pool_staged_tma"),
    ("planes", [synth.batchnorm(64, 7), synth.relu(), synth.avgpool(7, 7)], (65, 64, 7, 7), None, "pool_planes"),
    ("planes_even", [synth.relu(), synth.maxpool(8, 8)], (3, C, 8, 8), None, "pool_planes"),
    ("seq_fast", synth.synthetic51(4, batch=64, C=C, H=20).layers, (64, C, 20, 20), {"force_tile_planes": 1},
     "sequence_staged_tma"),
    ("seq_inplace", synth.synthetic51(4, batch=64, C=C, H=20).layers, (64, C, 20, 20), None, "sequence_staged_tma"),
    ("seq_inplace_wide", synth.synthetic51(3, batch=8, C=C, H=100).layers, (8, C, 100, 100), None,
     "sequence_staged_tma"),
    # planes 129..224 wide: one plane per CTA, two column segments per row with halo lanes
    ("seq_inplace_2seg", synth.synthetic51(3, batch=2, C=C, H=16).layers, (2, C, 16, 160), None,
     "sequence_staged_tma"),
    # rows of 16 lane groups fill a 16-lane segment: edge selects instead of -inf pads -- two-step
    # sweeps (equal row parts) and the one-step kernel (odd height: unequal parts)
    ("seq_inplace_edge", synth.synthetic51(3, batch=8, C=C, H=24).layers, (8, C, 24, 64), None,
     "sequence_staged_tma"),
    ("seq_inplace_onestep", synth.synthetic51(3, batch=8, C=C, H=23).layers, (8, C, 23, 64), None,
     "sequence_staged_tma"),
    ("seq_halo", synth.synthetic51(5, batch=2, C=C, H=64).layers, (2, C, 64, 64), {"force_rows_per_task": 7},
     "sequence_staged_tma"),
    # halo (band) tiles swept in place: planes that do not fit whole under the budget
    ("seq_inplace_bands", synth.synthetic51(7, batch=1, C=C, H=100).layers, (1, C, 100, 64),
     {"smem_budget_bytes": 16384}, "sequence_staged_tma"),
    ("seq_inplace_bands_2seg", synth.synthetic51(4, batch=1, C=2, H=80).layers, (1, 2, 80, 224),
     {"smem_budget_bytes": 40960}, "sequence_staged_tma"),
    ("seq_generic", [synth.maxpool(3, 1, 1), synth.relu(), synth.avgpool(2, 2), synth.batchnorm(C, 8),
                     synth.maxpool(3, 2, 1)], (64, C, 24, 22), {"force_tile_planes": 1}, "sequence_staged_tma"),
]


def main():
    only = sys.argv[1:]
    dev = torch.device("cuda:0")
    for name, layers, shape, opts, kname in FAMILIES:
        if only and name not in only:
            continue
        n_ops = sum(1 for L in layers if L.kind == "add")
        shapes = oracle.layer_shapes(layers, shape, n_ops)
        x, ops = U.make_inputs(layers, shape, n_ops, 17, shapes)
        plan = bs.bs_plan_create(layers, shape, opts)
        li = bs.bs_plan_query_launch(plan, 0)
        assert li["kernel_name"] == kname, (name, li["kernel_name"])
        xd = [torch.from_numpy(t).to(dev) for t in [x] + ops]
        out = torch.empty(bs.bs_plan_query(plan)["out"], device=dev)
        bs.bs_execute_ex(plan, xd, out)
        torch.cuda.synchronize()
        U.check(out.cpu().numpy(), oracle.run_bf(layers, x, ops), layers, name)
        print(f"{name}: {kname} grid {li['grid']} block {li['block']} smem {li['smem_bytes']} OK", flush=True)
        del xd, out
        bs.bs_plan_destroy(plan)             # plan-owned device memory freed before exit (leak check)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()                 # torch's cached blocks too
    print("ALL OK")


if __name__ == "__main__":
    main()
