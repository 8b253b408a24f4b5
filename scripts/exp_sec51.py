"""PAPER.md §5.1 on B200: time the synthetic network of 1-40 <MaxPool3x3/s1/p1, BN, ReLU> blocks
(fig:eval:synthetic_scaling) under the paper's three sequence policies (1 step per sequence,
<= 5 steps, unrestricted) against torch eager layer-by-layer on the same GPU.

usage: python scripts/exp_sec51.py [OUT.jsonl] [N C H] [depths,comma,separated] [--no-eager]
(CUDA-graph bursts over rotating buffers > L2; default shape (128, 64, 56, 56))
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F

import paper_1804_08378_b200 as bs
import synth

argv = [a for a in sys.argv[1:] if not a.startswith("--")]
out_path = argv[0] if argv and argv[0] != "-" else None
N, C, H = (int(argv[1]), int(argv[2]), int(argv[3])) if len(argv) >= 4 else (128, 64, 56)
DEPTHS = [int(v) for v in argv[4].split(",")] if len(argv) >= 5 else [1, 2, 4, 8, 12, 16, 17, 20, 24, 32, 40]
EAGER = "--no-eager" not in sys.argv
EXTRA = json.loads(os.environ.get("BS_SEC51_OPTS", "{}"))   # extra plan options (dev sweeps)
dev = torch.device("cuda")
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]


def time_graph(fn, nset, reps=3):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for q in range(nset):
            fn(q)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for q in range(nset):
            fn(q)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        g.replay()
        a.record(st)
        for _ in range(reps):
            g.replay()
        b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (reps * nset)


rows = []
for depth in DEPTHS:
    case = synth.synthetic51(depth, batch=N, C=C, H=H)
    nbytes = 2 * 4 * math.prod(case.shape)
    nset = max(2, int(math.ceil(4 * l2 / nbytes)) + 1)
    xs = [synth.uniform_torch(case.input_seed + q, case.shape, device=dev) for q in range(nset)]
    ys = [torch.empty(case.shape, device=dev) for _ in range(nset)]
    res = {"depth": depth, "shape": list(case.shape), "alg_bytes": nbytes}
    for policy, name in ((1, "1_step"), (5, "max_5_steps"), (-1, "unrestricted"), (0, "planner")):
        plan = bs.bs_plan_create(case.layers, case.shape, {"max_steps_per_sequence": policy, **EXTRA})
        info = bs.bs_plan_query(plan)
        ms = time_graph(lambda q: bs.bs_execute(plan, xs[q], ys[q]), nset)
        li = bs.bs_plan_query_launch(plan, 0)
        res[name] = {"ms": ms, "sequences": info["n_sequences"], "alg_gbs": nbytes / ms / 1e6,
                     "us_per_block": 1e3 * ms / depth, "first_seq_steps": li["groups_per_warp"] if li["kernel"] == 7 else 1,
                     "tile_rows": li["tile_rows"], "tile_planes": li["tile_planes"], "smem": li["smem_bytes"]}
        del plan
    bns = [(torch.from_numpy(L.mean).to(dev), torch.from_numpy(L.var).to(dev), torch.from_numpy(L.gamma).to(dev),
            torch.from_numpy(L.beta).to(dev), L.eps) for L in case.layers if L.kind == "batchnorm"]

    def eager(q):
        t = xs[q]
        for (m, v, g, b, eps) in bns:
            t = F.max_pool2d(t, 3, 1, 1)
            t = F.batch_norm(t, m, v, g, b, False, 0.0, eps)
            t = F.relu(t)
        return t
    if EAGER:
        res["torch_eager"] = {"ms": time_graph(eager, nset)}
        for name in ("1_step", "max_5_steps", "unrestricted", "planner"):
            res[name]["speedup_vs_torch"] = res["torch_eager"]["ms"] / res[name]["ms"]
    res["unrestricted_vs_1_step"] = res["1_step"]["ms"] / res["unrestricted"]["ms"]
    res["planner_vs_1_step"] = res["1_step"]["ms"] / res["planner"]["ms"]
    rows.append(res)
    print(json.dumps(res), flush=True)
    if out_path:
        with open(out_path, "a") as f:
            f.write(json.dumps(res) + "\n")
    del xs, ys
