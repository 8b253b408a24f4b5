"""Time the §5.1 network (depth D, unrestricted policy) under several plan options."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_08378_b200 as bs
import synth
depth = int(sys.argv[1])
case = synth.synthetic51(depth)
dev = torch.device("cuda")
nset = 3
xs = [synth.uniform_torch(case.input_seed + q, case.shape, device=dev) for q in range(nset)]
ys = [torch.empty(case.shape, device=dev) for _ in range(nset)]
for a in sys.argv[2:]:
    o = json.loads(a)
    plan = bs.bs_plan_create(case.layers, case.shape, o)
    li = bs.bs_plan_query_launch(plan, 0)
    for q in range(nset):
        bs.bs_execute(plan, xs[q], ys[q])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(5):
        for q in range(nset):
            bs.bs_execute(plan, xs[q], ys[q])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (5 * nset)
    print(json.dumps({"depth": depth, "opts": o, "us": ms * 1e3, "us_per_block": ms * 1e3 / depth, "grid": li["grid"],
                      "tile_planes": li["outputs_per_group"], "launches": bs.bs_plan_query(plan)["n_launches"]}), flush=True)
