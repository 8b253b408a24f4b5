"""Run one stack of a workload a few times (for ncu): python scripts/prof_one.py WL IDX REPS"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_1804_08378_b200 as bs

wl, idx, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 3
case = synth.workload(wl)[idx]
plan = bs.bs_plan_create(case.layers, case.shape)
info = bs.bs_plan_query(plan)
xs = [synth.uniform_torch(case.input_seed + k, case.shape, device="cuda") for k in range(2)]
y = torch.empty(info["out"], device="cuda")
for r in range(reps):
    bs.bs_execute(plan, xs[r % 2], y)
torch.cuda.synchronize()
print(case.name, bs.bs_plan_query_launch(plan, 0))
