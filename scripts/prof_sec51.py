"""Run the §5.1 network once or a few times (for ncu): python scripts/prof_sec51.py DEPTH POLICY REPS"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_1804_08378_b200 as bs

depth, policy, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
case = synth.synthetic51(depth)
plan = bs.bs_plan_create(case.layers, case.shape, {"max_steps_per_sequence": policy})
x = synth.uniform_torch(case.input_seed, case.shape, device="cuda")
y = torch.empty(case.shape, device="cuda")
for r in range(reps):
    bs.bs_execute(plan, x, y)
torch.cuda.synchronize()
print(bs.bs_plan_query(plan), bs.bs_plan_query_launch(plan, 0))
