"""One stack, fused (libbrainslug) then layer-by-layer (torch eager), for an ncu DRAM-bytes
comparison ("DRAM bytes per stack vs a layer-by-layer baseline").
usage: python scripts/prof_lbl.py WORKLOAD IDX"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F
import synth
import paper_1804_08378_b200 as bs

wl, idx = sys.argv[1], int(sys.argv[2])
case = synth.workload(wl)[idx]
plan = bs.bs_plan_create(case.layers, case.shape)
x = synth.uniform_torch(case.input_seed, case.shape, device="cuda")
y = torch.empty(bs.bs_plan_query(plan)["out"], device="cuda")
torch.cuda.synchronize()
bs.bs_execute(plan, x, y)                       # fused: one launch
torch.cuda.synchronize()
t = x
for L in case.layers:                           # layer by layer: one launch per layer
    if L.kind == "batchnorm":
        t = F.batch_norm(t, torch.from_numpy(L.mean).cuda(), torch.from_numpy(L.var).cuda(),
                         torch.from_numpy(L.gamma).cuda(), torch.from_numpy(L.beta).cuda(), False, 0.0, L.eps)
    elif L.kind == "relu":
        t = F.relu(t)
    elif L.kind == "maxpool":
        t = F.max_pool2d(t, L.kernel, L.stride, L.padding)
    elif L.kind == "avgpool":
        t = F.avg_pool2d(t, L.kernel, L.stride, L.padding, count_include_pad=L.count_include_pad)
torch.cuda.synchronize()
print(case.name, case.shape, "fused vs torch max |diff|", (t - y).abs().max().item())
