"""Debug: VGG-16 s1 at batch 64 -- does image 63 of the output match the oracle after graph steps?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import paper_1804_08378_b200 as bs
from tests import _util as U
oracle.build()
dev = torch.device("cuda")
cases = synth.workload("vgg16")
c = cases[0]
plan = bs.bs_plan_create(c.layers, c.shape)
chw = int(np.prod(c.shape[1:]))
x = synth.uniform_torch(c.input_seed, c.shape, device=dev)
torch.cuda.synchronize()
for n in (0, 62, 63):
    xn = synth.uniform_np(c.input_seed, chw, start=n * chw)
    same = np.array_equal(x[n].cpu().numpy().ravel().view(np.uint32), xn.view(np.uint32))
    print("input image", n, "torch==numpy:", same, flush=True)
y = torch.empty(bs.bs_plan_query(plan)["out"], device=dev)
bs.bs_execute(plan, x, y)
torch.cuda.synchronize()
for n in (0, 31, 62, 63):
    ref = oracle.run_bf(c.layers, x[n:n+1].cpu().numpy())
    try:
        U.check(y[n:n+1].cpu().numpy(), ref, c.layers, f"image {n} (input from the GPU tensor)")
        print("image", n, "ok vs oracle(GPU input)", flush=True)
    except AssertionError as e:
        print("FAIL", str(e)[:300], flush=True)
    xn = synth.uniform_np(c.input_seed, chw, start=n * chw).reshape((1,) + c.shape[1:])
    ref2 = oracle.run_bf(c.layers, xn)
    print("   oracle(numpy input) == oracle(GPU input):", np.array_equal(ref, ref2), flush=True)
# fmaxf / max.f32 semantics with signed zeros
a = torch.tensor([-0.0, 0.0, -0.0, 0.0], device=dev)
b = torch.tensor([0.0, -0.0, -0.0, 0.0], device=dev)
print("torch.maximum(-0,+0) sign bits:", torch.signbit(torch.maximum(a, b)).tolist())
