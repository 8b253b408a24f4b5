"""PAPER.md §5.2 (fig:eval_total_gpu_time) on B200: whole torchvision networks, eager
PyTorch vs the same network with every stack replaced by a BrainSlugStack (frontend.optimize),
batch 128, fp32, random weights (no checkpoints offline).  Convolutions / linear layers run in
cuDNN / cuBLAS in both arms; only the stacks differ.  Context, not the headline.

usage: python scripts/exp_networks.py [OUT.jsonl]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torchvision

from paper_1804_08378_b200 import frontend

out_path = sys.argv[1] if len(sys.argv) > 1 else None
torch.backends.cudnn.benchmark = True


def timed(fn, x, reps=10):
    with torch.no_grad():
        for _ in range(3):
            fn(x)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn(x)
        b.record()
        torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for net in ["alexnet", "vgg16", "resnet50", "densenet121"]:
    torch.manual_seed(0)
    m = getattr(torchvision.models, net)().eval().cuda()
    x = torch.randn(128, 3, 224, 224, device="cuda")
    t_eager = timed(m, x)
    gm = frontend.optimize(m)
    t_bs = timed(gm, x)
    with torch.no_grad():
        err = (gm(x) - m(x)).abs().max().item()
    s = frontend.summary(getattr(torchvision.models, net)().eval())
    r = {"net": net, "batch": 128, "eager_ms": t_eager, "brainslug_ms": t_bs, "speedup": t_eager / t_bs,
         "stacks": s["stacks"], "opt_layers": s["opt_layers"], "max_abs_diff": err}
    print(json.dumps(r), flush=True)
    if out_path:
        with open(out_path, "a") as f:
            f.write(json.dumps(r) + "\n")
    del m, gm
    torch.cuda.empty_cache()
