"""e2e probe: bs_execute_host_batch over the ResNet-50 step at several chunk counts, against
plain pinned copies of the same bytes on two streams (no kernels).  python scripts/e2e_probe.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1804_08378_b200 as bs

cases = synth.workload("resnet50")
counts = {}
for c in cases:
    counts[c.name] = counts.get(c.name, 0) + 1
inst = []
for c in cases:
    inst.append(c)
plans = {c.name: bs.bs_plan_create(c.layers, c.shape) for c in cases}
handles = [plans[c.name] for c in inst]
infos = [bs.bs_plan_query(h) for h in handles]
xs = [[torch.empty(c.shape, device="cuda")] for c in inst]
ys = [torch.empty(i["out"], device="cuda") for i in infos]
max_in = max(int(np.prod(c.shape)) for c in inst)
max_out = max(int(np.prod(i["out"])) for i in infos)
h_in = torch.empty(max_in).pin_memory()
h_out = torch.empty(max_out).pin_memory()
h2d = sum(int(np.prod(c.shape)) * 4 for c in inst)
d2h = sum(int(np.prod(i["out"])) * 4 for i in infos)
st = torch.cuda.Stream()
print("stacks", len(inst), "h2d GB", h2d / 1e9, "d2h GB", d2h / 1e9)


def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


for ch in (0, 2, 8, 31):
    t = timeit(lambda: bs.bs_execute_host_batch(handles, [[h_in]] * len(inst), [h_out] * len(inst), xs, ys, ch, st))
    print(f"batch n_chunks={ch}: {t*1e3:.1f} ms  {256/t:.0f} img/s")
for ch in (0, 8):
    def single():
        for h, x, y in zip(handles, xs, ys):
            bs.bs_execute_host(h, [h_in], h_out, x, y, ch, st)
    t = timeit(single)
    print(f"per-stack calls n_chunks={ch}: {t*1e3:.1f} ms  {256/t:.0f} img/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def copies():
    for x, y, i in zip(xs, ys, infos):
        n = x[0].numel(); m = y.numel()
        with torch.cuda.stream(s1):
            x[0].view(-1).copy_(h_in[:n], non_blocking=True)
        with torch.cuda.stream(s2):
            h_out[:m].copy_(y.view(-1), non_blocking=True)
t = timeit(copies)
print(f"plain copies both directions, two streams: {t*1e3:.1f} ms  {256/t:.0f} img/s")
def h2d_only():
    for x in xs:
        with torch.cuda.stream(s1):
            x[0].view(-1).copy_(h_in[:x[0].numel()], non_blocking=True)
t = timeit(h2d_only)
print(f"H2D only: {t*1e3:.1f} ms ({h2d/t/1e9:.1f} GB/s)")
def d2h_only():
    for y in ys:
        with torch.cuda.stream(s2):
            h_out[:y.numel()].copy_(y.view(-1), non_blocking=True)
t = timeit(d2h_only)
print(f"D2H only: {t*1e3:.1f} ms ({d2h/t/1e9:.1f} GB/s)")
