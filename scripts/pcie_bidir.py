import torch, time
n = 256 << 20
hb1 = torch.empty(n // 4).pin_memory(); hb2 = torch.empty(n // 4).pin_memory()
d1 = torch.empty(n // 4, device="cuda"); d2 = torch.empty(n // 4, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - t0
for r in range(3):
    h = t(lambda: d1.copy_(hb1, non_blocking=True))
    d = t(lambda: hb2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d1.copy_(hb1, non_blocking=True)
        with torch.cuda.stream(s2): hb2.copy_(d2, non_blocking=True)
    b = t(both)
    print(f"H2D {n/h/1e9:.1f} GB/s  D2H {n/d/1e9:.1f} GB/s  both {2*n/b/1e9:.1f} GB/s total ({b*1e3:.2f} ms vs {max(h,d)*1e3:.2f})")
