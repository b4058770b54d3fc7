python - <<'PY'
import torch, time
d = torch.device("cuda", 0)
for mb in (80, 160):
    n = mb * 1000 * 1000 // 8
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    g = torch.empty(n, dtype=torch.float64, device=d)
    for name, f in (("h2d", lambda: g.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(g, non_blocking=True))):
        f(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(10): f()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 10
        print(mb, "MB", name, "%.1f GB/s" % (n * 8 / dt / 1e9))
# bidirectional: 80 MB H2D on one stream, 160 MB D2H on another
h1 = torch.empty(10_000_000, dtype=torch.float64).pin_memory(); g1 = torch.empty_like(h1, device=d)
h2 = torch.empty(20_000_000, dtype=torch.float64).pin_memory(); g2 = torch.empty_like(h2, device=d)
s1, s2 = torch.cuda.Stream(d), torch.cuda.Stream(d)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): g1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(g2, non_blocking=True)
torch.cuda.synchronize()
print("bidir 80 MB in + 160 MB out: %.2f ms/step" % ((time.perf_counter() - t) / 10 * 1e3))
PY
