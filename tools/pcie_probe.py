"""Raw pinned-memory copy bandwidth of the box (bounds the host-buffer e2e figure of bench.py)."""
import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n // 4, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n // 4, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
a = t(lambda: d.copy_(h, non_blocking=True))
b = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
c = t(both)
print(f"H2D 1 GiB: {n / a / 1e9:.1f} GB/s   D2H 256 MiB: {n / 4 / b / 1e9:.1f} GB/s   both concurrently: {c * 1e3:.1f} ms (H2D-equivalent {n / c / 1e9:.1f} GB/s)")
for mb in (16, 64, 256):
    m = mb << 20
    x = t(lambda: [d[i * m:(i + 1) * m].copy_(h[i * m:(i + 1) * m], non_blocking=True) for i in range(n // m)], 3)
    print(f"H2D in {mb} MiB pieces: {n / x / 1e9:.1f} GB/s")
