"""PCIe copy bandwidth on this box: pinned H2D / D2H, one vs two streams, alone and together."""
import torch, time
dev = torch.device("cuda", 0)
n = 63_332_880
h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device=dev)
h2 = torch.empty(31_400_000, dtype=torch.uint8).pin_memory(); d2 = torch.empty(31_400_000, dtype=torch.uint8, device=dev)
s = [torch.cuda.Stream(dev) for _ in range(4)]
def run(fn, reps=20):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
def h2d1():
    with torch.cuda.stream(s[0]): d.copy_(h, non_blocking=True)
def h2d2():
    half = n // 2
    with torch.cuda.stream(s[0]): d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s[1]): d[half:].copy_(h[half:], non_blocking=True)
def h2d4():
    q = n // 4
    for i in range(4):
        with torch.cuda.stream(s[i]): d[i*q:(i+1)*q].copy_(h[i*q:(i+1)*q], non_blocking=True)
def d2h1():
    with torch.cuda.stream(s[2]): h2.copy_(d2, non_blocking=True)
def both():
    h2d1(); d2h1()
for name, fn, b in (("H2D 1 stream", h2d1, n), ("H2D 2 streams", h2d2, n), ("H2D 4 streams", h2d4, n), ("D2H 1 stream", d2h1, h2.numel()), ("H2D+D2H together", both, n)):
    t = run(fn)
    print(f"{name:18s} {t*1e3:7.3f} ms  {b/t/1e9:6.1f} GB/s (H2D bytes)")
