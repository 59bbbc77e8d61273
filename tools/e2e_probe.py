"""Streamed e2e (fwa_b200_backbone_forward_frames, f64 host buffers) of N F60 frames, ms per
frame by wall clock, next to the PCIe floor (one frame's H2D and D2H bytes copied concurrently).
FWA_B200_DEBUG_SCHEDULE_ONLY=1 skips the blocks: copies + schedule alone."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2301_08739_b200 as F
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st)
ctx = F.Context(0, stream=st.cuda_stream)
cfg = F.FwaConfig()
ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
ps = F.make_pillars(F.SCENES["F60"], 42)
n = ps.size()
pin = dict(pin_memory=True)
h_c = torch.from_numpy(ps.coords).pin_memory(); h_f = torch.from_numpy(ps.features).pin_memory()
h_o = [torch.empty((n, 128), dtype=torch.float32, **pin) for _ in range(2)]
h_k = [torch.empty(n, dtype=torch.int32, **pin) for _ in range(2)]
h_d = torch.empty(n, dtype=torch.int32, **pin); h_b = torch.empty(8, dtype=torch.int32, **pin)
def call(k):
    fr = [(h_c.data_ptr(), h_f.data_ptr(), n, h_o[i & 1].data_ptr(), h_k[i & 1].data_ptr(), h_d.data_ptr(), h_b.data_ptr()) for i in range(k)]
    return ctx.run_frames_ptrs(fr, True, cfg)
call(3); torch.cuda.synchronize()
for k in (10, 40):
    t0 = time.perf_counter(); call(k); dt = time.perf_counter() - t0
    print(f"{k} frames: {dt / k * 1e3:.4f} ms/frame")
d_f = torch.empty(h_f.numel(), dtype=torch.float64, device=dev); d_o = torch.empty((n, 128), dtype=torch.float32, device=dev)
s2 = torch.cuda.Stream(dev)
def floor(reps=10):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps):
        d_f.copy_(h_f.view(-1), non_blocking=True)
        with torch.cuda.stream(s2): h_o[0].copy_(d_o, non_blocking=True)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
print(f"floor (H2D 62.4 MB + D2H 31.2 MB concurrently): {floor():.4f} ms; H2D alone:", end=" ")
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10): d_f.copy_(h_f.view(-1), non_blocking=True)
torch.cuda.synchronize(); print(f"{(time.perf_counter() - t0) / 10 * 1e3:.4f} ms")
