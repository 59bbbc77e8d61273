"""A/B timing of library builds: F60 frame, 8 blocks, device-resident forward (CUDA graph
replay), L2 flushed before each step; prints ms/frame.  FWA_B200_LIB selects the .so."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2301_08739_b200 as F
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
name = sys.argv[2] if len(sys.argv) > 2 else "F60"
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st)
ctx = F.Context(0, stream=st.cuda_stream)
cfg = F.FwaConfig()
ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
ps = F.make_pillars(F.SCENES[name], 42)
n = ps.size()
dc = torch.from_numpy(ps.coords).to(dev); df = torch.from_numpy(ps.features.astype(np.float32)).to(dev)
do = torch.empty((n, 128), dtype=torch.float32, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
fn = lambda: ctx.forward_device(dc.data_ptr(), df.data_ptr(), [0, n], cfg, do.data_ptr())
for _ in range(5):
    flush.zero_(); fn()
torch.cuda.synchronize()
tot = 0.0
for _ in range(steps):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); fn(); b.record(st)
    torch.cuda.synchronize()
    tot += a.elapsed_time(b)
ctx.set_profiling(True); fn(); p = ctx.profile(); ctx.set_profiling(False)
print(f"{os.path.basename(os.environ.get('FWA_B200_LIB', 'default'))}: {tot / steps:.4f} ms/frame  "
      f"block {p['block_fused'][0] / max(1, p['block_fused'][1]) * 1e3:.1f} us  schedule {p['schedule'][0] * 1e3:.1f} us")
