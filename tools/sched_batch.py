"""The config-3 batch (64 F60-spec frames, 3.94 M pillars) schedule only
(FWA_B200_DEBUG_SCHEDULE_ONLY=1 skips the blocks): for an ncu launch list / per-kernel
split of the window sort at batch scale.  argv[1]: frames (default 64)."""
import os, sys
os.environ.setdefault("FWA_B200_DEBUG_SCHEDULE_ONLY", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2301_08739_b200 as F
nf = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st)
ctx = F.Context(0, stream=st.cuda_stream)
cfg = F.FwaConfig()
ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
frames = [F.make_pillars(F.SCENES["F60"], 42 + i) for i in range(nf)]
off = np.cumsum([0] + [f.size() for f in frames]).tolist()
dc = torch.from_numpy(np.concatenate([f.coords for f in frames])).to(dev)
df = torch.from_numpy(np.concatenate([f.features for f in frames]).astype(np.float32)).to(dev)
do = torch.empty((off[-1], 128), dtype=torch.float32, device=dev)
fn = lambda: ctx.forward_device(dc.data_ptr(), df.data_ptr(), off, cfg, do.data_ptr())
for _ in range(3):
    fn()
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); fn(); b.record(st); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(f"{nf} frames, {off[-1]} pillars: schedule-only forward {np.median(ts):.3f} ms (graph replay, median of 10)")
