"""In-graph time of the schedule + PE alone (FWA_B200_DEBUG_SCHEDULE_ONLY=1 skips the blocks)."""
import os, sys
os.environ["FWA_B200_DEBUG_SCHEDULE_ONLY"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2301_08739_b200 as F
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
ctx = F.Context(0, stream=stream.cuda_stream, precision="bf16")
ps = F.make_pillars(F.SCENES["F60"], 42)
n = ps.size()
cfg = F.FwaConfig()
ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
d_coords = torch.from_numpy(ps.coords).to(dev)
d_feats = torch.from_numpy(ps.features.astype(np.float32)).to(dev)
d_out = torch.empty((n, 128), dtype=torch.float32, device=dev)
d_kept = torch.empty(n, dtype=torch.int32, device=dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for _ in range(5):
    ctx.forward_device(d_coords.data_ptr(), d_feats.data_ptr(), [0, n], cfg, d_out.data_ptr(), d_kept.data_ptr())
tot = 0.0
for _ in range(50):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    ctx.forward_device(d_coords.data_ptr(), d_feats.data_ptr(), [0, n], cfg, d_out.data_ptr(), d_kept.data_ptr())
    b.record(stream)
    b.synchronize()
    tot += a.elapsed_time(b)
print(f"schedule + PE only (graph, L2 flushed): {tot / 50 * 1e3:.1f} us")
