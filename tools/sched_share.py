"""Device forward time vs number of blocks (F60, graph replay, L2 flushed): the
intercept is the schedule + PE + launch overhead, the slope the per-block time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2301_08739_b200 as F
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
ctx = F.Context(0, stream=stream.cuda_stream, precision="bf16")
ps = F.make_pillars(F.SCENES["F60"], 42)
n = ps.size()
d_coords = torch.from_numpy(ps.coords).to(dev)
d_feats = torch.from_numpy(ps.features.astype(np.float32)).to(dev)
d_out = torch.empty((n, 128), dtype=torch.float32, device=dev)
d_kept = torch.empty(n, dtype=torch.int32, device=dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
res = {}
noflush = "--noflush" in sys.argv
for nb in (1, 2, 4, 8):
    cfg = F.FwaConfig(n_blocks=nb)
    ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
    for _ in range(5):
        ctx.forward_device(d_coords.data_ptr(), d_feats.data_ptr(), [0, n], cfg, d_out.data_ptr(), d_kept.data_ptr())
    tot = 0.0
    for _ in range(30):
        if not noflush:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ctx.forward_device(d_coords.data_ptr(), d_feats.data_ptr(), [0, n], cfg, d_out.data_ptr(), d_kept.data_ptr())
        b.record(stream)
        b.synchronize()
        tot += a.elapsed_time(b)
    res[nb] = tot / 30
    print(f"n_blocks {nb}: {res[nb] * 1e3:.1f} us")
slope = (res[8] - res[1]) / 7
print(f"per block {slope * 1e3:.1f} us, intercept (schedule + PE + first-block extra) {(res[1] - slope) * 1e3:.1f} us")
