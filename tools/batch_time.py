"""Config 3 on one GPU: 64 F60-spec frames (seeds 42..105) batched through one device-resident
forward; prints ms per batch (median of 5, L2 flushed) for the library in FWA_B200_LIB (A/B)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2301_08739_b200 as F
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st)
nfr = int(sys.argv[1]) if len(sys.argv) > 1 else 64
frames = [F.make_pillars(F.SCENES["F60"], 42 + i) for i in range(nfr)]
coords = np.concatenate([f.coords for f in frames]); feats = np.concatenate([f.features.astype(np.float32) for f in frames])
off = [0]
for f in frames: off.append(off[-1] + f.size())
n = off[-1]
cfg = F.FwaConfig()
ctx = F.Context(0, stream=st.cuda_stream, precision="bf16"); ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
dc = torch.from_numpy(coords).to(dev); df = torch.from_numpy(feats).to(dev)
do = torch.empty((n, 128), dtype=torch.float32, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
fn = lambda: ctx.forward_device(dc.data_ptr(), df.data_ptr(), off, cfg, do.data_ptr())
for _ in range(2): flush.zero_(); fn()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); fn(); b.record(st); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
lib = os.path.basename(os.environ.get("FWA_B200_LIB", "default"))
print(f"{lib}: {np.median(ts):.3f} ms per {nfr}-frame batch ({n / np.median(ts) / 1e3:.1f} M pillars/s)")
