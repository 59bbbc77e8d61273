"""Device time of the fp32 check mode (FWA_PREC_FP32, SIMT fp32 kernels) and of the bf16 fast
path on the F60 frame (device-resident, graph replay, L2 flushed): ms/frame."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2301_08739_b200 as F
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st)
ps = F.make_pillars(F.SCENES["F60"], 42)
n = ps.size()
cfg = F.FwaConfig()
blob = F.init_backbone_params(cfg, 42)
dc = torch.from_numpy(ps.coords).to(dev); df = torch.from_numpy(ps.features.astype(np.float32)).to(dev)
do = torch.empty((n, 128), dtype=torch.float32, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
for prec in ("fp32", "bf16"):
    ctx = F.Context(0, stream=st.cuda_stream, precision=prec)
    ctx.load_params(cfg, blob)
    fn = lambda: ctx.forward_device(dc.data_ptr(), df.data_ptr(), [0, n], cfg, do.data_ptr())
    for _ in range(3):
        flush.zero_(); fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(f"{prec}: {np.median(ts):.3f} ms/frame F60 ({n / np.median(ts) / 1e3:.1f} M pillars/s)")
