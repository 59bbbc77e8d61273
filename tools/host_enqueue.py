"""Host-side enqueue cost of the eager device-resident forward (F60): per call wall time of
fwa_b200_backbone_forward_device (alternating output buffers: no graph replay), and the GPU
time of the same calls.  A host enqueue slower than the GPU work leaves the GPU idle."""
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
dc = torch.from_numpy(ps.coords).to(dev); df = torch.from_numpy(ps.features.astype(np.float32)).to(dev)
outs = [torch.empty((n, 128), dtype=torch.float32, device=dev) for _ in range(2)]
for i in range(4):
    ctx.forward_device(dc.data_ptr(), df.data_ptr(), [0, n], cfg, outs[i % 2].data_ptr())
torch.cuda.synchronize()
K = 30
t_host = []
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record(st)
t0 = time.perf_counter()
for i in range(K):
    t1 = time.perf_counter()
    ctx.forward_device(dc.data_ptr(), df.data_ptr(), [0, n], cfg, outs[i % 2].data_ptr())
    t_host.append(time.perf_counter() - t1)
b.record(st)
t_enq = time.perf_counter() - t0
torch.cuda.synchronize()
gpu = a.elapsed_time(b) / K
print(f"eager: host enqueue {1e3 * np.mean(t_host):.3f} ms/call (min {1e3 * np.min(t_host):.3f}), "
      f"GPU {gpu:.3f} ms/frame back to back, enqueue loop {1e3 * t_enq / K:.3f} ms/call")
