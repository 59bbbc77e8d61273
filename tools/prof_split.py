import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2301_08739_b200 as F
from paper_2301_08739_b200.split import DeviceRunner, partition_groups, split_forward_a2a
ps = F.make_pillars(F.SCENES["F250"], 42)
cfg = F.FwaConfig()
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
ctx = F.Context(0, stream=st.cuda_stream)
ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
dev = torch.device("cuda", 0)
dc = torch.from_numpy(ps.coords).to(dev); df = torch.from_numpy(ps.features.astype(np.float32)).to(dev)
def T(f, n=3):
    for _ in range(2): f()
    torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(n): r=f()
    torch.cuda.synchronize(); return (time.perf_counter()-t)/n*1e3, r
r = DeviceRunner(ctx, dc, df, cfg)
t, K = T(lambda: r.begin()); print("begin ms", t)
ng = K // 69; ranges, per = partition_groups(ng, 1)
t, tabs = T(lambda: r.exchange_tables_all(8, ranges, per, 69, 0, 1)); print("tables ms", t)
y = torch.zeros((K, 128), device=dev)
t, _ = T(lambda: r.block(1, 0, ng, r.x_buffer(), y)); print("block ms", t)
t, snd = T(lambda: r.pack(y, tabs[0][0])); print("pack ms", t)
rcv = torch.empty_like(snd)
t, _ = T(lambda: rcv.copy_(snd)); print("copy ms", t)
t, _ = T(lambda: r.unpack(rcv, tabs[0][2], r.x_buffer())); print("unpack ms", t)
t, _ = T(lambda: split_forward_a2a(r, 8, 69, 1, 0, lambda d, s: d.copy_(s), lambda d, s, a, b: d.copy_(s), lambda n: torch.empty((n,128), device=dev))); print("a2a total ms", t)
