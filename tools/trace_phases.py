"""Run one F60 backbone forward with FWA_B200_TRACE=1 and print per-phase SM-clock
durations of the tcgen05 kernels (last traced block)."""
import ctypes as C, os, sys
os.environ["FWA_B200_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_08739_b200 as F
ctx = F.Context(0)
cfg = F.FwaConfig()
ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
ps = F.make_pillars(F.SCENES["F60"], 42)
ps32 = F.PillarSet(ps.coords, ps.features.astype(np.float32))
for _ in range(3):
    ctx.run_backbone(ps32, cfg)
buf = np.zeros(2 * 148 * 64, np.uint64)
F.lib().fwa_b200_debug_trace.argtypes = [C.c_void_p, C.c_void_p]
rc = F.lib().fwa_b200_debug_trace(ctx._h, buf.ctypes.data)
assert rc == 0, rc
t = buf.reshape(2, 148, 64).astype(np.int64)
def rel(a, cta): return (a - t[a_k][cta][0]) if False else a
for k, name in ((0, "ln1_qkv"), (1, "outproj_ffn")):
    print(f"== {name} (SM clocks relative to CTA start; cta 0 / 77 / 147)")
    for cta in (0, 77, 147):
        row = t[k][cta]
        base = row[0]
        nz = [(i, int(v - base)) for i, v in enumerate(row) if v]
        print(f"cta {cta}: " + " ".join(f"{i}:{v}" for i, v in nz))
