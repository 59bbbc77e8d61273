"""FWA_B200_TRACE=1: per-phase SM-clock durations of the fused block kernel (last
f32-input block of an F60 forward), for a few CTAs and the first units."""
import ctypes as C, os, sys
os.environ["FWA_B200_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_08739_b200 as F
ctx = F.Context(0, precision=sys.argv[1] if len(sys.argv) > 1 else "bf16")
cfg = F.FwaConfig()
ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
ps = F.make_pillars(F.SCENES["F60"], 42)
ps32 = F.PillarSet(ps.coords, ps.features.astype(np.float32))
for _ in range(3):
    ctx.run_backbone(ps32, cfg)
buf = np.zeros(2 * 148 * 64, np.uint64)
F.lib().fwa_b200_debug_trace.argtypes = [C.c_void_p, C.c_void_p]
assert F.lib().fwa_b200_debug_trace(ctx._h, buf.ctypes.data) == 0
t = buf.reshape(2, 148, 64).astype(np.int64)[0]
g = buf.reshape(2, 148, 64).astype(np.int64)[0]
e0 = g[:, 63].min()
def st(col): v = (g[:, col] - e0) / 1e3; return f"min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us"
print("fused kernel, global timer relative to the first CTA entry (us):")
for col, nm in ((63, "entry"), (60, "griddep_wait done"), (59, "weights landed"), (61, "unit loop done"), (62, "exit")):
    print(f"  {nm:18s} {st(col)}")
names = ["start", "ln1_ld", "ln1", "qkv", "ep", "att_pre", "halo", "att_post", "P", "ln2", "Ua", "ffn2a", "Ub", "ffn2b", "O", "out"]
for cta in (0, 1, 40, 41, 146, 147):
    row = t[cta]
    print(f"cta {cta}: setup {row[1] - row[0] if row[1] else 0}")
    for u in range(3):
        if 1 + 16 * u + 15 >= 49: break
        b = 1 + 16 * u
        if not row[b]:
            break
        ks = sorted((int(row[b + k]), k) for k in range(0, 16) if row[b + k])
        seg = [(names[k], t - tp) for (tp, _), (t, k) in zip(ks, ks[1:])]
        print("   u%d total %d: " % (u, int(row[b + 15] - row[b])) + " ".join(f"{n}={v}" for n, v in seg))

clk = (t[:, 49] - t[:, 0]).astype(np.float64)
ns = (g[:, 61] - g[:, 59]).astype(np.float64)
ok = (clk > 0) & (ns > 0)
print(f"SM clock inside the unit loop: median {np.median(clk[ok] / ns[ok]) * 1e3:.0f} MHz "
      f"(min {np.min(clk[ok] / ns[ok]) * 1e3:.0f}, max {np.max(clk[ok] / ns[ok]) * 1e3:.0f})")
