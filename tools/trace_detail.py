"""FWA_B200_TRACE=1 with a detail-trace variant of the fused kernel (slots 33.. = marks of
unit 1, see the variant source): prints each mark's SM clock relative to mark 0 for a
few CTA pairs.  Usage: FWA_B200_LIB=<variant .so> python tools/trace_detail.py name0 name1 ..."""
import ctypes as C, os, sys
os.environ["FWA_B200_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_08739_b200 as F
ctx = F.Context(0, precision="bf16")
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
names = sys.argv[1:]
for cta in range(0, 148, 1):
    row = t[cta]
    if not row[33]:
        continue
    marks = [(k, int(row[33 + k] - row[33])) for k in range(len(names)) if row[33 + k]]
    if cta in (0, 1, 40, 41, 100, 101, 146, 147):
        print(f"cta {cta}: " + " ".join(f"{names[k]}={v}" for k, v in marks))
# pairs on one clock (globaltimer variants: ns): both ranks relative to rank 0's mark 0
if os.environ.get("GT"):
    for cta in (0, 40, 100, 146):
        r0, r1 = t[cta], t[cta + 1]
        print(f"pair {cta // 2} ns, rank0: " + " ".join(f"{names[k]}={int(r0[33 + k] - r0[33])}" for k in range(len(names)) if r0[33 + k]))
        print(f"pair {cta // 2} ns, rank1: " + " ".join(f"{names[k]}={int(r1[33 + k] - r0[33])}" for k in range(len(names)) if r1[33 + k]))
# medians over CTAs of each rank
for rk in (0, 1):
    rows = t[rk::2]
    rows = rows[rows[:, 33] != 0]
    med = [int(np.median(rows[:, 33 + k] - rows[:, 33])) if np.all(rows[:, 33 + k] != 0) else -1 for k in range(len(names))]
    print(f"median rank {rk}: " + " ".join(f"{n}={v}" for n, v in zip(names, med)))
