"""Large single frames (F200, F250) through run_backbone: finite features, kept set == the NumPy sort oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_08739_b200 as F
import oracle as O
ctx = F.Context(0, precision="bf16")
cfg = F.FwaConfig()
ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
for name in ("F200", "F250"):
    ps = F.make_pillars(F.SCENES[name], 42)
    t = time.time(); r = ctx.run_backbone(ps, cfg); dt = time.time() - t
    w = 9 * 0.32
    p0 = O.np_sort(ps.coords, w, w, 0, 0)
    n = ps.size(); nk = (n // 69) * 69
    print(name, n, r.features.shape, np.all(np.isfinite(r.features)), np.array_equal(r.kept_indices, np.sort(p0[:nk])), f"{dt*1e3:.1f} ms")
