"""racecheck target: one small fused block (G 69) -- the shared-memory hazard checker is slow."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_08739_b200 as F
ctx = F.Context(0, precision="bf16")
cfg = F.FwaConfig(n_blocks=1)
ctx.load_params(cfg, F.init_backbone_params(cfg, 3))
ps = F.make_pillars(F.SceneSpec(4, 200, 300, 2.0, 40.0, 40.0, 300, 2), 5)
r = ctx.run_backbone(ps, cfg)
print("ok", r.features.shape, bool(np.all(np.isfinite(r.features))))
