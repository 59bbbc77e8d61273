"""bf16 backbone max relative error against the golden D128 features (for A/B of numerics
variants via FWA_B200_LIB)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2301_08739_b200 as F
import oracle as O

g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "backbone_d128.npz"))
s = [float(x) for x in g["scene"]]
scene = F.SceneSpec(int(s[0]), int(s[1]), int(s[2]), s[3], s[4], s[5], int(s[6]), int(s[7]))
ps = F.make_pillars(scene, int(g["scene_seed"]))
cfg = F.FwaConfig()
ctx = F.Context(0, precision="bf16")
ctx.load_params(cfg, F.init_backbone_params(cfg, int(g["param_seed"])))
r = ctx.run_backbone(ps, cfg)
print("bf16 max_rel_err vs golden:", O.max_rel_err(r.features, g["features"]),
      "mean abs diff:", float(np.abs(r.features - g["features"]).mean()))
