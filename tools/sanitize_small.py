"""compute-sanitizer target: small backbones through every fused-kernel shape (G 16..128),
the frame stream and the split path -- memcheck / racecheck / synccheck find nothing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_08739_b200 as F
ctx = F.Context(0, precision="bf16")
for G in (69, 16, 33, 100, 128):
    cfg = F.FwaConfig(group_size=G, n_blocks=2)
    ctx.load_params(cfg, F.init_backbone_params(cfg, 3))
    ps = F.make_pillars(F.SceneSpec(8, 200, 300, 2.0, 60.0, 60.0, 800, 2), 5)
    r = ctx.run_backbone(ps, cfg)
    assert np.all(np.isfinite(r.features))
cfg = F.FwaConfig(n_blocks=2)
ctx.load_params(cfg, F.init_backbone_params(cfg, 3))
frames = [F.make_pillars(F.SceneSpec(8, 200, 300, 2.0, 60.0, 60.0, 800, 2), s) for s in (1, 2, 3)]
outs = ctx.run_frames(frames, cfg)
print("ok", [o.features.shape for o in outs])
