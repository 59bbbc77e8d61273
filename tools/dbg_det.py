"""Debug: determinism of run_backbone across calls and against the stream API, per precision."""
import numpy as np, sys
sys.path.insert(0, '.')
import paper_2301_08739_b200 as F
prec = sys.argv[1]
with_wide = "--wide" in sys.argv
ctx = F.Context(0, precision=prec)
cfg = F.FwaConfig(n_blocks=4)
ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
frames = [F.make_pillars(F.SCENES[s], seed) for s, seed in (("F10", 1), ("F30", 2), ("F10", 3), ("PINNED", 4), ("F30", 5))]
if with_wide:
    rng = np.random.default_rng(9)
    frames.insert(2, F.PillarSet(rng.uniform(-5000, 5000, size=(3000, 2)), rng.normal(size=(3000, 128))))
ref = [ctx.run_backbone(ps, cfg) for ps in frames]
bad = 0
for rep in range(3):
    for i, ps in enumerate(frames):
        r = ctx.run_backbone(ps, cfg)
        if not (np.array_equal(r.kept_indices, ref[i].kept_indices) and np.array_equal(r.features, ref[i].features)):
            bad += 1; print("run_backbone differs", rep, i)
    outs = ctx.run_frames(frames, cfg)
    for i, o in enumerate(outs):
        if not (np.array_equal(o.kept_indices, ref[i].kept_indices) and np.array_equal(o.features, ref[i].features)):
            bad += 1; print("stream differs", rep, i)
print(prec, "wide" if with_wide else "", "bad", bad)
