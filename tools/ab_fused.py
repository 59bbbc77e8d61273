"""A/B: fused CTA-pair block kernel (precision "bf16") vs the three-kernel pipeline
("bf16_3k") vs the reference port, on F30 (1 block) and F60 (8 blocks); prints errors
and device time per frame."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2301_08739_b200 as F

def run(name, nb, check_port):
    ps = F.make_pillars(F.SCENES[name], 42)
    cfg = F.FwaConfig(n_blocks=nb)
    blob = F.init_backbone_params(cfg, 42)
    outs = {}
    for prec in ("bf16_3k", "bf16"):
        ctx = F.Context(0, precision=prec)
        ctx.load_params(cfg, blob)
        r = ctx.run_backbone(ps, cfg)
        outs[prec] = r
        t0 = time.perf_counter()
        for _ in range(5):
            r2 = ctx.run_backbone(ps, cfg)
        dt = (time.perf_counter() - t0) / 5
        print(f"{name} nb={nb} {prec}: host-api {dt*1e3:.2f} ms  det={np.array_equal(r2.features, r.features)}", flush=True)
    a, b = outs["bf16_3k"].features, outs["bf16"].features
    print(f"{name}: fused vs 3k max_rel_err {O.max_rel_err(b, a):.3e}  kept eq {np.array_equal(outs['bf16'].kept_indices, outs['bf16_3k'].kept_indices)}", flush=True)
    bad = np.argwhere(~np.isclose(b, a, rtol=5e-2, atol=5e-2))
    print("  mismatching rows:", np.unique(bad[:, 0]).size if bad.size else 0, bad[:5].tolist(), flush=True)
    if check_port:
        w = O.port_run_backbone(ps.coords, ps.features.astype(np.float32), O.make_cfg(n_blocks=nb), blob)
        print(f"{name}: fused vs port {O.max_rel_err(b, w['features']):.3e}; 3k vs port {O.max_rel_err(a, w['features']):.3e}", flush=True)

run("F30", 1, True)
run("F60", 8, False)
