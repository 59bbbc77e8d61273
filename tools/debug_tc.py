"""Debug driver: one bf16 fast-path block on random rows (run under compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_08739_b200 as F
import oracle as O
G = int(sys.argv[1]) if len(sys.argv) > 1 else 69
rng = np.random.default_rng(0)
rec = F.init_backbone_params(F.FwaConfig(group_size=G), 3)[:16 + 4 * 132480]
ng = 3
f = rng.normal(size=(ng * G, 128)).astype(np.float32)
pe = (0.3 * rng.normal(size=(ng * G, 128))).astype(np.float32)
ctx = F.Context(0, precision="bf16")
try:
    got = ctx.fwa_block_forward(f, pe, rec, ng)
    want = O.port_block_forward(f, pe, ng, rec)
    print("rel err", O.max_rel_err(got, want))
    print("got[0,:8]", got[0, :8]); print("want[0,:8]", want[0, :8])
except Exception as e:
    print("ERROR", type(e).__name__, e)
