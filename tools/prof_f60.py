"""Run the F60 backbone a few times through the host API (profiling driver)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_08739_b200 as F
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ps = F.make_pillars(F.SCENES["F60"], 42)
cfg = F.FwaConfig()
ctx = F.Context(0, precision=prec)
ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
for _ in range(n):
    ctx.run_backbone(ps, cfg)
print("done")
