"""Run GPU pillarization of the F60 point cloud a few times (profiling driver)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_08739_b200 as F
scene = F.SCENES["F60"]
xy, f = F.generate_points(scene, 42)
w = F.pillar_params(scene.f_in, 128, 42)
ctx = F.Context(0)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    ps = ctx.pillarize(xy, f, 0.32, w)
print("pillars", ps.size())
