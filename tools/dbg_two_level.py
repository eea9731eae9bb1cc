import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1505_00077_b200 as g
G = np.load("/root/repo/tests/golden/gpf_golden.npz")
img, ref = G["two_level_sr30/in"], G["two_level_sr30/out"]
out, fb = g.gpf_filter_gpf(img, g.spatial_params(2.0), g.range_params(30.0, 20))
np.set_printoptions(precision=3, suppress=True, linewidth=160)
print(out - ref)
plan = g.Plan(8, 8, 2.0, 30.0, 20)
o32, _ = plan.filter_host(img.astype(np.float32))
print(o32 - ref)
