import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1505_00077_b200._lib as L
if len(sys.argv) > 1:
    L.LIB_PATH = sys.argv[1]
import paper_1505_00077_b200 as g
G = np.load("/root/repo/tests/golden/gpf_golden.npz")
img, ref = G["two_level_sr30/in"], G["two_level_sr30/out"]
out, fb = g.gpf_filter_gpf(img, g.spatial_params(2.0), g.range_params(30.0, 20))
print(sys.argv[1:], "max err", np.abs(out - ref).max())
out, fb = g.gpf_filter_gpf(img, g.spatial_params(2.0), g.range_params(30.0, 19))
print("N=19 (runtime-N build) err vs N=20 golden (expected small-ish):", np.abs(out - ref).max())
