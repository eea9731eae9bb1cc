"""Times tools/one_frame-like runs against alternative builds of the library (diagnostics)."""
import sys, ctypes
sys.path.insert(0, "/root/repo")
import paper_1505_00077_b200._lib as L
if len(sys.argv) > 1:
    L.LIB_PATH = sys.argv[1]
import torch
from paper_1505_00077_b200 import gpf, synth
w = 8192
img = synth.rects_image(w, w, 1024, 10.0, 3)
d_in = torch.from_numpy(img).cuda(); d_out = torch.empty_like(d_in)
plan = gpf.Plan(w, w, 5.0, 30.0, 20)
s = torch.cuda.current_stream().cuda_stream
plan.filter_device(d_in, d_out, 1, None, s)
plan.set_profiling(True)
for _ in range(3): plan.filter_device(d_in, d_out, 1, None, s)
torch.cuda.synchronize()
print(sys.argv[1:] or ["default"], {k: round(v / 3, 3) for k, v in plan.stage_times().items()})
