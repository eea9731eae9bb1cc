"""Runs `reps` device-resident frames of the plan API (for ncu launch lists)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1505_00077_b200 import gpf, synth
w = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
ss = float(sys.argv[2]) if len(sys.argv) > 2 else 5.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
img = synth.rects_image(w, w, max(1, w * w // 65536), 10.0, 3)
d_in = torch.from_numpy(img).cuda(); d_out = torch.empty_like(d_in)
plan = gpf.Plan(w, w, ss, 30.0, 20)
s = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    plan.filter_device(d_in, d_out, 1, None, s)
torch.cuda.synchronize()
print("ok", float(d_out.mean()))
