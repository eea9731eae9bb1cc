"""Times the GPU exact filter on the C3 frame at each sigma_s (diagnostic)."""
import sys
import time
sys.path.insert(0, "/root/repo")
import torch
from paper_1505_00077_b200 import gpf, synth
cfg = synth.CONFIGS[3]
img = synth.make(cfg)
d_in = torch.from_numpy(img).cuda()
d_out = torch.empty_like(d_in)
s = torch.cuda.current_stream().cuda_stream
for ss in cfg.sigma_s:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gpf.exact_device(d_in, d_out, cfg.width, cfg.height, ss, cfg.sigma_r, stream=s)
    torch.cuda.synchronize()
    print(f"sigma_s {ss}: {time.perf_counter() - t0:.3f} s")
