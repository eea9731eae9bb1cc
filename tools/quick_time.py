"""Quick device-resident timing of the plan API (dev tool, not the bench)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1505_00077_b200 import gpf, synth
sizes = [(512, 512), (2048, 2048), (8192, 8192)] if len(sys.argv) < 2 else [tuple(map(int, a.split("x"))) for a in sys.argv[1:]]
for (w, h) in sizes:
    img = synth.rects_image(w, h, max(1, w * h // 65536), 10.0, 3)
    d_in = torch.from_numpy(img).cuda(); d_out = torch.empty_like(d_in)
    for ss in (2.0, 5.0, 50.0):
        plan = gpf.Plan(w, h, ss, 30.0, 20)
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(2): plan.filter_device(d_in, d_out, 1, None, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); n = 3
        for _ in range(n): plan.filter_device(d_in, d_out, 1, None, s)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(f"{w}x{h} ss={ss}: {ms:.3f} ms  {w*h/ms/1e3:.1f} Mpix/s  {ms*1e9/(w*h):.1f} ps/px  ws={plan.workspace_bytes/2**30:.2f} GiB", flush=True)
        plan.close()
