"""Times the bench's e2e leg alone (5 host threads, one per sigma_s plan, pinned
host frames through gpf_b200_filter_f32_host) against an optional alternative build."""
import sys, threading, time
sys.path.insert(0, "/root/repo")
import paper_1505_00077_b200._lib as L
if len(sys.argv) > 1:
    L.LIB_PATH = sys.argv[1]
import torch
from paper_1505_00077_b200 import gpf, synth
cfg = synth.CONFIGS[3]
img = synth.make(cfg)
plans = [gpf.Plan(cfg.width, cfg.height, s, cfg.sigma_r, 20) for s in cfg.sigma_s]
h_in = torch.from_numpy(img).pin_memory().numpy()
outs = [torch.empty_like(torch.from_numpy(img)).pin_memory().numpy() for _ in plans]
def run(n):
    def w(p, o):
        for _ in range(n):
            p.filter_host(h_in, o)
    ts = [threading.Thread(target=w, args=(p, o)) for p, o in zip(plans, outs)]
    t0 = time.perf_counter()
    for t in ts: t.start()
    for t in ts: t.join()
    return time.perf_counter() - t0
run(1)
n = 4
dt = run(n) / n
print(sys.argv[1:] or ["default"], f"e2e {5 * img.size / dt / 1e6:.0f} Mpix/s  ({dt * 1e3:.1f} ms/step)")
t0 = time.perf_counter(); plans[0].filter_host(h_in, outs[0]); print(f"single call {1e3 * (time.perf_counter() - t0):.2f} ms")
