"""Five-frame bench step (bench.py's C3 mix) issued three ways, same frames and
plans: (a) five streams, launches in stream order (bench.py); (b) the same
launches interleaved kernel by kernel across the streams; (c) one CUDA graph per
step captured from (a). Prints Mpix/s of each. usage: python tools/graph_step.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_1505_00077_b200 import gpf, synth  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = synth.CONFIGS[3]
W = H = cfg.width
frames = [synth.make(cfg, k) for k in range(len(cfg.sigma_s))]
d_ins = [torch.from_numpy(f).cuda() for f in frames]
outs = [torch.empty_like(d) for d in d_ins]
plans = [gpf.Plan(W, H, s, cfg.sigma_r, cfg.degree) for s in cfg.sigma_s]
streams = [torch.cuda.Stream() for _ in plans]
main = torch.cuda.current_stream()
px = W * H * len(plans)


def step():
    for i, (p, st) in enumerate(zip(plans, streams)):
        p.filter_device(d_ins[i], outs[i], 1, None, st.cuda_stream)


def timed(fn, n):
    for st in streams:
        st.wait_stream(main)
    for _ in range(3):
        fn()
    for st in streams:
        main.wait_stream(st)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for st in streams:
        st.wait_stream(main)
    for _ in range(n):
        fn()
    for st in streams:
        main.wait_stream(st)
    b.record(main)
    torch.cuda.synchronize()
    return px * n / (a.elapsed_time(b) / 1e3) / 1e6


r_streams = timed(step, steps)
# (c) graph of one step: capture on a side stream, the five streams forked from it
cap = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
for st in streams:
    st.wait_stream(main)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=cap):
    for st in streams:
        st.wait_stream(cap)
    step()
    for st in streams:
        cap.wait_stream(st)
torch.cuda.synchronize()
r_graph = timed(g.replay, steps)
r_streams2 = timed(step, steps)
print({"streams": round(r_streams, 1), "graph": round(r_graph, 1), "streams_again": round(r_streams2, 1)})
