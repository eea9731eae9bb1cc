"""Timeline of the bench mix: the five C3 sigma_s frames on five streams (as
bench.py runs them), with stage events recorded between every plan's kernels
(gpf_b200_plan_stage_marks). Prints, per stage, how much of the wall time it
was running on at least one stream and which stages overlapped it.

usage: python tools/timeline.py [steps] [size]   (writes gpurun_out/timeline.json)
"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_1505_00077_b200 import gpf, synth  # noqa: E402

STAGES = ("mean", "carry", "colpass", "rowscan", "rowpass")
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = synth.CONFIGS[3]
W = H = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.width
if W != cfg.width:
    cfg = synth.scaled(cfg, W, H)
frames = [synth.make(cfg, k) for k in range(len(cfg.sigma_s))]
d_ins = [torch.from_numpy(f).cuda() for f in frames]
outs = [torch.empty_like(d) for d in d_ins]
plans = [gpf.Plan(W, H, s, cfg.sigma_r, cfg.degree) for s in cfg.sigma_s]
streams = [torch.cuda.Stream() for _ in plans]
main = torch.cuda.current_stream()


def step():
    for i, (p, st) in enumerate(zip(plans, streams)):
        p.filter_device(d_ins[i], outs[i], 1, None, st.cuda_stream)


for st in streams:
    st.wait_stream(main)
for _ in range(3):
    step()
torch.cuda.synchronize()
for p in plans:
    p.set_profiling(True)
ref = torch.cuda.Event(enable_timing=True)
end = torch.cuda.Event(enable_timing=True)
ref.record(main)
for st in streams:
    st.wait_stream(main)
for _ in range(steps):
    step()
for st in streams:
    main.wait_stream(st)
end.record(main)
torch.cuda.synchronize()
total = ref.elapsed_time(end)
# intervals per stream: consecutive marks (stage s starts at mark i, ends at mark i+1)
iv = []
for k, p in enumerate(plans):
    marks = p.stage_marks(ref.cuda_event)
    for (s0, t0), (_, t1) in zip(marks, marks[1:]):
        if s0 >= 0:
            iv.append((k, STAGES[s0], t0, t1))
# sweep-line concurrency
edges = sorted({t for _, _, a, b in iv for t in (a, b)} | {0.0, total})
busy = {s: 0.0 for s in STAGES}
pair = {}
running_hist = {}
for a, b in zip(edges, edges[1:]):
    if b <= a:
        continue
    act = [s for _, s, t0, t1 in iv if t0 <= a and t1 >= b]
    kinds = sorted(set(act))
    for s in kinds:
        busy[s] += b - a
    key = "+".join(f"{s}x{act.count(s)}" for s in kinds) or "idle"
    pair[key] = pair.get(key, 0.0) + (b - a)
    running_hist[len(act)] = running_hist.get(len(act), 0.0) + (b - a)
res = {
    "steps": steps, "frames_per_step": len(plans), "wall_ms": round(total, 3),
    "ms_per_frame": round(total / steps / len(plans), 4),
    "busy_ms_per_step": {s: round(v / steps, 3) for s, v in busy.items()},
    "streams_running_ms_per_step": {str(k): round(v / steps, 3) for k, v in sorted(running_hist.items())},
    "top_overlaps_ms_per_step": dict(sorted(((k, round(v / steps, 3)) for k, v in pair.items()),
                                            key=lambda kv: -kv[1])[:25]),
    "intervals": [(k, s, round(a, 4), round(b, 4)) for k, s, a, b in iv],
}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/timeline.json", "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "intervals"}, indent=1))
