#!/usr/bin/env python3
"""Benchmark of the B200 GPF hot path (BASELINE.json metric: Mpixel/s of the
sigma_s-independent Gauss-polynomial bilateral filter, and % of roofline).

Workload (BASELINE config 3): one 8192x8192 fp32 frame of the seeded
generator (1024 rectangles, noise 10), sigma_r 30, N = 20, recursive backend,
mean centering; a STEP filters it at every sigma_s of the sweep
{2, 5, 10, 20, 50} (5 frames = 335.5 Mpixel per GPU), one plan and stream per
sigma_s. Inputs are 256 MiB per frame (> 126 MB L2), so no L2 flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 runs one process per GPU under torch.distributed.run (weak scaling:
every rank filters its own frame sweep; no collective on the data path);
time = max over ranks of the CUDA-event time of the K steps.

--impl reference times the reference's own CPU implementation
(oracle/_ref/libgpfilter_ref.so, compiled unmodified from the reference
sources; the oracle port if that build is absent) on the box's host cores, on
a bounded sample of the same workload (one 2048x2048 frame of the generator at
each sigma_s per step, ~5 s on 16 cores).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpixel/s of Gauss-poly bilateral (sigma_s-independent) and % of HBM/FP32 roofline"
UNIT = "Mpixel/s"
CFG_ID = 3
SAMPLE_W = SAMPLE_H = 2048  # 5 sigma_s x 4.2 MP: ~5 s per pass of the reference on 16 cores


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-mse", action="store_true",
                    help="skip the (untimed) MSE-vs-exact report, e.g. for ncu launch lists")
    ap.add_argument("--workload", choices=["c3", "c4"], default="c3",
                    help="c3 (default, the metric's config): 8192^2 sigma_s sweep, replicas per GPU; "
                         "c4: 64 frames x 3 channels of 3840x2160 sharded across the GPUs")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def relaunch_under_torchrun(args):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port", "29531",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        # samples under load: the timed region keeps the GPU busy throughout
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------- CPU leg
def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_reference_run(sigmas, sigma_r, degree, steps, threads):
    """Times the reference CPU implementation on the bounded sample; returns
    (Mpix/s, seconds per step, kind)."""
    import numpy as np

    from oracle.oracle import LIB_REF, Oracle, Reference
    from paper_1505_00077_b200 import synth
    img = synth.rects_image(SAMPLE_W, SAMPLE_H, 16, 10.0, CFG_ID * 1000 + 7).astype(np.float64)
    if os.path.exists(LIB_REF):
        ref = Reference()
        ref.set_num_threads(threads)
        kind = "reference"

        def one(ss):
            st, _, _ = ref.gpf(img, ss, sigma_r, degree)
            assert st == 0
    else:
        orc = Oracle()
        kind = "port"

        def one(ss):
            orc.gpf(img, ss, sigma_r, degree, threads=threads)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        for ss in sigmas:
            one(ss)
        times.append(time.perf_counter() - t0)
    per_step = statistics.median(times)
    return len(sigmas) * SAMPLE_W * SAMPLE_H / per_step / 1e6, per_step, kind


def algorithmic_bytes_per_px(pairs: int) -> dict:
    """HBM bytes each stage must move per pixel (fp32 frames, N+2 = 2*pairs
    planes; carries every 32 samples: 32 B per (pair, line, chunk) = pairs B/px).
      mean       f                                   4
      col_carry  seeds: f in, EM out; carries: EM in, CA out   4 + 8 + 8 + pairs
      colpass    EM + CA in; V + AH out              8 + pairs + 8 pairs + pairs
      row_scan   AH in, CH out                       2 pairs
      rowpass    V + CH + f in; out                  8 pairs + pairs + 4 + 4
    (ncu dram__bytes of each launch agree to within 3%: profiles/r01_v26_traffic.csv)"""
    return {"mean": 4, "col_carry": 20 + pairs, "colpass": 8 + 10 * pairs, "row_scan": 2 * pairs,
            "rowpass": 9 * pairs + 8}


def algorithmic_flops_per_px(pairs: int) -> dict:
    """FP32 FLOPs each stage issues per pixel (FMA = 2), P = plane pairs.
    One IIR step of one plane in the output-aligned section basis (DESIGN.md
    section 3): two sections advanced, 3 FMA each, in each direction = 24;
    emits with normalised weights (causal 1 FMA, or ADD + FMA where the other
    direction's parked value is added; anticausal MUL + FMA, or 2 FMA) ~6;
    i.e. ~30 per plane, 60 per pair. Strip/chunk dot products: 4 FMA per
    plane. Contraction: 2 FMA + 2 MUL per plane.
      carries    seeds ~20 + per pair: planes 2 MUL, dots 16          18 P + 20
      colpass    per pair: planes 2, sweeps 60, row dots 16           78 P
      row_scan   per pair: one chain step per 32 pixels              ~P
      rowpass    per pair: sweeps 60, contraction 12                  72 P + 10"""
    return {"mean": 1, "col_carry": 18 * pairs + 20, "colpass": 78 * pairs, "row_scan": pairs,
            "rowpass": 72 * pairs + 10}


def fp32_peak_tflops(peaks: dict) -> float:
    """Nominal FP32 FMA peak: 148 SMs x 128 FMA/clk x 2 FLOP x max SM clock."""
    return 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12


def roofline_of(px: int, ms: float, bpp: int, fpp: int, hbm_gbs: float, fp32_tf: float) -> dict:
    """Achieved vs the slower of HBM bytes and FP32 FLOPs (north_star)."""
    t_hbm = bpp * px / (hbm_gbs * 1e9)
    t_fp = fpp * px / (fp32_tf * 1e12)
    if t_hbm >= t_fp:
        ach = bpp * px / (ms / 1e3) / 1e9
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_gbs, "unit": "GB/s",
                "frac": round(ach / hbm_gbs, 4)}
    ach = fpp * px / (ms / 1e3) / 1e12
    return {"bound": "fp32", "achieved": round(ach, 2), "peak": round(fp32_tf, 1), "unit": "TFLOP/s",
            "frac": round(ach / fp32_tf, 4)}


# ------------------------------------------------------------- B200 leg
def bench_b200(args):
    import numpy as np
    import torch

    from paper_1505_00077_b200 import gpf, synth

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.CONFIGS[CFG_ID]
    W, H, sigmas, sr, N = cfg.width, cfg.height, cfg.sigma_s, cfg.sigma_r, cfg.degree
    img = synth.make(cfg)
    px = W * H
    d_in = torch.from_numpy(img).cuda()
    plans = [gpf.Plan(W, H, s, sr, N) for s in sigmas]
    outs = [torch.empty_like(d_in) for _ in sigmas]
    d_fb = torch.zeros(len(sigmas), dtype=torch.int64, device="cuda")
    streams = [torch.cuda.Stream() for _ in sigmas]
    main = torch.cuda.current_stream()

    # The five sigma_s frames run concurrently on five streams. (GPF_BENCH_CHAIN=1
    # instead chains them -- frame j starts when frame j-1's column half is done,
    # via gpf_b200_filter_f32_ev -- measured slower: 12.0 vs 13.8 Gpix/s.)
    pipelined = os.environ.get("GPF_BENCH_CHAIN", "0") == "1"
    front = [torch.cuda.Event() for _ in sigmas]
    for ev, st in zip(front, streams):
        ev.record(st)  # creates the events
    chain = {"prev": None}

    # A step enqueues the five frames; steps follow each other on the streams
    # without a join in between (the timed region is still bracketed by a
    # device-wide synchronize), so one frame's tail overlaps the next step.
    join_each_step = os.environ.get("GPF_BENCH_JOIN", "0") == "1"

    def step():
        for i, (plan, out, st) in enumerate(zip(plans, outs, streams)):
            if pipelined and chain["prev"] is not None:
                st.wait_event(chain["prev"])
            plan.filter_device(d_in, out, 1, d_fb[i:i + 1], st.cuda_stream,
                               front[i].cuda_event if pipelined else None)
            chain["prev"] = front[i]
        if join_each_step:
            for st in streams:
                main.wait_stream(st)

    for st in streams:
        st.wait_stream(main)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for st in streams:
        st.wait_stream(main)  # every stream starts after e0
    for _ in range(args.steps):
        step()
    for st in streams:
        main.wait_stream(st)  # e1 after every stream's last frame
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    ms_step = ms / args.steps
    frames = len(sigmas)
    value = world * frames * px / (ms_step / 1e3) / 1e6
    fallbacks = d_fb.cpu().tolist()

    # GPF's error against the exact O(sigma_s^2) filter (north_star: reported
    # alongside), full frame, metrics::compare definitions; outside the timed region
    mse = {}
    d_ex = torch.empty_like(d_in)
    for s_, out in zip(sigmas, [] if args.no_mse else outs):
        gpf.exact_device(d_in, d_ex, W, H, s_, sr, stream=main.cuda_stream)
        rep = gpf.compare_device(d_ex, out, W, H, 0, main.cuda_stream)
        mse[f"{s_:g}"] = {"mse": round(rep["mse"], 4), "mse_db": round(rep["mse_db"], 3),
                          "max_abs": round(rep["max_abs"], 4)}
    del d_ex

    # sigma_s independence: each plan alone on one stream
    per_sigma = {}
    for s, plan, out in zip(sigmas, plans, outs):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        plan.filter_device(d_in, out, 1, None, main.cuda_stream)
        a.record(main)
        for _ in range(3):
            plan.filter_device(d_in, out, 1, None, main.cuda_stream)
        b.record(main)
        torch.cuda.synchronize()
        per_sigma[f"{s:g}"] = round(a.elapsed_time(b) / 3, 4)

    # per-stage timing of one plan (sigma_s = 5) on one stream: dominant kernel
    p5 = plans[sigmas.index(5.0)]
    p5.set_profiling(True)
    reps = max(3, min(args.steps, 10))
    for _ in range(reps):
        p5.filter_device(d_in, outs[0], 1, None, main.cuda_stream)
    torch.cuda.synchronize()
    stage_ms = {k: v / reps for k, v in p5.stage_times().items()}
    p5.set_profiling(False)
    pairs = (N + 3) // 2
    bpp = algorithmic_bytes_per_px(pairs)
    fpp = algorithmic_flops_per_px(pairs)
    dom = max(stage_ms, key=stage_ms.get)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    fp32_tf = fp32_peak_tflops(peaks)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        t = json.load(open(tpath))
        if t.get("width") == W and t.get("height") == H and dom in t.get("bytes_per_launch", {}):
            traffic = t["bytes_per_launch"][dom]
    roof = roofline_of(px, stage_ms[dom], bpp[dom], fpp[dom], hbm_peak, fp32_tf)
    fp_k = fpp[dom] * px / (stage_ms[dom] / 1e3) / 1e12
    # whole step: all stages' bytes and FLOPs against the same peaks
    design_bpp, design_fpp = sum(bpp.values()), sum(fpp.values())
    step = roofline_of(px * frames, ms_step, design_bpp, design_fpp, hbm_peak, fp32_tf)
    model_bpp = 8 * (N + 2) + 12  # SURVEY 8(d) streaming model
    model_frac = (model_bpp * px * frames / (ms_step / 1e3) / 1e9) / hbm_peak
    roofline = dict(roof, kernel=dom, traffic=traffic, algorithmic_bytes_per_px=bpp[dom],
                    algorithmic_flops_per_px=fpp[dom],
                    fp32={"achieved_tflops": round(fp_k, 2), "peak_tflops": round(fp32_tf, 1),
                          "frac": round(fp_k / fp32_tf, 4),
                          "peak_source": "nominal 148 SM x 128 FMA/clk x 2 x sm_max_mhz"},
                    peak_source="MEASURED_PEAKS.json hbm_gbs (burst copy)",
                    step=dict(step, bytes_per_px=design_bpp, flops_per_px=design_fpp,
                              what="all stages of the step, slower of HBM bytes and FP32 FLOPs"),
                    step_model_frac=round(model_frac, 4),
                    step_model=f"SURVEY 8(d): {model_bpp} B/px at HBM peak")

    # end to end through the C ABI: pinned host fp32 in -> host fp32 out
    # One host thread per sigma_s plan (the C call releases the GIL; each plan
    # owns its streams), so one frame's upload/download overlaps the others'
    # compute. Every step still moves its input H2D and its output D2H.
    import threading
    h_in = torch.from_numpy(img).pin_memory()
    h_in_np = h_in.numpy()
    h_outs = [torch.empty_like(h_in).pin_memory() for _ in plans]
    h_outs_np = [o.numpy() for o in h_outs]
    e2e_steps = max(3, min(args.steps, 10))  # amortise the pipeline fill (first upload) and drain (last download)

    def host_run(n):
        errs = []

        def worker(plan, o):
            try:
                for _ in range(n):
                    plan.filter_host(h_in_np, o)
            except Exception as e:  # surfaced below
                errs.append(e)
        ths = [threading.Thread(target=worker, args=(p, o)) for p, o in zip(plans, h_outs_np)]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        if errs:
            raise errs[0]
        return time.perf_counter() - t0

    host_run(1)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e2e_s = host_run(e2e_steps) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": round(world * frames * px / e2e_s / 1e6, 1), "unit": UNIT,
           "h2d_bytes_per_step": frames * px * 4, "d2h_bytes_per_step": frames * px * 4 + frames * 8,
           "api": "gpf_b200_filter_f32_host (pinned host fp32 in/out, one call per sigma_s per step, "
                   f"{frames} host threads, one per sigma_s plan)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        thr = cpu_threads()
        v, sec, kind = cpu_reference_run(sigmas, sr, N, 2, thr)
        cpu = {"value": round(v, 3), "unit": UNIT, "cores": thr, "kind": kind,
               "sample": f"{SAMPLE_W}x{SAMPLE_H} generator frame at sigma_s {list(sigmas)}, "
                         f"sigma_r {sr}, N {N}; median of 2 passes of {sec:.1f} s of CPU work"}

    launches = args.steps * frames * plans[0].launches_per_frame
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic (seeded generator, SURVEY.md 8(d))",
        "config": {"workload": f"C3: {W}x{H} fp32 rects1024 noise10, sigma_r {sr}, N {N}, "
                               f"sigma_s sweep {list(sigmas)} = {frames} frames/step/GPU",
                   "frames_per_step_per_gpu": frames, "pixels_per_frame": px,
                   "l2": "inputs larger than L2 (256 MiB per frame, 126 MB L2); no flush",
                   "parallelism": f"frame replicas x{world}, no collective"},
        "sigma_s_ms_per_frame": per_sigma,
        "mse_vs_exact": {"per_sigma_s": mse, "pixels": px,
                         "what": "GPF output vs the exact O(sigma_s^2) bilateral (gpf_b200_exact_f32), "
                                 "full frame, metrics::compare (mse, 10 log10 mse, max |d|)"},
        "stage_ms_per_frame": {k: round(v, 4) for k, v in stage_ms.items()},
        "roofline": roofline,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "gpu_launches": launches,
        "fallbacks": fallbacks,
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


# ------------------------------------------------------------- C4 frame batch
def build_c4_frames(d_in, first: int, cfg):
    """Problems first .. first+len(d_in)-1 of C4 (problem i = frame i // 3,
    channel i % 3) on the device: the synth gradient + the channel's rectangle
    layer drifted 4 px per frame + N(0, noise^2) (torch-seeded per problem),
    clipped to [0, 255]."""
    import numpy as np
    import torch

    from paper_1505_00077_b200 import synth
    H, W = cfg.height, cfg.width
    base = cfg.cid * 1000
    layers = [torch.from_numpy(synth._rect_layer(np.random.default_rng(base + c), W, H, 48)).float().cuda()
              for c in range(cfg.channels)]
    x = torch.arange(W, device="cuda", dtype=torch.float32) / max(1, W - 1)
    y = torch.arange(H, device="cuda", dtype=torch.float32) / max(1, H - 1)
    grad = 32.0 * (x[None, :] + y[:, None])
    g = torch.Generator(device="cuda")
    for k in range(d_in.shape[0]):
        i = first + k
        fr, ch = divmod(i, cfg.channels)
        dx = min(4 * fr, W)
        img = grad.clone()
        img[:, dx:] += layers[ch][:, :W - dx]
        g.manual_seed(base + fr * 3 + ch + 500)
        img += cfg.noise * torch.randn((H, W), generator=g, device="cuda")
        d_in[k] = img.clamp_(0.0, 255.0)


def bench_c4(args):
    import torch

    from paper_1505_00077_b200 import gpf, shard, synth

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.CONFIGS[4]
    W, H, ss, sr, N = cfg.width, cfg.height, cfg.sigma_s[0], cfg.sigma_r, cfg.degree
    n_items = cfg.frames * cfg.channels
    first, stop = shard.shard_range(n_items, rank, world)
    n_loc = stop - first
    px = W * H
    d_in = torch.empty((max(n_loc, 1), H, W), dtype=torch.float32, device="cuda")
    build_c4_frames(d_in[:n_loc], first, cfg)
    d_out = torch.empty_like(d_in)
    d_fb = torch.zeros(max(n_loc, 1), dtype=torch.int64, device="cuda")
    # frames per launch: large batches keep every pass several waves deep (the
    # single stream has no other work to fill a batch's tail)
    plan = gpf.Plan(W, H, ss, sr, N, batch=max(1, min(n_loc, int(os.environ.get("GPF_C4_BATCH", "48")))))
    st = torch.cuda.current_stream()

    def step():
        if n_loc:
            plan.filter_device(d_in, d_out, n_loc, d_fb, st.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    ms_local = e0.elapsed_time(e1)
    clk = clocks.stop()
    if world > 1:
        torch.distributed.barrier()
    secs, fallbacks = shard.reduce_job(ms_local / 1e3, d_fb[:n_loc].cpu().tolist(), n_items, rank,
                                       world, device="cuda")
    ms_step = secs * 1e3 / args.steps
    value = n_items * px / (ms_step / 1e3) / 1e6

    # per-stage timing of one frame (dominant kernel) and the roofline
    plan.set_profiling(True)
    reps = 3
    for _ in range(reps):
        plan.filter_device(d_in, d_out, 1, None, st.cuda_stream)
    torch.cuda.synchronize()
    stage_ms = {k: v / reps for k, v in plan.stage_times().items()}
    plan.set_profiling(False)
    pairs = (N + 3) // 2
    bpp, fpp = algorithmic_bytes_per_px(pairs), algorithmic_flops_per_px(pairs)
    dom = max(stage_ms, key=stage_ms.get)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak, fp32_tf = peaks.get("hbm_gbs", 6650.0), fp32_peak_tflops(peaks)
    roof = roofline_of(px, stage_ms[dom], bpp[dom], fpp[dom], hbm_peak, fp32_tf)
    step_roof = roofline_of(n_items * px, ms_step, sum(bpp.values()), sum(fpp.values()),
                            hbm_peak * world, fp32_tf * world)
    roofline = dict(roof, kernel=dom, traffic=None, algorithmic_bytes_per_px=bpp[dom],
                    algorithmic_flops_per_px=fpp[dom],
                    peak_source="MEASURED_PEAKS.json hbm_gbs (burst copy)",
                    step=dict(step_roof, what=f"whole job on {world} GPU(s), peaks x {world}"))

    # end to end: this rank's frames from pinned host memory through the
    # pipelined host entry (H2D of frame f+1 overlaps compute of f), every step
    h_in = d_in[:max(n_loc, 1)].cpu().pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    h_in_np, h_out_np = h_in.numpy(), h_out.numpy()
    if n_loc:
        plan.filter_host(h_in_np[:n_loc], h_out_np[:n_loc])
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e2e_steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        if n_loc:
            plan.filter_host(h_in_np[:n_loc], h_out_np[:n_loc])
    e2e_s, _ = shard.reduce_job((time.perf_counter() - t0) / e2e_steps, [0] * n_loc, n_items, rank,
                                world, device="cuda")
    e2e = {"value": round(n_items * px / e2e_s / 1e6, 1), "unit": UNIT,
           "h2d_bytes_per_step": n_items * px * 4, "d2h_bytes_per_step": n_items * (px * 4 + 8),
           "api": "gpf_b200_filter_f32_host (pinned host fp32 in/out, all local frames per call, "
                  "H2D/compute/D2H pipelined inside)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        thr = cpu_threads()
        v, sec, kind = cpu_reference_run((ss,), sr, N, 3, thr)
        cpu = {"value": round(v, 3), "unit": UNIT, "cores": thr, "kind": kind,
               "sample": f"{SAMPLE_W}x{SAMPLE_H} generator frame at sigma_s {ss}, sigma_r {sr}, N {N} "
                         f"({sec:.1f} s of CPU work)"}
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic (C4 generator on device: drifting rectangles + seeded noise)",
        "config": {"workload": f"C4: {cfg.frames} frames x {cfg.channels} channels of {W}x{H} fp32, "
                               f"sigma_s {ss}, sigma_r {sr}, N {N}; {n_items} independent problems "
                               f"sharded contiguously ({shard.shard_sizes(n_items, world)})",
                   "l2": "inputs larger than L2 (33 MB per problem x %d per GPU); no flush" % n_loc,
                   "parallelism": f"frame shards x{world}, no collective on the data path"},
        "stage_ms_per_frame": {k: round(v, 4) for k, v in stage_ms.items()},
        "roofline": roofline,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "gpu_launches": args.steps * n_loc * plan.launches_per_frame,
        "fallbacks_total": int(sum(fallbacks)),
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def bench_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1505_00077_b200 import synth
    cfg = synth.CONFIGS[4 if args.workload == "c4" else CFG_ID]
    thr = cpu_threads()
    cpu_reference_run(cfg.sigma_s, cfg.sigma_r, cfg.degree, args.warmup, thr) if args.warmup else None
    v, sec, kind = cpu_reference_run(cfg.sigma_s, cfg.sigma_r, cfg.degree, args.steps, thr)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 1),
        "higher_is_better": True, "scaling": "strong" if args.workload == "c4" else "weak",
        "vs_baseline": None, "dtype": "fp64",
        "data": "synthetic (seeded generator, SURVEY.md 8(d))",
        "config": {"workload": f"C{cfg.cid} sample: {SAMPLE_W}x{SAMPLE_H} generator frame, sigma_r "
                               f"{cfg.sigma_r}, N {cfg.degree}, sigma_s sweep {list(cfg.sigma_s)}",
                   "parallelism": f"{thr} host threads (gpf_set_num_threads)"},
        "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": thr, "kind": kind,
                         "sample": f"{SAMPLE_W}x{SAMPLE_H} x {len(cfg.sigma_s)} sigma_s per step"},
        "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    if args.impl == "reference":
        bench_reference(args)
    elif args.workload == "c4":
        bench_c4(args)
    else:
        bench_b200(args)


if __name__ == "__main__":
    main()
