#!/usr/bin/env python3
"""Benchmark of the B200 GPF hot path (BASELINE.json metric: Mpixel/s of the
sigma_s-independent Gauss-polynomial bilateral filter, and % of roofline).

Workload (BASELINE config 3): 8192x8192 fp32 frames of the seeded generator
(1024 rectangles, noise 10), sigma_r 30, N = 20, recursive backend, mean
centering. A STEP filters five frames, frame k of the C3 batch at sigma_s[k]
of the sweep {2, 5, 10, 20, 50} (335.5 Mpixel per GPU), one plan and stream
per sigma_s. Inputs are 256 MiB per frame (> 126 MB L2), so no L2 flush is
needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 runs one process per GPU under torch.distributed.run: the frame batch
is sharded, rank r filtering frames 5r .. 5r+4 (weak scaling, no collective on
the data path); time = max over ranks of the CUDA-event time of the K steps.
`--workload c4` shards BASELINE C4's 192 problems instead (strong scaling).

--impl reference times the reference's own CPU implementation
(oracle/_ref/libgpfilter_ref.so, compiled unmodified from the reference
sources; the oracle port if that build is absent) on the box's host cores, on
the bench's own frames: each step filters one full 8192x8192 C3 frame at the
next sigma_s of the sweep.

Besides `value` (device-resident fp32 frames), the line carries:
  roofline   the dominant kernel and the whole step against SURVEY 8(d)'s
             algorithmic bytes (188 B/px per frame; 96 B/px for the row pass)
  e2e        pinned host fp32 frames through gpf_b200_filter_f32_host
  e2e_dropin the reference's own call, gpf_filter_gpf on fp64 host images
             (what the reference's `gpf bench` times), per frame
  fp64_exact the reference-exact fp64 precision mode on BASELINE C5 / C2
  parity     max |out - reference| on the golden reference samples of the
             bench's own frames (tests/golden/baseline_samples.npz)
  cpu_baseline  the reference on one full C3 frame (nproc threads) and a
             2048^2 crop (1 thread)
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
# reference arm: wall-time budget of the K timed steps (seconds), the frame is banded to fit
REF_BUDGET_S = 150.0
GOLDEN = os.path.join(ROOT, "tests", "golden", "baseline_samples.npz")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-mse", action="store_true",
                    help="skip the (untimed) MSE-vs-exact report, e.g. for ncu launch lists")
    ap.add_argument("--no-extras", action="store_true",
                    help="only the timed device-resident step (no e2e / drop-in / fp64 / parity legs)")
    ap.add_argument("--workload", choices=["c3", "c4"], default="c3",
                    help="c3 (default, the metric's config): 8192^2 sigma_s sweep, 5 frames per GPU; "
                         "c4: 64 frames x 3 channels of 3840x2160 sharded across the GPUs")
    ap.add_argument("--size", type=int, default=0,
                    help="frame side override (functional runs only; the metric is quoted at 8192)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="every rank on GPU 0 with gloo for the scalar reductions (functional "
                         "multi-rank run on one GPU; not a performance number)")
    ap.add_argument("--selftest-cpu", action="store_true",
                    help="CPU-only check of the launch / reduction plumbing with a stub filter (gloo)")
    return ap.parse_args(argv)


# ------------------------------------------------------------ process plumbing
def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def relaunch_under_torchrun(args, port: int = 29531):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(int(os.environ.get("GPF_BENCH_PORT", port))), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


class Job:
    """One rank of the job: device selection, process group, and the scalar
    reductions after the timed region (only scalars cross ranks)."""

    def __init__(self, backend: str | None, device: str | None):
        self.rank, self.world, self.local = dist_env()
        self.device = device
        self.pg = False
        if self.world > 1:
            import torch
            import torch.distributed as dist
            kw = {}
            if backend == "nccl":
                kw["device_id"] = torch.device("cuda", self.local)
            dist.init_process_group(backend, **kw)
            self.pg = True

    def barrier(self):
        if self.pg:
            import torch.distributed as dist
            dist.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return float(x)
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(x)], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return float(x)
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(x)], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg:
            import torch.distributed as dist
            dist.destroy_process_group()


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
        sm, smax, pw, reasons = [], [], [], set()
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
            try:
                pw.append(float(parts[2]))
            except ValueError:
                pass
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        # samples under load: the timed region keeps the GPU busy throughout
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "power_w": statistics.median(pw) if pw else None,
                "reasons": sorted(reasons)}


# ------------------------------------------------------------- CPU leg
def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_filter(threads: int):
    """(kind, fn(img, sigma_s, sigma_r, degree)): the unmodified reference
    library when built (oracle/_ref), else the oracle port."""
    from oracle.oracle import LIB_REF, Oracle, Reference
    if os.path.exists(LIB_REF):
        ref = Reference()
        ref.set_num_threads(threads)

        def run(img, ss, sr, deg):
            st, out, fb = ref.gpf(img, ss, sr, deg)
            assert st == 0
            return out, fb
        return "reference", run
    orc = Oracle()

    def run_port(img, ss, sr, deg):
        out, fb, _ = orc.gpf(img, ss, sr, deg, threads=threads)
        return out, fb
    return "port", run_port


def cpu_baseline_leg(cfg, frames) -> dict:
    """The reference on the host cores: one full frame of the bench's batch at
    nproc threads (the same config as `value`), and a 2048^2 crop at 1 thread."""
    thr = cpu_threads()
    kind, run = reference_filter(thr)
    img0 = frames[0].astype("float64")
    t0 = time.perf_counter()
    run(img0, cfg.sigma_s[0], cfg.sigma_r, cfg.degree)
    sec = time.perf_counter() - t0
    px = img0.size
    out = {"value": round(px / sec / 1e6, 3), "unit": UNIT, "cores": thr, "kind": kind,
           "cpu_model": cpu_model(),
           "sample": f"one full {img0.shape[1]}x{img0.shape[0]} C3 frame (frame 0) at sigma_s "
                     f"{cfg.sigma_s[0]:g}, sigma_r {cfg.sigma_r:g}, N {cfg.degree}, {thr} threads: "
                     f"{sec:.1f} s"}
    kind1, run1 = reference_filter(1)
    crop = img0[:2048, :2048].copy()
    t0 = time.perf_counter()
    run1(crop, cfg.sigma_s[0], cfg.sigma_r, cfg.degree)
    sec1 = time.perf_counter() - t0
    out["single_thread"] = {"value": round(crop.size / sec1 / 1e6, 3), "unit": UNIT, "cores": 1,
                            "sample": f"2048x2048 crop of frame 0, 1 thread: {sec1:.1f} s"}
    return out


# ------------------------------------------------------- roofline model
def model_bytes_per_px(degree: int) -> dict:
    """SURVEY 8(d) algorithmic HBM bytes per pixel (fp32 frames, N+2 planes):
    the step reads f for the mean (4) and for the planes (4), writes and reads
    every plane once between the separable passes (2 x 4 (N+2)) and writes the
    output (4): 8 (N+2) + 12 = 188 at N = 20. The row pass's share: it reads
    the N+2 column-pass planes (4 (N+2)), the input f for the fallback rule (4)
    and writes the output (4): 4 (N+2) + 8 = 96."""
    planes = degree + 2
    return {"step": 8 * planes + 12, "rowpass": 4 * planes + 8, "colpass": 4 * planes + 4,
            "col_carry": 4, "row_scan": 0, "mean": 4}


def design_bytes_per_px(pairs: int) -> dict:
    """HBM bytes each stage of THIS implementation moves per pixel (P = plane
    pairs; carries every 32 samples: 32 B per (pair, line, chunk) = P B/px).
      mean       f                                          4
      col_carry  seeds: f in, EM out; carries: EM in, CA out   4 + 8 + 8 + P
      colpass    EM + CA in; V + AH out                     8 + P + 8P + P
      row_scan   AH in, CH out                              2P
      rowpass    V + CH + f in; out                         8P + P + 4 + 4
    (ncu dram__bytes per launch: profiles/ncu_traffic.json)"""
    return {"mean": 4, "col_carry": 20 + pairs, "colpass": 8 + 10 * pairs, "row_scan": 2 * pairs,
            "rowpass": 9 * pairs + 8}


def algorithmic_flops_per_px(pairs: int) -> dict:
    """FP32 FLOPs each stage issues per pixel (FMA = 2), P = plane pairs.
    One IIR step of one plane in the output-aligned section basis (DESIGN.md
    section 3): two sections advanced, 3 FMA each, in each direction = 24;
    emits ~6; i.e. ~30 per plane, 60 per pair. Strip/chunk dot products: 4 FMA
    per plane. Contraction on G-scaled planes: two packed FMAs
    per plane pair (joint Horner of Q and P = Q'), i.e. 2 FMA per plane.
      carries    seeds ~20 + per pair: planes 2 MUL, dots 16          18 P + 20
      colpass    per pair: planes 2 MUL + 2 (1/n!), sweeps 60, dots 16 80 P
      row_scan   per pair: one chain step per 32 pixels              ~P
      rowpass    per pair: sweeps 60, contraction 8; setup ~12        68 P + 12"""
    return {"mean": 1, "col_carry": 18 * pairs + 20, "colpass": 80 * pairs, "row_scan": pairs,
            "rowpass": 68 * pairs + 12}


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


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def load_traffic(w: int, h: int):
    """ncu dram__bytes per launch of each stage (profiles/ncu_traffic.json)."""
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(tpath):
        return None
    t = json.load(open(tpath))
    if t.get("width") != w or t.get("height") != h:
        return None
    return t


def roofline_block(px, frames, ms_step, stage_ms, degree, w, h) -> dict:
    """`roofline` key: the dominant kernel against its SURVEY 8(d) share of the
    algorithmic bytes, the whole step against 8(d)'s 188 B/px (the headline
    fraction), and the implementation's own traffic beside them."""
    pairs = (degree + 3) // 2
    model = model_bytes_per_px(degree)
    design = design_bytes_per_px(pairs)
    fpp = algorithmic_flops_per_px(pairs)
    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6460.5)
    hbm_src = ("MEASURED_PEAKS.json hbm_gbs (burst copy)" if "hbm_gbs" in peaks
               else "B200_PROFILING.md fallback")
    fp32_tf = fp32_peak_tflops(peaks)
    heavy = [k for k in ("colpass", "rowpass") if k in stage_ms]
    dom = max(heavy, key=stage_ms.get) if heavy else max(stage_ms, key=stage_ms.get)
    k_ms = stage_ms[dom]
    # both heavy passes against their own 8(d) shares (the dominant one is `frac`)
    per_kernel = {}
    for k in heavy:
        rk = roofline_of(px, stage_ms[k], model[k], fpp[k], hbm_peak, fp32_tf)
        per_kernel[k] = {"ms": round(stage_ms[k], 4), "achieved": rk["achieved"], "frac": rk["frac"],
                         "algorithmic_bytes_per_px": model[k]}
    roof = roofline_of(px, k_ms, model[dom], fpp[dom], hbm_peak, fp32_tf)
    fp_k = fpp[dom] * px / (k_ms / 1e3) / 1e12
    traffic = load_traffic(w, h)
    t_launch = traffic["bytes_per_launch"].get(dom) if traffic else None
    t_step = sum(traffic["bytes_per_launch"].values()) if traffic else None
    step = roofline_of(px * frames, ms_step, model["step"], sum(fpp.values()), hbm_peak, fp32_tf)
    return dict(
        roof, kernel=dom, kernel_ms=round(k_ms, 4), traffic=t_launch,
        algorithmic_bytes_per_px=model[dom],
        algorithmic_what=(f"SURVEY 8(d) share of the {dom}: " +
                          ("N+2 plane reads 4(N+2) + f 4 + out 4" if dom == "rowpass"
                           else "f 4 + N+2 plane writes 4(N+2)")),
        kernels=per_kernel,
        traffic_over_algorithmic=round(t_launch / (model[dom] * px), 3) if t_launch else None,
        design_bytes_per_px=design[dom], algorithmic_flops_per_px=fpp[dom],
        fp32={"achieved_tflops": round(fp_k, 2), "peak_tflops": round(fp32_tf, 1),
              "frac": round(fp_k / fp32_tf, 4),
              "peak_source": "nominal 148 SM x 128 FMA/clk x 2 x sm_max_mhz"},
        peak_source=hbm_src,
        step=dict(step, bytes_per_px=model["step"],
                  what="whole step at SURVEY 8(d)'s 188 B/px per frame (headline fraction)",
                  traffic_bytes_per_px=round(t_step / px, 1) if t_step else None,
                  traffic_over_algorithmic=round(t_step / (model["step"] * px), 3) if t_step else None,
                  design_bytes_per_px=sum(design.values())))


# ------------------------------------------------------------- B200 leg
def golden_parity(outs, sigmas, n_frames) -> dict | None:
    """max |out - reference| on the committed reference samples of the bench's
    frames (frame k at sigma_s[k]; tests/golden/make_baseline_samples.py)."""
    import numpy as np
    if not os.path.exists(GOLDEN):
        return None
    g = np.load(GOLDEN)
    res, worst = {}, 0.0
    for k in range(n_frames):
        key = f"c3_f{k}_ss{int(sigmas[k])}"
        if f"{key}/samples" not in g.files:
            continue
        ref = g[f"{key}/samples"]
        s = int(g[f"{key}/meta"][0])
        got = outs[k][::s, ::s].double().cpu().numpy()
        d = float(np.abs(got - ref).max())
        worst = max(worst, d)
        res[f"{sigmas[k]:g}"] = {"max_abs": float(f"{d:.3e}"), "samples": int(ref.size),
                                 "ref_fallbacks": int(g[f"{key}/meta"][1])}
    return {"per_sigma_s": res, "max_abs": float(f"{worst:.3e}"), "tol": 1e-3,
            "what": "fp32 outputs of the timed step vs the unmodified reference (oracle/_ref) "
                    "on a stride-64 grid of every frame (tests/golden/baseline_samples.npz); "
                    "every pixel is compared in tests/test_gpu_fullsize.py"}


def dropin_leg(frames, sigmas, cfg, steps) -> dict:
    """The reference's own call, gpf_filter_gpf, on fp64 host images (the
    reference's `gpf bench` protocol, proj/tools/gpf_cli.cpp:241-258): every
    call copies the frame H2D, filters it and returns a new host image."""
    import ctypes as C

    import numpy as np

    from paper_1505_00077_b200 import _lib, gpf
    L = _lib.lib()
    imgs = [gpf.Image.from_array(f.astype(np.float64)) for f in frames]
    sps = [gpf.spatial_params(s) for s in sigmas]
    rp = gpf.range_params(cfg.sigma_r, cfg.degree)

    def call(i):
        out = C.c_void_p()
        fb = C.c_longlong(-1)
        st = L.gpf_filter_gpf(imgs[i].h, C.byref(sps[i]), C.byref(rp), 1, 1, C.byref(fb), C.byref(out))
        if st != 0:
            raise RuntimeError(L.gpf_last_error().decode())
        L.gpf_image_destroy(out)
        return gpf.last_precision(), gpf.last_device_ms()

    for i in range(len(frames)):  # first call per frame: plan + buffers (cached afterwards)
        call(i)
    t0 = time.perf_counter()
    dev_ms, precs = 0.0, set()
    for _ in range(steps):
        for i in range(len(frames)):
            p, ms = call(i)
            precs.add(p)
            dev_ms += ms
    sec = (time.perf_counter() - t0) / steps
    px = sum(f.size for f in frames)

    # the same calls from one host thread per frame (a serving process with
    # several callers): the engine pipelines one call's upload and another's
    # download against the kernels of a third (dropin.cpp call slots)
    def worker(i, n):
        for _ in range(n):
            call(i)
    import threading
    ths = [threading.Thread(target=worker, args=(i, 1)) for i in range(len(frames))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker, args=(i, steps)) for i in range(len(frames))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    csec = (time.perf_counter() - t0) / steps
    return {"value": round(px / sec / 1e6, 1), "unit": UNIT, "ms_per_step": round(sec * 1e3, 2),
            "device_ms_per_step": round(dev_ms / steps, 3), "precision": sorted(precs),
            "h2d_bytes_per_step": px * 8, "d2h_bytes_per_step": px * 8 + 8 * len(frames),
            "api": "gpf_filter_gpf (reference C ABI): fp64 host image in, new fp64 host image out, "
                   f"one call per frame, {len(frames)} frames per step, AUTO precision",
            "concurrent": {"value": round(px / csec / 1e6, 1), "unit": UNIT,
                           "ms_per_step": round(csec * 1e3, 2), "host_threads": len(frames),
                           "what": "the same calls, one host thread per frame calling concurrently"}}


def fp64_leg(steps) -> dict:
    """The reference-exact fp64 mode through gpf_filter_gpf on BASELINE C5 (and
    C2): the configs whose reference series leaves the input range."""
    import ctypes as C

    import numpy as np

    from paper_1505_00077_b200 import _lib, gpf, synth
    L = _lib.lib()
    res = {}
    for cid in (5, 2):
        cfg = synth.CONFIGS[cid]
        img = gpf.Image.from_array(synth.make(cfg).astype(np.float64))
        sp, rp = gpf.spatial_params(cfg.sigma_s[0]), gpf.range_params(cfg.sigma_r, cfg.degree)

        def call():
            out = C.c_void_p()
            fb = C.c_longlong(-1)
            st = L.gpf_filter_gpf(img.h, C.byref(sp), C.byref(rp), 1, 1, C.byref(fb), C.byref(out))
            if st != 0:
                raise RuntimeError(L.gpf_last_error().decode())
            L.gpf_image_destroy(out)
            return gpf.last_device_ms()

        call()
        t0 = time.perf_counter()
        dev = [call() for _ in range(steps)]
        sec = (time.perf_counter() - t0) / steps
        px = cfg.width * cfg.height
        res[f"C{cid}"] = {"e2e": round(px / sec / 1e6, 1), "device": round(px / (min(dev) / 1e3) / 1e6, 1),
                          "unit": UNIT, "device_ms": round(min(dev), 3), "precision": gpf.last_precision(),
                          "frame": f"{cfg.width}x{cfg.height}, sigma_s {cfg.sigma_s[0]:g}, "
                                   f"sigma_r {cfg.sigma_r:g}, max|H| {gpf.last_max_abs_h():.2f}"}
    return res


def bench_b200(args):
    import numpy as np
    import torch

    from paper_1505_00077_b200 import gpf, synth

    rank, world, local = dist_env()
    dev_index = 0 if args.share_gpu else local
    torch.cuda.set_device(dev_index)
    job = Job("gloo" if args.share_gpu else "nccl", None if args.share_gpu else "cuda")
    cfg = synth.CONFIGS[CFG_ID]
    W = H = args.size or cfg.width
    if args.size:
        cfg = synth.scaled(cfg, W, H)
    sigmas, sr, N = cfg.sigma_s, cfg.sigma_r, cfg.degree
    n_fr = len(sigmas)
    # this rank's shard of the frame batch: frames n_fr*rank .. n_fr*rank + n_fr - 1
    frames = [synth.make(cfg, n_fr * rank + k) for k in range(n_fr)]
    px = W * H
    d_ins = [torch.from_numpy(f).cuda() for f in frames]
    plans = [gpf.Plan(W, H, s, sr, N) for s in sigmas]
    outs = [torch.empty_like(d) for d in d_ins]
    d_fb = torch.zeros(n_fr, dtype=torch.int64, device="cuda")
    streams = [torch.cuda.Stream() for _ in sigmas]
    main = torch.cuda.current_stream()

    # A step enqueues the five frames on five streams; steps follow each other
    # on the streams without a join in between (the timed region is bracketed
    # by a device-wide synchronize), so one frame's tail overlaps the next step.
    def step():
        for i, (plan, st) in enumerate(zip(plans, streams)):
            plan.filter_device(d_ins[i], outs[i], 1, d_fb[i:i + 1], st.cuda_stream)

    for st in streams:
        st.wait_stream(main)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    job.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev_index)
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
    ms = job.max(ms)
    job.barrier()
    ms_step = ms / args.steps
    value = world * n_fr * px / (ms_step / 1e3) / 1e6
    launches = args.steps * n_fr * plans[0].launches_per_frame
    fallbacks = d_fb.cpu().tolist()
    parity = golden_parity(outs, sigmas, n_fr) if (rank == 0 and not args.size) else None

    # GPF's error against the exact O(sigma_s^2) filter (north_star: reported
    # alongside), full frame, metrics::compare definitions; outside the timed region
    mse = {}
    if not args.no_mse and not args.no_extras:
        d_ex = torch.empty_like(d_ins[0])
        for k, (s_, out) in enumerate(zip(sigmas, outs)):
            gpf.exact_device(d_ins[k], d_ex, W, H, s_, sr, stream=main.cuda_stream)
            rep = gpf.compare_device(d_ex, out, W, H, 0, main.cuda_stream)
            mse[f"{s_:g}"] = {"mse": round(rep["mse"], 4), "mse_db": round(rep["mse_db"], 3),
                              "max_abs": round(rep["max_abs"], 4)}
        del d_ex

    # sigma_s independence: each plan alone on one stream
    per_sigma = {}
    for k, (s, plan) in enumerate(zip(sigmas, plans)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        plan.filter_device(d_ins[k], outs[k], 1, None, main.cuda_stream)
        a.record(main)
        for _ in range(3):
            plan.filter_device(d_ins[k], outs[k], 1, None, main.cuda_stream)
        b.record(main)
        torch.cuda.synchronize()
        per_sigma[f"{s:g}"] = round(a.elapsed_time(b) / 3, 4)

    # per-stage timing of one plan (sigma_s = 5) on one stream: dominant kernel
    k5 = list(sigmas).index(5.0)
    p5 = plans[k5]
    p5.set_profiling(True)
    reps = max(3, min(args.steps, 10))
    for _ in range(reps):
        p5.filter_device(d_ins[k5], outs[k5], 1, None, main.cuda_stream)
    torch.cuda.synchronize()
    stage_ms = {k: v / reps for k, v in p5.stage_times().items()}
    p5.set_profiling(False)
    roofline = roofline_block(px, n_fr, ms_step, stage_ms, N, W, H)

    e2e = dropin = fp64 = None
    if not args.no_extras:
        # end to end through the C ABI: pinned host fp32 in -> host fp32 out.
        # One host thread per sigma_s plan (the C call releases the GIL; each
        # plan owns its streams), so one frame's upload/download overlaps the
        # others' compute. Every step moves its inputs H2D and outputs D2H.
        import threading
        h_ins = [torch.from_numpy(f).pin_memory().numpy() for f in frames]
        h_outs = [torch.empty((H, W), dtype=torch.float32).pin_memory().numpy() for _ in frames]
        e2e_steps = max(3, min(args.steps, 10))

        def host_run(n):
            errs = []

            def worker(plan, i):
                try:
                    for _ in range(n):
                        plan.filter_host(h_ins[i], h_outs[i])
                except Exception as e:  # surfaced below
                    errs.append(e)
            ths = [threading.Thread(target=worker, args=(p, i)) for i, p in enumerate(plans)]
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
        job.barrier()
        e2e_s = job.max(host_run(e2e_steps) / e2e_steps)
        e2e = {"value": round(world * n_fr * px / e2e_s / 1e6, 1), "unit": UNIT,
               "h2d_bytes_per_step": n_fr * px * 4, "d2h_bytes_per_step": n_fr * px * 4 + n_fr * 8,
               "api": "gpf_b200_filter_f32_host (pinned host fp32 in/out, one call per sigma_s per "
                      f"step, {n_fr} host threads, one per sigma_s plan)"}
        # the reference's own call on fp64 host images
        for p in plans:
            p.close()
        del outs
        torch.cuda.empty_cache()
        dsteps = max(1, min(args.steps, 3))
        dropin = dropin_leg(frames, sigmas, cfg, dsteps)
        dropin["value"] = round(job.sum(dropin["value"]), 1)
        dropin["concurrent"]["value"] = round(job.sum(dropin["concurrent"]["value"]), 1)
        if rank == 0 and world == 1 and not args.size:
            fp64 = fp64_leg(max(1, min(args.steps, 3)))
        gpf.dropin_release()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(cfg, frames)

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic (seeded generator, SURVEY.md 8(d))",
        "config": {"workload": f"C3: {W}x{H} fp32 rects{cfg.rects} noise10, sigma_r {sr:g}, N {N}; "
                               f"frame k of the C3 batch at sigma_s[k] of {list(sigmas)} = {n_fr} "
                               "frames/step/GPU",
                   "frames_per_step_per_gpu": n_fr, "pixels_per_frame": px,
                   "l2": "inputs larger than L2 (256 MiB per frame, 126 MB L2); no flush",
                   "parallelism": f"frame batch sharded x{world} (rank r: frames {n_fr}r..{n_fr}r+"
                                  f"{n_fr - 1}), no collective on the data path"
                                  + ("; all ranks on GPU 0 (functional run)" if args.share_gpu else "")},
        "sigma_s_ms_per_frame": per_sigma,
        "mse_vs_exact": {"per_sigma_s": mse, "pixels": px,
                         "what": "GPF output vs the exact O(sigma_s^2) bilateral (gpf_b200_exact_f32), "
                                 "full frame, metrics::compare (mse, 10 log10 mse, max |d|)"},
        "stage_ms_per_frame": {k: round(v, 4) for k, v in stage_ms.items()},
        "roofline": roofline,
        "parity": parity,
        "e2e": e2e,
        "e2e_dropin": dropin,
        "fp64_exact": fp64,
        "cpu_baseline": cpu,
        "gpu_launches": launches,
        "fallbacks": fallbacks,
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    job.close()


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
    dev_index = 0 if args.share_gpu else local
    torch.cuda.set_device(dev_index)
    job = Job("gloo" if args.share_gpu else "nccl", None if args.share_gpu else "cuda")
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
    job.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev_index)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    ms_local = e0.elapsed_time(e1)
    clk = clocks.stop()
    job.barrier()
    secs, fallbacks = shard.reduce_job(ms_local / 1e3, d_fb[:n_loc].cpu().tolist(), n_items, rank,
                                       world, device=job.device)
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
    roofline = roofline_block(px, n_items / world, ms_step, stage_ms, N, W, H)

    # end to end: this rank's frames from pinned host memory through the
    # pipelined host entry (H2D of frame f+1 overlaps compute of f), every step
    e2e = None
    if not args.no_extras:
        h_in = d_in[:max(n_loc, 1)].cpu().pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        h_in_np, h_out_np = h_in.numpy(), h_out.numpy()
        if n_loc:
            plan.filter_host(h_in_np[:n_loc], h_out_np[:n_loc])
        torch.cuda.synchronize()
        job.barrier()
        e2e_steps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            if n_loc:
                plan.filter_host(h_in_np[:n_loc], h_out_np[:n_loc])
        e2e_s = job.max((time.perf_counter() - t0) / e2e_steps)
        e2e = {"value": round(n_items * px / e2e_s / 1e6, 1), "unit": UNIT,
               "h2d_bytes_per_step": n_items * px * 4, "d2h_bytes_per_step": n_items * (px * 4 + 8),
               "api": "gpf_b200_filter_f32_host (pinned host fp32 in/out, all local frames per call, "
                      "H2D/compute/D2H pipelined inside)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        thr = cpu_threads()
        kind, run = reference_filter(thr)
        img = d_in[0].double().cpu().numpy()
        t0 = time.perf_counter()
        run(img, ss, sr, N)
        sec = time.perf_counter() - t0
        cpu = {"value": round(px / sec / 1e6, 3), "unit": UNIT, "cores": thr, "kind": kind,
               "cpu_model": cpu_model(),
               "sample": f"one full C4 problem (frame 0, channel 0, {W}x{H}) at sigma_s {ss:g}, "
                         f"sigma_r {sr:g}, N {N}: {sec:.1f} s"}
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
    job.close()


# ------------------------------------------------------------- reference arm
def bench_reference(args):
    """The reference's own CPU implementation on the bench's frames: step s
    filters frame k = s mod 5 of the C3 batch at sigma_s[k] with all host
    threads -- the whole frame, or, when K whole frames would not finish in
    about REF_BUDGET_S, a full-width band of rows of it (the reference's cost
    per pixel does not depend on the frame height; the band moves down the
    frame from step to step). Warm-up steps page the library and the frames in
    on a 512-row full-width band and time it to size the band. Under torchrun
    only rank 0 runs."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    from paper_1505_00077_b200 import synth
    cfg = synth.CONFIGS[4 if args.workload == "c4" else CFG_ID]
    thr = cpu_threads()
    kind, run = reference_filter(thr)
    if args.workload == "c4":
        imgs = [synth.make(cfg, 0, 0).astype("float64")]
        sig = [cfg.sigma_s[0]]
    else:
        n = args.size or cfg.width
        c = synth.scaled(cfg, n, n) if args.size else cfg
        imgs = [synth.make(c, k).astype("float64") for k in range(len(cfg.sigma_s))]
        sig = list(cfg.sigma_s)
    h, w = imgs[0].shape
    cal_rows = min(h, 512)
    t_cal = None
    for _ in range(max(1, args.warmup)):
        t0 = time.perf_counter()
        run(np.ascontiguousarray(imgs[0][:cal_rows]), sig[0], cfg.sigma_r, cfg.degree)
        t_cal = time.perf_counter() - t0
    # rows per step: whole frames if K of them fit the budget, else a band
    # (calibrated on a full-width band, with a 1.3x margin)
    est_frame_s = 1.3 * t_cal * h / cal_rows
    rows = h
    if args.steps * est_frame_s > REF_BUDGET_S:
        rows = int(h * REF_BUDGET_S / (args.steps * est_frame_s)) // 64 * 64
        rows = max(256, min(h, rows))
    times, px = [], 0
    for s in range(args.steps):
        k = s % len(imgs)
        r0 = (s * rows) % h if rows < h else 0
        r0 = min(r0, h - rows)
        band = imgs[k] if rows == h else np.ascontiguousarray(imgs[k][r0:r0 + rows])
        t0 = time.perf_counter()
        run(band, sig[k], cfg.sigma_r, cfg.degree)
        times.append(time.perf_counter() - t0)
        px += band.size
    total = sum(times)
    v = px / total / 1e6
    sample = (f"{args.steps} full {w}x{h} frames" if rows == h else
              f"{args.steps} full-width bands of {rows} rows ({w}x{rows}) of the {w}x{h} frames, "
              f"the band moving down the frame")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 1),
        "higher_is_better": True, "scaling": "strong" if args.workload == "c4" else "weak",
        "vs_baseline": None, "dtype": "fp64",
        "data": "synthetic (seeded generator, SURVEY.md 8(d))",
        "config": {"workload": (f"C{cfg.cid}: {w}x{h} frame k of the batch at sigma_s[k] per step "
                                f"(k = step mod {len(imgs)}; {'whole frame' if rows == h else f'{rows}-row band'}), "
                                f"sigma_r {cfg.sigma_r:g}, N {cfg.degree}, sigma_s {sig}"),
                   "parallelism": f"{thr} host threads (gpf_set_num_threads)"},
        "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": thr, "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"{sample} ({total:.1f} s)"},
        "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- CPU self-test
def selftest_cpu(args):
    """The launch and reduction plumbing of the B200 leg with a stub filter:
    torchrun relaunch, gloo process group, frame shard per rank, max-over-ranks
    time, whole-job value. No GPU and no library involved."""
    import numpy as np
    rank, world, _ = dist_env()
    job = Job("gloo", None)
    n_fr, n = 5, args.size or 64
    frames = [np.full((n, n), float(n_fr * rank + k), np.float32) for k in range(n_fr)]
    job.barrier()
    t0 = time.perf_counter()
    acc = 0.0
    for _ in range(args.steps):
        for f in frames:
            acc += float(np.cumsum(f, axis=0)[-1].sum())  # stub work
    ms = job.max((time.perf_counter() - t0) * 1e3)
    total_frames = job.sum(n_fr)
    ms_step = ms / args.steps
    line = {"metric": METRIC, "value": round(world * n_fr * n * n / (ms_step / 1e3) / 1e6, 3),
            "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "scaling": "weak", "selftest": True,
            "frames_total": int(total_frames), "checksum": job.sum(acc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    job.close()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    if args.selftest_cpu:
        selftest_cpu(args)
    elif args.impl == "reference":
        bench_reference(args)
    elif args.workload == "c4":
        bench_c4(args)
    else:
        bench_b200(args)


if __name__ == "__main__":
    main()
