"""bench.py contract: helper arithmetic on CPU; one short run of each workload
on the GPU, checking the JSON line's keys and their consistency."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_roofline_helpers():
    import bench
    bpp, fpp = bench.design_bytes_per_px(11), bench.algorithmic_flops_per_px(11)
    assert sum(bpp.values()) == 282 and bpp["rowpass"] == 107
    model = bench.model_bytes_per_px(20)
    assert model["step"] == 188 and model["rowpass"] == 96
    assert bench.fp32_peak_tflops({"sm_max_mhz": 1965.0}) == pytest.approx(74.4, abs=0.05)
    r = bench.roofline_of(1000, 1.0, 100, 10, 1000.0, 74.4)  # HBM-bound
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["achieved"] == pytest.approx(0.1)
    r = bench.roofline_of(1000, 1.0, 1, 10 ** 9, 1000.0, 74.4)  # FLOP-bound
    assert r["bound"] == "fp32" and r["unit"] == "TFLOP/s"


def test_roofline_block_uses_survey_bytes(monkeypatch):
    import bench
    px = 10 ** 6
    monkeypatch.setattr(bench, "load_traffic", lambda w, h: {"bytes_per_launch": {"rowpass": 96 * px * 2}})
    r = bench.roofline_block(px, 5, 1.0, {"rowpass": 0.5, "colpass": 0.4}, 20, 1000, 1000)
    assert r["kernel"] == "rowpass" and r["algorithmic_bytes_per_px"] == 96
    assert r["traffic_over_algorithmic"] == 2.0
    assert r["step"]["bytes_per_px"] == 188
    assert r["achieved"] == pytest.approx(96 * px / 0.5e-3 / 1e9, rel=1e-3)


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_multirank_plumbing_cpu():
    """bench.py --gpus 2 relaunches itself under torch.distributed.run, builds a
    gloo group, shards the frame batch (5 frames per rank) and reduces the time
    (max over ranks) and the frame count (sum) -- with a stub filter on CPU."""
    env = dict(os.environ, GPF_BENCH_PORT=str(_free_port()))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--selftest-cpu",
                          "--steps", "3", "--warmup", "1", "--size", "32"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["frames_total"] == 10 and d["selftest"]
    # per-rank frames hold their global index: ranks 0 and 1 sum 0..9 over 32 x 32 x 3 steps
    assert d["checksum"] == pytest.approx(sum(range(10)) * 32 * 32 * 3)
    assert d["value"] > 0


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "cpu_baseline",
        "gpu_launches", "clocks"}


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["c3", "c4"])
def test_bench_json_line(gpu, workload):
    d = _run("--workload", workload, "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-mse")
    if workload == "c3":
        assert d["parity"]["max_abs"] <= 1e-3 and d["e2e_dropin"]["value"] > 0
        assert d["fp64_exact"]["C5"]["precision"] == "fp64"
    assert KEYS <= set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["scaling"] == ("weak" if workload == "c3" else "strong")
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r) and 0 < r["frac"] < 1
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


@pytest.mark.gpu
def test_bench_reference_arm(gpu):
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--size", "1024")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_bench_two_ranks_one_gpu(gpu):
    """The N > 1 code path end to end (relaunch, sharded frames, reductions) with
    both ranks on GPU 0 and gloo for the scalars: a functional run, not a number."""
    env = dict(os.environ, GPF_BENCH_PORT=str(_free_port()))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--share-gpu",
                          "--size", "1024", "--steps", "2", "--warmup", "3", "--no-cpu-baseline",
                          "--no-mse"], capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e_dropin"]["value"] > 0 and d["fallbacks"] == [0] * 5
