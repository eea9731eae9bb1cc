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
    bpp, fpp = bench.algorithmic_bytes_per_px(11), bench.algorithmic_flops_per_px(11)
    assert sum(bpp.values()) == 282 and bpp["rowpass"] == 107
    assert bench.fp32_peak_tflops({"sm_max_mhz": 1965.0}) == pytest.approx(74.4, abs=0.05)
    r = bench.roofline_of(1000, 1.0, 100, 10, 1000.0, 74.4)  # HBM-bound
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["achieved"] == pytest.approx(0.1)
    r = bench.roofline_of(1000, 1.0, 1, 10 ** 9, 1000.0, 74.4)  # FLOP-bound
    assert r["bound"] == "fp32" and r["unit"] == "TFLOP/s"


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
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1
