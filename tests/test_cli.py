"""gpf_b200 command-line front end (filter / compare / bench; the reference
CLI's flags and CSV protocol, proj/tools/gpf_cli.cpp). Argument errors run on
CPU; the filtering runs are GPU tests."""
import csv
import os
import subprocess

import numpy as np
import pytest

from paper_1505_00077_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1505_00077_b200", "gpf_b200")


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True)


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(CLI):
        subprocess.run(["make", "-s", "-C", os.path.dirname(CLI)], check=True)
    return CLI


def test_cli_argument_errors(cli, tmp_path):
    r = run("filter", "--input", "x.pgm")
    assert r.returncode == 1 and "error: --output: is required" in r.stderr
    r = run("filter", "--input", "x", "--output", "y", "--method", "median", "--sigma-s", "2",
            "--sigma-r", "30")
    assert r.returncode == 1 and "--method" in r.stderr
    r = run("filter", "--input", str(tmp_path / "missing.pgm"), "--output", "y", "--method", "gpf",
            "--sigma-s", "2", "--sigma-r", "30")
    assert r.returncode == 1 and r.stderr.startswith("error: --input: cannot open")
    r = run("bench", "--input", "x", "--method", "gpf", "--sigma-s-list", "2,-1", "--sigma-r", "30",
            "--degree", "20", "--backend", "recursive", "--csv", "o.csv")
    assert r.returncode == 1 and "--sigma-s-list" in r.stderr
    r = run("kernel-error")
    assert r.returncode == 1 and "error: --sigma-r: is required" in r.stderr
    r = run("kernel-error", "--sigma-r", "30", "--degree", "20", "--tau-list", "0,40", "--range", "255:0",
            "--step", "1", "--which", "both", "--csv", str(tmp_path / "k.csv"))
    assert r.returncode == 1 and "error: --range: expected LO:HI with LO < HI" in r.stderr
    assert run("--version").stdout.strip().endswith("b200")


def test_cli_kernel_error_csv(cli, reference, tmp_path):
    """kernel-error (host only): the reference CLI's CSV (proj/tools/gpf_cli.cpp:165-199),
    values equal to the reference library's gpf_kernel_sup_error."""
    path = tmp_path / "k.csv"
    r = run("kernel-error", "--sigma-r", "30", "--degree", "12", "--tau-list", "0,40,-100.5", "--range",
            "0:255", "--step", "0.5", "--which", "both", "--csv", str(path))
    assert r.returncode == 0, r.stderr
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["tau", "approx", "sup_error"]
    assert [(a, b) for a, b, _ in rows[1:]] == [("0.0", "gp"), ("0.0", "taylor"), ("40.0", "gp"), ("40.0", "taylor"),
                                                ("-100.5", "gp"), ("-100.5", "taylor")]
    for tau, ap, v in rows[1:]:
        st, want = reference.kernel("sup_error", 30.0, 12, float(tau), 0.0, 255.0, 0.5, 0 if ap == "gp" else 1)
        assert st == 0 and float(v) == want
    assert rows[1][2] == "0.0"
    r = run("kernel-error", "--sigma-r", "30", "--degree", "12", "--tau-list", "40", "--range", "0:255",
            "--step", "1", "--which", "taylor", "--csv", str(path))
    assert r.returncode == 0 and [x[1] for x in csv.reader(open(path))][1:] == ["taylor"]


@pytest.mark.gpu
def test_cli_filter_compare_bench(cli, gpu, reference, tmp_path):
    img = np.round(synth.rects_image(96, 64, 6, 10.0, 3)).astype(np.float64)
    src = tmp_path / "in.pgm"
    gpu.gpf.write_pgm(img, str(src))
    out = tmp_path / "out.pgm"
    r = run("filter", "--input", str(src), "--output", str(out), "--method", "gpf", "--sigma-s", "3",
            "--sigma-r", "30")
    assert r.returncode == 0, r.stderr
    st, ref, _ = reference.gpf(img, 3.0, 30.0, 20)
    want = np.frombuffer(reference.encode_pgm(ref)[-96 * 64:], np.uint8).astype(int)
    got = np.frombuffer(out.read_bytes()[-96 * 64:], np.uint8).astype(int)
    assert np.abs(got - want).max() <= 1 and (got == want).mean() > 0.999  # rounding ties only
    ex = tmp_path / "ex.pgm"
    assert run("filter", "--input", str(src), "--output", str(ex), "--method", "exact", "--sigma-s",
               "2", "--sigma-r", "30").returncode == 0
    r = run("compare", "--ref", str(ex), "--test", str(out), "--exclude-border", "2")
    assert r.returncode == 0 and r.stdout.startswith("mse=")
    fields = dict(kv.split("=") for kv in r.stdout.split())
    rep = gpu.gpf_compare(gpu.gpf.read_pgm(str(ex)), gpu.gpf.read_pgm(str(out)), 2)
    assert float(fields["mse"]) == pytest.approx(rep["mse"], rel=1e-12)
    assert int(fields["pixels"]) == rep["pixels"] == 92 * 60
    table = tmp_path / "bench.csv"
    r = run("bench", "--input", str(src), "--method", "gpf,exact,taylor", "--sigma-s-list", "2,4.5",
            "--sigma-r", "30", "--degree", "20", "--backend", "recursive", "--repeats", "2",
            "--warmup", "1", "--csv", str(table))
    assert r.returncode == 0, r.stderr
    rows = list(csv.reader(open(table)))
    assert rows[0] == ["method", "backend", "sigma_s", "sigma_r", "degree", "pixels", "repeats",
                       "median_seconds"]
    assert [(x[0], x[2]) for x in rows[1:]] == [("gpf", "2.0"), ("gpf", "4.5"), ("exact", "2.0"),
                                              ("exact", "4.5"), ("taylor", "2.0"), ("taylor", "4.5")]
    assert all(x[1] == "recursive" and x[3] == "30.0" and x[4] == "20" and x[5] == str(96 * 64)
               and x[6] == "2" and float(x[7]) > 0 for x in rows[1:])
    # the direct backend through the CLI (reference flags --backend / --window / --boundary)
    dout = tmp_path / "direct.pgm"
    r = run("filter", "--input", str(src), "--output", str(dout), "--method", "gpf", "--sigma-s", "2",
            "--sigma-r", "30", "--backend", "direct", "--window", "4", "--boundary", "reflect")
    assert r.returncode == 0, r.stderr
    st, ref, _ = reference.gpf(img, 2.0, 30.0, 20, backend=0, window_radius=4, boundary=1)
    want = np.frombuffer(reference.encode_pgm(ref)[-96 * 64:], np.uint8).astype(int)
    got = np.frombuffer(dout.read_bytes()[-96 * 64:], np.uint8).astype(int)
    assert st == 0 and np.abs(got - want).max() <= 1 and (got == want).mean() > 0.999
