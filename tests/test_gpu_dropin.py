"""The drop-in entry's machinery (dropin.cpp, capi.cpp) and the plan entries'
robustness fixes: precision modes, plan cache, per-frame conditioning flags,
misaligned device pointers, failed re-batching, device restore."""
import numpy as np
import pytest

from paper_1505_00077_b200 import synth

pytestmark = pytest.mark.gpu

TOL = 1e-3


def test_precision_modes_and_envelope(gpu, oracle):
    """AUTO picks fp32 inside the envelope and the reference-exact fp64 mode
    outside it; both forced modes run; the limit is the documented one."""
    assert gpu.fp32_h_limit() == pytest.approx(7.0)
    inside = synth.rects_image(256, 192, 8, 10.0, 3).astype(np.float64)   # sigma_r 40: max|H| ~ 3.7
    outside = synth.checker_image(256, 192, 5.0, 4).astype(np.float64)    # sigma_r 10: max|H| 12.75
    for img, sr, want in ((inside, 40.0, "fp32"), (outside, 10.0, "fp64")):
        ref, rfb, tc = oracle.gpf(img, 4.0, sr, 20)
        for mode in ("auto", "fp32", "fp64"):
            gpu.set_precision(mode)
            try:
                out, fb = gpu.gpf_filter_gpf(img, gpu.spatial_params(4.0), gpu.range_params(sr, 20))
            finally:
                gpu.set_precision("auto")
            ran = gpu.last_precision()
            assert ran == (want if mode == "auto" else mode)
            if mode == "auto":
                hm = max(img.max() - tc, tc - img.min()) / sr
                assert gpu.last_max_abs_h() == pytest.approx(hm, rel=1e-12)
            if ran == "fp64" or want == "fp32":
                assert fb == rfb and np.abs(out - ref).max() <= TOL, (mode, want)


def test_fp64_mode_large_degree(gpu, oracle):
    """Degrees above the fp32 kernels' limit (48) run the fp64 mode (<= 62)."""
    img = synth.rects_image(64, 48, 4, 10.0, 5).astype(np.float64)
    for deg in (49, 62):
        ref, rfb, _ = oracle.gpf(img, 3.0, 60.0, deg)
        out, fb = gpu.gpf_filter_gpf(img, gpu.spatial_params(3.0), gpu.range_params(60.0, deg))
        assert gpu.last_precision() == "fp64"
        assert fb == rfb and np.abs(out - ref).max() <= 1e-9
    with pytest.raises(gpu.GpfError):
        gpu.gpf_filter_gpf(img, gpu.spatial_params(3.0), gpu.range_params(60.0, 63))
    gpu.set_precision("fp32")
    try:
        with pytest.raises(gpu.GpfError):
            gpu.gpf_filter_gpf(img, gpu.spatial_params(3.0), gpu.range_params(60.0, 49))
    finally:
        gpu.set_precision("auto")


def test_fp64_mode_matches_reference_goldens(gpu, golden):
    """The fp64 mode replays the reference's arithmetic: the golden cases agree
    to round-off (only exp() differs), far inside the bar."""
    gpu.set_precision("fp64")
    try:
        for name in [str(n) for n in golden["__names__"]]:
            img = golden[f"{name}/in"]
            ss, sr, deg, cen, ks = golden[f"{name}/params"]
            out, fb = gpu.gpf_filter_gpf(img, gpu.spatial_params(ss, kernel_scale=ks),
                                         gpu.range_params(sr, int(deg)), centering=int(cen))
            ref = golden[f"{name}/out"]
            assert fb == int(golden[f"{name}/fb"]), name
            assert np.abs(out - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max()), name
    finally:
        gpu.set_precision("auto")


def test_dropin_repeated_call_allocates_nothing(gpu):
    """A second call with the same shape and parameters reuses the cached plan,
    buffers and pinned images: device free memory is unchanged."""
    import torch
    img = synth.rects_image(1024, 768, 16, 10.0, 8).astype(np.float64)
    sp, rp = gpu.spatial_params(5.0), gpu.range_params(30.0, 20)
    a, _ = gpu.gpf_filter_gpf(img, sp, rp)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    b, _ = gpu.gpf_filter_gpf(img, sp, rp)
    free1 = torch.cuda.mem_get_info()[0]
    assert free1 == free0
    np.testing.assert_array_equal(a, b)
    gpu.dropin_release()
    assert torch.cuda.mem_get_info()[0] > free1


def test_checked_entry_flags(gpu):
    """gpf_b200_filter_f32_checked flags exactly the frames outside the fp32
    envelope, computed on the device from each frame."""
    import torch
    w, h = 320, 200
    good = synth.rects_image(w, h, 8, 10.0, 1)                       # sigma_r 10: rects ~ up to 15
    calm = np.clip(good * 0.2 + 100.0, 0, 255).astype(np.float32)    # narrow range: inside
    frames = np.stack([calm, good, calm])
    plan = gpu.Plan(w, h, 3.0, 10.0, 20, batch=2)
    d_in = torch.from_numpy(frames).cuda()
    d_out = torch.empty_like(d_in)
    d_ill = torch.full((3,), -1, dtype=torch.int32, device="cuda")
    plan.filter_device_checked(d_in, d_out, 3, None, d_ill, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    hm = [max(f.max() - f.astype(np.float64).mean(), f.astype(np.float64).mean() - f.min()) / 10.0
          for f in frames]
    want = [int(v > gpu.fp32_h_limit()) for v in hm]
    assert d_ill.cpu().tolist() == want and want == [0, 1, 0]


def test_misaligned_device_input(gpu):
    """A frame starting 4 bytes past a 16-B boundary: no vector
    load faults, same result as the aligned copy."""
    import torch
    w, h = 256, 64
    img = torch.from_numpy(synth.rects_image(w, h, 4, 10.0, 2)).cuda()
    buf = torch.empty(w * h + 1, device="cuda")
    buf[1:].copy_(img.reshape(-1))
    mis = buf[1:].view(h, w)
    assert mis.data_ptr() % 16 == 4
    plan = gpu.Plan(w, h, 3.0, 30.0, 20)
    s = torch.cuda.current_stream().cuda_stream
    a, b = torch.empty_like(img), torch.empty_like(img)
    plan.filter_device(img, a, 1, None, s)
    plan.filter_device(mis, b, 1, None, s)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_failed_rebatch_keeps_plan_usable(gpu):
    """plan_set_batch that cannot allocate returns an error and leaves the
    plan's previous workspace intact."""
    import ctypes as C
    import torch
    from paper_1505_00077_b200 import _lib
    w = h = 4096
    plan = gpu.Plan(w, h, 3.0, 30.0, 20)
    st = _lib.lib().gpf_b200_plan_set_batch(plan.h, 100000)  # petabytes
    assert st != 0
    img = torch.from_numpy(synth.rects_image(512, 512, 4, 10.0, 2)).cuda()
    img = torch.nn.functional.interpolate(img[None, None], size=(h, w))[0, 0].contiguous()
    out = torch.empty_like(img)
    plan.filter_device(img, out, 1, None, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    del C


def test_plan_create_restores_current_device(gpu):
    import ctypes as C
    import torch
    from paper_1505_00077_b200 import _lib
    torch.cuda.set_device(0)
    sp, rp = gpu.spatial_params(2.0), gpu.range_params(30.0, 20)
    h = C.c_void_p()
    assert _lib.lib().gpf_b200_plan_create(64, 64, C.byref(sp), C.byref(rp), 1, 0, C.byref(h)) == 0
    assert torch.cuda.current_device() == 0
    _lib.lib().gpf_b200_plan_destroy(h)
    # the fp32 plan entries reject degrees above their kernels' limit with one message
    with pytest.raises(gpu.GpfError, match="48"):
        gpu.Plan(64, 64, 2.0, 30.0, 49)


@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (5, 1), (2, 33), (33, 2), (31, 65), (64, 32),
                                   (1, 1000), (1000, 1), (97, 131)])
def test_fp64_mode_shapes(gpu, oracle, shape):
    """The fp64 mode's row tiles (32 rows x 32-column chunks) and column
    threads at every edge: partial tiles, single rows / columns."""
    img = np.random.default_rng(sum(shape) + 7).uniform(0, 255, size=shape)
    ref, rfb, _ = oracle.gpf(img, 2.0, 12.0, 20)
    gpu.set_precision("fp64")
    try:
        out, fb = gpu.gpf_filter_gpf(img, gpu.spatial_params(2.0), gpu.range_params(12.0, 20))
    finally:
        gpu.set_precision("auto")
    assert fb == rfb
    assert np.abs(out - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max()), shape


@pytest.mark.parametrize("mode", ["fp32", "fp64"])
@pytest.mark.parametrize("deg", [0, 1, 2])
def test_low_degrees(gpu, oracle, mode, deg):
    img = synth.rects_image(70, 45, 4, 10.0, 3 + deg).astype(np.float64)
    ref, rfb, _ = oracle.gpf(img, 3.0, 40.0, deg)
    gpu.set_precision(mode)
    try:
        out, fb = gpu.gpf_filter_gpf(img, gpu.spatial_params(3.0), gpu.range_params(40.0, deg))
    finally:
        gpu.set_precision("auto")
    assert fb == rfb and np.abs(out - ref).max() <= TOL


def test_dropin_concurrent_host_threads(gpu):
    """gpf_filter_gpf from several host threads at once (the engine serialises
    calls per device): every thread gets its sequential result, in both modes."""
    import threading
    cases = [(synth.rects_image(200 + 8 * k, 150, 6, 10.0, 30 + k).astype(np.float64),
              2.0 + k, 30.0 if k % 2 == 0 else 10.0) for k in range(6)]
    seq = [gpu.gpf_filter_gpf(img, gpu.spatial_params(ss), gpu.range_params(sr)) for img, ss, sr in cases]
    got = [None] * len(cases)

    def work(i):
        img, ss, sr = cases[i]
        for _ in range(3):
            got[i] = gpu.gpf_filter_gpf(img, gpu.spatial_params(ss), gpu.range_params(sr))
    ths = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for (a, fa), (b, fb) in zip(seq, got):
        assert fa == fb
        np.testing.assert_array_equal(a, b)


def test_stage_timing_and_timeline(gpu):
    """Per-stage profiling of a plan (bench.py's stage times, tools/timeline.py):
    stage_times sums every recorded stage, stage_marks returns the timeline --
    stages 0..4 then the end marker per launch group, non-decreasing times after
    the caller's reference event -- and consumes the events."""
    import torch

    w, h = 512, 384
    img = torch.from_numpy(synth.rects_image(w, h, 8, 10.0, 11)).cuda()
    out = torch.empty_like(img)
    plan = gpu.Plan(w, h, 3.0, 30.0, 20)
    try:
        st = torch.cuda.current_stream()
        plan.set_profiling(True)
        plan.filter_device(img, out, 1, None, st.cuda_stream)
        times = plan.stage_times()
        assert set(times) == set(plan.STAGES) and all(v > 0 for v in times.values()), times
        ref = torch.cuda.Event(enable_timing=True)
        ref.record(st)
        for _ in range(2):
            plan.filter_device(img, out, 1, None, st.cuda_stream)
        marks = plan.stage_marks(ref.cuda_event)
        assert [s for s, _ in marks] == [0, 1, 2, 3, 4, -1] * 2, marks
        ts = [t for _, t in marks]
        assert ts[0] >= 0 and all(b >= a for a, b in zip(ts, ts[1:])), ts
        assert plan.stage_marks(ref.cuda_event) == []  # consumed
    finally:
        plan.set_profiling(False)
        plan.close()


@pytest.mark.gpu
def test_dropin_concurrent_large_frames_pipeline(gpu):
    """Concurrent calls on >= 4 MP frames (the band/pixel-range D2H path of the
    call slots), fp32 and fp64 modes mixed: every thread's result is bitwise its
    sequential one, fallback counts included."""
    import threading
    cases = [(synth.rects_image(2048, 2048, 64, 15.0, 700 + k).astype(np.float64), 5.0 + k,
              30.0 if k % 2 == 0 else 10.0) for k in range(4)]
    seq = [gpu.gpf_filter_gpf(img, gpu.spatial_params(ss), gpu.range_params(sr)) for img, ss, sr in cases]
    got = [None] * len(cases)
    errs = []

    def work(i):
        try:
            img, ss, sr = cases[i]
            for _ in range(2):
                got[i] = gpu.gpf_filter_gpf(img, gpu.spatial_params(ss), gpu.range_params(sr))
        except Exception as e:  # surfaced below
            errs.append(e)
    ths = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    for (a, fa), (b, fb) in zip(seq, got):
        assert fa == fb
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("shape,deg,ss", [((97, 131), 20, 2.0), ((64, 64), 7, 0.7), ((33, 200), 49, 6.0),
                                          ((300, 40), 20, 25.0), ((1, 77), 3, 3.0), ((520, 515), 20, 9.0)])
def test_fp64_chunked_equals_sequential_bitwise(gpu, shape, deg, ss, monkeypatch):
    """The chunked fp64 passes (anticausal states recorded per 32-sample chunk,
    chunks restarted from them) against the literal sequential replay
    (GPF_B200_F64_SEQUENTIAL=1): same operations in the same order, equal bits."""
    img = np.random.default_rng(shape[0] * 1000 + shape[1]).uniform(0, 255, size=shape)
    gpu.set_precision("fp64")
    try:
        out, fb = gpu.gpf_filter_gpf(img, gpu.spatial_params(ss), gpu.range_params(11.0, deg))
        monkeypatch.setenv("GPF_B200_F64_SEQUENTIAL", "1")
        seq, fbs = gpu.gpf_filter_gpf(img, gpu.spatial_params(ss), gpu.range_params(11.0, deg))
    finally:
        gpu.set_precision("auto")
    assert fb == fbs
    assert np.array_equal(out.view(np.uint64), seq.view(np.uint64)), shape


def test_filter_batch_one_shot(gpu, oracle):
    """gpf_b200_filter_batch (SURVEY 8(b)'s plan-less device entry): equals the plan
    entry bitwise, holds the bar against the oracle, allocates nothing on a repeated
    call, keeps several parameter sets cached and rejects what the plan entry rejects."""
    import torch

    w, h, n = 160, 96, 3
    frames = np.stack([synth.rects_image(w, h, 6, 10.0, 20 + k) for k in range(n)]).astype(np.float32)
    d_in = torch.from_numpy(frames).cuda()
    d_out = torch.empty_like(d_in)
    d_fb = torch.zeros(n, dtype=torch.int64, device="cuda")
    sp, rp = gpu.spatial_params(4.0), gpu.range_params(35.0, 20)
    gpu.filter_batch_device(d_in, d_out, w, h, n, sp, rp, 1, d_fb)
    torch.cuda.synchronize()
    out = d_out.cpu().numpy()
    plan = gpu.Plan(w, h, 4.0, 35.0, 20)
    d_ref = torch.empty_like(d_in)
    plan.filter_device(d_in, d_ref, n)
    torch.cuda.synchronize()
    plan.close()
    assert np.array_equal(out, d_ref.cpu().numpy())
    for k in range(n):
        ref, rfb, _ = oracle.gpf(frames[k].astype(np.float64), 4.0, 35.0, 20)
        assert int(d_fb[k]) == rfb and np.abs(out[k] - ref).max() <= TOL
    # a second parameter set, then the first again: both stay cached, nothing is allocated
    sp2 = gpu.spatial_params(9.0)
    gpu.filter_batch_device(d_in, d_out, w, h, n, sp2, rp)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for s in (sp, sp2, sp):
        gpu.filter_batch_device(d_in, d_out, w, h, n, s, rp, 1, d_fb)
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] == free0
    assert np.array_equal(d_out.cpu().numpy(), out)
    gpu.filter_batch_device(d_in, d_out, w, h, 0, sp, rp)  # empty batch: nothing to do
    with pytest.raises(gpu.GpfError, match="sigma_s"):
        gpu.filter_batch_device(d_in, d_out, w, h, n, gpu.spatial_params(-1.0), rp)
    with pytest.raises(gpu.GpfError, match="48"):
        gpu.filter_batch_device(d_in, d_out, w, h, n, sp, gpu.range_params(35.0, 49))
    gpu.dropin_release()
