"""Host-side mirror of the reference's GPF interface over the B200 C ABI.

``gpf_filter_gpf`` follows ``gpf_filter_gpf`` of the reference C ABI
(proj/include/gpfilter/gpfilter.h:100-107, proj/src/capi.cpp:176-192): same
parameter structs and defaults, same status codes; a non-OK status raises
``GpfError`` carrying the status and the library's ``gpf_last_error`` text.

``Plan`` is the batched device-resident entry (gpfilter_b200.h): fp32 frames
already in HBM, addressed by raw device pointers or torch CUDA tensors.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import (GPF_BACKEND_DIRECT, GPF_BACKEND_RECURSIVE, GPF_BOUNDARY_REFLECT,  # noqa: F401
                   GPF_BOUNDARY_REPLICATE, GPF_BOUNDARY_ZERO, RangeParams, SpatialParams)


class GpfError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        self.detail = detail
        name = _lib.lib().gpf_status_name(status).decode()
        super().__init__(f"{name}: {detail}")


def _check(status: int) -> None:
    if status != _lib.GPF_OK:
        raise GpfError(status, _lib.lib().gpf_last_error().decode())


def spatial_params(sigma_s: float = 2.0, window_radius: int = 0,
                   boundary: int = GPF_BOUNDARY_REPLICATE,
                   kernel_scale: float = 1.0) -> SpatialParams:
    sp = SpatialParams()
    _lib.lib().gpf_spatial_params_init(C.byref(sp))
    sp.sigma_s, sp.window_radius, sp.boundary, sp.kernel_scale = (
        sigma_s, window_radius, boundary, kernel_scale)
    return sp


def range_params(sigma_r: float = 30.0, degree: int = 20) -> RangeParams:
    rp = RangeParams()
    _lib.lib().gpf_range_params_init(C.byref(rp))
    rp.sigma_r, rp.degree = sigma_r, degree
    return rp


class Image:
    """Owning handle of a gpf_image (row-major doubles)."""

    def __init__(self, handle: C.c_void_p):
        self.h = handle

    @classmethod
    def from_array(cls, a: np.ndarray) -> "Image":
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise ValueError("image must be 2-D (height, width)")
        hdl = C.c_void_p()
        _check(_lib.lib().gpf_image_create(a.shape[1], a.shape[0], C.byref(hdl)))
        img = cls(hdl)
        img.view()[...] = a
        return img

    @property
    def shape(self):
        L = _lib.lib()
        return (L.gpf_image_height(self.h), L.gpf_image_width(self.h))

    def view(self) -> np.ndarray:
        h, w = self.shape
        ptr = _lib.lib().gpf_image_data(self.h)
        return np.ctypeslib.as_array(ptr, shape=(h * w,)).reshape(h, w)

    def numpy(self) -> np.ndarray:
        return self.view().copy()

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().gpf_image_destroy(self.h)
                self.h = None
        except Exception:  # interpreter shutdown: module globals may already be gone
            pass


def gpf_filter_gpf(img: np.ndarray, sp: SpatialParams | None = None, rp: RangeParams | None = None,
                   backend: int = GPF_BACKEND_RECURSIVE, centering: int = 1):
    """Constant-time Gauss-polynomial bilateral filter on the GPU.

    Returns ``(out, fallback_count)``; raises GpfError on a non-OK status.
    """
    sp = sp or spatial_params()
    rp = rp or range_params()
    src = Image.from_array(img)
    out = C.c_void_p()
    fb = C.c_longlong(-1)
    _check(_lib.lib().gpf_filter_gpf(src.h, C.byref(sp), C.byref(rp), backend, centering,
                                     C.byref(fb), C.byref(out)))
    res = Image(out)
    return res.numpy(), fb.value


def gpf_gaussian_recursive(img: np.ndarray, sigma_s: float, kernel_scale: float = 1.0) -> np.ndarray:
    """Single-plane recursive Gaussian (reference gpf_gaussian_recursive)."""
    src = Image.from_array(img)
    out = C.c_void_p()
    _check(_lib.lib().gpf_gaussian_recursive(src.h, sigma_s, kernel_scale, C.byref(out)))
    return Image(out).numpy()


def gpf_gaussian_direct(img: np.ndarray, sp: SpatialParams | None = None) -> np.ndarray:
    """Single-plane windowed Gaussian (reference gpf_gaussian_direct), fp64 on the GPU."""
    sp = sp or spatial_params()
    src = Image.from_array(img)
    out = C.c_void_p()
    _check(_lib.lib().gpf_gaussian_direct(src.h, C.byref(sp), C.byref(out)))
    return Image(out).numpy()


GPF_RANGE_APPROX_GAUSS_POLY, GPF_RANGE_APPROX_TAYLOR = 0, 1


def kernel_gauss(t: float, tau: float, sigma_r: float) -> float:
    """exp(-(t - tau)^2 / 2 sigma_r^2) (reference gpf_kernel_gauss)."""
    v = C.c_double()
    _check(_lib.lib().gpf_kernel_gauss(t, tau, sigma_r, C.byref(v)))
    return v.value


def kernel_gauss_poly(t: float, tau: float, sigma_r: float, degree: int) -> float:
    """Degree-N Gauss-polynomial range kernel (reference gpf_kernel_gauss_poly)."""
    v = C.c_double()
    _check(_lib.lib().gpf_kernel_gauss_poly(t, tau, sigma_r, degree, C.byref(v)))
    return v.value


def kernel_taylor(t: float, tau: float, sigma_r: float, degree: int) -> float:
    """Degree-N Taylor range kernel (reference gpf_kernel_taylor)."""
    v = C.c_double()
    _check(_lib.lib().gpf_kernel_taylor(t, tau, sigma_r, degree, C.byref(v)))
    return v.value


def kernel_sup_error(sigma_r: float, degree: int, tau: float, low: float, high: float, step: float,
                     which: int = GPF_RANGE_APPROX_GAUSS_POLY) -> float:
    """sup |exact - approximation| over the closed grid (reference gpf_kernel_sup_error)."""
    v = C.c_double()
    _check(_lib.lib().gpf_kernel_sup_error(sigma_r, degree, tau, low, high, step, which, C.byref(v)))
    return v.value


def gpf_filter_taylor(img: np.ndarray, sp: SpatialParams | None = None, rp: RangeParams | None = None,
                      backend: int = GPF_BACKEND_RECURSIVE):
    """Taylor-polynomial baseline (reference gpf_filter_taylor), on the GPU.
    Returns ``(out, fallback_count)``."""
    sp = sp or spatial_params()
    rp = rp or range_params()
    src = Image.from_array(img)
    out = C.c_void_p()
    fb = C.c_longlong(-1)
    _check(_lib.lib().gpf_filter_taylor(src.h, C.byref(sp), C.byref(rp), backend, C.byref(fb),
                                        C.byref(out)))
    return Image(out).numpy(), fb.value


def gpf_filter_exact(img: np.ndarray, sp: SpatialParams | None = None,
                     rp: RangeParams | None = None) -> np.ndarray:
    """Exact brute-force bilateral filter (reference gpf_filter_exact), on the GPU."""
    sp = sp or spatial_params()
    rp = rp or range_params()
    src = Image.from_array(img)
    out = C.c_void_p()
    _check(_lib.lib().gpf_filter_exact(src.h, C.byref(sp), C.byref(rp), C.byref(out)))
    return Image(out).numpy()


def _report(rep) -> dict:
    return {"mse": rep.mse, "mse_db": rep.mse_db, "max_abs": rep.max_abs, "pixels": rep.pixels}


def gpf_compare(ref: np.ndarray, test: np.ndarray, exclude_border: int = 0) -> dict:
    """Error statistics (reference gpf_compare / metrics::compare)."""
    a, b = Image.from_array(ref), Image.from_array(test)
    rep = _lib.ErrorReport()
    _check(_lib.lib().gpf_compare(a.h, b.h, exclude_border, C.byref(rep)))
    return _report(rep)


def exact_device(d_in, d_out, width: int, height: int, sigma_s: float, sigma_r: float,
                 count: int = 1, boundary: int = GPF_BOUNDARY_REPLICATE, stream: int = 0) -> None:
    """Exact bilateral of `count` fp32 device frames (gpf_b200_exact_f32), on `stream`."""
    sp = spatial_params(sigma_s, boundary=boundary)
    rp = range_params(sigma_r)
    _check(_lib.lib().gpf_b200_exact_f32(_ptr(d_in), _ptr(d_out), width, height, count, C.byref(sp),
                                         C.byref(rp), stream))


def filter_batch_device(d_in, d_out, width: int, height: int, count: int,
                        sp: SpatialParams | None = None, rp: RangeParams | None = None,
                        centering: int = 1, d_fallbacks=None, stream: int = 0) -> None:
    """gpf_b200_filter_batch: `count` contiguous device fp32 frames, no plan handle
    (the library caches one per device, size and parameter set). Enqueued on `stream`."""
    sp = sp or spatial_params()
    rp = rp or range_params()
    fb = _ptr(d_fallbacks) if d_fallbacks is not None else None
    _check(_lib.lib().gpf_b200_filter_batch(_ptr(d_in), _ptr(d_out), width, height, count, C.byref(sp),
                                            C.byref(rp), centering, fb, stream))


def compare_device(d_ref, d_test, width: int, height: int, exclude_border: int = 0,
                   stream: int = 0) -> dict:
    """gpf_compare on fp32 device images (synchronises `stream`)."""
    rep = _lib.ErrorReport()
    _check(_lib.lib().gpf_b200_compare_f32(_ptr(d_ref), _ptr(d_test), width, height, exclude_border,
                                           C.byref(rep), stream))
    return _report(rep)


def read_pgm(path: str) -> np.ndarray:
    """gpf_read_pgm: P5/P2 file -> float64 array (raises GpfError with the PGM status)."""
    out = C.c_void_p()
    _check(_lib.lib().gpf_read_pgm(path.encode(), C.byref(out)))
    return Image(out).numpy()


def decode_pgm(data: bytes) -> np.ndarray:
    out = C.c_void_p()
    buf = C.create_string_buffer(data, len(data))
    _check(_lib.lib().gpf_decode_pgm(buf, len(data), C.byref(out)))
    return Image(out).numpy()


def encode_pgm(img: np.ndarray) -> bytes:
    src = Image.from_array(img)
    p = C.POINTER(C.c_uint8)()
    n = C.c_size_t()
    _check(_lib.lib().gpf_encode_pgm(src.h, C.byref(p), C.byref(n)))
    try:
        return bytes(p[:n.value])
    finally:
        _lib.lib().gpf_free_bytes(p)


def write_pgm(img: np.ndarray, path: str) -> None:
    src = Image.from_array(img)
    _check(_lib.lib().gpf_write_pgm(src.h, path.encode()))


PRECISIONS = {"auto": _lib.PRECISION_AUTO, "fp32": _lib.PRECISION_FP32, "fp64": _lib.PRECISION_FP64}


def set_precision(mode: str) -> None:
    """Precision of gpf_filter_gpf: "auto" (default), "fp32" or "fp64" (gpfilter_b200.h)."""
    _check(_lib.lib().gpf_b200_set_precision(PRECISIONS[mode]))


def get_precision() -> str:
    inv = {v: k for k, v in PRECISIONS.items()}
    return inv[_lib.lib().gpf_b200_get_precision()]


def last_precision() -> str | None:
    """Mode ("fp32"/"fp64") this thread's last gpf_filter_gpf call ran."""
    return {1: "fp32", 2: "fp64"}.get(_lib.lib().gpf_b200_last_precision())


def last_max_abs_h() -> float:
    return _lib.lib().gpf_b200_last_max_abs_h()


def last_device_ms() -> float:
    """Device time of the filter kernels of this thread's last gpf_filter_gpf call."""
    return _lib.lib().gpf_b200_last_device_ms()


def fp32_h_limit(degree: int | None = None) -> float:
    """The fp32 envelope (max|H| up to which AUTO runs the fp32 kernels) at
    `degree`, or at the default degree 20."""
    if degree is None:
        return _lib.lib().gpf_b200_fp32_h_limit()
    return _lib.lib().gpf_b200_fp32_h_limit_degree(int(degree))


def dropin_release() -> None:
    _lib.lib().gpf_b200_dropin_release()


def set_num_threads(n: int) -> None:
    _check(_lib.lib().gpf_set_num_threads(n))


def get_num_threads() -> int:
    return _lib.lib().gpf_get_num_threads()


def _ptr(x) -> int:
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    raise TypeError("expected a device pointer (int) or a torch CUDA tensor")


class Plan:
    """Device workspace for filtering fp32 frames of one size/parameter set."""

    def __init__(self, width: int, height: int, sigma_s: float, sigma_r: float, degree: int = 20,
                 kernel_scale: float = 1.0, centering: int = 1, device: int = -1, batch: int = 1):
        self.width, self.height = width, height
        sp = spatial_params(sigma_s, kernel_scale=kernel_scale)
        rp = range_params(sigma_r, degree)
        self.h = C.c_void_p()
        _check(_lib.lib().gpf_b200_plan_create(width, height, C.byref(sp), C.byref(rp),
                                               centering, device, C.byref(self.h)))
        if batch > 1:
            _check(_lib.lib().gpf_b200_plan_set_batch(self.h, batch))

    STAGES = ("mean", "col_carry", "colpass", "row_scan", "rowpass")

    def set_profiling(self, enable: bool) -> None:
        """Record CUDA events between this plan's kernels (per-stage timing)."""
        _check(_lib.lib().gpf_b200_plan_set_profiling(self.h, 1 if enable else 0))

    def stage_times(self) -> dict:
        """Milliseconds per stage accumulated since profiling was enabled (syncs)."""
        buf = (C.c_float * len(self.STAGES))()
        n = _lib.lib().gpf_b200_plan_stage_times(self.h, buf, len(self.STAGES))
        return {self.STAGES[i]: float(buf[i]) for i in range(n)}

    def stage_marks(self, ref_event: int, max_marks: int = 4096) -> list:
        """[(stage, ms after ref_event)] of the recorded stage events (stage -1 =
        end of a launch group); `ref_event` is a cudaEvent_t handle. Syncs."""
        t = (C.c_float * max_marks)()
        st = (C.c_int * max_marks)()
        n = _lib.lib().gpf_b200_plan_stage_marks(self.h, C.c_void_p(ref_event), t, st, max_marks)
        return [(int(st[i]), float(t[i])) for i in range(n)]

    @property
    def workspace_bytes(self) -> int:
        return _lib.lib().gpf_b200_plan_workspace_bytes(self.h)

    @property
    def launches_per_frame(self) -> int:
        return _lib.lib().gpf_b200_plan_launches_per_frame(self.h)

    def filter_device(self, d_in, d_out, count: int = 1, d_fallbacks=None, stream: int = 0,
                      front_done: int | None = None) -> None:
        """Enqueue `count` frames (device fp32 in -> device fp32 out) on `stream`.
        `front_done` (a cudaEvent_t handle, e.g. torch.cuda.Event().cuda_event)
        is recorded once the last frame's column half is enqueued."""
        fb = _ptr(d_fallbacks) if d_fallbacks is not None else None
        _check(_lib.lib().gpf_b200_filter_f32_ev(self.h, _ptr(d_in), _ptr(d_out), count, fb, stream,
                                                 front_done))

    def filter_device_checked(self, d_in, d_out, count: int, d_fallbacks, d_ill,
                              stream: int = 0) -> None:
        """filter_device plus per-frame ill-conditioned flags (int32 device array):
        1 where the frame lies outside the fp32 envelope (gpf_b200_filter_f32_checked)."""
        fb = _ptr(d_fallbacks) if d_fallbacks is not None else None
        _check(_lib.lib().gpf_b200_filter_f32_checked(self.h, _ptr(d_in), _ptr(d_out), count, fb,
                                                      _ptr(d_ill), stream))

    def filter_host(self, h_in: np.ndarray, h_out: np.ndarray | None = None, stream: int = 0):
        """Host fp32 frames -> host fp32 frames (copies inside). Returns (out, fallbacks)."""
        a = np.ascontiguousarray(h_in, dtype=np.float32)
        count = a.size // (self.width * self.height)
        if count * self.width * self.height != a.size:
            raise ValueError("input size is not a whole number of frames")
        out = h_out if h_out is not None else np.empty_like(a)
        if out.dtype != np.float32 or out.size != a.size or not out.flags.c_contiguous:
            raise ValueError("h_out must be a C-contiguous float32 array of the input's size")
        fb = (C.c_longlong * max(count, 1))()
        _check(_lib.lib().gpf_b200_filter_f32_host(self.h, a.ctypes.data, out.ctypes.data, count,
                                                   fb, stream))
        return out, list(fb)[:count]

    def close(self) -> None:
        if getattr(self, "h", None):
            _lib.lib().gpf_b200_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: module globals may already be gone
            pass
