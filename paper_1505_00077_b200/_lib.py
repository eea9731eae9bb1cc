"""ctypes binding of libgpfilter_b200.so (the in-tree C-ABI library).

There is no Python or CPU compute path behind these bindings: if the shared
library is missing or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# GPF_B200_LIB: an alternative build of the same library (A/B timing); there is no fallback
LIB_PATH = os.environ.get("GPF_B200_LIB") or os.path.join(PKG_DIR, "libgpfilter_b200.so")

# gpf_status values (include/gpfilter/gpfilter.h)
GPF_OK = 0
GPF_ERR_INVALID_ARGUMENT = 1
GPF_ERR_IO = 2
GPF_ERR_SIGMA_TOO_SMALL = 3
GPF_ERR_PGM_BAD_MAGIC, GPF_ERR_PGM_BAD_DIMS, GPF_ERR_PGM_BAD_MAXVAL = 4, 5, 6
GPF_ERR_PGM_TRUNCATED, GPF_ERR_PGM_BAD_PIXEL = 7, 8
GPF_ERR_UNKNOWN = 9

GPF_BOUNDARY_REPLICATE, GPF_BOUNDARY_REFLECT, GPF_BOUNDARY_ZERO = 0, 1, 2
GPF_BACKEND_DIRECT, GPF_BACKEND_RECURSIVE = 0, 1

# Every symbol include/gpfilter/*.h declares.
EXPORTED = (
    "gpf_status_name", "gpf_last_error", "gpf_version",
    "gpf_image_create", "gpf_image_destroy", "gpf_image_width", "gpf_image_height",
    "gpf_image_data", "gpf_image_cdata",
    "gpf_spatial_params_init", "gpf_range_params_init",
    "gpf_filter_gpf", "gpf_gaussian_recursive", "gpf_gaussian_direct", "gpf_filter_exact", "gpf_compare",
    "gpf_kernel_gauss", "gpf_kernel_gauss_poly", "gpf_kernel_taylor", "gpf_kernel_sup_error",
    "gpf_filter_taylor", "gpf_read_pgm", "gpf_decode_pgm", "gpf_write_pgm", "gpf_encode_pgm",
    "gpf_free_bytes",
    "gpf_set_num_threads", "gpf_get_num_threads",
    "gpf_b200_plan_create", "gpf_b200_plan_destroy", "gpf_b200_plan_set_batch",
    "gpf_b200_plan_set_profiling", "gpf_b200_plan_stage_times", "gpf_b200_plan_stage_marks", "gpf_b200_plan_workspace_bytes",
    "gpf_b200_plan_launches_per_frame", "gpf_b200_filter_f32", "gpf_b200_filter_f32_ev",
    "gpf_b200_filter_f32_host", "gpf_b200_exact_f32", "gpf_b200_compare_f32",
    "gpf_b200_set_precision", "gpf_b200_get_precision", "gpf_b200_last_precision",
    "gpf_b200_last_max_abs_h", "gpf_b200_fp32_h_limit", "gpf_b200_fp32_h_limit_degree", "gpf_b200_dropin_release", "gpf_b200_exp_cr",
    "gpf_b200_last_device_ms", "gpf_b200_filter_f32_checked", "gpf_b200_filter_batch",
)

# gpf_b200_precision (include/gpfilter/gpfilter_b200.h)
PRECISION_AUTO, PRECISION_FP32, PRECISION_FP64 = 0, 1, 2


class SpatialParams(C.Structure):
    """gpf_spatial_params (reference gpfilter.h:75-80)."""
    _fields_ = [("sigma_s", C.c_double), ("window_radius", C.c_int),
                ("boundary", C.c_int), ("kernel_scale", C.c_double)]


class ErrorReport(C.Structure):
    """gpf_error_report (reference gpfilter.h:149-154)."""
    _fields_ = [("mse", C.c_double), ("mse_db", C.c_double), ("max_abs", C.c_double),
                ("pixels", C.c_longlong)]


class RangeParams(C.Structure):
    """gpf_range_params (reference gpfilter.h:82-85)."""
    _fields_ = [("sigma_r", C.c_double), ("degree", C.c_int)]


def build() -> None:
    """Compile libgpfilter_b200.so for sm_100a (nvcc cross-compiles; no GPU needed)."""
    subprocess.run(["make", "-s", "-j8", "-C", PKG_DIR], check=True)


def _declare(lib: C.CDLL) -> C.CDLL:
    vp, dp = C.c_void_p, C.POINTER(C.c_double)
    pvp = C.POINTER(vp)
    lib.gpf_status_name.restype = C.c_char_p
    lib.gpf_status_name.argtypes = [C.c_int]
    lib.gpf_last_error.restype = C.c_char_p
    lib.gpf_version.restype = C.c_char_p
    lib.gpf_image_create.argtypes = [C.c_int, C.c_int, pvp]
    lib.gpf_image_destroy.argtypes = [vp]
    lib.gpf_image_width.argtypes = [vp]
    lib.gpf_image_height.argtypes = [vp]
    lib.gpf_image_data.restype = dp
    lib.gpf_image_data.argtypes = [vp]
    lib.gpf_image_cdata.restype = dp
    lib.gpf_image_cdata.argtypes = [vp]
    lib.gpf_spatial_params_init.argtypes = [C.POINTER(SpatialParams)]
    lib.gpf_range_params_init.argtypes = [C.POINTER(RangeParams)]
    lib.gpf_filter_gpf.argtypes = [vp, C.POINTER(SpatialParams), C.POINTER(RangeParams), C.c_int,
                                   C.c_int, C.POINTER(C.c_longlong), pvp]
    lib.gpf_gaussian_recursive.argtypes = [vp, C.c_double, C.c_double, pvp]
    lib.gpf_b200_exp_cr.argtypes = [C.c_void_p, C.c_void_p, C.c_longlong]
    lib.gpf_gaussian_direct.argtypes = [vp, C.POINTER(SpatialParams), pvp]
    pd = C.POINTER(C.c_double)
    lib.gpf_kernel_gauss.argtypes = [C.c_double, C.c_double, C.c_double, pd]
    lib.gpf_kernel_gauss_poly.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, pd]
    lib.gpf_kernel_taylor.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, pd]
    lib.gpf_kernel_sup_error.argtypes = [C.c_double, C.c_int, C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.c_int, pd]
    lib.gpf_filter_exact.argtypes = [vp, C.POINTER(SpatialParams), C.POINTER(RangeParams), pvp]
    lib.gpf_read_pgm.argtypes = [C.c_char_p, pvp]
    lib.gpf_decode_pgm.argtypes = [C.c_void_p, C.c_size_t, pvp]
    lib.gpf_write_pgm.argtypes = [vp, C.c_char_p]
    lib.gpf_encode_pgm.argtypes = [vp, C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(C.c_size_t)]
    lib.gpf_free_bytes.argtypes = [C.POINTER(C.c_uint8)]
    lib.gpf_filter_taylor.argtypes = [vp, C.POINTER(SpatialParams), C.POINTER(RangeParams), C.c_int,
                                      C.POINTER(C.c_longlong), pvp]
    lib.gpf_compare.argtypes = [vp, vp, C.c_int, C.POINTER(ErrorReport)]
    lib.gpf_b200_exact_f32.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, C.POINTER(SpatialParams),
                                       C.POINTER(RangeParams), vp]
    lib.gpf_b200_compare_f32.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, C.POINTER(ErrorReport), vp]
    lib.gpf_set_num_threads.argtypes = [C.c_int]
    lib.gpf_b200_plan_create.argtypes = [C.c_int, C.c_int, C.POINTER(SpatialParams),
                                         C.POINTER(RangeParams), C.c_int, C.c_int, pvp]
    lib.gpf_b200_plan_destroy.argtypes = [vp]
    lib.gpf_b200_plan_set_batch.argtypes = [vp, C.c_int]
    lib.gpf_b200_plan_set_profiling.argtypes = [vp, C.c_int]
    lib.gpf_b200_plan_stage_times.argtypes = [vp, C.POINTER(C.c_float), C.c_int]
    lib.gpf_b200_plan_stage_marks.argtypes = [vp, vp, C.POINTER(C.c_float), C.POINTER(C.c_int), C.c_int]
    lib.gpf_b200_plan_workspace_bytes.restype = C.c_size_t
    lib.gpf_b200_plan_workspace_bytes.argtypes = [vp]
    lib.gpf_b200_plan_launches_per_frame.argtypes = [vp]
    lib.gpf_b200_filter_f32.argtypes = [vp, vp, vp, C.c_int, vp, vp]
    lib.gpf_b200_filter_f32_ev.argtypes = [vp, vp, vp, C.c_int, vp, vp, vp]
    lib.gpf_b200_filter_f32_host.argtypes = [vp, vp, vp, C.c_int, C.POINTER(C.c_longlong), vp]
    lib.gpf_b200_set_precision.argtypes = [C.c_int]
    lib.gpf_b200_last_max_abs_h.restype = C.c_double
    lib.gpf_b200_fp32_h_limit.restype = C.c_double
    lib.gpf_b200_fp32_h_limit_degree.restype = C.c_double
    lib.gpf_b200_fp32_h_limit_degree.argtypes = [C.c_int]
    lib.gpf_b200_last_device_ms.restype = C.c_float
    lib.gpf_b200_filter_f32_checked.argtypes = [vp, vp, vp, C.c_int, vp, vp, vp]
    lib.gpf_b200_filter_batch.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, C.POINTER(SpatialParams),
                                          C.POINTER(RangeParams), C.c_int, vp, vp]
    return lib


_LIB: C.CDLL | None = None


def lib() -> C.CDLL:
    """The loaded library. Raises (never falls back) if it is absent."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() or "
                f"`make -C {PKG_DIR}` (there is no CPU fallback)")
        _LIB = _declare(C.CDLL(LIB_PATH))
    return _LIB
