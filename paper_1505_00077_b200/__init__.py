"""B200-native Gauss-polynomial O(1) bilateral filter (arXiv 1505.00077 GPF path).

The compute path is libgpfilter_b200.so (hand-written sm_100a kernels behind a
C ABI that mirrors the reference's gpf_filter_gpf). This package is the thin
host-side binding; it never computes the filter on the CPU.
"""
from . import gpf  # noqa: F401
from ._lib import LIB_PATH, build  # noqa: F401
from .gpf import (GpfError, Image, Plan, compare_device, exact_device, gpf_compare,  # noqa: F401
                  gpf_filter_exact, gpf_filter_gpf, gpf_filter_taylor, gpf_gaussian_recursive, get_num_threads,
                  gpf_gaussian_direct, kernel_gauss, kernel_gauss_poly, kernel_taylor, kernel_sup_error,
                  range_params, set_num_threads, spatial_params, set_precision, get_precision,
                  last_precision, last_max_abs_h, last_device_ms, fp32_h_limit, dropin_release,
                  filter_batch_device)

__all__ = ["GpfError", "Image", "Plan", "gpf_filter_gpf", "gpf_gaussian_recursive", "gpf_gaussian_direct",
           "kernel_gauss", "kernel_gauss_poly", "kernel_taylor", "kernel_sup_error",
           "gpf_filter_exact", "gpf_filter_taylor", "gpf_compare", "exact_device", "compare_device",
           "range_params", "spatial_params", "set_num_threads", "get_num_threads", "build",
           "LIB_PATH", "set_precision", "get_precision", "last_precision", "last_max_abs_h",
           "fp32_h_limit", "dropin_release", "last_device_ms", "filter_batch_device"]
