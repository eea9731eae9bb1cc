"""TEST INFRASTRUCTURE ONLY -- ctypes front-end for the CPU checkers.

* ``Oracle``  wraps ``oracle/liboracle.so`` (the plain-C fp64 restatement in
  ``gpf_oracle.c``, each function citing the reference file:line it follows).
* ``Reference`` wraps ``oracle/_ref/libgpfilter_ref.so``: the unmodified
  reference library compiled from ``/root/reference/proj`` by
  ``oracle/Makefile`` (C ABI of ``proj/include/gpfilter/gpfilter.h``).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module. The product path (``paper_1505_00077_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libgpfilter_ref.so")

_dp = C.POINTER(C.c_double)


def build() -> None:
    """Compile the checkers (the reference only when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _as_c(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """fp64 restatement of gpf() on the recursive backend."""

    def __init__(self, path: str = LIB_ORACLE):
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        lib.oracle_mean.restype = C.c_double
        lib.oracle_mean.argtypes = [_dp, C.c_longlong]
        lib.oracle_kernel_mass_1d.restype = C.c_double
        lib.oracle_kernel_mass_1d.argtypes = [C.c_double, C.c_int]
        lib.oracle_deriche_coeffs.argtypes = [C.c_double, _dp, _dp, _dp]
        lib.oracle_recursive_gaussian.restype = C.c_int
        lib.oracle_recursive_gaussian.argtypes = [_dp, C.c_int, C.c_int, C.c_double,
                                                  C.c_double, _dp, C.c_int]
        lib.oracle_gpf.restype = C.c_int
        lib.oracle_gpf.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                   C.c_int, C.c_int, C.c_double, C.c_double, _dp,
                                   C.POINTER(C.c_longlong), _dp, C.c_int]
        lib.oracle_exact_bilateral_at.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_int,
                                                  C.c_int, C.c_double, C.c_double,
                                                  C.POINTER(C.c_longlong), C.c_longlong, _dp]
        self.lib = lib

    def mean(self, img: np.ndarray) -> float:
        a = _as_c(img)
        return self.lib.oracle_mean(a.ctypes.data_as(_dp), a.size)

    def kernel_mass_1d(self, sigma: float, radius: int) -> float:
        return self.lib.oracle_kernel_mass_1d(sigma, radius)

    def deriche_coeffs(self, sigma: float):
        nc, na, d = (np.zeros(4) for _ in range(3))
        self.lib.oracle_deriche_coeffs(sigma, nc.ctypes.data_as(_dp), na.ctypes.data_as(_dp),
                                       d.ctypes.data_as(_dp))
        return nc, na, d

    def recursive_gaussian(self, img: np.ndarray, sigma_s: float, kernel_scale: float = 1.0,
                           threads: int = 1) -> np.ndarray:
        a = _as_c(img)
        out = np.empty_like(a)
        rc = self.lib.oracle_recursive_gaussian(a.ctypes.data_as(_dp), a.shape[1], a.shape[0],
                                                sigma_s, kernel_scale, out.ctypes.data_as(_dp),
                                                threads)
        if rc != 0:
            raise ValueError(f"oracle_recursive_gaussian rc={rc}")
        return out

    def gpf(self, img: np.ndarray, sigma_s: float, sigma_r: float, degree: int = 20,
            centering: int = 1, kernel_scale: float = 1.0, threads: int = 1,
            midpoint=(0.0, 255.0)):
        """Returns (out, fallback_count, t_c)."""
        a = _as_c(img)
        out = np.empty_like(a)
        fb = C.c_longlong(0)
        tc = C.c_double(0)
        rc = self.lib.oracle_gpf(a.ctypes.data_as(_dp), a.shape[1], a.shape[0], sigma_s,
                                 kernel_scale, sigma_r, degree, centering, midpoint[0],
                                 midpoint[1], out.ctypes.data_as(_dp), C.byref(fb),
                                 C.byref(tc), threads)
        if rc != 0:
            raise ValueError(f"oracle_gpf rc={rc}")
        return out, fb.value, tc.value

    def exact_bilateral_at(self, img: np.ndarray, sigma_s: float, sigma_r: float,
                           idx: np.ndarray, radius: int | None = None, boundary: int = 0,
                           kernel_scale: float = 1.0) -> np.ndarray:
        a = _as_c(img)
        if radius is None:
            radius = int(np.ceil(3.0 * sigma_s))
        ix = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty(ix.size)
        self.lib.oracle_exact_bilateral_at(a.ctypes.data_as(_dp), a.shape[1], a.shape[0],
                                           sigma_s, radius, boundary, kernel_scale, sigma_r,
                                           ix.ctypes.data_as(C.POINTER(C.c_longlong)), ix.size,
                                           out.ctypes.data_as(_dp))
        return out


class Reference:
    """The unmodified reference ``libgpfilter`` through its own C ABI."""

    GPF_BACKEND_DIRECT = 0
    GPF_BACKEND_RECURSIVE = 1

    class SpatialParams(C.Structure):
        _fields_ = [("sigma_s", C.c_double), ("window_radius", C.c_int),
                    ("boundary", C.c_int), ("kernel_scale", C.c_double)]

    class RangeParams(C.Structure):
        _fields_ = [("sigma_r", C.c_double), ("degree", C.c_int)]

    def __init__(self, path: str = LIB_REF):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = C.CDLL(path)
        vp = C.c_void_p
        lib.gpf_image_create.argtypes = [C.c_int, C.c_int, C.POINTER(vp)]
        lib.gpf_image_destroy.argtypes = [vp]
        lib.gpf_image_data.restype = _dp
        lib.gpf_image_data.argtypes = [vp]
        lib.gpf_image_cdata.restype = _dp
        lib.gpf_image_cdata.argtypes = [vp]
        lib.gpf_last_error.restype = C.c_char_p
        lib.gpf_filter_gpf.argtypes = [vp, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                       C.POINTER(C.c_longlong), C.POINTER(vp)]
        lib.gpf_filter_exact.argtypes = [vp, C.c_void_p, C.c_void_p, C.POINTER(vp)]
        lib.gpf_gaussian_recursive.argtypes = [vp, C.c_double, C.c_double, C.POINTER(vp)]
        lib.gpf_set_num_threads.argtypes = [C.c_int]
        self.lib = lib

    def _img(self, a: np.ndarray):
        h, w = a.shape
        p = C.c_void_p()
        assert self.lib.gpf_image_create(w, h, C.byref(p)) == 0
        buf = np.ctypeslib.as_array(self.lib.gpf_image_data(p), shape=(h * w,))
        buf[:] = np.asarray(a, dtype=np.float64).ravel()
        return p

    def _take(self, p, shape) -> np.ndarray:
        out = np.ctypeslib.as_array(self.lib.gpf_image_cdata(p), shape=(shape[0] * shape[1],))
        res = out.copy().reshape(shape)
        self.lib.gpf_image_destroy(p)
        return res

    def set_num_threads(self, n: int) -> None:
        self.lib.gpf_set_num_threads(n)

    def gpf(self, img: np.ndarray, sigma_s: float, sigma_r: float, degree: int = 20,
            centering: int = 1, kernel_scale: float = 1.0, backend: int = 1,
            window_radius: int = 0, boundary: int = 0):
        """Returns (status, out or None, fallback_count)."""
        sp = self.SpatialParams(sigma_s, window_radius, boundary, kernel_scale)
        rp = self.RangeParams(sigma_r, degree)
        src = self._img(img)
        out = C.c_void_p()
        fb = C.c_longlong(-1)
        st = self.lib.gpf_filter_gpf(src, C.byref(sp), C.byref(rp), backend, centering,
                                     C.byref(fb), C.byref(out))
        self.lib.gpf_image_destroy(src)
        if st != 0:
            return st, None, fb.value
        return st, self._take(out, img.shape), fb.value

    class ErrorReport(C.Structure):
        _fields_ = [("mse", C.c_double), ("mse_db", C.c_double), ("max_abs", C.c_double),
                    ("pixels", C.c_longlong)]

    def compare(self, ref: np.ndarray, test: np.ndarray, exclude_border: int = 0):
        """Reference gpf_compare (capi.cpp:288-301): (status, report dict or None)."""
        self.lib.gpf_compare.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(self.ErrorReport)]
        a, b = self._img(ref), self._img(test)
        rep = self.ErrorReport()
        st = self.lib.gpf_compare(a, b, exclude_border, C.byref(rep))
        self.lib.gpf_image_destroy(a)
        self.lib.gpf_image_destroy(b)
        if st != 0:
            return st, None
        return st, {"mse": rep.mse, "mse_db": rep.mse_db, "max_abs": rep.max_abs, "pixels": rep.pixels}

    def gaussian_direct(self, img: np.ndarray, sigma_s: float, window_radius: int = 0,
                        boundary: int = 0, kernel_scale: float = 1.0):
        """Reference gpf_gaussian_direct (capi.cpp:209-217): (status, out or None)."""
        self.lib.gpf_gaussian_direct.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        sp = self.SpatialParams(sigma_s, window_radius, boundary, kernel_scale)
        src = self._img(img)
        out = C.c_void_p()
        st = self.lib.gpf_gaussian_direct(src, C.byref(sp), C.byref(out))
        self.lib.gpf_image_destroy(src)
        if st != 0:
            return st, None
        return st, self._take(out, img.shape)

    def kernel(self, name: str, *args):
        """Reference gpf_kernel_<name> (capi.cpp:230-286) with the C argument order:
        (status, value)."""
        fn = getattr(self.lib, "gpf_kernel_" + name)
        sig = {"gauss": [C.c_double] * 3, "gauss_poly": [C.c_double] * 3 + [C.c_int],
               "taylor": [C.c_double] * 3 + [C.c_int],
               "sup_error": [C.c_double, C.c_int] + [C.c_double] * 4 + [C.c_int]}[name]
        fn.argtypes = sig + [C.POINTER(C.c_double)]
        v = C.c_double(float("nan"))
        st = fn(*args, C.byref(v))
        return st, v.value

    def taylor(self, img: np.ndarray, sigma_s: float, sigma_r: float, degree: int = 20,
               backend: int = 1):
        """Reference gpf_filter_taylor (capi.cpp:194-207): (status, out or None, fallbacks)."""
        self.lib.gpf_filter_taylor.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                               C.POINTER(C.c_longlong), C.POINTER(C.c_void_p)]
        sp = self.SpatialParams(sigma_s, 0, 0, 1.0)
        rp = self.RangeParams(sigma_r, degree)
        src = self._img(img)
        out = C.c_void_p()
        fb = C.c_longlong(-1)
        st = self.lib.gpf_filter_taylor(src, C.byref(sp), C.byref(rp), backend, C.byref(fb),
                                        C.byref(out))
        self.lib.gpf_image_destroy(src)
        if st != 0:
            return st, None, fb.value
        return st, self._take(out, img.shape), fb.value

    def exact(self, img: np.ndarray, sigma_s: float, sigma_r: float, boundary: int = 0) -> np.ndarray:
        sp = self.SpatialParams(sigma_s, 0, boundary, 1.0)
        rp = self.RangeParams(sigma_r, 20)
        src = self._img(img)
        out = C.c_void_p()
        st = self.lib.gpf_filter_exact(src, C.byref(sp), C.byref(rp), C.byref(out))
        self.lib.gpf_image_destroy(src)
        assert st == 0
        return self._take(out, img.shape)

    def decode_pgm(self, data: bytes):
        """Reference gpf_decode_pgm: (status, array or None, last_error)."""
        self.lib.gpf_decode_pgm.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]
        self.lib.gpf_image_width.argtypes = [C.c_void_p]
        self.lib.gpf_image_height.argtypes = [C.c_void_p]
        buf = C.create_string_buffer(data, len(data))
        out = C.c_void_p()
        st = self.lib.gpf_decode_pgm(buf, len(data), C.byref(out))
        if st != 0:
            return st, None, self.last_error()
        w, h = self.lib.gpf_image_width(out), self.lib.gpf_image_height(out)
        return st, self._take(out, (h, w)), ""

    def encode_pgm(self, img: np.ndarray) -> bytes:
        self.lib.gpf_encode_pgm.argtypes = [C.c_void_p, C.POINTER(C.POINTER(C.c_uint8)),
                                            C.POINTER(C.c_size_t)]
        self.lib.gpf_free_bytes.argtypes = [C.POINTER(C.c_uint8)]
        src = self._img(img)
        p = C.POINTER(C.c_uint8)()
        n = C.c_size_t()
        assert self.lib.gpf_encode_pgm(src, C.byref(p), C.byref(n)) == 0
        out = bytes(p[:n.value])
        self.lib.gpf_free_bytes(p)
        self.lib.gpf_image_destroy(src)
        return out

    def last_error(self) -> str:
        return self.lib.gpf_last_error().decode()
