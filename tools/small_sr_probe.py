"""Probe: GPU vs oracle at small sigma_r (outside the BASELINE configs), with
the oracle's per-pixel cancellation factor kappa (oracle_gpf_kappa)."""
import ctypes as C
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from oracle.oracle import Oracle
from paper_1505_00077_b200 import gpf, synth

o = Oracle()
dp = C.POINTER(C.c_double)
o.lib.oracle_gpf_kappa.argtypes = [dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                   dp, dp, C.c_int]
for sr in (1.0, 3.0, 8.0):
    for ss in (2.0, 6.0):
        img = np.ascontiguousarray(synth.rects_image(96, 64, 8, 10.0, 77).astype(np.float64))
        ref, rfb, _ = o.gpf(img, ss, sr, 20)
        out, fb = gpf.gpf_filter_gpf(img, gpf.spatial_params(ss), gpf.range_params(sr, 20))
        kap = np.zeros_like(img); r2 = np.zeros_like(img)
        o.lib.oracle_gpf_kappa(img.ctypes.data_as(dp), 96, 64, ss, 1.0, sr, 20, r2.ctypes.data_as(dp),
                               kap.ctypes.data_as(dp), 1)
        d = np.abs(out - ref)
        i = np.unravel_index(d.argmax(), d.shape)
        print(f"sr {sr} ss {ss}: fb {fb}/{rfb}; max {d.max():.3e} at {i} (ref {ref[i]:.2f}, kappa {kap[i]:.3g}); "
              f"max over kappa<=10: {d[kap <= 10].max():.3e}; max kappa {kap.max():.3g}")
