"""Times the unmodified reference (oracle/_ref) on the host: full 8192^2 C3
frame at nproc threads, and a 2048^2 sample at 1 thread; prints the CPU model."""
import os, sys, time, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Reference
from paper_1505_00077_b200 import synth
model = next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")), "?")
ref = Reference()
res = {"cpu_model": model, "nproc": os.cpu_count()}
cfg = synth.CONFIGS[3]
img = synth.make(cfg).astype(np.float64)
for thr in (os.cpu_count(),):
    ref.set_num_threads(thr)
    t0 = time.time(); ref.gpf(img, 2.0, 30.0, 20); res[f"c3_8192_t{thr}_s"] = time.time() - t0
small = img[:2048, :2048].copy()
for thr in (1, os.cpu_count()):
    ref.set_num_threads(thr)
    t0 = time.time(); ref.gpf(small, 2.0, 30.0, 20); res[f"c3_2048_t{thr}_s"] = time.time() - t0
print(json.dumps(res))
