"""Time the GPU subsample-mask generation (bb_subsample_masks_gpu) for T trees."""
import argparse, ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1609_06119_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--a", type=int, default=300_000)
ap.add_argument("--b", type=int, default=700_000)
ap.add_argument("--trees", type=int, default=32)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = _lib.FitConfigC(**_lib.pcg_config(0))
words = (a.a + a.b + 31) // 32
bits = np.zeros(words * a.trees, np.uint32)
for r in range(a.reps):
    t0 = time.perf_counter()
    _lib.check(_lib.lib().bb_subsample_masks_gpu(_lib.context(), a.a, a.b, 0.5, a.trees, C.byref(cfg), _lib.ptr(bits)))
    dt = time.perf_counter() - t0
    print(f"masks: {a.trees} trees {dt*1e3:.1f} ms = {dt*1e3/a.trees:.3f} ms/tree")
