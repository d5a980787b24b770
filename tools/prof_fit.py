"""Small fit driver for profiling (ncu) and quick timing: a few trees of a config."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1609_06119_b200 import FitConfig, fit_forest
from paper_1609_06119_b200.datagen import CONFIGS, make_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--trees", type=int, default=4)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--host-masks", action="store_true")
a = ap.parse_args()
spec = dict(CONFIGS[a.config])
X, y, w, _ = make_config(a.config, n=a.n)
cfg = FitConfig(n_trees=a.trees, depth=spec["depth"], shrinkage=spec.get("shrinkage", 0.1),
                subsample=spec.get("subsample", 0.5), binning_levels=spec["binning_levels"], seed=0)
for r in range(a.reps):
    f = fit_forest(X, y, w, cfg, profile=True, host_masks=a.host_masks)
    ti = f.fit_info
    print({k: round(v, 3) for k, v in ti["timing_ms"].items()}, "hist launches", ti["hist_launches"],
          "avg hist ms", round(ti["timing_ms"]["hist_kernels"] / max(1, ti["hist_launches"]), 4))
