"""Device time of full fits (cfg2 by default) under the current env: median
of --reps fits after one warm-up; --host-masks precomputes the masks."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1609_06119_b200 import FitConfig, fit_forest
from paper_1609_06119_b200.datagen import CONFIGS, make_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--trees", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--host-masks", action="store_true")
ap.add_argument("--tag", default="")
a = ap.parse_args()
spec = dict(CONFIGS[a.config])
X, y, w, _ = make_config(a.config)
T = a.trees or spec["trees"]
cfg = FitConfig(n_trees=T, depth=spec["depth"], shrinkage=spec.get("shrinkage", 0.1),
                subsample=spec.get("subsample", 0.5), binning_levels=spec["binning_levels"], seed=0)
ts = []
for r in range(a.reps + 1):
    f = fit_forest(X, y, w, cfg, host_masks=a.host_masks)
    ts.append(f.fit_info["timing_ms"]["device_total"])
ts = ts[1:]
print(f"{a.tag} {a.config} T={T} host_masks={a.host_masks} device ms: median {np.median(ts):.2f} all {[round(t, 2) for t in ts]}")
