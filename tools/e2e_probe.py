import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1609_06119_b200 import FitConfig, fit_forest
from paper_1609_06119_b200.datagen import CONFIGS, make_config
spec = dict(CONFIGS["cfg3"]); X, y, w, _ = make_config("cfg3")
cfg = FitConfig(n_trees=spec["trees"], depth=spec["depth"], shrinkage=spec.get("shrinkage", 0.1), subsample=spec.get("subsample", 0.5), binning_levels=spec["binning_levels"], seed=0)
for r in range(4):
    t0 = time.perf_counter(); f = fit_forest(X, y, w, cfg); dt = time.perf_counter() - t0
    tm = f.fit_info["timing_ms"]
    print(f"wall {dt*1e3:.1f} ms; lib total {tm['total']:.1f} device {tm['device_total']:.1f} upload {tm['upload']:.1f} binning {tm['binning']:.1f} trees {tm['trees']:.1f} download {tm['download']:.1f}")
