import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1609_06119_b200 import FitConfig, fit_forest, predict_batch
rng = np.random.default_rng(0)
Xs = rng.normal(size=(200_000, 40)).astype(np.float32); y = (Xs[:, 0] + Xs[:, 3] > 0).astype(int)
forest = fit_forest(Xs, y, None, FitConfig(n_trees=1000, depth=3, binning_levels=8, seed=0))
X = rng.normal(size=(10_000_000, 40)).astype(np.float32)
for r in range(4):
    t0 = time.perf_counter(); p = predict_batch(forest, X); dt = time.perf_counter() - t0
    print(f"apply e2e {X.shape[0]/dt/1e6:.1f} M rows/s ({dt*1e3:.1f} ms)")
