"""Write a GPU-fitted model file for the cross-implementation fixture
(tests/golden/gpu_model.json): run on a B200, then copy the outputs from
gpurun_out/ into tests/golden/.  test_api_cpu.py loads the document with the
reference's model_io and checks its predictions."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1609_06119_b200 import bridge

rng = np.random.default_rng(21)
X = rng.normal(size=(4000, 5))
X[rng.random(X.shape) < 0.04] = np.nan
X[:, 3] = np.round(X[:, 3] * 2)
y = (np.nan_to_num(X[:, 0]) - 0.7 * np.nan_to_num(X[:, 2]) + 0.4 * rng.normal(size=4000) > 0).astype(int)
w = rng.uniform(0.5, 2.0, 4000)
trees, depth, seed = 12, 4, 5
m = bridge.fit(X, y, w, trees=trees, depth=depth, seed=seed)
os.makedirs("gpurun_out", exist_ok=True)
m.save("gpurun_out/gpu_model.json")
np.savez_compressed("gpurun_out/gpu_model_inputs.npz", X=X, y=y, w=w, trees=trees, depth=depth, seed=seed,
                    pred=m.predict(X))
print("written")
