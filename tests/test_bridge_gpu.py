"""The array-in/array-out binding (paper_1609_06119_b200.bridge) on the GPU,
case by case against the contract of binboost_bridge
(/root/reference/pkg/bridge/src/binboost_bridge/__init__.py:25-176): fit,
predict, save/load, close semantics, importance dispatch and concurrency.
The validation messages that need no GPU are in test_api_cpu.py."""

from __future__ import annotations

import os
import threading

import numpy as np
import pytest

from paper_1609_06119_b200 import FitConfig, bridge, fit_forest, predict_batch
from paper_1609_06119_b200.analysis import gain_importance, individual_importance, roc_auc

pytestmark = pytest.mark.gpu


def _xor(n=4000, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.uniform(-1, 1, (n, 2))
    y = ((X[:, 0] > 0) ^ (X[:, 1] > 0)).astype(int)
    return X, y


@pytest.fixture(scope="module")
def small_model():
    rng = np.random.default_rng(3)
    X = rng.normal(size=(3000, 4))
    y = (X[:, 0] + 0.5 * X[:, 1] + 0.3 * rng.normal(size=3000) > 0).astype(int)
    return bridge.fit(X, y, trees=15, depth=3, seed=1), X, y


def test_xor_reaches_high_training_auc():
    X, y = _xor()
    m = bridge.fit(X, y, trees=60, depth=2, shrinkage=0.3, seed=2)
    assert roc_auc(m.predict(X), y) > 0.95


def test_defaults_and_hyperparameters_echoed():
    X, y = _xor(800)
    m = bridge.fit(X, y)
    assert m.config == FitConfig()
    m2 = bridge.fit(X, y, trees=7, depth=2, shrinkage=0.5, subsample=0.8, binning_levels=5, seed=9)
    assert m2.config == FitConfig(n_trees=7, depth=2, shrinkage=0.5, subsample=0.8, binning_levels=5, seed=9)
    assert m2.n_features == 2 and len(m2.forest.trees) == 7


@pytest.mark.parametrize("kw", [dict(trees=0), dict(depth=0), dict(shrinkage=0.0), dict(shrinkage=1.5),
                                dict(subsample=0.0), dict(binning_levels=0)])
def test_invalid_hyperparameters_rejected(kw):
    X, y = _xor(200)
    with pytest.raises(ValueError):
        bridge.fit(X, y, **kw)


def test_weights_pass_through_to_engine():
    X, y = _xor(2000)
    w = np.random.default_rng(1).uniform(0.2, 3.0, y.size)
    m = bridge.fit(X, y, w, trees=5, seed=4)
    e = fit_forest(X, y, w, FitConfig(n_trees=5, seed=4))
    np.testing.assert_array_equal(m.predict(X), predict_batch(e, X))


def test_predict_matches_engine_and_edge_shapes(small_model):
    m, X, _ = small_model
    np.testing.assert_array_equal(m.predict(X), predict_batch(m.forest, X))
    assert m.predict(np.empty((0, 4))).shape == (0,)
    assert m.predict(np.empty(0)).shape == (0,)
    with pytest.raises(ValueError, match="expects 4 features"):
        m.predict(np.zeros((3, 5)))
    with pytest.raises(ValueError, match="2-d"):
        m.predict(np.zeros(4))
    Xn = X[:50].copy()
    Xn[::3, 1] = np.nan
    p = m.predict(Xn)
    assert np.all(np.isfinite(p)) and np.all((p > 0) & (p < 1))


def test_save_load_roundtrip_and_errors(small_model, tmp_path):
    m, X, _ = small_model
    path = str(tmp_path / "m.json")
    m.save(path)
    m2 = bridge.load(path)
    np.testing.assert_array_equal(m2.predict(X), m.predict(X))
    path2 = str(tmp_path / "m2.json")
    m2.save(path2)
    assert open(path).read() == open(path2).read()
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    with pytest.raises(ValueError):
        bridge.load(str(bad))
    with pytest.raises((FileNotFoundError, OSError)):
        bridge.load(str(tmp_path / "missing.json"))


def test_close_semantics(small_model, tmp_path):
    X, y = _xor(500)
    m = bridge.fit(X, y, trees=3)
    m.close()
    m.close()  # idempotent
    for call in (lambda: m.predict(X), lambda: m.save(str(tmp_path / "x.json")), lambda: m.config,
                 lambda: m.importance("gain")):
        with pytest.raises(RuntimeError, match="model handle is closed"):
            call()
    with bridge.fit(X, y, trees=3) as m3:
        m3.predict(X[:5])
    with pytest.raises(RuntimeError, match="model handle is closed"):
        m3.predict(X[:5])


def test_importance_dispatch(small_model):
    m, X, y = small_model
    np.testing.assert_array_equal(m.importance("gain"), gain_importance(m.forest).scores)
    np.testing.assert_array_equal(m.importance("individual", row=X[0]), individual_importance(m.forest, X[0]).scores)
    with pytest.raises(ValueError, match="no extra arguments"):
        m.importance("gain", row=X[0])
    with pytest.raises(ValueError, match="requires row="):
        m.importance("individual")
    with pytest.raises(ValueError, match="requires X= and y="):
        m.importance("elimination")
    with pytest.raises(ValueError, match="unknown importance method"):
        m.importance("shap")
    el = m.importance("elimination", X=X[:1500], y=y[:1500])
    assert el.shape == (4,) and np.all(np.isfinite(el))


def test_concurrent_predictions_match_serial(small_model):
    m, X, _ = small_model
    want = m.predict(X)
    out = [None] * 8

    def work(k):
        out[k] = m.predict(X)

    th = [threading.Thread(target=work, args=(k,)) for k in range(8)]
    [t.start() for t in th]
    [t.join() for t in th]
    for o in out:
        np.testing.assert_array_equal(o, want)


def test_gpu_written_model_fixture_is_current(golden_dir, tmp_path):
    """tests/golden/gpu_model.json was written by this binding on a B200
    (tools/gen_gpu_model.py); refitting the same inputs reproduces it byte
    for byte, and its stored predictions.  test_api_cpu.py loads the same
    document with the reference's model_io and predicts the same values."""
    z = np.load(os.path.join(golden_dir, "gpu_model_inputs.npz"))
    m = bridge.fit(z["X"], z["y"], z["w"], trees=int(z["trees"]), depth=int(z["depth"]), seed=int(z["seed"]))
    path = str(tmp_path / "g.json")
    m.save(path)
    assert open(path).read() == open(os.path.join(golden_dir, "gpu_model.json")).read()
    np.testing.assert_array_equal(m.predict(z["X"]), z["pred"])
