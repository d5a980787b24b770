"""Pin the oracle (oracle/binboost_np.py, float64 mode) to the golden vectors
the unmodified reference produced (tests/golden/gen_golden.py).  CPU only."""

from __future__ import annotations

import hashlib
import json
import math

import numpy as np
import pytest

import oracle
from paper_1609_06119_b200.datagen import make_config


def sha(a) -> str:
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


def _assert_forest(orc, g, T=None):
    T = int(g["n_trees"]) if T is None else T
    for name in ("feature", "cut_bin", "threshold", "gain", "valid", "node_weight", "node_purity"):
        np.testing.assert_array_equal(getattr(orc, name)[:T], g[name][:T], err_msg=name)
    assert orc.leaf_hashes[:T] == list(g["leaf_hashes"][:T])
    assert orc.mask_hashes[:T] == list(g["mask_hashes"][:T])


def test_kats(golden_dir):
    k = json.load(open(f"{golden_dir}/kats.json"))
    assert oracle.fit_boundaries(np.arange(1.0, 9.0), 2).tolist() == k["bounds_1to8_L2"]
    assert oracle.fit_boundaries(np.array([5.0, 5, 5, 5]), 1).tolist() == k["bounds_5555_L1"]
    assert oracle.fit_boundaries(np.array([1.0, 2, np.nan, np.inf, 3, 4]), 1).tolist() == k["bounds_mixed_L1"]
    probe = np.array([np.nan if v is None else v for v in k["to_bin_probe"]])
    assert oracle.bin_codes(oracle.fit_boundaries(np.arange(1.0, 9.0), 2), probe).tolist() == k["to_bin_codes"]
    from oracle.binboost_np import _g_arr
    for sl, bl, sr, br, g in k["gain_kats"]:
        a = lambda s, b: _g_arr(np.array([s]), np.array([b]))[0]  # noqa: E731
        assert a(sl, bl) + a(sr, br) - a(sl + sr, bl + br) == g


def test_binning_golden(golden_dir):
    g = np.load(f"{golden_dir}/binning_random.npz")
    vals = np.split(g["values"], np.cumsum(g["lengths"])[:-1])
    bnds = np.split(g["boundaries"], np.cumsum(g["bound_lengths"])[:-1])
    codes = np.split(g["codes"], np.cumsum(g["lengths"])[:-1])
    for col, L, b_ref, c_ref in zip(vals, g["levels"], bnds, codes):
        b = oracle.fit_boundaries(col, int(L))
        np.testing.assert_array_equal(b, b_ref)
        np.testing.assert_array_equal(oracle.bin_codes(b, col), c_ref)


def test_small_fits_golden(golden_dir):
    z = np.load(f"{golden_dir}/small_fits.npz")
    for i in range(len({k.split("__")[0] for k in z.files})):
        g = {k.split("__", 1)[1]: z[k] for k in z.files if k.startswith(f"c{i}__")}
        T, D, eta, alpha, L, seed = g["config"]
        orc = oracle.fit_forest(g["X"], g["y"], g.get("w"), n_trees=int(T), depth=int(D), shrinkage=float(eta),
                                subsample=float(alpha), levels=int(L), seed=int(seed))
        assert orc.f0 == float(g["f0"])
        np.testing.assert_array_equal(orc.boundaries, g["boundaries"])
        _assert_forest(orc, g)
        np.testing.assert_array_equal(oracle.predict(orc, g["X"][g["pred_rows"]]), g["pred"])


def test_cfg1_golden(golden_dir):
    g = np.load(f"{golden_dir}/cfg1_fit.npz")
    X, y, w, kw = make_config("cfg1")
    orc = oracle.fit_forest(X, y, w, n_trees=kw["trees"], depth=kw["depth"], shrinkage=kw["shrinkage"],
                            subsample=kw["subsample"], levels=kw["binning_levels"], seed=kw["seed"])
    np.testing.assert_array_equal(orc.boundaries, g["boundaries"])
    _assert_forest(orc, g)
    np.testing.assert_array_equal(oracle.predict(orc, X[g["pred_rows"]]), g["pred"])


def test_cfg2_slice_golden_prefix(golden_dir):
    g = np.load(f"{golden_dir}/cfg2_slice_fit.npz")
    X, y, w, _ = make_config("cfg2", n=200_000)
    T = 8  # trees are a deterministic prefix (reference tests/test_boosting.py:161-169)
    orc = oracle.fit_forest(X, y, w, n_trees=T, depth=3, shrinkage=0.1, subsample=0.5, levels=8, seed=0)
    np.testing.assert_array_equal(orc.boundaries, g["boundaries"])
    _assert_forest(orc, g, T)


def test_apply_golden(golden_dir):
    g = np.load(f"{golden_dir}/apply_cfg4_slice.npz")
    X, _, _, _ = make_config("cfg4", n=20_000)
    T = g["feature"].shape[0]
    orc = oracle.OracleForest(f0=0.0, levels=8, depth=3, shrinkage=1.0, boundaries=g["boundaries"],
                              feature=g["feature"], cut_bin=g["cut_bin"], threshold=g["threshold"],
                              gain=np.zeros((T, 7)), valid=np.ones((T, 7), bool), node_weight=g["node_weight"],
                              node_purity=np.zeros((T, 15)))
    np.testing.assert_array_equal(oracle.predict(orc, X), g["pred"])


def test_fixed_point_matches_float_cuts_on_cfg1_slice():
    """The GPU's fixed-point arithmetic (predicted exactly by the oracle's
    fixed-point mode) chooses the reference's cuts wherever the argmax is not
    a near-tie."""
    X, y, w, _ = make_config("cfg1", n=30_000)
    a = oracle.fit_forest(X, y, w, n_trees=15, depth=3, shrinkage=0.1, subsample=0.5, levels=8, seed=0)
    b = oracle.fit_forest(X, y, w, n_trees=15, depth=3, shrinkage=0.1, subsample=0.5, levels=8, seed=0,
                          fixed_point=True)
    assert a.leaf_hashes == b.leaf_hashes
    np.testing.assert_array_equal(a.feature, b.feature)
    np.testing.assert_array_equal(a.cut_bin, b.cut_bin)
    assert np.max(np.abs(oracle.predict(a, X[:2000]) - oracle.predict(b, X[:2000]))) < 1e-9


@pytest.mark.parametrize("w,S", [(1.0, 32), (1.5, 31), (0.5, 33), (2.0, 31), (17.3, 27), (0.0, 32)])
def test_fixed_point_shift(w, S):
    from oracle.binboost_np import fixed_point_shift
    assert fixed_point_shift(w) == S
    if w > 0:
        assert w * 2.0 ** S <= 2.0 ** 32
