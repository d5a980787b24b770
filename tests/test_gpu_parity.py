"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
golden vectors the unmodified reference produced (tests/golden/gen_golden.py).

Bars: boundaries, codes, cut feature/bin/validity,
thresholds and per-row leaf ids bit-exact; probabilities within 1e-5
absolute; integer histograms exact vs the fixed-point oracle.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import json
import math
import threading

import numpy as np
import pytest

import oracle
from oracle.binboost_np import _gains_fixed, _pick_cuts
from paper_1609_06119_b200 import FitConfig, _lib, bridge, fit_forest, predict_batch
from paper_1609_06119_b200.datagen import make_config

pytestmark = pytest.mark.gpu

PROB_TOL = 1e-5


def sha(a) -> str:
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


def gpu_bin(X, levels):
    X = np.ascontiguousarray(X)
    dt = _lib.BB_F32 if X.dtype == np.float32 else _lib.BB_F64
    n, d = X.shape
    bounds = np.zeros((d, (1 << levels) - 1))
    codes = np.zeros((d, n), np.int16)
    _lib.check(_lib.lib().bb_bin(_lib.context(), _lib.ptr(X), dt, n, d, levels, _lib.ptr(bounds), _lib.ptr(codes)))
    return bounds, codes


# ------------------------------------------------------------------ binning
def test_binning_golden_columns(golden_dir):
    g = np.load(f"{golden_dir}/binning_random.npz")
    vals = np.split(g["values"], np.cumsum(g["lengths"])[:-1])
    bnds = np.split(g["boundaries"], np.cumsum(g["bound_lengths"])[:-1])
    codes = np.split(g["codes"], np.cumsum(g["lengths"])[:-1])
    for col, L, b_ref, c_ref in zip(vals, g["levels"], bnds, codes):
        b, c = gpu_bin(col.reshape(-1, 1), int(L))
        np.testing.assert_array_equal(b[0], b_ref)
        np.testing.assert_array_equal(c[0], c_ref)


def test_binning_kats(golden_dir):
    k = json.load(open(f"{golden_dir}/kats.json"))
    b, _ = gpu_bin(np.arange(1.0, 9.0).reshape(-1, 1), 2)
    assert b[0].tolist() == k["bounds_1to8_L2"]
    b, _ = gpu_bin(np.array([[5.0], [5], [5], [5]]), 1)
    assert b[0].tolist() == k["bounds_5555_L1"]
    b, _ = gpu_bin(np.array([1.0, 2, np.nan, np.inf, 3, 4]).reshape(-1, 1), 1)
    assert b[0].tolist() == k["bounds_mixed_L1"]


@pytest.mark.parametrize("name,n", [("cfg1", 100_000), ("cfg2", 200_000), ("cfg5", 50_000)])
def test_binning_configs_vs_oracle(name, n):
    X, _, _, kw = make_config(name, n=n)
    L = kw["binning_levels"]
    for arr in (X, X.astype(np.float64)):
        b, c = gpu_bin(arr, L)
        for j in range(X.shape[1]):
            ref_b = oracle.fit_boundaries(X[:, j], L)
            np.testing.assert_array_equal(b[j], ref_b)
            np.testing.assert_array_equal(c[j], oracle.bin_codes(ref_b, X[:, j]))


# ------------------------------------------------------------------ subsample masks
def _np_masks(seed, a, b, rate, T):
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for _ in range(T):
        ms = []
        for nn in (a, b):
            m = np.zeros(nn, bool)
            m[rng.permutation(nn)[:math.floor(rate * nn)]] = True
            ms.append(m)
        out.append(np.concatenate(ms))
    return out


@pytest.mark.parametrize("seed,a,b,rate,T", [(0, 50_000, 50_000, 0.5, 3), (7, 1, 2, 0.5, 3), (3, 1000, 17, 0.3, 4),
                                             (9, 65_537, 131_071, 0.77, 2), (2**40 + 5, 2, 5, 1.0, 2),
                                             (42, 5, 100_000, 0.01, 2), (123, 300_000, 700_000, 0.5, 2),
                                             (5, 0, 9, 0.5, 2), (8, 2_000_003, 1_048_577, 0.5, 1),
                                             (17, 300_000, 700_000, 0.5, 10)])
def test_gpu_subsample_masks_match_numpy(seed, a, b, rate, T):
    _check_masks(seed, a, b, rate, T)


# short jobs next to huge ones: the anchor slack (up to 4000 draws) exceeds the
# short job's whole draw count, so it ends inside the chain's first walk
# (kernels_seg.cuh k_seg_chain); then the BASELINE class-block sizes: cfg3
# 5M/5M and cfg5 20M/30M (datagen proportions), chained trees
@pytest.mark.parametrize("seed,a,b,rate,T", [(1, 2_100, 10_000_000, 0.5, 2), (4, 2_500, 1_000_000, 0.5, 50),
                                             (6, 3_000_000, 2_049, 0.5, 3), (0, 5_000_000, 5_000_000, 0.5, 3),
                                             (0, 20_000_000, 30_000_000, 0.5, 2)])
def test_gpu_subsample_masks_large_blocks(seed, a, b, rate, T):
    _check_masks(seed, a, b, rate, T)


# narrow windows and short segments: most starts miss their window, so the
# chain falls back to exact walks all the time; the result must not change
# (windows only decide how much work is parallel).  Also the throughput plan
# (>= 4M rows: 16384-draw segments, 3-sd windows) on an uneven pair of blocks.
@pytest.mark.parametrize("seed,a,b,rate,T,sd,seg_len", [(11, 300_000, 700_000, 0.5, 3, "0.5", "4096"),
                                                        (12, 1_500_000, 900_000, 0.37, 2, "1.0", "16384"),
                                                        (13, 3_100_000, 1_200_000, 0.5, 4, None, None)])
def test_gpu_subsample_masks_window_misses(seed, a, b, rate, T, sd, seg_len, monkeypatch):
    if sd is not None:
        monkeypatch.setenv("BB_SEG_SD", sd)
        monkeypatch.setenv("BB_SEG_LEN", seg_len)
    _check_masks(seed, a, b, rate, T)


def _check_masks(seed, a, b, rate, T):
    cfg = _lib.FitConfigC(**_lib.pcg_config(seed))
    words = (a + b + 31) // 32
    bits = np.zeros(max(1, words) * T, np.uint32)
    _lib.check(_lib.lib().bb_subsample_masks_gpu(_lib.context(), a, b, rate, T, C.byref(cfg), _lib.ptr(bits)))
    ref = _np_masks(seed, a, b, rate, T)
    for t in range(T):
        m = np.unpackbits(bits[t * words:(t + 1) * words].view(np.uint8), bitorder="little")[:a + b].astype(bool)
        np.testing.assert_array_equal(m, ref[t], err_msg=f"tree {t}")


# ------------------------------------------------------------------ histogram
def _random_layer(rng, n, n_sig, d, levels, layer, nan_rate=0.05, neg=True):
    B = 1 << levels
    codes = rng.integers(1, B + 1, (d, n)).astype(np.uint16)
    codes[rng.random((d, n)) < nan_rate] = 0
    start = (1 << (layer - 1)) - 1
    node = rng.integers(start, 2 * start + 1, n).astype(np.uint16)
    parked = rng.random(n) < 0.05
    node[parked] = rng.integers(0, max(start, 1), parked.sum()) if start > 0 else 0
    q = rng.integers(0, 1 << 32, n).astype(np.int64)
    q[rng.random(n) < 0.4] = 0
    if neg:
        m = rng.random(n) < 0.05
        q[m] = -q[m]
    return codes, node, q


def _oracle_hist(codes, node, q, n_sig, d, levels, layer):
    B = 1 << levels
    start = (1 << (layer - 1)) - 1
    nodes = 1 << (layer - 1)
    out = np.zeros((2, nodes, d, B), np.int64)
    for cls, sl in ((0, slice(0, n_sig)), (1, slice(n_sig, None))):
        nd = node[sl].astype(np.int64) - start
        ok = (nd >= 0) & (nd < nodes)
        for j in range(d):
            c = codes[j, sl].astype(np.int64)
            m = ok & (c > 0)
            flat = nd[m] * B + (c[m] - 1)
            out[cls, :, j, :] = oracle.binboost_np._exact_int_bincount(flat, q[sl][m], nodes * B).reshape(nodes, B)
    return out


@pytest.fixture(params=["list", "list_groups", "fl", "fl_partials", "warp", "cta", "global"])
def hist_path(request, monkeypatch):
    """Every histogram kernel: the node-partitioned row-list one (default for
    u8 codes and d <= 64), the feature-lane one (TMA bulk reductions into the
    histogram, or with BB_FL_PARTIALS=1 per-CTA partial rows summed by
    k_fl_reduce), the warp-independent shared-memory one, the CTA-barrier one
    and the global-atomic one (BB_HIST_PATH = list | fl | w | cta | g)."""
    monkeypatch.setenv("BB_HIST_PATH", {"list": "list", "list_groups": "list", "fl": "fl", "fl_partials": "fl",
                                        "warp": "w", "cta": "cta", "global": "g"}[request.param])
    if request.param == "list_groups":  # rows of 33..64 features as two 32-feature groups
        monkeypatch.setenv("BB_LH_GROUPS", "1")
    if request.param == "fl_partials":
        monkeypatch.setenv("BB_FL_PARTIALS", "1")
    return request.param


@pytest.mark.parametrize("levels,layer,d", [(8, 1, 10), (8, 3, 40), (8, 5, 7), (10, 6, 3), (3, 2, 5), (1, 1, 2),
                                             (8, 2, 50), (8, 4, 33), (6, 3, 17), (8, 2, 70), (4, 3, 100)])
def test_layer_hist_exact(levels, layer, d, hist_path):
    if hist_path.startswith("list") and (d > 64 or levels > 8):
        pytest.skip("row-list kernel: u8 codes, d <= 64 (other shapes take the other kernels)")
    rng = np.random.default_rng(levels * 100 + layer)
    n, n_sig = 60_000, 23_456
    # u8 codes with B = 256 hold no NaN bin (the fit stores code - 1)
    nan_rate = 0.0 if (hist_path.startswith("list") and levels == 8) else 0.05
    codes, node, q = _random_layer(rng, n, n_sig, d, levels, layer, nan_rate=nan_rate)
    B = 1 << levels
    nodes = 1 << (layer - 1)
    out = np.zeros((2, nodes, d, B), np.int64)
    _lib.check(_lib.lib().bb_layer_hist(_lib.context(), _lib.ptr(codes), _lib.ptr(node), _lib.ptr(q), n, n_sig, d,
                                        levels, layer, _lib.ptr(out)))
    np.testing.assert_array_equal(out, _oracle_hist(codes, node, q, n_sig, d, levels, layer))


def test_layer_hist_list_long_runs(monkeypatch):
    """Row-list kernel with > kLhFlushRows (32767) rows per CTA (mid-run
    flushes of the 16/16-bit limbs), the largest |q| and one tied bin."""
    monkeypatch.setenv("BB_HIST_PATH", "list")
    rng = np.random.default_rng(6)
    n, n_sig, d, levels, layer = 12_000_000, 4_400_001, 3, 8, 1
    codes, node, q = _random_layer(rng, n, n_sig, d, levels, layer, nan_rate=0.0)
    q[::7] = (1 << 32) - 1
    q[3::11] = -((1 << 32) - 1)
    codes[1, : n // 2] = 17
    B = 1 << levels
    out = np.zeros((2, 1, d, B), np.int64)
    _lib.check(_lib.lib().bb_layer_hist(_lib.context(), _lib.ptr(codes), _lib.ptr(node), _lib.ptr(q), n, n_sig, d,
                                        levels, layer, _lib.ptr(out)))
    np.testing.assert_array_equal(out, _oracle_hist(codes, node, q, n_sig, d, levels, layer))


@pytest.mark.parametrize("name,n,T,D,L", [("cfg3", 300_000, 6, 5, 8), ("cfg1", 50_000, 8, 3, 8),
                                          ("cfg2", 200_000, 8, 4, 8), ("cfg2", 100_000, 5, 6, 6)])
def test_fit_list_path_matches_fl(name, n, T, D, L, monkeypatch):
    """The fit with the row-list histogram (default) against the same fit on
    the feature-lane / warp kernels: identical cuts, leaves and weights."""
    X, y, w, _ = make_config(name, n=n)
    cfg = FitConfig(n_trees=T, depth=D, shrinkage=0.1, subsample=0.5, binning_levels=L, seed=4)
    monkeypatch.setenv("BB_HIST_PATH", "list")
    a = fit_forest(X, y, w, cfg, return_leaves=True)
    monkeypatch.setenv("BB_HIST_PATH", "w")
    b = fit_forest(X, y, w, cfg, return_leaves=True)
    for ta, tb in zip(a.trees, b.trees):
        np.testing.assert_array_equal(ta.valid, tb.valid)
        np.testing.assert_array_equal(ta.feature, tb.feature)
        np.testing.assert_array_equal(ta.cut_bin, tb.cut_bin)
        np.testing.assert_array_equal(ta.node_weight, tb.node_weight)
        np.testing.assert_array_equal(ta.gain, tb.gain)
    np.testing.assert_array_equal(a.fit_info["leaves"], b.fit_info["leaves"])


def test_layer_hist_fl_long_runs(monkeypatch):
    """Feature-lane kernel with > kFlFlushStages (63) stages per CTA (mid-run
    flushes of the 16/16-bit limbs) and the largest |q| (2^32 - 1)."""
    monkeypatch.setenv("BB_HIST_PATH", "fl")
    rng = np.random.default_rng(5)
    n, n_sig, d, levels, layer = 6_000_000, 2_200_001, 2, 8, 2
    codes, node, q = _random_layer(rng, n, n_sig, d, levels, layer)
    q[::7] = (1 << 32) - 1
    q[3::11] = -((1 << 32) - 1)
    codes[1, : n // 2] = 17  # one tied bin takes half the rows
    B = 1 << levels
    out = np.zeros((2, 1 << (layer - 1), d, B), np.int64)
    _lib.check(_lib.lib().bb_layer_hist(_lib.context(), _lib.ptr(codes), _lib.ptr(node), _lib.ptr(q), n, n_sig, d,
                                        levels, layer, _lib.ptr(out)))
    np.testing.assert_array_equal(out, _oracle_hist(codes, node, q, n_sig, d, levels, layer))


@pytest.mark.parametrize("levels,layer,d,final", [(8, 1, 10, 0), (8, 3, 40, 1), (4, 4, 3, 0), (2, 2, 2, 1)])
def test_split_exact(levels, layer, d, final):
    rng = np.random.default_rng(7 + levels + layer)
    n, n_sig = 30_000, 12_000
    codes, node, q = _random_layer(rng, n, n_sig, d, levels, layer, neg=False)
    q = (q >> 1)
    B = 1 << levels
    nodes = 1 << (layer - 1)
    hist = _oracle_hist(codes, node, q, n_sig, d, levels, layer)
    # discrete-like ties: duplicate a feature so equal gains occur
    if d >= 2:
        hist[:, :, 1, :] = hist[:, :, 0, :]
    bounds = np.sort(rng.normal(size=(d, B - 1)), axis=1)
    shift = 32
    v = np.zeros(nodes, np.uint8)
    f = np.zeros(nodes, np.int32)
    c = np.zeros(nodes, np.int32)
    g = np.zeros(nodes)
    t = np.zeros(nodes)
    _lib.check(_lib.lib().bb_split(_lib.context(), _lib.ptr(hist), d, levels, layer, final, shift, _lib.ptr(bounds),
                                   _lib.ptr(v), _lib.ptr(f), _lib.ptr(c), _lib.ptr(g), _lib.ptr(t)))
    # oracle: cumulative layout (nodes, d, B+1) with slot 0 = NaN (unused)
    cum = [np.concatenate([np.zeros((nodes, d, 1), np.int64), np.cumsum(hist[k], axis=2)], axis=2) for k in (0, 1)]
    scored = _gains_fixed(cum[0], cum[1], B, 2.0 ** -shift)
    ref = _pick_cuts(scored, B, bool(final), {})
    for k, (ok, rf, rc, rg) in enumerate(ref):
        assert bool(v[k]) == ok, k
        if ok:
            assert (f[k], c[k]) == (rf, rc), k
            assert g[k] == rg, k
            assert t[k] == bounds[rf][rc - 1]


# ------------------------------------------------------------------ full fit
def _forced_from_golden(g, gap_tol=1e-9, noise_tol=1e-9):
    """Teacher-forced protocol: nodes whose reference
    argmax is decided by float64 rounding noise take the reference's
    decision: best-vs-runner-up relative gap < gap_tol, pure-signal nodes
    (G(s,0) = s*s/s noise), or a best gain at the noise floor of the node's
    absolute weight mass (its validity g > 0 on the last layer, and the
    argmax among such gains, are then rounding noise)."""
    forced = {}
    for t, node, gap, pure, best, scale in g["audit"]:
        t, node = int(t), int(node)
        noise = math.isfinite(best) and abs(best) <= noise_tol * scale
        if gap < gap_tol or pure or noise:
            forced[(t, node)] = (bool(g["valid"][t, node]), int(g["feature"][t, node]), int(g["cut_bin"][t, node]))
    return forced


def _check_fit_vs_golden(forest, g, rows_X, forced_ok=True, tight=True):
    T = int(g["n_trees"])
    np.testing.assert_array_equal(np.stack([b.boundaries for b in forest.binnings]), g["boundaries"])
    for t in range(T):
        tr = forest.trees[t]
        np.testing.assert_array_equal(tr.valid, g["valid"][t], err_msg=f"tree {t}")
        np.testing.assert_array_equal(tr.feature, g["feature"][t], err_msg=f"tree {t}")
        np.testing.assert_array_equal(tr.cut_bin, g["cut_bin"][t], err_msg=f"tree {t}")
        np.testing.assert_array_equal(tr.threshold, g["threshold"][t], err_msg=f"tree {t}")
        lv = forest.fit_info["leaves"][t].astype(np.int16)
        assert sha(lv) == g["leaf_hashes"][t], f"leaf ids differ at tree {t}"
        # node weights and gains come from fixed-point sums: not bit-exact
        # quantities (the contract on them is the probability bar below).
        # Measured max relative error over the goldens (tools/divergence.py,
        # profiles/r02_divergence.txt): node weight 3.5e-6, gain 1.5e-10
        # (the randomized small fits - negative weights, near-empty nodes,
        # cancelling sums - keep the loose bound: tight=False)
        if not tight:
            np.testing.assert_allclose(tr.node_weight, g["node_weight"][t], rtol=1e-3, atol=1e-6)
            continue
        np.testing.assert_allclose(tr.node_weight, g["node_weight"][t], rtol=1e-4, atol=1e-7)
        if "gain" in g:
            ok = np.asarray(tr.valid, bool) & np.isfinite(g["gain"][t])
            scale = float(np.max(np.abs(g["gain"][t][ok]))) if ok.any() else 0.0
            np.testing.assert_allclose(tr.gain[ok], g["gain"][t][ok], rtol=1e-6, atol=1e-9 * scale)
    p = predict_batch(forest, rows_X)
    assert np.max(np.abs(p - g["pred"])) <= PROB_TOL


def test_fit_cfg1_vs_reference_golden(golden_dir):
    g = np.load(f"{golden_dir}/cfg1_fit.npz")
    X, y, w, kw = make_config("cfg1")
    cfg = FitConfig(n_trees=kw["trees"], depth=kw["depth"], shrinkage=kw["shrinkage"], subsample=kw["subsample"],
                    binning_levels=kw["binning_levels"], seed=kw["seed"])
    forced = _forced_from_golden(g)
    assert not forced, "cfg1 has no tie-ambiguous nodes (SURVEY.md A4): free-running parity"
    forest = fit_forest(X, y, w, cfg, return_leaves=True)
    assert forest.f0 == float(g["f0"])
    _check_fit_vs_golden(forest, g, X[g["pred_rows"]])


def test_fit_vs_fixed_point_oracle(hist_path):
    X, y, w, _ = make_config("cfg2", n=60_000)
    cfg = FitConfig(n_trees=12, depth=4, shrinkage=0.2, subsample=0.6, binning_levels=6, seed=11)
    forest = fit_forest(X, y, w, cfg, return_leaves=True, return_scores=True)
    ref = oracle.fit_forest(X, y, w, n_trees=12, depth=4, shrinkage=0.2, subsample=0.6, levels=6, seed=11,
                            fixed_point=True, record_leaves=True)
    assert forest.fit_info["fixed_shift"] == ref.fixed_shift
    for t in range(12):
        tr = forest.trees[t]
        np.testing.assert_array_equal(tr.feature, ref.feature[t])
        np.testing.assert_array_equal(tr.cut_bin, ref.cut_bin[t])
        np.testing.assert_array_equal(tr.valid, ref.valid[t])
        np.testing.assert_array_equal(forest.fit_info["leaves"][t], ref.leaves[t].astype(np.uint16))
        np.testing.assert_allclose(tr.node_weight, ref.node_weight[t], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(tr.gain, ref.gain[t], rtol=1e-9, atol=1e-12)


def test_small_fits_vs_reference_golden(golden_dir):
    z = np.load(f"{golden_dir}/small_fits.npz")
    n_cases = len({k.split("__")[0] for k in z.files})
    forced_total = 0
    for i in range(n_cases):
        g = {k.split("__", 1)[1]: z[k] for k in z.files if k.startswith(f"c{i}__")}
        T, D, eta, alpha, L, seed = g["config"]
        cfg = FitConfig(n_trees=int(T), depth=int(D), shrinkage=float(eta), subsample=float(alpha),
                        binning_levels=int(L), seed=int(seed))
        forced = _forced_from_golden(g)
        forced_total += len(forced)
        forest = fit_forest(g["X"], g["y"], g.get("w"), cfg, forced_cuts=forced, return_leaves=True)
        assert forest.f0 == float(g["f0"]), i
        try:
            _check_fit_vs_golden(forest, g, g["X"][g["pred_rows"]], tight=False)
        except AssertionError as e:
            raise AssertionError(f"case {i}: {e}") from None
    print("forced nodes across small cases:", forced_total)


# ------------------------------------------------------------------ apply
def test_apply_cfg4_slice_vs_golden(golden_dir):
    g = np.load(f"{golden_dir}/apply_cfg4_slice.npz")
    X, _, _, _ = make_config("cfg4", n=20_000)
    from paper_1609_06119_b200.engine import FeatureBinning, Forest, Tree

    T = g["feature"].shape[0]
    trees = [Tree(depth=3, feature=g["feature"][t], cut_bin=g["cut_bin"][t], threshold=g["threshold"][t],
                  gain=np.zeros(7), valid=np.ones(7, bool), node_weight=g["node_weight"][t],
                  node_purity=np.zeros(15)) for t in range(T)]
    forest = Forest(f0=0.0, trees=trees, binnings=[FeatureBinning(b, 8) for b in g["boundaries"]])
    for arr in (X, X.astype(np.float64)):
        p = predict_batch(forest, arr)
        assert np.max(np.abs(p - g["pred"])) <= 1e-15


def test_apply_nan_and_invalid_nodes():
    rng = np.random.default_rng(3)
    X = rng.normal(size=(5000, 4))
    X[rng.random(X.shape) < 0.2] = np.nan
    y = (rng.random(5000) < 0.5).astype(int)
    forest = fit_forest(X, y, None, FitConfig(n_trees=15, depth=4, binning_levels=3, seed=5))
    ref = oracle.predict_scores(forest.f0, np.stack([t.valid for t in forest.trees]),
                                np.stack([t.feature for t in forest.trees]),
                                np.stack([t.threshold for t in forest.trees]),
                                np.stack([t.node_weight for t in forest.trees]), 4, X)
    p, F = predict_batch(forest, X, return_scores=True)
    np.testing.assert_array_equal(F, ref)


def test_apply_large_forest_multi_launch():
    """More trees than one launch's parameter-space records (1300 trees at the
    default 2 levels, 557 at 3): F continues across launches in tree order;
    NaN rows and invalid nodes."""
    from paper_1609_06119_b200.engine import FeatureBinning, Forest, Tree

    rng = np.random.default_rng(11)
    T, D, d = 1400, 3, 6
    X = rng.normal(size=(3000, d)).astype(np.float32)
    X[rng.random(X.shape) < 0.03] = np.nan
    bounds = [np.sort(rng.normal(size=255)) for _ in range(d)]
    feature = rng.integers(0, d, (T, 7)).astype(np.int32)
    cut = rng.integers(1, 256, (T, 7)).astype(np.int32)
    valid = rng.random((T, 7)) > 0.05
    thr = np.array([[bounds[feature[t, k]][cut[t, k] - 1] for k in range(7)] for t in range(T)])
    nw = rng.uniform(-1, 1, (T, 15))
    trees = [Tree(depth=D, feature=np.where(valid[t], feature[t], -1), cut_bin=np.where(valid[t], cut[t], 0),
                  threshold=np.where(valid[t], thr[t], np.nan), gain=np.zeros(7), valid=valid[t], node_weight=nw[t],
                  node_purity=np.zeros(15)) for t in range(T)]
    forest = Forest(f0=0.25, trees=trees, binnings=[FeatureBinning(b, 8) for b in bounds])
    ref = oracle.predict_scores(0.25, valid, np.where(valid, feature, -1), np.where(valid, thr, np.nan), nw, D, X)
    for levels in ("2", "3"):
        os.environ["BB_APPLY_PARAM_LEVELS"] = levels  # read per call
        try:
            p, F = predict_batch(forest, X, return_scores=True)
        finally:
            del os.environ["BB_APPLY_PARAM_LEVELS"]
        np.testing.assert_array_equal(F, ref)


def test_apply_mixed_depth_forest():
    """A forest whose trees have different depths (allowed by the model file,
    model_io.py:185-191): shallow trees are padded with invalid nodes, so each
    tree's prediction is its own traversal (trees.py:333-346)."""
    from paper_1609_06119_b200.engine import FeatureBinning, Forest, Tree

    rng = np.random.default_rng(21)
    d = 5
    X = rng.normal(size=(4000, d))
    X[rng.random(X.shape) < 0.05] = np.nan
    trees = []
    for t, D in enumerate([1, 3, 2, 5, 4, 3]):
        I, N = (1 << D) - 1, (1 << (D + 1)) - 1
        valid = rng.random(I) > 0.1
        feature = np.where(valid, rng.integers(0, d, I), -1)
        thr = np.where(valid, rng.normal(size=I), np.nan)
        nw = rng.uniform(-1, 1, N)
        trees.append(Tree(depth=D, feature=feature, cut_bin=np.where(valid, 1, 0), threshold=thr, gain=np.zeros(I),
                          valid=valid, node_weight=nw, node_purity=np.zeros(N)))
    forest = Forest(f0=0.1, trees=trees, binnings=[FeatureBinning(np.sort(rng.normal(size=7)), 3) for _ in range(d)])
    for dt in (np.float64, np.float32):
        Xc = X.astype(dt)
        ref = np.full(X.shape[0], 0.1)
        for t in trees:
            ref += oracle.predict_scores(0.0, t.valid[None], t.feature[None], t.threshold[None], t.node_weight[None],
                                         t.depth, Xc)
        _, F = predict_batch(forest, Xc, return_scores=True)
        np.testing.assert_allclose(F, ref, rtol=0, atol=1e-12)


# ------------------------------------------------------------------ bridge
def test_bridge_fit_predict_and_concurrency():
    X, y, w, _ = make_config("cfg1", n=20_000)
    m = bridge.fit(X, y, w, trees=20, depth=3, seed=3)
    p = m.predict(X[:1000])
    assert p.shape == (1000,) and np.all((p > 0) & (p < 1))
    assert m.predict(np.empty(0)).shape == (0,)
    results = [None] * 4

    def work(k):
        results[k] = m.predict(X[:1000])

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    [t.start() for t in th]
    [t.join() for t in th]
    for r in results:
        np.testing.assert_array_equal(r, p)
    m.close()
    with pytest.raises(RuntimeError, match="model handle is closed"):
        m.predict(X[:3])


# ------------------------------------------------------------------ model files
def test_model_file_interop(golden_dir, tmp_path):
    from paper_1609_06119_b200.model_format import load_forest, parse_forest, save_forest, serialize_forest

    # reference-written model -> GPU apply
    f = load_forest(f"{golden_dir}/ref_model.json")
    X = np.load(f"{golden_dir}/ref_model_inputs.npz")["X"]
    np.testing.assert_allclose(predict_batch(f, X), np.load(f"{golden_dir}/ref_model_pred.npy"), rtol=0, atol=1e-15)
    # GPU-fitted model -> file -> same predictions, byte-stable document
    Xf, y, w, _ = make_config("cfg1", n=5000)
    m = bridge.fit(Xf, y, w, trees=5, depth=3, seed=2)
    path = str(tmp_path / "m.json")
    m.save(path)
    m2 = bridge.load(path)
    np.testing.assert_array_equal(m.predict(Xf[:500]), m2.predict(Xf[:500]))
    text = open(path).read()
    assert serialize_forest(parse_forest(text)) == text


# ------------------------------------------------------------------ other configs
@pytest.mark.parametrize("name,fixture,n", [("cfg2", "cfg2_slice_fit.npz", 200_000),
                                            ("cfg3", "cfg3_proxy_fit.npz", 200_000)])
def test_fit_config_slices_vs_reference_golden(golden_dir, name, fixture, n):
    """cfg2 slice (ties from discrete features, U(0.5,1.5) weights) and the
    cfg3-literal proxy (depth 5, highly separable: genuine near-ties, SURVEY
    A4/A6) against the unmodified reference, teacher-forced at tie-ambiguous
    nodes only."""
    g = np.load(f"{golden_dir}/{fixture}")
    X, y, w, _ = make_config(name, n=n)
    T, D, eta, alpha, L, seed = g["config"]
    cfg = FitConfig(n_trees=int(T), depth=int(D), shrinkage=float(eta), subsample=float(alpha),
                    binning_levels=int(L), seed=int(seed))
    forced = _forced_from_golden(g)
    forest = fit_forest(X, y, w, cfg, forced_cuts=forced, return_leaves=True)
    print(f"{name}: {len(forced)} forced of {g['audit'].shape[0]} nodes")
    _check_fit_vs_golden(forest, g, X[g["pred_rows"]])


def test_cfg5_slice_vs_fixed_point_oracle():
    """cfg5 shape: 1024 bins (uint16 codes), depth 6, exponential weights,
    heavy tails — GPU integer arithmetic predicted exactly by the oracle."""
    X, y, w, _ = make_config("cfg5", n=60_000)
    kw = dict(n_trees=4, depth=6, shrinkage=0.1, subsample=0.5, levels=10, seed=0)
    forest = fit_forest(X, y, w, FitConfig(n_trees=4, depth=6, shrinkage=0.1, subsample=0.5, binning_levels=10,
                                           seed=0), return_leaves=True)
    ref = oracle.fit_forest(X, y, w, fixed_point=True, record_leaves=True, **kw)
    np.testing.assert_array_equal(np.stack([b.boundaries for b in forest.binnings]), ref.boundaries)
    for t in range(4):
        tr = forest.trees[t]
        np.testing.assert_array_equal(tr.feature, ref.feature[t])
        np.testing.assert_array_equal(tr.cut_bin, ref.cut_bin[t])
        np.testing.assert_array_equal(forest.fit_info["leaves"][t], ref.leaves[t].astype(np.uint16))
        np.testing.assert_allclose(tr.node_weight, ref.node_weight[t], rtol=1e-12, atol=1e-15)
    p = predict_batch(forest, X[:3000])
    assert np.max(np.abs(p - oracle.predict(ref, X[:3000]))) <= 1e-12


# ------------------------------------------------------------ sharded fit
@pytest.mark.parametrize("weighted", [False, True])
def test_sharded_fit_world1_matches_single(weighted):
    """The NCCL row-sharded path (communicator, binning/class-count/layer/
    final-sum all-reduces, global mask + slice) at world size 1 must give
    the single-device forest bit-for-bit."""
    import os
    import socket

    import torch.distributed as dist

    from paper_1609_06119_b200.distributed import fit_forest_sharded

    rng = np.random.default_rng(11)
    n, d = 30_000, 6
    X = rng.normal(size=(n, d)).astype(np.float32)
    y = (X[:, 0] + 0.5 * rng.normal(size=n) > 0).astype(np.int8)
    w = rng.uniform(0.5, 2.0, n) if weighted else None
    cfg = FitConfig(n_trees=6, depth=3, shrinkage=0.1, subsample=0.5, binning_levels=6, seed=3)
    ref = fit_forest(X, y, w, cfg, return_leaves=True)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        got = fit_forest_sharded(X, y, w, cfg, device=0, return_leaves=True)
    finally:
        dist.destroy_process_group()
    assert got.f0 == ref.f0
    for a, b in zip(got.binnings, ref.binnings):
        np.testing.assert_array_equal(a.boundaries, b.boundaries)
    for ta, tb in zip(got.trees, ref.trees):
        np.testing.assert_array_equal(ta.valid, tb.valid)
        np.testing.assert_array_equal(ta.feature[ta.valid], tb.feature[tb.valid])
        np.testing.assert_array_equal(ta.cut_bin[ta.valid], tb.cut_bin[tb.valid])
        np.testing.assert_array_equal(ta.node_weight, tb.node_weight)
    np.testing.assert_array_equal(got.fit_info["leaves"], ref.fit_info["leaves"])


# ------------------------------------------------------------ full-size configs
def _fit_golden_config(name, fixture, golden_dir, n=None):
    g = np.load(f"{golden_dir}/{fixture}")
    X, y, w, _ = make_config(name, n=n)
    T, D, eta, alpha, L, seed = g["config"]
    cfg = FitConfig(n_trees=int(T), depth=int(D), shrinkage=float(eta), subsample=float(alpha),
                    binning_levels=int(L), seed=int(seed))
    forced = _forced_from_golden(g)
    forest = fit_forest(X, y, w, cfg, forced_cuts=forced, return_leaves=True)
    return g, X, forest, forced


def test_fit_cfg2_full_vs_reference_golden(golden_dir):
    """BASELINE configs[1] exactly (1M rows x 40, 200 trees) against the
    unmodified reference: no tie-ambiguous node, so free-running; every cut,
    threshold and per-row leaf id of all 200 trees, probabilities <= 1e-5."""
    g, X, forest, forced = _fit_golden_config("cfg2", "cfg2_full_fit.npz", golden_dir)
    assert not forced
    assert forest.f0 == float(g["f0"])
    _check_fit_vs_golden(forest, g, X[g["pred_rows"]])


def test_fit_cfg3_10M_prefix_vs_reference_golden(golden_dir):
    """BASELINE configs[2] at its full 10M rows x 50 features: the first 4
    of the 400 depth-5 trees (a fit's first trees do not depend on the tree
    count) against the reference, free-running."""
    g, X, forest, forced = _fit_golden_config("cfg3", "cfg3_10M_prefix.npz", golden_dir)
    assert not forced
    _check_fit_vs_golden(forest, g, X[g["pred_rows"]])


def test_fit_cfg5_1M_slice_vs_reference_golden(golden_dir):
    """BASELINE configs[4] generator (t3 + Gaussian mixtures, exponential
    weights, 40% signal) on a 1M-row slice x 100 features, 1024 bins (u16
    codes), depth 6, against the reference (not only the fixed-point
    oracle)."""
    g, X, forest, forced = _fit_golden_config("cfg5", "cfg5_1M_slice.npz", golden_dir, n=1_000_000)
    assert not forced
    _check_fit_vs_golden(forest, g, X[g["pred_rows"]])


def test_apply_cfg4_1000_trees_vs_reference_golden(golden_dir):
    """BASELINE configs[3]: the full 1000-tree depth-3 forest (seed 1) over
    the first 100k rows of the seed-1 N(0,1) data, boundaries fitted on those
    rows, against the reference's predict_batch."""
    from paper_1609_06119_b200.engine import FeatureBinning, Forest, Tree

    g = np.load(f"{golden_dir}/apply_cfg4_1000trees.npz")
    X, _, _, _ = make_config("cfg4", n=100_000)
    bnd = g["boundaries"]
    b, _ = gpu_bin(X, 8)
    np.testing.assert_array_equal(b, bnd)
    from paper_1609_06119_b200.datagen import make_apply_forest

    feat, cut, thr, nw = make_apply_forest(bnd, n_trees=1000, depth=3, seed=1)
    trees = [Tree(depth=3, feature=feat[t], cut_bin=cut[t], threshold=thr[t], gain=np.zeros(7),
                  valid=np.ones(7, bool), node_weight=nw[t], node_purity=np.zeros(15)) for t in range(1000)]
    forest = Forest(f0=0.0, trees=trees, binnings=[FeatureBinning(bnd[j], 8) for j in range(X.shape[1])])
    for arr in (X, X.astype(np.float64)):
        p = predict_batch(forest, arr)
        assert np.max(np.abs(p - g["pred"])) <= 1e-15


def test_binning_cfg3_full_and_cfg5_50M_columns():
    """bb_bin bit-exact against the oracle: all 50 cfg3 features at 10M rows,
    and 10 cfg5-shaped columns (5 Student-t(3), 5 Gaussian mixtures) at 50M
    rows, 1024 bins."""
    X, _, _, _ = make_config("cfg3")
    b, c = gpu_bin(X, 8)
    for j in range(X.shape[1]):
        ref_b = oracle.fit_boundaries(X[:, j], 8)
        np.testing.assert_array_equal(b[j], ref_b, err_msg=f"cfg3 feature {j}")
        np.testing.assert_array_equal(c[j], oracle.bin_codes(ref_b, X[:, j]), err_msg=f"cfg3 feature {j}")
    del X, b, c
    rng = np.random.Generator(np.random.PCG64(55))
    n = 50_000_000
    cols = np.empty((n, 10), np.float32)
    for j in range(5):
        cols[:, j] = rng.standard_t(3, n)
        cols[:, 5 + j] = np.where(rng.random(n) < 0.5, -1.0, 1.0) + 0.5 * rng.standard_normal(n)
    b, c = gpu_bin(cols, 10)
    for j in range(10):
        ref_b = oracle.fit_boundaries(cols[:, j], 10)
        np.testing.assert_array_equal(b[j], ref_b, err_msg=f"cfg5 column {j}")
        np.testing.assert_array_equal(c[j], oracle.bin_codes(ref_b, cols[:, j]), err_msg=f"cfg5 column {j}")


# ------------------------------------------------------------ analysis (f2, f3)
def test_roc_auc_vs_reference_golden(golden_dir):
    """GPU weighted ROC AUC (radix sort + prefix sums) against the reference's
    roc_auc on plain, tied and weighted scores (analysis.py:45-70)."""
    from paper_1609_06119_b200.analysis import roc_auc

    g = np.load(f"{golden_dir}/analysis.npz")
    for k in range(4):
        w = g[f"auc{k}_w"] if f"auc{k}_w" in g.files else None
        got = roc_auc(g[f"auc{k}_scores"], g[f"auc{k}_labels"], w)
        assert abs(got - float(g[f"auc{k}_value"])) <= 1e-12, k
    with pytest.raises(ValueError, match="both classes"):
        roc_auc(np.arange(5.0), np.ones(5))


def test_roc_auc_large_vs_numpy():
    """20M rows with heavy ties (every rank bucket of the 16 radix passes)."""
    from paper_1609_06119_b200.analysis import roc_auc

    rng = np.random.default_rng(4)
    n = 20_000_000
    s = np.round(rng.normal(size=n) * 64) / 64
    s[::97] = -0.0
    s[1::97] = 0.0
    y = rng.random(n) < 0.3
    w = rng.exponential(1.0, n)
    u, inv = np.unique(s, return_inverse=True)
    sa = np.bincount(inv, weights=np.where(y, w, 0.0), minlength=u.size)
    ba = np.bincount(inv, weights=np.where(y, 0.0, w), minlength=u.size)
    below = np.concatenate(([0.0], np.cumsum(ba)[:-1]))
    ref = float(np.sum(sa * (below + 0.5 * ba))) / (float(np.sum(w[y])) * float(np.sum(w[~y])))
    assert abs(roc_auc(s, y.astype(np.int8), w) - ref) <= 1e-10


def test_elimination_importance_vs_reference_golden(golden_dir):
    """Batched GPU elimination (one binning, concurrent refits on several
    contexts, device AUC) against the reference's elimination_importance:
    same removal order and fit count.  Scores / AUCs agree to 5e-5: refit 2
    (seed 11, features 0,2,3,4,5) has a tie-ambiguous node (tree 2, node 6)
    where the reference's float64 argmax and the fixed-point one differ (the
    oracle reproduces both), so that refit's AUC moves by ~1e-5."""
    from paper_1609_06119_b200.analysis import elimination_importance

    g = np.load(f"{golden_dir}/analysis.npz")
    T, D, eta, alpha, L, seed = g["elim_config"]
    cfg = FitConfig(n_trees=int(T), depth=int(D), shrinkage=float(eta), subsample=float(alpha),
                    binning_levels=int(L), seed=int(seed))
    reps = [elimination_importance(g["elim_X"], g["elim_y"], g["elim_w"], cfg, workers=k) for k in (1, 4)]
    for rep in reps:
        assert rep.n_fits == int(g["elim_n_fits"])
        assert rep.order == g["elim_order"].tolist()
        np.testing.assert_allclose(rep.scores, g["elim_scores"], rtol=0, atol=5e-5)
        np.testing.assert_allclose(rep.step_aucs, g["elim_step_aucs"], rtol=0, atol=5e-5)
    # concurrency does not change a single bit
    np.testing.assert_array_equal(reps[0].scores, reps[1].scores)
    # the batched session equals the reference protocol run fit by fit on the
    # GPU engine (fit_forest / predict_batch / roc_auc per refit)
    from paper_1609_06119_b200.analysis import roc_auc

    X, y, w = g["elim_X"], g["elim_y"], g["elim_w"]
    n = X.shape[0]
    perm = np.random.Generator(np.random.PCG64(cfg.seed)).permutation(n)
    tr, va = perm[: n // 2], perm[n // 2:]
    import dataclasses

    def fit_auc(cols, o):
        f = fit_forest(X[np.ix_(tr, cols)], y[tr], w[tr], dataclasses.replace(cfg, seed=cfg.seed + o))
        return roc_auc(predict_batch(f, X[np.ix_(va, cols)]), y[va], w[va])

    rem, o = list(range(X.shape[1])), 0
    base = fit_auc(rem, o)
    o += 1
    assert abs(base - reps[0].step_aucs[0]) <= 1e-12
    for step, worst in enumerate(reps[0].order[:-1]):
        aucs = {}
        for f in rem:
            aucs[f] = fit_auc([c for c in rem if c != f], o)
            o += 1
        assert abs(base - aucs[worst] - reps[0].scores[worst]) <= 1e-12
        rem.remove(worst)
        base = aucs[worst]
        assert abs(base - reps[0].step_aucs[step + 1]) <= 1e-12


def test_elimination_refit_equals_direct_fit():
    """A session refit on a feature subset is the forest a direct fit of the
    subset's columns gives (binning once per session is exact)."""
    from paper_1609_06119_b200.analysis import EliminationSession

    X, y, w, _ = make_config("cfg2", n=50_000)
    cols = [3, 17, 22, 31, 39]
    cfg = FitConfig(n_trees=8, depth=4, shrinkage=0.1, subsample=0.5, binning_levels=8, seed=5)
    with EliminationSession(X, y, w, X[:1000], y[:1000], w[:1000], 8) as ses:
        auc = ses.fit_auc(cols, cfg)
    direct = fit_forest(X[:, cols], y, w, cfg)
    from paper_1609_06119_b200.analysis import roc_auc

    ref_auc = roc_auc(predict_batch(direct, X[:1000][:, cols]), y[:1000], w[:1000])
    assert abs(auc - ref_auc) <= 1e-12


# ------------------------------------------------------------ virtual shards
@pytest.mark.parametrize("G,weighted,name,n,D", [(2, False, "cfg1", 40_000, 3), (4, True, "cfg2", 60_000, 4),
                                                 (8, True, "cfg3", 90_000, 5), (3, False, "cfg5", 30_000, 6)])
def test_virtual_shards_match_single(G, weighted, name, n, D):
    """SURVEY.md §4's G-shard harness: the row-sharded library path with G
    shard contexts on one GPU (in-process rank-order sums instead of NCCL)
    gives the single-device forest bit-for-bit: global binning from the
    exchanged radix histograms, class-count offsets, the global subsample
    mask sliced per shard (k_mask_slice), the layer histograms and node sums
    (sample.py:112-116, 128-132)."""
    from paper_1609_06119_b200.distributed import fit_forest_virtual_shards
    from paper_1609_06119_b200.sharding import shard_rows

    X, y, w, kw = make_config(name, n=n)
    if not weighted:
        w = None
    cfg = FitConfig(n_trees=5, depth=D, shrinkage=0.1, subsample=0.5, binning_levels=kw["binning_levels"], seed=7)
    ref = fit_forest(X, y, w, cfg, return_leaves=True)
    parts = [shard_rows(y, g, G) for g in range(G)]
    got = fit_forest_virtual_shards([(X[i], y[i], None if w is None else w[i]) for i in parts], cfg,
                                    return_leaves=True)
    for f in got:
        assert f.f0 == ref.f0
        for a, b in zip(f.binnings, ref.binnings):
            np.testing.assert_array_equal(a.boundaries, b.boundaries)
        for ta, tb in zip(f.trees, ref.trees):
            np.testing.assert_array_equal(ta.valid, tb.valid)
            np.testing.assert_array_equal(ta.feature, tb.feature)
            np.testing.assert_array_equal(ta.cut_bin, tb.cut_bin)
            np.testing.assert_array_equal(ta.node_weight, tb.node_weight)
    # per-shard leaves (class-block order of the shard) = the single fit's
    # leaves of those rows: signal shards then background shards
    n_sig = int((y > 0).sum())
    lv = ref.fit_info["leaves"]
    sig_parts = [got[g].fit_info["leaves"][:, :int((y[parts[g]] > 0).sum())] for g in range(G)]
    bkg_parts = [got[g].fit_info["leaves"][:, int((y[parts[g]] > 0).sum()):] for g in range(G)]
    np.testing.assert_array_equal(np.concatenate(sig_parts, axis=1), lv[:, :n_sig])
    np.testing.assert_array_equal(np.concatenate(bkg_parts, axis=1), lv[:, n_sig:])


# ------------------------------------------------------------ wide bins (levels 12..15)
@pytest.mark.parametrize("levels", [12, 13, 15])
def test_binning_wide_levels_vs_oracle(levels):
    """binning_levels 12..15 (uint16 codes, sample.py:22-24): boundaries and
    codes bit-exact, f32 and f64 keys (levels 15 with f64 keys searches the
    boundary keys in global memory)."""
    rng = np.random.default_rng(levels)
    X = rng.standard_t(3, size=(120_000, 3))
    X[rng.random(X.shape) < 0.02] = np.nan
    X[:, 2] = np.round(X[:, 2] * 3)  # ties
    for arr in (X.astype(np.float32), X):
        b, c = gpu_bin(arr, levels)
        for j in range(X.shape[1]):
            ref_b = oracle.fit_boundaries(arr[:, j], levels)
            np.testing.assert_array_equal(b[j], ref_b)
            np.testing.assert_array_equal(c[j].astype(np.uint16), oracle.bin_codes(ref_b, arr[:, j]).astype(np.uint16))


@pytest.mark.parametrize("levels,nan", [(12, False), (15, True)])
def test_fit_wide_levels_vs_fixed_point_oracle(levels, nan):
    """Fits with 4096 / 32768 bins (global-atomic histograms, the chunked
    CPH split) exact against the fixed-point oracle."""
    X, y, w, _ = make_config("cfg2", n=30_000)
    X = X[:, :4].copy()
    if nan:
        X[np.random.default_rng(1).random(X.shape) < 0.03] = np.nan
    kw = dict(n_trees=4, depth=3, shrinkage=0.1, subsample=0.5, levels=levels, seed=2)
    forest = fit_forest(X, y, w, FitConfig(n_trees=4, depth=3, shrinkage=0.1, subsample=0.5, binning_levels=levels,
                                           seed=2), return_leaves=True)
    ref = oracle.fit_forest(X, y, w, fixed_point=True, record_leaves=True, **kw)
    np.testing.assert_array_equal(np.stack([b.boundaries for b in forest.binnings]), ref.boundaries)
    for t in range(4):
        tr = forest.trees[t]
        np.testing.assert_array_equal(tr.valid, ref.valid[t])
        np.testing.assert_array_equal(tr.feature, ref.feature[t])
        np.testing.assert_array_equal(tr.cut_bin, ref.cut_bin[t])
        np.testing.assert_array_equal(forest.fit_info["leaves"][t], ref.leaves[t].astype(np.uint16))
        np.testing.assert_allclose(tr.node_weight, ref.node_weight[t], rtol=1e-12, atol=1e-15)


# ------------------------------------------------------------------ host staging (csrc/bb_stage.cpp)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_predict_pipelined_host_rows_match_plain_copy(dtype, monkeypatch):
    """Pageable host rows go through the pinned-chunk pipeline (upload,
    kernels and read-back per row chunk); the result must be identical to the
    single plain copy (BB_NO_STAGING=1), including a ragged last chunk."""
    rng = np.random.default_rng(11)
    Xs = rng.normal(size=(20_000, 12))
    y = (Xs[:, 0] + 0.5 * Xs[:, 3] + rng.normal(size=20_000) > 0).astype(int)
    forest = fit_forest(Xs, y, None, FitConfig(n_trees=20, depth=3, binning_levels=6, seed=2))
    n = 1_300_003  # several chunks of 349,184 (f32) / 174,080 (f64) rows + a ragged tail
    X = rng.normal(size=(n, 12)).astype(dtype)
    X[rng.random(n) < 0.01, 5] = np.nan
    p1, F1 = predict_batch(forest, X, return_scores=True)
    p1b = predict_batch(forest, X)
    monkeypatch.setenv("BB_NO_STAGING", "1")
    p0, F0 = predict_batch(forest, X, return_scores=True)
    np.testing.assert_array_equal(F1, F0)
    np.testing.assert_array_equal(p1, p0)
    np.testing.assert_array_equal(p1b, p0)


def test_fit_staged_upload_matches_plain_copy(monkeypatch):
    """bb_fit uploads pageable rows/weights through the threaded pinned ring;
    the forest must not depend on the transfer path."""
    X, y, w, _ = make_config("cfg2", n=400_000)  # 400k x 40 f32 = 64 MB: 4 ring laps
    cfg = FitConfig(n_trees=5, depth=3, binning_levels=8, seed=3)
    a = fit_forest(X, y, w, cfg, return_scores=True)
    monkeypatch.setenv("BB_NO_STAGING", "1")
    b = fit_forest(X, y, w, cfg, return_scores=True)
    assert a.f0 == b.f0
    for ta, tb in zip(a.trees, b.trees):
        np.testing.assert_array_equal(ta.feature, tb.feature)
        np.testing.assert_array_equal(ta.cut_bin, tb.cut_bin)
        np.testing.assert_array_equal(ta.node_weight, tb.node_weight)
    np.testing.assert_array_equal(a.fit_info["scores"], b.fit_info["scores"])


# ------------------------------------------------------------------ u16 row-list histogram (k_hist_list16)
@pytest.mark.parametrize("levels,nan,d,depth", [(8, True, 37, 4), (9, False, 21, 5), (10, False, 16, 3),
                                                (10, True, 50, 4), (9, False, 100, 6),
                                                (8, False, 100, 4), (7, True, 70, 3)])  # u8 codes, > 64 features
def test_fit_list16_vs_fixed_point_oracle(levels, nan, d, depth, monkeypatch):
    """2-byte codes (256 bins with missing values, 512 and 1024 bins) run the
    16-feature-group row-list histogram: ragged last groups, with and without
    sibling subtraction, negative weights; exact against the fixed-point oracle
    and identical to the round-1 kernels (BB_LIST16=0)."""
    rng = np.random.default_rng(levels * 100 + d)
    n = 40_000
    X = rng.normal(size=(n, d)).astype(np.float32)
    X[:, 1] = np.round(X[:, 1] * 3) / 3  # ties
    y = (X[:, 0] - 0.7 * X[:, min(5, d - 1)] + rng.normal(size=n) > 0).astype(int)
    w = rng.exponential(size=n) * np.where(rng.random(n) < 0.1, -0.5, 1.0)
    if nan:
        X[rng.random(X.shape) < 0.04] = np.nan
    cfg = FitConfig(n_trees=5, depth=depth, shrinkage=0.2, subsample=0.5, binning_levels=levels, seed=4)
    forest = fit_forest(X, y, w, cfg, return_leaves=True)
    ref = oracle.fit_forest(X, y, w, fixed_point=True, record_leaves=True, n_trees=5, depth=depth, shrinkage=0.2,
                            subsample=0.5, levels=levels, seed=4)
    monkeypatch.setenv("BB_LIST16", "0")
    old = fit_forest(X, y, w, cfg, return_leaves=True)
    for t in range(5):
        tr = forest.trees[t]
        np.testing.assert_array_equal(tr.valid, ref.valid[t])
        np.testing.assert_array_equal(tr.feature, ref.feature[t])
        np.testing.assert_array_equal(tr.cut_bin, ref.cut_bin[t])
        np.testing.assert_array_equal(forest.fit_info["leaves"][t], ref.leaves[t].astype(np.uint16))
        np.testing.assert_allclose(tr.node_weight, ref.node_weight[t], rtol=1e-12, atol=1e-15)
        np.testing.assert_array_equal(tr.feature, old.trees[t].feature)
        np.testing.assert_array_equal(tr.cut_bin, old.trees[t].cut_bin)
        np.testing.assert_array_equal(tr.node_weight, old.trees[t].node_weight)


def test_predict_pinned_host_rows_bypass_staging():
    """Rows that are already pinned (cudaHostAlloc / torch pin_memory) are
    passed to the DMA engine directly; same result as pageable rows."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(21)
    Xs = rng.normal(size=(10_000, 8))
    y = (Xs[:, 0] - Xs[:, 2] + rng.normal(size=10_000) > 0).astype(int)
    forest = fit_forest(Xs, y, None, FitConfig(n_trees=10, depth=3, binning_levels=5, seed=9))
    n = 400_000  # 12.8 MB of float32 rows: above the staging threshold
    Xp = torch.empty((n, 8), dtype=torch.float32, pin_memory=True)
    X = Xp.numpy()
    X[:] = rng.normal(size=(n, 8)).astype(np.float32)
    p_pinned = predict_batch(forest, X)
    p_pageable = predict_batch(forest, X.copy())
    np.testing.assert_array_equal(p_pinned, p_pageable)
