"""Seeded synthetic inputs for the five BASELINE configurations.

The paper's physics dataset is not available (no network), so the BASELINE
configs stand in for it.  Every generator draws from
``np.random.Generator(np.random.PCG64(seed))`` in a fixed call order, casts
features to float32, and returns ``(X, y01, weights_or_None, fit_kwargs)``.
``y01`` uses the binding's 0/1 label convention (reference
``pkg/bridge/src/binboost_bridge/__init__.py:45-47``).

``n`` may be overridden to produce a smaller slice with the same shape of
distribution (used by parity tests at oracle-friendly sizes).
"""

from __future__ import annotations

import numpy as np

__all__ = ["CONFIGS", "make_config", "make_apply_forest"]

# Fit hyper-parameters per config (BASELINE.json "configs").
CONFIGS = {
    "cfg1": dict(n=100_000, d=10, trees=100, depth=3, shrinkage=0.1, subsample=0.5, binning_levels=8, seed=0),
    "cfg2": dict(n=1_000_000, d=40, trees=200, depth=3, shrinkage=0.1, subsample=0.5, binning_levels=8, seed=0),
    "cfg3": dict(n=10_000_000, d=50, trees=400, depth=5, shrinkage=0.05, subsample=0.5, binning_levels=8, seed=0),
    "cfg4": dict(n=100_000_000, d=40, trees=1000, depth=3, binning_levels=8),
    "cfg5": dict(n=50_000_000, d=100, trees=500, depth=6, shrinkage=0.1, subsample=0.5, binning_levels=10, seed=0),
}


def _ar1_gaussian(rng, n, d, chunk=1 << 20):
    """Unit-variance AR(1) features, corr 0.5 between neighbours, float32."""
    X = np.empty((n, d), dtype=np.float32)
    c = np.sqrt(0.75)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        z = rng.standard_normal((hi - lo, d))
        for k in range(1, d):
            z[:, k] = 0.5 * z[:, k - 1] + c * z[:, k]
        X[lo:hi] = z
    return X


def _cfg1_like(seed, n, d):
    # cfg1/cfg3: exact 50/50 labels, AR(1) latent, signal shift 0.3*k/10
    # (literal reading of BASELINE.json configs[0]; recorded in DESIGN.md).
    rng = np.random.Generator(np.random.PCG64(seed))
    n_sig = n // 2
    y = rng.permutation(np.concatenate([np.ones(n_sig, np.int8), np.zeros(n - n_sig, np.int8)]))
    X = _ar1_gaussian(rng, n, d)
    shift = (0.3 * np.arange(d) / 10.0).astype(np.float32)
    X[y == 1] += shift
    return X, y, None


def _cfg2(seed, n):
    rng = np.random.Generator(np.random.PCG64(seed))
    y = (rng.random(n) < 0.3).astype(np.int8)
    X = np.empty((n, 40), dtype=np.float32)
    sig = y == 1
    g = rng.standard_normal((n, 20))
    g[sig] += 0.05 * (np.arange(20) + 1)
    X[:, :20] = g
    e = rng.exponential(1.0, (n, 10))
    e[sig] *= 1.0 / 0.8
    X[:, 20:30] = e
    X[:, 30:40] = rng.integers(0, 16, (n, 10)).astype(np.float32)
    w = rng.uniform(0.5, 1.5, n)
    return X, y, w


def _cfg4(seed, n, d=40, chunk=1 << 20, threads=None):
    """N(0,1) rows; chunk c of 2^20 rows comes from PCG64(seed) jumped c
    times (chunk 0 is the plain seed-1 stream), so the 100M-row apply set is
    generated in parallel and any prefix is reproducible on its own."""
    from concurrent.futures import ThreadPoolExecutor
    import os

    X = np.empty((n, d), dtype=np.float32)
    base = np.random.PCG64(seed)

    def fill(c):
        lo, hi = c * chunk, min(n, (c + 1) * chunk)
        X[lo:hi] = np.random.Generator(base.jumped(c) if c else np.random.PCG64(seed)).standard_normal((hi - lo, d))

    nc = (n + chunk - 1) // chunk
    with ThreadPoolExecutor(max_workers=threads or min(32, os.cpu_count() or 1)) as pool:
        list(pool.map(fill, range(nc)))
    return X, None, None


def _cfg5(seed, n, d=100, chunk=1 << 20):
    rng = np.random.Generator(np.random.PCG64(seed))
    y = (rng.random(n) < 0.4).astype(np.int8)
    w = rng.exponential(1.0, n)
    shifted = rng.choice(d, 30, replace=False)
    sigma = np.where(np.arange(d) < 50, np.sqrt(3.0), np.sqrt(1.25))
    shift = np.zeros(d)
    shift[shifted] = 0.2 * sigma[shifted]
    X = np.empty((n, d), dtype=np.float32)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        m = hi - lo
        t = rng.standard_t(3, (m, 50))
        comp = rng.random((m, 50)) < 0.5
        mix = np.where(comp, -1.0, 1.0) + 0.5 * rng.standard_normal((m, 50))
        blk = np.concatenate([t, mix], axis=1)
        blk += y[lo:hi, None] * shift[None, :]
        X[lo:hi] = blk
    return X, y, w


def make_config(name: str, n: int | None = None):
    """Return ``(X float32 (n,d), y01 int8 (n,), weights float64 or None, fit_kwargs)``."""
    spec = dict(CONFIGS[name])
    rows = spec.pop("n") if n is None else int(n)
    if n is not None:
        spec.pop("n")
    d = spec.pop("d")
    if name == "cfg1":
        X, y, w = _cfg1_like(0, rows, d)
    elif name == "cfg3":
        X, y, w = _cfg1_like(3, rows, d)
    elif name == "cfg2":
        X, y, w = _cfg2(2, rows)
    elif name == "cfg4":
        X, y, w = _cfg4(1, rows, d)
    elif name == "cfg5":
        X, y, w = _cfg5(5, rows, d)
    else:
        raise KeyError(name)
    return X, y, w, spec


def make_apply_forest(boundaries: np.ndarray, n_trees: int = 1000, depth: int = 3, seed: int = 1):
    """cfg4 forest: every internal node valid, feature
    uniform over the features, cut_bin uniform in 1..B-1, leaf weights
    U(-1, 1), internal weights 0, f0 = 0.  ``boundaries`` is (d, B-1).

    Returns plain arrays: feature (T, I) int32, cut_bin (T, I) int32,
    threshold (T, I) float64, node_weight (T, N) float64.
    """
    rng = np.random.Generator(np.random.PCG64(seed + 1000))
    d, bm1 = boundaries.shape
    n_int = (1 << depth) - 1
    n_nodes = (1 << (depth + 1)) - 1
    feature = rng.integers(0, d, (n_trees, n_int)).astype(np.int32)
    cut_bin = rng.integers(1, bm1 + 1, (n_trees, n_int)).astype(np.int32)
    threshold = boundaries[feature, cut_bin - 1]
    node_weight = np.zeros((n_trees, n_nodes))
    node_weight[:, n_int:] = rng.uniform(-1.0, 1.0, (n_trees, n_nodes - n_int))
    return feature, cut_bin, threshold, node_weight
