"""Engine-level drop-in for the reference's ``binboost`` hot path.

Same names, argument meaning and error behaviour as the reference engine
(``/root/reference/pkg/src/binboost``):

- ``FitConfig``      boosting.py:36-57
- ``FeatureBinning`` binning.py:18-49
- ``Cut`` / ``Tree`` trees.py:43-91
- ``Forest``         boosting.py:60-73
- ``fit_forest``     boosting.py:117-173  -> C-ABI ``bb_fit`` (GPU)
- ``predict_batch``  boosting.py:196-219  -> C-ABI ``bb_predict`` (GPU)
- ``predict``        boosting.py:222-227

All arithmetic runs in the CUDA library; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = ["FitConfig", "FeatureBinning", "Cut", "Tree", "Forest", "fit_forest", "fit_forest_device",
           "predict_batch", "predict"]

WEIGHT_EPS = 1e-12  # trees.py:39-40


@dataclass(frozen=True)
class FitConfig:
    """Hyperparameters of one forest fit (boosting.py:36-57)."""

    n_trees: int = 100
    depth: int = 3
    shrinkage: float = 0.1
    subsample: float = 0.5
    binning_levels: int = 8
    seed: int = 0

    def __post_init__(self) -> None:
        if self.n_trees < 1:
            raise ValueError("n_trees must be >= 1")
        if self.depth < 1:
            raise ValueError("depth must be >= 1")
        if not 0.0 < self.shrinkage <= 1.0:
            raise ValueError("shrinkage must be in (0, 1]")
        if not 0.0 < self.subsample <= 1.0:
            raise ValueError("subsample must be in (0, 1]")
        if self.binning_levels < 1:
            raise ValueError("binning_levels must be >= 1")


@dataclass(frozen=True)
class FeatureBinning:
    """Bin boundaries for one feature (binning.py:18-49)."""

    boundaries: np.ndarray
    levels: int

    def __post_init__(self) -> None:
        if self.levels < 1:
            raise ValueError("levels must be a positive integer")
        bounds = np.asarray(self.boundaries, dtype=np.float64)
        object.__setattr__(self, "boundaries", bounds)
        if bounds.ndim != 1 or bounds.size != self.n_bins - 1:
            raise ValueError(
                f"expected {self.n_bins - 1} boundaries for {self.levels} levels, got {bounds.size}"
            )
        if not np.all(np.isfinite(bounds)):
            raise ValueError("boundaries must be finite")
        if np.any(np.diff(bounds) < 0):
            raise ValueError("boundaries must be non-decreasing")

    @property
    def n_bins(self) -> int:
        return 1 << self.levels


@dataclass
class Cut:
    """Best split of one node: go left iff bin <= cut_bin (trees.py:43-55)."""

    feature: int
    cut_bin: int
    threshold: float
    gain: float
    valid: bool

    @staticmethod
    def none() -> "Cut":
        return Cut(feature=-1, cut_bin=0, threshold=math.nan, gain=0.0, valid=False)


@dataclass
class Tree:
    """Heap-indexed tree (trees.py:58-91)."""

    depth: int
    feature: np.ndarray
    cut_bin: np.ndarray
    threshold: np.ndarray
    gain: np.ndarray
    valid: np.ndarray
    node_weight: np.ndarray
    node_purity: np.ndarray

    @property
    def n_internal(self) -> int:
        return (1 << self.depth) - 1

    @property
    def n_nodes(self) -> int:
        return (1 << (self.depth + 1)) - 1

    def cuts(self) -> list[Cut]:
        return [
            Cut(feature=int(self.feature[i]), cut_bin=int(self.cut_bin[i]), threshold=float(self.threshold[i]),
                gain=float(self.gain[i]), valid=bool(self.valid[i]))
            for i in range(self.n_internal)
        ]


@dataclass
class Forest:
    """A fitted model (boosting.py:60-73).  ``fit_info`` carries GPU-side
    diagnostics (fixed-point shift, timings, optional per-tree leaf ids)."""

    f0: float
    trees: list
    binnings: list
    shrinkage: float = 1.0
    config: FitConfig | None = None
    fit_info: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def n_features(self) -> int:
        return len(self.binnings)


def _as_features(X) -> tuple[np.ndarray, int]:
    arr = np.asarray(X)
    if arr.dtype == np.float32:
        return np.ascontiguousarray(arr), _lib.BB_F32
    return np.ascontiguousarray(arr, dtype=np.float64), _lib.BB_F64


def fit_forest(X, y, weights=None, config: FitConfig | None = None, *, forced_cuts=None,
               return_leaves: bool = False, return_scores: bool = False, profile: bool = False,
               host_masks: bool = False, device: int = 0) -> Forest:
    """Fit a boosted forest on raw rows (boosting.py:117-173) on the GPU.

    forced_cuts: optional {(tree, heap_node): (valid, feature, cut_bin)} for
    the teacher-forced parity protocol.
    return_leaves: record every tree's final node per row (class-block
    order) in ``forest.fit_info["leaves"]`` (T, n) uint16.
    """
    cfg = config or FitConfig()
    X, xdt = _as_features(X)
    if X.ndim != 2:
        raise ValueError("X must be 2-d (n_events, n_features)")
    n, d = X.shape
    y = np.asarray(y)
    # labels = where(y > 0, 1, -1) (boosting.py:142-144) as one boolean pass
    is_sig = y > 0
    n_pos = int(np.count_nonzero(is_sig))
    if not 0 < n_pos < is_sig.size:
        raise ValueError("training data must contain both classes")
    if y.shape != (n,):
        raise ValueError(f"y has shape {y.shape}, expected ({n},)")
    w = None
    if weights is not None:
        w = np.ascontiguousarray(weights, dtype=np.float64)
        if w.shape != (n,):
            raise ValueError(f"weights has shape {w.shape}, expected ({n},)")
        if not np.all(np.isfinite(w)):
            raise ValueError("user weights must be finite")
    if d == 0:
        raise ValueError("X must have at least one feature")
    y01 = np.ascontiguousarray(is_sig).view(np.int8)

    return _fit_native(X, xdt, False, n, d, y01, False, w, False, cfg, forced_cuts=forced_cuts,
                       return_leaves=return_leaves, return_scores=return_scores,
                       profile=int(profile) | (2 if host_masks else 0), device=device)


def fit_forest_device(x_ptr: int, x_dtype: str, n: int, d: int, y01_ptr: int, w_ptr: int | None,
                      config: FitConfig | None = None, *, profile: bool = False, device: int = 0) -> Forest:
    """fit_forest on inputs already resident in device memory (raw CUDA
    pointers, e.g. torch ``data_ptr()``): X row-major float32/float64,
    y01 int8 (>0 signal), w float64 or None.  Used by bench.py's HBM leg."""
    cfg = config or FitConfig()
    xdt = _lib.BB_F32 if x_dtype == "float32" else _lib.BB_F64
    return _fit_native(C.c_void_p(x_ptr), xdt, True, n, d, C.c_void_p(y01_ptr), True,
                       None if w_ptr is None else C.c_void_p(w_ptr), True, cfg, profile=profile, device=device)


def _fit_native(X, xdt, x_dev, n, d, y01, y_dev, w, w_dev, cfg, *, forced_cuts=None, return_leaves=False,
                return_scores=False, profile=False, device=0, ctx=None, f0_override=math.nan) -> Forest:
    def p(a):
        return a if (a is None or isinstance(a, C.c_void_p)) else _lib.ptr(a)

    L, D, T = cfg.binning_levels, cfg.depth, cfg.n_trees
    B, I, N = 1 << L, (1 << D) - 1, (1 << (D + 1)) - 1
    c = _lib.FitConfigC(n_trees=T, depth=D, binning_levels=L, flags=int(profile), shrinkage=cfg.shrinkage,
                        subsample=cfg.subsample, f0_override=f0_override, **_lib.pcg_config(cfg.seed))
    bounds = np.zeros((d, B - 1))
    feat = np.zeros((T, I), np.int32)
    cut = np.zeros((T, I), np.int32)
    valid = np.zeros((T, I), np.uint8)
    thr = np.zeros((T, I))
    gain = np.zeros((T, I))
    nw = np.zeros((T, N))
    pur = np.zeros((T, N))
    f0 = np.zeros(1)
    shift = np.zeros(1, np.int32)
    n_sig = np.zeros(1, np.int64)
    timing = np.zeros(16)
    leaves = np.zeros((T, n), np.uint16) if return_leaves else None
    scores = np.zeros(n) if return_scores else None
    out = _lib.FitOutC(*[_lib.ptr(a) for a in (bounds, feat, cut, valid, thr, gain, nw, pur, f0, shift, n_sig,
                                                 leaves, scores, timing)])
    forced_arr, n_forced = None, 0
    if forced_cuts:
        items = sorted(forced_cuts.items())
        forced_arr = (_lib.ForcedCutC * len(items))(
            *[_lib.ForcedCutC(int(t), int(nd), int(bool(v[0])), int(v[1]), int(v[2])) for (t, nd), v in items])
        n_forced = len(items)
    ctx = ctx or _lib.context(device)
    _lib.check(_lib.lib().bb_fit(ctx, p(X), xdt, int(x_dev), n, d, p(y01), int(y_dev), p(w), int(w_dev), C.byref(c),
                                 C.cast(forced_arr, C.c_void_p) if forced_arr is not None else None, n_forced,
                                 C.byref(out)))
    binnings = [FeatureBinning(boundaries=bounds[j].copy(), levels=L) for j in range(d)]
    trees = [
        Tree(depth=D, feature=feat[t].copy(), cut_bin=cut[t].copy(), threshold=thr[t].copy(), gain=gain[t].copy(),
             valid=valid[t].astype(bool), node_weight=nw[t].copy(), node_purity=pur[t].copy())
        for t in range(T)
    ]
    info = dict(fixed_shift=int(shift[0]), n_sig=int(n_sig[0]),
                timing_ms=dict(upload=timing[0], binning=timing[1], trees=timing[2], download=timing[3],
                               total=timing[4], device_total=timing[5], hist_kernels=timing[6],
                               masks_host=timing[9]),
                hist_launches=int(timing[7]), kernel_launches=int(timing[8]))
    if return_leaves:
        info["leaves"] = leaves
    if return_scores:
        info["scores"] = scores
    return Forest(f0=float(f0[0]), trees=trees, binnings=binnings, shrinkage=cfg.shrinkage, config=cfg,
                  fit_info=info)


def _pad(a: np.ndarray, size: int, fill) -> np.ndarray:
    out = np.full(size, fill, dtype=a.dtype)
    out[: a.shape[0]] = a
    return out


def _forest_struct(forest: Forest):
    """Packs the forest for bb_predict.  Trees of a mixed-depth forest (the
    model format allows it, model_io.py:185-191) are padded to the deepest
    tree: a shallow tree's leaves become invalid internal nodes, where the
    traversal stops (trees.py:333-346), so its predictions are unchanged."""
    T = len(forest.trees)
    depth = max(t.depth for t in forest.trees) if T else 1
    I, N = (1 << depth) - 1, (1 << (depth + 1)) - 1
    if T:
        for k, t in enumerate(forest.trees):
            fv = np.asarray(t.feature)[np.asarray(t.valid, dtype=bool)]
            if fv.size and (fv.min() < 0 or fv.max() >= forest.n_features):
                raise ValueError(f"tree {k}: cut feature out of range for a model with {forest.n_features} features")
        feat = np.ascontiguousarray(np.stack([_pad(np.where(t.valid, t.feature, 0), I, 0) for t in forest.trees]),
                                    dtype=np.int32)
        valid = np.ascontiguousarray(np.stack([_pad(np.asarray(t.valid, dtype=np.uint8), I, 0) for t in forest.trees]),
                                     dtype=np.uint8)
        thr = np.ascontiguousarray(np.stack([_pad(np.asarray(t.threshold, dtype=np.float64), I, 0.0)
                                             for t in forest.trees]), dtype=np.float64)
        nw = np.ascontiguousarray(np.stack([_pad(np.asarray(t.node_weight, dtype=np.float64), N, 0.0)
                                            for t in forest.trees]), dtype=np.float64)
    else:
        feat = np.zeros((0, I), np.int32)
        valid = np.zeros((0, I), np.uint8)
        thr = np.zeros((0, I))
        nw = np.zeros((0, N))
    keep = (feat, valid, thr, nw)
    s = _lib.ForestC(n_trees=T, depth=depth, n_features=forest.n_features, reserved0=0, f0=float(forest.f0),
                     feature=_lib.ptr(feat), valid=_lib.ptr(valid), threshold=_lib.ptr(thr), node_weight=_lib.ptr(nw))
    return s, keep


def predict_batch(forest: Forest, X, threads: int = 1, *, return_scores: bool = False, device: int = 0):
    """Signal probabilities for a batch of raw rows (boosting.py:196-219).

    ``threads`` is accepted for API compatibility (the GPU kernel is
    row-parallel; results never depend on it)."""
    X, xdt = _as_features(X)
    if X.ndim != 2:
        raise ValueError("X must be 2-d (n_events, n_features)")
    if X.shape[1] != forest.n_features:
        raise ValueError(f"model expects {forest.n_features} features, rows have {X.shape[1]}")
    if X.shape[0] == 0:
        return (np.empty(0), np.empty(0)) if return_scores else np.empty(0)
    if threads < 1:
        raise ValueError("threads must be >= 1")
    s, keep = _forest_struct(forest)
    n = X.shape[0]
    p = np.empty(n)
    F = np.empty(n) if return_scores else None
    ctx = _lib.context(device)
    _lib.check(_lib.lib().bb_predict(ctx, C.byref(s), _lib.ptr(X), xdt, 0, n, X.shape[1], _lib.ptr(p), _lib.ptr(F), 0))
    del keep
    return (p, F) if return_scores else p


def predict_batch_device(forest: Forest, x_ptr: int, x_dtype: str, n: int, d: int, out_ptr: int, *,
                         scores_ptr: int | None = None, device: int = 0) -> None:
    """predict_batch on device-resident rows: X row-major float32/float64 at
    ``x_ptr``, probabilities written to the float64 device array ``out_ptr``."""
    if d != forest.n_features:
        raise ValueError(f"model expects {forest.n_features} features, rows have {d}")
    s, keep = _forest_struct(forest)
    xdt = _lib.BB_F32 if x_dtype == "float32" else _lib.BB_F64
    ctx = _lib.context(device)
    _lib.check(_lib.lib().bb_predict(ctx, C.byref(s), C.c_void_p(x_ptr), xdt, 1, n, d, C.c_void_p(out_ptr),
                                     None if scores_ptr is None else C.c_void_p(scores_ptr), 1))
    del keep


def predict(forest: Forest, row) -> float:
    """Signal probability of a single feature vector (boosting.py:222-227)."""
    row = np.asarray(row, dtype=np.float64)
    if row.ndim != 1:
        raise ValueError("row must be 1-d")
    return float(predict_batch(forest, row.reshape(1, -1))[0])
