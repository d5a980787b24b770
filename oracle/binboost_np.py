"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference hot path.

Restates, function by function, the algorithm of the reference package
``binboost`` (``/root/reference/pkg/src/binboost``; citations are
``file:line`` there).  Two accumulation modes:

``fixed_point=False`` (default)
    float64 arithmetic in the reference's exact operation order (per-slot
    sequential sums = ``np.bincount``, sequential ``np.cumsum``, the same
    gain expression), so results are bit-identical to the reference.
    Pinned by ``tests/test_oracle_golden.py`` against golden vectors the
    unmodified reference produced.

``fixed_point=True``
    the deterministic integer arithmetic the CUDA path uses (DESIGN.md
    §Fixed point): per-row effective weight and response are quantised to
    ``q = rint(x * 2**S)`` (int64) and every histogram / node sum is an exact
    integer sum, so GPU histograms and cuts are predicted exactly.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may use this module.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np
from scipy.special import expit

WEIGHT_EPS = 1e-12  # trees.py:39-40


# --------------------------------------------------------------------------
# binning  (binning.py)
# --------------------------------------------------------------------------

def fit_boundaries(values: np.ndarray, levels: int) -> np.ndarray:
    """Equal-frequency boundaries: sorted finite values at floor(k*M/B),
    k = 1..B-1 (binning.py:52-71).  An all-non-finite column gets the zero
    placeholder the engine uses (boosting.py:146-155)."""
    arr = np.asarray(values, dtype=np.float64).ravel()
    finite = arr[np.isfinite(arr)]
    n_bins = 1 << levels
    if finite.size == 0:
        return np.zeros(n_bins - 1)
    finite = np.sort(finite)
    idx = (np.arange(1, n_bins, dtype=np.int64) * finite.size) // n_bins
    return finite[idx]


def bin_codes(boundaries: np.ndarray, values: np.ndarray) -> np.ndarray:
    """1 + #{boundaries <= v}; NaN -> 0 (binning.py:74-79)."""
    arr = np.asarray(values, dtype=np.float64)
    out = np.searchsorted(boundaries, arr, side="right").astype(np.int64) + 1
    out[np.isnan(arr)] = 0
    return out


# --------------------------------------------------------------------------
# subsample  (sample.py:120-132, rng from boosting.py:162)
# --------------------------------------------------------------------------

def subsample_masks(rng: np.random.Generator, n_sig: int, n_bkg: int, rate: float):
    """Signal block then background block: first floor(rate*n) entries of
    rng.permutation(n) are active (sample.py:128-132)."""
    out = []
    for n in (n_sig, n_bkg):
        k = math.floor(rate * n)
        m = np.zeros(n, dtype=bool)
        m[rng.permutation(n)[:k]] = True
        out.append(m)
    return out[0], out[1]


# --------------------------------------------------------------------------
# fixed-point scale (DESIGN.md §Fixed point; mirrored by csrc/bb_fit.cpp)
# --------------------------------------------------------------------------

def fixed_point_shift(max_abs_w: float) -> int:
    """S = 32 - ceil(log2(max|w|)): |w*bw| * 2**S <= 2**32 since bw <= 1."""
    if not max_abs_w > 0.0:
        return 32
    m, e = math.frexp(max_abs_w)  # max_abs_w = m * 2**e, m in [0.5, 1)
    ceil_log2 = e - 1 if m == 0.5 else e
    return 32 - ceil_log2


def _exact_int_bincount(idx: np.ndarray, q: np.ndarray, minlength: int) -> np.ndarray:
    """Exact int64 per-slot sums via two float64 bincounts of 26-bit limbs."""
    q = q.astype(np.int64)
    lo = (q & ((1 << 26) - 1)).astype(np.float64)
    hi = (q >> 26).astype(np.float64)
    s_lo = np.bincount(idx, weights=lo, minlength=minlength)
    s_hi = np.bincount(idx, weights=hi, minlength=minlength)
    return (s_hi.astype(np.int64) << 26) + s_lo.astype(np.int64)


# --------------------------------------------------------------------------
# split search
# --------------------------------------------------------------------------

def _g_arr(s, b):
    """G(s,b) = s^2/(s+b) where s+b > 0 else 0 (trees.py:131-136)."""
    den = s + b
    out = np.zeros_like(den)
    ok = den > 0.0
    out[ok] = s[ok] * s[ok] / den[ok]
    return out


def _gains_float(cum_s, cum_b, n_bins):
    """Candidate gains exactly as find_best_cuts computes them
    (trees.py:181-193).  cum_*: (nodes, d, B+1) float64."""
    left_s = cum_s[:, :, 1:n_bins]
    left_b = cum_b[:, :, 1:n_bins]
    right_s = cum_s[:, :, n_bins:] - left_s
    right_b = cum_b[:, :, n_bins:] - left_b
    feasible = ((left_s + left_b) > 0) & ((right_s + right_b) > 0)
    gains = _g_arr(left_s, left_b) + _g_arr(right_s, right_b) - _g_arr(left_s + right_s, left_b + right_b)
    return np.where(feasible, gains, -np.inf)


def _g_fixed(s_q, b_q, scale):
    den_q = s_q + b_q
    out = np.zeros(den_q.shape)
    ok = den_q > 0
    s = s_q[ok].astype(np.float64) * scale
    den = den_q[ok].astype(np.float64) * scale
    out[ok] = (s * s) / den
    return out


def _gains_fixed(cum_s, cum_b, n_bins, scale):
    """Fixed-point gains, the definition csrc/bb_split.cu implements:
    integer left/right/total sums, each G term from exactly converted
    doubles, gain = (G_L + G_R) - G_T."""
    ls = cum_s[:, :, 1:n_bins]
    lb = cum_b[:, :, 1:n_bins]
    ts = np.broadcast_to(cum_s[:, :, n_bins:], ls.shape)
    tb = np.broadcast_to(cum_b[:, :, n_bins:], lb.shape)
    rs = ts - ls
    rb = tb - lb
    feasible = ((ls + lb) > 0) & ((rs + rb) > 0)
    gains = (_g_fixed(ls, lb, scale) + _g_fixed(rs, rb, scale)) - _g_fixed(ts, tb, scale)
    return np.where(feasible, gains, -np.inf)


def _pick_cuts(scored, n_bins, final_layer, forced_layer):
    """argmax over flat (feature, cut_bin-1), first max wins; valid iff
    g > 0 or (g == 0 and not final) (trees.py:193-204)."""
    nodes = scored.shape[0]
    flat = scored.reshape(nodes, -1)
    best = np.argmax(flat, axis=1)
    out = []
    for node in range(nodes):
        if node in forced_layer:
            ok, f, c = forced_layer[node]
            if ok:
                g = float(flat[node, f * (n_bins - 1) + (c - 1)])
                out.append((True, int(f), int(c), g))
            else:
                out.append((False, -1, 0, 0.0))
            continue
        g = float(flat[node, best[node]])
        if math.isfinite(g) and (g > 0.0 or (g == 0.0 and not final_layer)):
            f, c = divmod(int(best[node]), n_bins - 1)
            out.append((True, f, c + 1, g))
        else:
            out.append((False, -1, 0, 0.0))
    return out


def _audit_layer(scored, mass, cum_s_total, tree_i, start, mass_b_total):
    """Per node: best gain, runner-up DISTINCT gain, relative gap, pure-signal
    flag, node absolute-mass scale (SURVEY.md §7 hard part 2, §8(c)
    teacher-forced protocol)."""
    recs = []
    flat = scored.reshape(scored.shape[0], -1)
    for node in range(flat.shape[0]):
        row = flat[node]
        fin = row[np.isfinite(row)]
        scale = float(np.max(mass[node])) if mass.shape[1] else 0.0
        if fin.size == 0:
            recs.append(dict(tree=tree_i, node=start + node, best=None, second=None, gap=math.inf, pure_signal=False,
                             scale=scale))
            continue
        best = float(fin.max())
        below = fin[fin < best]
        second = float(below.max()) if below.size else None
        if second is None:
            gap = math.inf
        else:
            gap = (best - second) / max(abs(best), 1e-300)
        pure = bool(np.all(mass_b_total[node] == 0.0) and np.any(cum_s_total[node] != 0.0))
        recs.append(dict(tree=tree_i, node=start + node, best=best, second=second, gap=gap, pure_signal=pure,
                         scale=scale))
    return recs


# --------------------------------------------------------------------------
# forest
# --------------------------------------------------------------------------

@dataclass
class OracleForest:
    f0: float
    levels: int
    depth: int
    shrinkage: float
    boundaries: np.ndarray          # (d, B-1) float64
    feature: np.ndarray             # (T, 2^D-1) int32, -1 where invalid
    cut_bin: np.ndarray             # (T, 2^D-1) int32
    threshold: np.ndarray           # (T, 2^D-1) float64, NaN where invalid
    gain: np.ndarray                # (T, 2^D-1) float64
    valid: np.ndarray               # (T, 2^D-1) bool
    node_weight: np.ndarray         # (T, 2^(D+1)-1) float64, shrinkage applied
    node_purity: np.ndarray         # (T, 2^(D+1)-1) float64
    fixed_shift: int | None = None
    leaf_hashes: list = field(default_factory=list)
    leaves: list = field(default_factory=list)
    mask_hashes: list = field(default_factory=list)
    audit: list = field(default_factory=list)

    @property
    def n_trees(self) -> int:
        return self.feature.shape[0]


def _hash(arr: np.ndarray) -> str:
    return hashlib.sha1(np.ascontiguousarray(arr).tobytes()).hexdigest()


def fit_forest(
    X,
    y,
    weights=None,
    n_trees=100,
    depth=3,
    shrinkage=0.1,
    subsample=0.5,
    levels=8,
    seed=0,
    *,
    fixed_point=False,
    forced=None,
    record_leaves=False,
    hash_leaves=True,
    audit=False,
    masks=None,
):
    """Restatement of ``fit_forest`` (boosting.py:117-173) with ``fit_tree``
    (trees.py:247-315) inlined.

    forced: {(tree, node): (valid, feature, cut_bin)} overrides the argmax at
    those nodes (teacher-forced parity protocol).
    masks: optional list of (mask_sig, mask_bkg) per tree instead of the RNG.
    """
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2:
        raise ValueError("X must be 2-d (n_events, n_features)")
    y = np.asarray(y)
    labels = np.where(y > 0, 1, -1)  # boosting.py:142
    if not ((labels == 1).any() and (labels == -1).any()):
        raise ValueError("training data must contain both classes")
    n, d = X.shape
    B = 1 << levels
    width = B + 1
    forced = forced or {}

    bounds = np.stack([fit_boundaries(X[:, j], levels) for j in range(d)]) if d else np.zeros((0, B - 1))
    codes = np.empty((n, d), dtype=np.int64)
    for j in range(d):
        codes[:, j] = bin_codes(bounds[j], X[:, j])  # sample.py:109-110

    sig = labels > 0  # sample.py:112-114
    blocks_codes = [np.ascontiguousarray(codes[sig]), np.ascontiguousarray(codes[~sig])]
    w_all = np.ones(n) if weights is None else np.asarray(weights, dtype=np.float64)
    if w_all.shape != (n,):
        raise ValueError(f"weights has shape {w_all.shape}, expected ({n},)")
    if not np.all(np.isfinite(w_all)):
        raise ValueError("user weights must be finite")
    blocks_w = [w_all[sig].copy(), w_all[~sig].copy()]
    block_label = [1, -1]

    # prior (boosting.py:76-83): numpy pairwise sums of user weights
    w_sig = float(np.sum(blocks_w[0]))
    w_bkg = float(np.sum(blocks_w[1]))
    f0 = 0.0 if (w_sig <= 0.0 or w_bkg <= 0.0) else 0.5 * math.log(w_sig / w_bkg)
    scores = [np.full(len(blocks_w[0]), f0), np.full(len(blocks_w[1]), f0)]

    S = fixed_point_shift(float(np.max(np.abs(w_all)))) if fixed_point else None
    two_s = float(2.0 ** S) if fixed_point else None
    inv_two_s = float(2.0 ** -S) if fixed_point else None

    rng = np.random.Generator(np.random.PCG64(seed))
    n_int = (1 << depth) - 1
    n_nodes = (1 << (depth + 1)) - 1
    T = n_trees
    out = OracleForest(
        f0=f0, levels=levels, depth=depth, shrinkage=shrinkage, boundaries=bounds,
        feature=np.full((T, n_int), -1, np.int32), cut_bin=np.zeros((T, n_int), np.int32),
        threshold=np.full((T, n_int), np.nan), gain=np.zeros((T, n_int)),
        valid=np.zeros((T, n_int), bool), node_weight=np.zeros((T, n_nodes)),
        node_purity=np.zeros((T, n_nodes)), fixed_shift=S,
    )

    for t in range(T):
        # _refresh_responses (boosting.py:109-114)
        resid, bw = [], []
        for k in range(2):
            lab = block_label[k]
            r = 2.0 * lab * expit(-2.0 * lab * scores[k])
            a = np.abs(r)
            resid.append(r)
            bw.append(a * (2.0 - a))
        # subsample (sample.py:120-132)
        if masks is not None:
            active = [np.asarray(masks[t][0], bool), np.asarray(masks[t][1], bool)]
        else:
            active = list(subsample_masks(rng, len(blocks_w[0]), len(blocks_w[1]), subsample))
        out.mask_hashes.append(_hash(np.concatenate(active)))

        if fixed_point:
            q_eff = [np.where(active[k], np.rint(blocks_w[k] * bw[k] * two_s), 0.0).astype(np.int64) for k in range(2)]
            q_resp = [np.where(active[k], np.rint(blocks_w[k] * resid[k] * two_s), 0.0).astype(np.int64) for k in range(2)]

        node_index = [np.zeros(len(blocks_w[0]), np.int64), np.zeros(len(blocks_w[1]), np.int64)]
        eff_c = [np.zeros(n_nodes), np.zeros(n_nodes)]
        resp_c = [np.zeros(n_nodes), np.zeros(n_nodes)]
        eff_q = [np.zeros(n_nodes, np.int64), np.zeros(n_nodes, np.int64)]
        resp_q = [np.zeros(n_nodes, np.int64), np.zeros(n_nodes, np.int64)]

        for layer in range(1, depth + 2):  # fit_tree layer loop, trees.py:275-295
            start = (1 << (layer - 1)) - 1
            count = 1 << (layer - 1)
            at = [active[k] & (node_index[k] >= start) for k in range(2)]
            # _node_sums (trees.py:231-244)
            for k in range(2):
                local = node_index[k][at[k]] - start
                if fixed_point:
                    eff_q[k][start:start + count] = _exact_int_bincount(local, q_eff[k][at[k]], count)
                    resp_q[k][start:start + count] = _exact_int_bincount(local, q_resp[k][at[k]], count)
                else:
                    w = blocks_w[k][at[k]]
                    eff_c[k][start:start + count] = np.bincount(local, weights=w * bw[k][at[k]], minlength=count)
                    resp_c[k][start:start + count] = np.bincount(local, weights=w * resid[k][at[k]], minlength=count)
            if layer > depth:
                break
            # accumulate_layer_histograms (trees.py:139-167)
            hists = []
            for k in range(2):
                local = node_index[k][at[k]] - start
                rows = blocks_codes[k][at[k]]
                if fixed_point:
                    h = np.zeros((count, d, width), np.int64)
                    qe = q_eff[k][at[k]]
                    for j in range(d):
                        h[:, j, :] = _exact_int_bincount(local * width + rows[:, j], qe, count * width).reshape(count, width)
                else:
                    eff = blocks_w[k][at[k]] * bw[k][at[k]]
                    h = np.zeros((count, d, width))
                    for j in range(d):
                        h[:, j, :] = np.bincount(local * width + rows[:, j], weights=eff, minlength=count * width).reshape(count, width)
                h[:, :, 1:] = np.cumsum(h[:, :, 1:], axis=2)
                hists.append(h)
            final = layer == depth
            if fixed_point:
                scored = _gains_fixed(hists[0], hists[1], B, inv_two_s)
            else:
                scored = _gains_float(hists[0], hists[1], B)
            if audit and not fixed_point:
                mass = np.abs(np.diff(hists[0][:, :, 1:], axis=2, prepend=0.0)).sum(axis=2) + \
                    np.abs(np.diff(hists[1][:, :, 1:], axis=2, prepend=0.0)).sum(axis=2)
                out.audit.extend(_audit_layer(scored, mass, hists[0][:, :, B], t, start, hists[1][:, :, B]))
            forced_layer = {node - start: v for (tt, node), v in forced.items() if tt == t and start <= node < start + count}
            cuts = _pick_cuts(scored, B, final, forced_layer)
            for local_i, (ok, f, c, g) in enumerate(cuts):
                if not ok:
                    continue
                i = start + local_i
                out.feature[t, i] = f
                out.cut_bin[t, i] = c
                out.threshold[t, i] = float(bounds[f][c - 1])  # from_bin_cut, binning.py:87-98
                out.gain[t, i] = g
                out.valid[t, i] = True
            # advance_node_indices (trees.py:207-228)
            ok_arr = np.array([c[0] for c in cuts], bool)
            feat = np.array([c[1] if c[0] else 0 for c in cuts], np.int64)
            cbin = np.array([c[2] for c in cuts], np.int64)
            for k in range(2):
                rows_i = np.flatnonzero(at[k])
                if rows_i.size == 0:
                    continue
                node = node_index[k][rows_i]
                local = node - start
                b = blocks_codes[k][rows_i, feat[local]]
                move = ok_arr[local] & (b != 0)
                child = 2 * node + 1 + (b > cbin[local])
                node_index[k][rows_i] = np.where(move, child, node)

        # node weights / purity (trees.py:297-304), shrinkage (boosting.py:168)
        if fixed_point:
            den_q = eff_q[0] + eff_q[1]
            num_q = resp_q[0] + resp_q[1]
            den = den_q.astype(np.float64) * inv_two_s
            num = num_q.astype(np.float64) * inv_two_s
            es = eff_q[0].astype(np.float64) * inv_two_s
        else:
            den = eff_c[0] + eff_c[1]
            num = resp_c[0] + resp_c[1]
            es = eff_c[0]
        nw = np.zeros(n_nodes)
        ok = np.abs(den) >= WEIGHT_EPS
        nw[ok] = num[ok] / den[ok]
        pur = np.zeros(n_nodes)
        pok = den >= WEIGHT_EPS
        pur[pok] = es[pok] / den[pok]
        nw *= shrinkage
        out.node_weight[t] = nw
        out.node_purity[t] = pur

        # score update over ALL rows via traverse_bins (boosting.py:170-171, trees.py:318-330)
        leaves = []
        for k in range(2):
            leaf = _traverse_bins(out, t, blocks_codes[k])
            scores[k] = scores[k] + nw[leaf]
            leaves.append(leaf)
        if record_leaves:
            out.leaves.append(np.concatenate(leaves).astype(np.int16))
        if hash_leaves:
            out.leaf_hashes.append(_hash(np.concatenate(leaves).astype(np.int16)))
    return out


def _traverse_bins(forest: OracleForest, t: int, codes: np.ndarray) -> np.ndarray:
    """Final node of every row over bin codes (trees.py:318-330)."""
    n = codes.shape[0]
    node = np.zeros(n, np.int64)
    rows = np.arange(n)
    valid, feature, cut = forest.valid[t], forest.feature[t], forest.cut_bin[t]
    for _ in range(forest.depth):
        vld = valid[node]
        f = np.where(vld, feature[node], 0)
        b = codes[rows, f]
        move = vld & (b != 0)
        child = 2 * node + 1 + (b > cut[node])
        node = np.where(move, child, node)
    return node


def _traverse_values(valid, feature, threshold, depth, X):
    """Final node per raw row: right iff v >= threshold; NaN stops
    (trees.py:333-346)."""
    n = X.shape[0]
    node = np.zeros(n, np.int64)
    rows = np.arange(n)
    for _ in range(depth):
        vld = valid[node]
        f = np.where(vld, feature[node], 0)
        v = X[rows, f]
        move = vld & ~np.isnan(v)
        child = 2 * node + 1 + (v >= threshold[node]).astype(np.int64)
        node = np.where(move, child, node)
    return node


def predict_scores(f0, valid, feature, threshold, node_weight, depth, X) -> np.ndarray:
    """F = f0 + sum of node weights in tree order (boosting.py:185-189)."""
    X = np.asarray(X, dtype=np.float64)
    F = np.full(X.shape[0], float(f0))
    for t in range(valid.shape[0]):
        F += node_weight[t][_traverse_values(valid[t], feature[t], threshold[t], depth, X)]
    return F


def _sigmoid2(f: float) -> float:
    """Branch-stable sigmoid(2F) with scalar math.exp (boosting.py:176-182)."""
    if f >= 0.0:
        return 1.0 / (1.0 + math.exp(-2.0 * f))
    e = math.exp(2.0 * f)
    return e / (1.0 + e)


def predict(forest: OracleForest, X, threads: int = 1) -> np.ndarray:
    """Signal probabilities (predict_batch, boosting.py:196-219)."""
    X = np.asarray(X, dtype=np.float64)
    if X.shape[0] == 0:
        return np.empty(0)

    def chunk(rows):
        F = predict_scores(forest.f0, forest.valid, forest.feature, forest.threshold,
                           forest.node_weight, forest.depth, rows)
        return np.array([_sigmoid2(f) for f in F])

    if threads <= 1 or X.shape[0] < 2 * threads:
        return chunk(X)
    from concurrent.futures import ThreadPoolExecutor
    parts = np.array_split(X, threads)
    with ThreadPoolExecutor(max_workers=threads) as pool:
        return np.concatenate(list(pool.map(chunk, parts)))
