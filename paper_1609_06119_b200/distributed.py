"""Row-sharded fit over NCCL: one process per GPU.

Every rank passes its own rows; the global training sample is the
concatenation of the ranks' rows in rank order, so the reference's class
blocks (sample.py:112-116) are rank 0's signal rows, rank 1's signal rows,
…, then the background rows in the same order.  ``sharding.shard_rows``
produces such a partition from one global array.

The library (bb_capi.cu, ``bb_ctx_init_comm``) then runs the whole fit with
four kinds of exchange, all on its own stream over the NCCL communicator:
binning (finite/NaN counts + one u32 radix histogram per select pass),
class counts (-> this rank's offsets in the global class blocks), the layer
histograms (int64 fixed-point, SUM — exact and order-free) and the final
node sums of each tree.  The subsample mask is drawn for the GLOBAL class
blocks (same PCG64 stream on every rank) and sliced to the local rows, so
the fitted forest is bit-identical to a single-device fit of the
concatenated rows, for any world size.

torch.distributed is the plumbing only: it carries the 128-byte NCCL unique
id from rank 0 and, for user weights, the per-class weight vectors needed to
reproduce the reference's prior exactly (``prior``, boosting.py:76-83).
"""

from __future__ import annotations

import ctypes as C
import math
import threading

import numpy as np

from . import _lib
from .engine import FitConfig, Forest, _as_features, _fit_native

__all__ = ["sharded_prior", "comm_context", "fit_forest_sharded", "fit_forest_virtual_shards"]

_comm_ctx: dict = {}
_comm_lock = threading.Lock()


def _dist():
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("fit_forest_sharded needs an initialised torch.distributed process group")
    return dist


def _pw_leaves(off: int, n: int, out: list) -> None:
    """numpy's pairwise-sum recursion (PW_BLOCKSIZE 128, 8-way unroll): the
    (offset, length) leaves in recursion order (bb_capi.cu pw_leaves)."""
    if n <= 128:
        out.append((off, n))
        return
    n2 = n // 2
    n2 -= n2 % 8
    _pw_leaves(off, n2, out)
    _pw_leaves(off + n2, n - n2, out)


def _leaf_sums(a: np.ndarray, leaves) -> np.ndarray:
    """numpy's sum of each <= 128-element leaf (8 accumulators, then the
    remainder in order), vectorised over leaves of equal length."""
    out = np.empty(len(leaves))
    by_len: dict = {}
    for k, (o, n) in enumerate(leaves):
        by_len.setdefault(n, []).append((k, o))
    for n, items in by_len.items():
        ks = np.array([k for k, _ in items])
        offs = np.array([o for _, o in items])
        blk = a[offs[:, None] + np.arange(n)[None, :]]
        if n < 8:
            res = np.zeros(len(items))
            for i in range(n):
                res = res + blk[:, i]
        else:
            r = blk[:, :8].copy()
            m = n - n % 8
            for i in range(8, m, 8):
                r += blk[:, i:i + 8]
            res = ((r[:, 0] + r[:, 1]) + (r[:, 2] + r[:, 3])) + ((r[:, 4] + r[:, 5]) + (r[:, 6] + r[:, 7]))
            for i in range(m, n):
                res = res + blk[:, i]
        out[ks] = res
    return out


def _pw_combine(n: int, leaf: np.ndarray, k: list) -> float:
    if n <= 128:
        v = float(leaf[k[0]])
        k[0] += 1
        return v
    n2 = n // 2
    n2 -= n2 % 8
    a = _pw_combine(n2, leaf, k)
    b = _pw_combine(n - n2, leaf, k)
    return a + b


def _global_pairwise(dist, group, a_local: np.ndarray) -> float:
    """np.sum (pairwise) of the concatenation of every rank's ``a_local`` in
    rank order, bit-exact, exchanging only each rank's <= 128-element head and
    tail and its sums of the recursion leaves that lie inside it (not the
    vectors: ~1/128 of the data)."""
    W = dist.get_world_size(group)
    info = [None] * W
    head, tail = a_local[:128].copy(), a_local[-128:].copy() if a_local.size else a_local[:0].copy()
    dist.all_gather_object(info, (int(a_local.size), head, tail), group=group)
    sizes = [x[0] for x in info]
    starts = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(starts[-1])
    if n == 0:
        return 0.0
    leaves = []
    _pw_leaves(0, n, leaves)
    me = dist.get_rank(group)
    s0, s1 = int(starts[me]), int(starts[me + 1])
    inside = [k for k, (o, m) in enumerate(leaves) if o >= s0 and o + m <= s1]
    mine = _leaf_sums(a_local, [(leaves[k][0] - s0, leaves[k][1]) for k in inside]) if inside else np.empty(0)
    parts = [None] * W
    dist.all_gather_object(parts, (inside, mine), group=group)
    leaf = np.full(len(leaves), np.nan)
    for ks, vs in parts:
        if len(ks):
            leaf[np.asarray(ks)] = vs
    # leaves crossing a rank boundary: every element is within 128 of a slice
    # end, so the gathered heads / tails hold it
    for k in np.flatnonzero(np.isnan(leaf)):
        o, m = leaves[k]
        vals = np.empty(m)
        for j in range(m):
            p = o + j
            r = int(np.searchsorted(starts, p, side="right") - 1)
            q = p - int(starts[r])
            h, t = info[r][1], info[r][2]
            vals[j] = h[q] if q < h.size else t[q - (sizes[r] - t.size)]
        leaf[k] = _leaf_sums(vals, [(0, m)])[0]
    return _pw_combine(n, leaf, [0])


def sharded_prior(w_local: np.ndarray | None, y01_local: np.ndarray, group=None) -> float:
    """The reference prior over the concatenated rows (boosting.py:76-83):
    0.5*log(sum w_sig / sum w_bkg) with numpy's pairwise sums taken over the
    GLOBAL class blocks in rank order, bit-identical to a single-process fit.
    NaN for unit weights: the library's exact count ratio is used then."""
    if w_local is None:
        return math.nan
    dist = _dist()
    sig = y01_local > 0
    w_sig = _global_pairwise(dist, group, np.ascontiguousarray(w_local[sig], dtype=np.float64))
    w_bkg = _global_pairwise(dist, group, np.ascontiguousarray(w_local[~sig], dtype=np.float64))
    if w_sig <= 0.0 or w_bkg <= 0.0:
        return 0.0
    return 0.5 * math.log(w_sig / w_bkg)


def _agree(dist, group, err: str | None) -> None:
    """Every rank validates its own rows, then all ranks learn whether any
    failed before the first collective of the fit, so a bad shard raises on
    every rank instead of leaving the others blocked in a collective."""
    flags = [None] * dist.get_world_size(group)
    dist.all_gather_object(flags, err, group=group)
    bad = [(r, e) for r, e in enumerate(flags) if e is not None]
    if bad:
        r, e = bad[0]
        raise ValueError(e if r == dist.get_rank(group) else f"rank {r} rejected its rows: {e}")


def _unique_id(dist, group) -> bytes:
    if dist.get_rank(group) == 0:
        import torch

        uid = bytes(torch.cuda.nccl.unique_id())
    else:
        uid = None
    box = [uid]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    if not isinstance(box[0], (bytes, bytearray)) or len(box[0]) != 128:
        raise RuntimeError("bad NCCL unique id from rank 0")
    return bytes(box[0])


def comm_context(device: int, group=None):
    """A library context bound to an NCCL communicator over ``group``
    (created once per (device, group); collective over the group)."""
    dist = _dist()
    key = (device, id(group))
    with _comm_lock:
        h = _comm_ctx.get(key)
        if h is not None:
            return h
    uid = _unique_id(dist, group)
    out = C.c_void_p()
    _lib.check(_lib.lib().bb_ctx_create(device, C.byref(out)))
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    _lib.check(_lib.lib().bb_ctx_init_comm(out, dist.get_rank(group), dist.get_world_size(group), buf))
    with _comm_lock:
        _comm_ctx[key] = out
    return out


def fit_forest_sharded(X, y, weights=None, config: FitConfig | None = None, *, group=None,
                       device: int | None = None, return_leaves: bool = False,
                       return_scores: bool = False) -> Forest:
    """fit_forest (boosting.py:117-173) over rows sharded across the ranks of
    ``group``: X/y/weights are THIS rank's rows.  Collective: every rank
    calls it with the same config; every rank gets the same Forest.
    ``fit_info['leaves'/'scores']`` cover the local rows (class-block order)."""
    dist = _dist()
    if device is None:
        import torch

        device = torch.cuda.current_device()
    cfg = config or FitConfig()
    err = None
    X, xdt = _as_features(X)
    n = d = 0
    y01 = w = None
    try:
        if X.ndim != 2:
            raise ValueError("X must be 2-d (n_events, n_features)")
        n, d = X.shape
        if n < 1:
            raise ValueError("every rank needs at least one row")
        y = np.asarray(y)
        if y.shape != (n,):
            raise ValueError(f"y has shape {y.shape}, expected ({n},)")
        y01 = np.ascontiguousarray(y > 0, dtype=np.int8)
        if weights is not None:
            w = np.ascontiguousarray(weights, dtype=np.float64)
            if w.shape != (n,):
                raise ValueError(f"weights has shape {w.shape}, expected ({n},)")
            if not np.all(np.isfinite(w)):
                raise ValueError("user weights must be finite")
    except ValueError as e:
        err = str(e)
    _agree(dist, group, err)
    f0 = sharded_prior(w, y01, group)
    ctx = comm_context(device, group)
    return _fit_native(X, xdt, False, n, d, y01, False, w, False, cfg, return_leaves=return_leaves,
                       return_scores=return_scores, device=device, ctx=ctx, f0_override=f0)


def fit_forest_virtual_shards(shards, config: FitConfig | None = None, *, device: int = 0,
                              return_leaves: bool = False) -> list:
    """The row-sharded fit with ``len(shards)`` shards in ONE process (and on
    one GPU): shard g = (X_g, y_g, w_g or None) is rank g's rows.  Each shard
    runs bb_fit in its own thread on its own context; the contexts share a
    virtual group whose all-reduces sum in host memory (bb_vgroup_*), so the
    library executes exactly the sharded code path (global binning from
    exchanged radix histograms, class offsets, global masks sliced to the
    local rows, per-layer histogram and node-sum reductions) without NCCL.
    Returns every shard's Forest (identical trees)."""
    cfg = config or FitConfig()
    G = len(shards)
    lib = _lib.lib()
    prep = []
    for X, y, w in shards:
        Xa, xdt = _as_features(X)
        y01 = np.ascontiguousarray(np.asarray(y) > 0, dtype=np.int8)
        wa = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
        prep.append((Xa, xdt, y01, wa))
    # the reference prior over the concatenated class blocks (boosting.py:76-83)
    f0 = math.nan
    if prep[0][3] is not None:
        ws = np.concatenate([p[3][p[2] > 0] for p in prep])
        wb = np.concatenate([p[3][p[2] <= 0] for p in prep])
        s_sig, s_bkg = float(np.sum(ws)), float(np.sum(wb))
        f0 = 0.0 if (s_sig <= 0.0 or s_bkg <= 0.0) else 0.5 * math.log(s_sig / s_bkg)
    grp = C.c_void_p()
    _lib.check(lib.bb_vgroup_create(G, C.byref(grp)))
    ctxs = []
    try:
        for g in range(G):
            h = C.c_void_p()
            _lib.check(lib.bb_ctx_create(device, C.byref(h)))
            ctxs.append(h)
            _lib.check(lib.bb_ctx_init_virtual(h, g, grp))
        out = [None] * G
        err = [None] * G

        def run(g):
            Xa, xdt, y01, wa = prep[g]
            try:
                out[g] = _fit_native(Xa, xdt, False, Xa.shape[0], Xa.shape[1], y01, False, wa, False, cfg,
                                     return_leaves=return_leaves, device=device, ctx=ctxs[g], f0_override=f0)
            except Exception as e:  # noqa: BLE001 - re-raised below
                err[g] = e

        th = [threading.Thread(target=run, args=(g,)) for g in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for e in err:
            if e is not None:
                raise e
        return out
    finally:
        for h in ctxs:
            lib.bb_ctx_destroy(h)
        lib.bb_vgroup_destroy(grp)
