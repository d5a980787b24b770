"""Generate golden fixtures by running the UNMODIFIED reference (binboost).

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/gen_golden.py [--big]

It imports ``binboost`` from /root/reference/pkg/src, runs it on seeded
inputs (datagen.py + small randomized cases in the style of the reference's
``tests/support.py:random_fit_sample``), and stores compact outputs under
tests/golden/.  Hooks record the per-tree subsample masks (sample.py:120-132),
the per-tree leaf ids (boosting.py:170-171) and a gain-margin audit of every
node (trees.py:170-204) without changing what the reference computes.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import binboost.boosting as bb  # noqa: E402
import binboost.trees as bt  # noqa: E402
from binboost.binning import bin_values, fit_binning  # noqa: E402
from binboost.boosting import FitConfig, predict_batch  # noqa: E402

from paper_1609_06119_b200.datagen import make_apply_forest, make_config  # noqa: E402


def sha(a) -> str:
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


class Recorder:
    """Wraps subsample / traverse_bins / find_best_cuts inside binboost.boosting
    and binboost.trees to observe (not alter) the fit."""

    def __init__(self):
        self.masks, self.leaves, self.audit = [], [], []
        self._pending = []
        self.tree = 0
        self._orig = (bb.subsample, bb.traverse_bins, bt.find_best_cuts)

    def __enter__(self):
        orig_sub, orig_trav, orig_find = self._orig
        rec = self

        def subsample(sample, rate, rng):
            orig_sub(sample, rate, rng)
            rec.masks.append(sha(np.concatenate([sample.signal.active, sample.background.active])))

        def traverse_bins(tree, bins):
            leaf = orig_trav(tree, bins)
            rec._pending.append(leaf)
            if len(rec._pending) == 2:
                rec.leaves.append(sha(np.concatenate(rec._pending).astype(np.int16)))
                rec._pending = []
                rec.tree += 1
            return leaf

        def find_best_cuts(hists, final_layer=False):
            cuts = orig_find(hists, final_layer)
            B = hists.n_bins
            cs, cb = hists.signal, hists.background
            ls, lb = cs[:, :, 1:B], cb[:, :, 1:B]
            rs, rb = cs[:, :, B:] - ls, cb[:, :, B:] - lb
            feas = ((ls + lb) > 0) & ((rs + rb) > 0)
            gains = bt._g_arr(ls, lb) + bt._g_arr(rs, rb) - bt._g_arr(ls + rs, lb + rb)
            scored = np.where(feas, gains, -np.inf).reshape(cs.shape[0], -1)
            start = cs.shape[0] - 1
            # node mass scale: sum over bins of |signal| + |background| weight
            # (per-bin masses from the cumulative histogram), max over features
            mass = np.abs(np.diff(cs[:, :, 1:], axis=2, prepend=0.0)).sum(axis=2) + \
                np.abs(np.diff(cb[:, :, 1:], axis=2, prepend=0.0)).sum(axis=2)
            for node in range(scored.shape[0]):
                fin = scored[node][np.isfinite(scored[node])]
                scale = float(np.max(mass[node])) if mass.shape[1] else 0.0
                if fin.size == 0:
                    rec.audit.append((rec.tree, start + node, math.inf, 0, math.nan, scale))
                    continue
                best = fin.max()
                below = fin[fin < best]
                gap = math.inf if below.size == 0 else (best - below.max()) / max(abs(best), 1e-300)
                pure = int(np.all(cb[node, :, B] == 0.0) and np.any(cs[node, :, B] != 0.0))
                rec.audit.append((rec.tree, start + node, float(gap), pure, float(best), scale))
            return cuts

        bb.subsample, bb.traverse_bins, bt.find_best_cuts = subsample, traverse_bins, find_best_cuts
        return self

    def __exit__(self, *exc):
        bb.subsample, bb.traverse_bins, bt.find_best_cuts = self._orig


def forest_arrays(forest):
    T = len(forest.trees)
    return dict(
        f0=np.float64(forest.f0),
        boundaries=np.stack([b.boundaries for b in forest.binnings]),
        feature=np.stack([t.feature for t in forest.trees]).astype(np.int32),
        cut_bin=np.stack([t.cut_bin for t in forest.trees]).astype(np.int32),
        threshold=np.stack([t.threshold for t in forest.trees]),
        gain=np.stack([t.gain for t in forest.trees]),
        valid=np.stack([t.valid for t in forest.trees]),
        node_weight=np.stack([t.node_weight for t in forest.trees]),
        node_purity=np.stack([t.node_purity for t in forest.trees]),
        n_trees=np.int64(T),
    )


def run_fit(X, y01, w, cfg: FitConfig, pred_rows):
    with Recorder() as rec:
        forest = bb.fit_forest(X, np.where(np.asarray(y01) > 0, 1, -1), w, cfg)
    arrs = forest_arrays(forest)
    arrs["mask_hashes"] = np.array(rec.masks)
    arrs["leaf_hashes"] = np.array(rec.leaves)
    # audit rows: tree, heap node, relative gap best vs runner-up distinct gain,
    # pure-signal flag, best gain, node absolute-mass scale
    arrs["audit"] = np.array(rec.audit, dtype=np.float64).reshape(-1, 6)
    arrs["pred_rows"] = pred_rows
    arrs["pred"] = predict_batch(forest, np.asarray(X, np.float64)[pred_rows])
    arrs["config"] = np.array([cfg.n_trees, cfg.depth, cfg.shrinkage, cfg.subsample, cfg.binning_levels, cfg.seed])
    return arrs


def small_case(rng):
    """Randomized tiny dataset in the spirit of tests/support.py:43-91:
    ties, NaN, +-inf, negative weights, varied levels/depth."""
    n = int(rng.integers(10, 400))
    d = int(rng.integers(1, 5))
    levels = int(rng.integers(1, 6))
    depth = int(rng.integers(1, 5))
    X = rng.normal(size=(n, d))
    for j in range(d):
        if rng.random() < 0.4:
            X[:, j] = np.round(X[:, j] * 2) / 2
        X[rng.random(n) < 0.1, j] = np.nan
        inf = rng.random(n) < 0.05
        X[inf, j] = np.where(rng.random(inf.sum()) < 0.5, np.inf, -np.inf)
    if rng.random() < 0.2:
        X[:, 0] = np.nan  # all-missing column -> placeholder binning
    y = rng.integers(0, 2, n)
    y[0], y[1] = 1, 0
    w = None
    if rng.random() < 0.7:
        w = rng.uniform(0.2, 2.0, n)
        if rng.random() < 0.5:
            w[rng.random(n) < 0.1] *= -1.0
    cfg = FitConfig(n_trees=int(rng.integers(1, 12)), depth=depth, shrinkage=float(rng.uniform(0.05, 1.0)),
                    subsample=float(rng.uniform(0.3, 1.0)), binning_levels=levels, seed=int(rng.integers(0, 1000)))
    return X, y, w, cfg


def gen_binning(out):
    rng = np.random.default_rng(11)
    cols, levels, bounds, codes = [], [], [], []
    for i in range(40):
        n = int(rng.integers(1, 3000))
        col = rng.normal(size=n) * 10.0 ** int(rng.integers(-3, 4))
        if i % 3 == 0:
            col = np.round(col)
        if i % 4 == 0:
            col[rng.random(n) < 0.1] = np.nan
        if i % 5 == 0:
            col[rng.random(n) < 0.05] = np.inf
            col[rng.random(n) < 0.05] = -np.inf
        if not np.isfinite(col).any():
            col[0] = 1.5
        L = int(rng.integers(1, 11))
        b = fit_binning(col, L).boundaries
        cols.append(col)
        levels.append(L)
        bounds.append(b)
        codes.append(bin_values(fit_binning(col, L), col))
    np.savez_compressed(
        out,
        lengths=np.array([len(c) for c in cols]),
        values=np.concatenate(cols),
        levels=np.array(levels),
        bound_lengths=np.array([len(b) for b in bounds]),
        boundaries=np.concatenate(bounds),
        codes=np.concatenate(codes),
    )


def gen_kats(out):
    """Known-answer vectors from the reference tests / SPEC (recomputed by
    the reference here, not transcribed)."""
    k = {}
    k["bounds_1to8_L2"] = fit_binning(np.arange(1.0, 9.0), 2).boundaries.tolist()
    k["bounds_5555_L1"] = fit_binning(np.array([5.0, 5, 5, 5]), 1).boundaries.tolist()
    k["bounds_mixed_L1"] = fit_binning(np.array([1.0, 2, np.nan, np.inf, 3, 4]), 1).boundaries.tolist()
    fb = fit_binning(np.arange(1.0, 9.0), 2)
    probe = [2.9, float("nan"), float("inf"), float("-inf"), 3.0, 5.0, 7.0, 100.0]
    k["to_bin_probe"] = [None if math.isnan(v) else v for v in probe]
    k["to_bin_codes"] = bin_values(fb, np.array(probe)).tolist()
    k["gain_kats"] = [
        [1.0, 0.0, 0.0, 1.0, bt.separation_gain(1.0, 0.0, 0.0, 1.0)],
        [1.0, 1.0, 1.0, 1.0, bt.separation_gain(1.0, 1.0, 1.0, 1.0)],
        [2.0, 0.0, 0.0, 2.0, bt.separation_gain(2.0, 0.0, 0.0, 2.0)],
    ]
    with open(out, "w") as fh:
        json.dump(k, fh, indent=1)


def gen_masks(out):
    """numpy Generator(PCG64(seed)).permutation-driven subsample masks
    (the reference's own RNG path, sample.py:120-132) for the C++/CUDA mask
    generator's parity test."""
    from binboost.sample import subsample

    class Blk:
        def __init__(self, n):
            self.active = np.ones(n, bool)

        @property
        def n_events(self):
            return self.active.size

    class Smp:
        def __init__(self, a, b):
            self.signal, self.background = Blk(a), Blk(b)

        def blocks(self):
            return ((1, self.signal), (-1, self.background))

    cases = [(0, 50_000, 50_000, 0.5, 4), (7, 1, 2, 0.5, 3), (3, 1000, 17, 0.3, 5), (123, 300_000, 700_000, 0.5, 2),
             (9, 65_537, 131_071, 0.77, 3), (2**40 + 5, 2, 5, 1.0, 2), (42, 5, 100_000, 0.01, 2)]
    rec = []
    first_masks = {}
    for seed, a, b, rate, trees in cases:
        rng = np.random.Generator(np.random.PCG64(seed))
        smp = Smp(a, b)
        hashes = []
        for t in range(trees):
            subsample(smp, rate, rng)
            m = np.concatenate([smp.signal.active, smp.background.active])
            hashes.append(sha(m))
            if t == 0 and a + b <= 200_000:
                first_masks[f"{seed}_{a}_{b}"] = np.packbits(m)
        st = np.random.PCG64(seed).state["state"]
        rec.append(dict(seed=seed, n_sig=a, n_bkg=b, rate=rate, trees=trees, hashes=hashes,
                        state=str(st["state"]), inc=str(st["inc"])))
    with open(out, "w") as fh:
        json.dump(rec, fh, indent=1)
    np.savez_compressed(out.replace(".json", "_first.npz"), **first_masks)


def gen_model_doc():
    """A reference-written JSON model (model_io.py format v1) plus inputs and
    its predictions, for the format-interop tests."""
    from binboost.model_io import serialize_forest

    rng = np.random.default_rng(3)
    X = rng.normal(size=(2000, 4))
    X[rng.random(X.shape) < 0.05] = np.nan
    y = np.where(rng.random(2000) < 0.4, 1, -1)
    f = bb.fit_forest(X, y, None, FitConfig(n_trees=5, depth=3, binning_levels=4, seed=1))
    with open(os.path.join(HERE, "ref_model.json"), "w") as fh:
        fh.write(serialize_forest(f))
    np.savez_compressed(os.path.join(HERE, "ref_model_inputs.npz"), X=X[:300])
    np.save(os.path.join(HERE, "ref_model_pred.npy"), predict_batch(f, X[:300]))


def gen_huge(which):
    """Full-size / near-full-size reference runs (tens of minutes on one core).
    Only compact outputs are stored: cuts, thresholds, node weights, per-tree
    leaf and mask hashes, the node audit and predictions on a row subset."""
    def slim(arrs):
        arrs.pop("node_purity", None)
        return arrs

    if "cfg2" in which:  # BASELINE configs[1] exactly: 1M rows x 40, 200 trees
        X, y, w, kw = make_config("cfg2")
        cfg = FitConfig(n_trees=200, depth=3, shrinkage=0.1, subsample=0.5, binning_levels=8, seed=0)
        np.savez_compressed(os.path.join(HERE, "cfg2_full_fit.npz"),
                            **slim(run_fit(X, y, w, cfg, np.arange(0, X.shape[0], 100))))
        print("cfg2 full done", flush=True)
    if "cfg3" in which:  # configs[2] at its full 10M rows, first 4 of 400 trees
        X, y, w, kw = make_config("cfg3")
        cfg = FitConfig(n_trees=4, depth=5, shrinkage=0.05, subsample=0.5, binning_levels=8, seed=0)
        np.savez_compressed(os.path.join(HERE, "cfg3_10M_prefix.npz"),
                            **slim(run_fit(X, y, w, cfg, np.arange(0, X.shape[0], 1000))))
        print("cfg3 prefix done", flush=True)
    if "cfg5" in which:  # configs[4] generator, 1M-row slice x 100 features, 1024 bins, depth 6
        X, y, w, kw = make_config("cfg5", n=1_000_000)
        cfg = FitConfig(n_trees=3, depth=6, shrinkage=0.1, subsample=0.5, binning_levels=10, seed=0)
        np.savez_compressed(os.path.join(HERE, "cfg5_1M_slice.npz"),
                            **slim(run_fit(X, y, w, cfg, np.arange(0, X.shape[0], 100))))
        print("cfg5 slice done", flush=True)
    if "cfg4" in which:  # configs[3]: the full 1000-tree depth-3 forest on the first 100k rows
        Xa, _, _, _ = make_config("cfg4", n=100_000)
        bnd = np.stack([fit_binning(Xa[:, j], 8).boundaries for j in range(Xa.shape[1])])
        feat, cut, thr, nw = make_apply_forest(bnd, n_trees=1000, depth=3, seed=1)
        forest = bb.Forest(
            f0=0.0,
            trees=[bt.Tree(depth=3, feature=feat[t], cut_bin=cut[t], threshold=thr[t], gain=np.zeros(7),
                           valid=np.ones(7, bool), node_weight=nw[t], node_purity=np.zeros(15)) for t in range(1000)],
            binnings=[fit_binning(Xa[:, j], 8) for j in range(Xa.shape[1])],
        )
        np.savez_compressed(os.path.join(HERE, "apply_cfg4_1000trees.npz"), boundaries=bnd,
                            pred=predict_batch(forest, Xa.astype(np.float64), threads=8))
        print("cfg4 forest done", flush=True)


def gen_analysis(out):
    """roc_auc on tied / weighted scores and a small elimination_importance
    run (analysis.py:45-70, 104-173) by the unmodified reference."""
    from binboost.analysis import elimination_importance, roc_auc

    rng = np.random.default_rng(17)
    arrs = {}
    for k, (n, ties, weighted) in enumerate([(1000, False, False), (5000, True, True), (20000, True, False),
                                            (777, False, True)]):
        s = rng.normal(size=n)
        if ties:
            s = np.round(s * 4) / 4
        lab = (rng.random(n) < 0.4).astype(np.int64)
        w = rng.uniform(0.1, 3.0, n) if weighted else None
        arrs[f"auc{k}_scores"] = s
        arrs[f"auc{k}_labels"] = lab
        if w is not None:
            arrs[f"auc{k}_w"] = w
        arrs[f"auc{k}_value"] = np.float64(roc_auc(s, lab, w))
    X, y, w, _ = make_config("cfg2", n=6000)
    X = X[:, [0, 5, 20, 25, 30, 35]]
    cfg = FitConfig(n_trees=12, depth=3, shrinkage=0.2, subsample=0.5, binning_levels=6, seed=9)
    rep = elimination_importance(X, y, w, cfg)
    arrs.update(elim_X=X, elim_y=y, elim_w=w, elim_scores=rep.scores, elim_order=np.array(rep.order),
                elim_step_aucs=np.array(rep.step_aucs), elim_n_fits=np.int64(rep.n_fits),
                elim_config=np.array([cfg.n_trees, cfg.depth, cfg.shrinkage, cfg.subsample, cfg.binning_levels,
                                      cfg.seed]))
    np.savez_compressed(out, **arrs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--analysis", action="store_true", help="only the roc_auc / elimination goldens")
    ap.add_argument("--big", action="store_true", help="also the cfg2 slice and cfg3 proxy (minutes)")
    ap.add_argument("--huge", nargs="*", default=None,
                    help="only the full-size runs: any of cfg2 cfg3 cfg4 cfg5 (default all; ~30 min)")
    args = ap.parse_args()
    if args.analysis:
        gen_analysis(os.path.join(HERE, "analysis.npz"))
        return
    if args.huge is not None:
        gen_huge(set(args.huge or ["cfg2", "cfg3", "cfg4", "cfg5"]))
        return

    gen_kats(os.path.join(HERE, "kats.json"))
    gen_binning(os.path.join(HERE, "binning_random.npz"))
    gen_masks(os.path.join(HERE, "masks.json"))
    gen_model_doc()

    rng = np.random.default_rng(2024)
    cases = {}
    for i in range(30):
        X, y, w, cfg = small_case(rng)
        arrs = run_fit(X, y, w, cfg, np.arange(X.shape[0]))
        arrs["X"] = X
        arrs["y"] = y
        if w is not None:
            arrs["w"] = w
        for key, v in arrs.items():
            cases[f"c{i}__{key}"] = v
    np.savez_compressed(os.path.join(HERE, "small_fits.npz"), **cases)

    X, y, w, kw = make_config("cfg1")
    cfg = FitConfig(n_trees=kw["trees"], depth=kw["depth"], shrinkage=kw["shrinkage"], subsample=kw["subsample"],
                    binning_levels=kw["binning_levels"], seed=kw["seed"])
    np.savez_compressed(os.path.join(HERE, "cfg1_fit.npz"), **run_fit(X, y, w, cfg, np.arange(0, X.shape[0], 20)))

    # cfg4-shaped apply slice: 100 trees over a 20k-row slice's boundaries
    Xa, _, _, _ = make_config("cfg4", n=20_000)
    bnd = np.stack([fit_binning(Xa[:, j], 8).boundaries for j in range(Xa.shape[1])])
    feat, cut, thr, nw = make_apply_forest(bnd, n_trees=100, depth=3, seed=1)
    forest = bb.Forest(
        f0=0.0,
        trees=[bt.Tree(depth=3, feature=feat[t], cut_bin=cut[t], threshold=thr[t], gain=np.zeros(7),
                       valid=np.ones(7, bool), node_weight=nw[t], node_purity=np.zeros(15)) for t in range(100)],
        binnings=[fit_binning(Xa[:, j], 8) for j in range(Xa.shape[1])],
    )
    np.savez_compressed(os.path.join(HERE, "apply_cfg4_slice.npz"), boundaries=bnd, feature=feat, cut_bin=cut,
                        threshold=thr, node_weight=nw, pred=predict_batch(forest, Xa.astype(np.float64)))

    if args.big:
        X, y, w, kw = make_config("cfg2", n=200_000)
        cfg = FitConfig(n_trees=30, depth=3, shrinkage=0.1, subsample=0.5, binning_levels=8, seed=0)
        np.savez_compressed(os.path.join(HERE, "cfg2_slice_fit.npz"), **run_fit(X, y, w, cfg, np.arange(0, X.shape[0], 50)))
        X, y, w, kw = make_config("cfg3", n=200_000)
        cfg = FitConfig(n_trees=150, depth=5, shrinkage=0.05, subsample=0.5, binning_levels=8, seed=0)
        np.savez_compressed(os.path.join(HERE, "cfg3_proxy_fit.npz"), **run_fit(X, y, w, cfg, np.arange(0, X.shape[0], 50)))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
