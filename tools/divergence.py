"""Free-running divergence report: the GPU fit,
NOT teacher-forced, against the reference's recorded fit on the same seeded
input (tests/golden/*_fit.npz): first tree whose cuts differ (and the node's
audited best-vs-runner-up gain gap), max |dp| and the AUC difference on the
golden's prediction rows."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1609_06119_b200 import FitConfig, fit_forest, predict_batch
from paper_1609_06119_b200.analysis import roc_auc
from paper_1609_06119_b200.datagen import make_config

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
for name, fixture, n in [("cfg3", "cfg3_proxy_fit.npz", 200_000), ("cfg2", "cfg2_full_fit.npz", None),
                         ("cfg3", "cfg3_10M_prefix.npz", None), ("cfg1", "cfg1_fit.npz", None)]:
    g = np.load(os.path.join(G, fixture))
    X, y, w, _ = make_config(name, n=n)
    T, D, eta, alpha, L, seed = g["config"]
    cfg = FitConfig(n_trees=int(T), depth=int(D), shrinkage=float(eta), subsample=float(alpha),
                    binning_levels=int(L), seed=int(seed))
    f = fit_forest(X, y, w, cfg)
    first = None
    for t in range(int(T)):
        tr = f.trees[t]
        bad = np.flatnonzero((tr.valid != g["valid"][t]) | (tr.feature != g["feature"][t]) |
                             (tr.cut_bin != g["cut_bin"][t]))
        if bad.size:
            node = int(bad[0])
            aud = [a for a in g["audit"] if int(a[0]) == t and int(a[1]) == node]
            gap = float(aud[0][2]) if aud else float("nan")
            first = (t, node, gap)
            break
    # node weights / gains of the trees that agree: max relative error vs the
    # reference's float64 values (the GPU's come from fixed-point sums)
    t_end = int(T) if first is None else first[0]
    nw_err = g_err = 0.0
    for t in range(t_end):
        ref_nw = g["node_weight"][t]
        den = np.maximum(np.abs(ref_nw), 1e-300)
        ok = np.abs(ref_nw) > 1e-12
        if ok.any():
            nw_err = max(nw_err, float(np.max(np.abs(f.trees[t].node_weight - ref_nw)[ok] / den[ok])))
        if "gain" in g.files:
            ref_g = g["gain"][t]
            okg = np.asarray(f.trees[t].valid, bool) & np.isfinite(ref_g) & (np.abs(ref_g) > 1e-12)
            if okg.any():
                g_err = max(g_err, float(np.max(np.abs(f.trees[t].gain - ref_g)[okg] / np.abs(ref_g)[okg])))
    rows = g["pred_rows"]
    p = predict_batch(f, X[rows])
    lab = y[rows]
    wr = None if w is None else w[rows]
    d_auc = roc_auc(p, lab, wr) - roc_auc(g["pred"], lab, wr)
    print(f"{fixture}: {int(T)} trees free-running; first divergent "
          f"{'none' if first is None else f'tree {first[0]} node {first[1]} (reference gain gap {first[2]:.2e})'}; "
          f"max|dp| {np.max(np.abs(p - g['pred'])):.3e}; dAUC {d_auc:+.3e} on {rows.size} rows; "
          f"max rel err over {t_end} agreeing trees: node weight {nw_err:.2e}"
          f"{'' if 'gain' not in g.files else f', gain {g_err:.2e}'}", flush=True)
