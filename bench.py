"""Benchmark of the FastBDT B200 hot path (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl b200|reference]

A step is one complete fit (binning + all trees, including the exact
subsample-mask generation) of the configured BASELINE workload — cfg2 by
default (BASELINE.json configs[1]: 1M rows x 40 fp32 features, 200 trees,
depth 3, 256 bins) on seeded synthetic data (datagen.py).  The metric is fit
rows*trees/s.

- value: inputs resident in HBM, device time from CUDA events recorded on
  the library's stream around each fit, summed over the K timed steps;
  max over ranks.  L2 is flushed (256 MiB write) between steps.
- e2e:   the same fit through the public API (engine.fit_forest) from pinned
  host arrays: H2D of X, y, w and the D2H of the fitted forest inside the
  timed region (device time from the library's own CUDA events).
- roofline: the level-wise histogram kernel (k_layer_hist), algorithmic
  bytes per launch = A_l*(d*b + 9) + nodes_l*d*B*16,
  averaged over the timed launches, / its CUDA-event duration.
- cpu_baseline / --impl reference: the oracle port (oracle/, a numpy
  restatement of the reference, bit-identical to it) timed on this host on
  a bounded sample (binning + 1 tree over the full rows), extrapolated to
  the full tree count.

Multi-GPU (N>1): every rank runs an independent full fit (replicas, weak
scaling); row-sharded fits with a per-layer NCCL allreduce are future work
(DESIGN.md §Multi-GPU).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-apply", action="store_true")
    ap.add_argument("--apply-rows", type=int, default=100_000_000, help="cfg4 rows for the apply leg")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        mask = 0
        for s in self.samples:
            mask |= s[2]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": [v for k, v in REASONS.items() if mask & k and v != "gpu_idle"], "samples": len(sm)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fit_kwargs(spec):
    from paper_1609_06119_b200 import FitConfig

    return FitConfig(n_trees=spec["trees"], depth=spec["depth"], shrinkage=spec["shrinkage"],
                     subsample=spec["subsample"], binning_levels=spec["binning_levels"], seed=spec["seed"])


def hist_algorithmic_bytes(n_active, d, levels, depth):
    """per layer A_l*(d*b + 9) + nodes_l*d*B*16 (b = code bytes)."""
    B = 1 << levels
    b = 1 if B <= 256 else 2
    tot = 0
    for layer in range(1, depth + 1):
        tot += n_active * (d * b + 9) + (1 << (layer - 1)) * d * B * 16
    return tot


def cpu_reference_step(X, y, w, spec, threads=1):
    """Oracle port: binning + 1 tree over the full rows; returns (bin_s, tree_s)."""
    import oracle

    t0 = time.perf_counter()
    oracle.fit_forest(X, y, w, n_trees=0, depth=spec["depth"], shrinkage=spec["shrinkage"],
                      subsample=spec["subsample"], levels=spec["binning_levels"], seed=spec["seed"],
                      hash_leaves=False)
    t1 = time.perf_counter()
    oracle.fit_forest(X, y, w, n_trees=1, depth=spec["depth"], shrinkage=spec["shrinkage"],
                      subsample=spec["subsample"], levels=spec["binning_levels"], seed=spec["seed"],
                      hash_leaves=False)
    t2 = time.perf_counter()
    t_bin = t1 - t0
    t_tree = max(1e-9, (t2 - t1) - t_bin)
    return t_bin, t_tree


def run_apply(args, rank, world, local, torch, dist):
    """cfg4 apply leg: rows/s of predict over a 1000-tree depth-3 forest
    (BASELINE.json configs[3]).  Rows ~ N(0,1) float32 generated on the
    device (seed 1); boundaries = 256-bin equal-frequency boundaries of the
    first 1M rows (GPU binning); forest from datagen.make_apply_forest."""
    import numpy as np

    from paper_1609_06119_b200 import _lib
    from paper_1609_06119_b200.datagen import make_apply_forest
    from paper_1609_06119_b200.engine import FeatureBinning, Forest, Tree, predict_batch, predict_batch_device

    n, d, T = args.apply_rows, 40, 1000
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    X = torch.randn((n, d), generator=g, device="cuda", dtype=torch.float32)
    head = X[: min(n, 1_000_000)].cpu().numpy()
    bnd = np.zeros((d, 255))
    codes = np.zeros((d, head.shape[0]), np.int16)
    _lib.check(_lib.lib().bb_bin(_lib.context(local), _lib.ptr(head), _lib.BB_F32, head.shape[0], d, 8,
                                 _lib.ptr(bnd), _lib.ptr(codes)))
    feat, cut, thr, nw = make_apply_forest(bnd, n_trees=T, depth=3, seed=1)
    trees = [Tree(depth=3, feature=feat[t], cut_bin=cut[t], threshold=thr[t], gain=np.zeros(7),
                  valid=np.ones(7, bool), node_weight=nw[t], node_purity=np.zeros(15)) for t in range(T)]
    forest = Forest(f0=0.0, trees=trees, binnings=[FeatureBinning(bnd[j], 8) for j in range(d)])
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(max(1, args.warmup)):
        predict_batch_device(forest, X.data_ptr(), "float32", n, d, out.data_ptr(), device=local)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        predict_batch_device(forest, X.data_ptr(), "float32", n, d, out.data_ptr(), device=local)
        e1.record(stream)  # bb_predict returns after its own stream synchronises
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    tot = sum(ms)
    if dist is not None:
        t = torch.tensor([tot], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t.item())
    value = world * n / (tot / args.steps / 1e3)
    peak, kind = measured_peak()
    alg = n * (4 * d + 8)
    achieved = alg / (tot / args.steps / 1e3) / 1e9
    visits = n * T * 3
    # e2e through the public API from pinned host memory on a 10M-row sample
    ne = min(n, 10_000_000)
    Xh = X[:ne].cpu().pin_memory().numpy()
    predict_batch(forest, Xh[:1000])
    e2e_ms = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        predict_batch(forest, Xh)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    del X, out
    torch.cuda.empty_cache()
    return {"metric": "apply rows/s", "value": value, "unit": "rows/s", "ms_per_step": tot / args.steps,
            "config": {"workload": "cfg4 apply", "rows": n, "features": d, "trees": T, "depth": 3,
                       "data": "synthetic N(0,1) float32 generated on device (seed 1)"},
            "roofline": {"bound": "issue", "kernel": "k_apply", "achieved": achieved, "peak": peak,
                         "peak_kind": kind, "unit": "GB/s", "frac": achieved / peak,
                         "alg_bytes_per_launch": alg, "node_visits_per_s": visits / (tot / args.steps / 1e3)},
            "e2e": {"value": ne / (statistics.mean(e2e_ms) / 1e3), "unit": "rows/s", "rows": ne,
                    "h2d_bytes_per_step": int(Xh.nbytes), "d2h_bytes_per_step": int(ne * 8),
                    "timing": "host wall clock around predict_batch (pinned input)"}}


def run_reference(args, rank, world):
    from paper_1609_06119_b200.datagen import CONFIGS, make_config

    if rank != 0:
        return
    spec = dict(CONFIGS[args.config])
    X, y, w, _ = make_config(args.config)
    n, T = X.shape[0], spec["trees"]
    vals = []
    for i in range(args.warmup + args.steps):
        t_bin, t_tree = cpu_reference_step(X, y, w, spec)
        if i >= args.warmup:
            vals.append((t_bin, t_tree))
    t_fit = [b + T * t for b, t in vals]
    value = n * T / statistics.mean(t_fit)
    sample = f"{args.config}: binning + 1 tree over all {n} rows per step, extrapolated to {T} trees"
    line = {
        "impl": "reference", "metric": "fit rows*trees/s", "value": value, "unit": "rows*trees/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(b + t for b, t in vals), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} fit", "rows": n, "features": X.shape[1], "trees": T,
                   "depth": spec["depth"], "bins": 1 << spec["binning_levels"]},
        "cpu_baseline": {"value": value, "unit": "rows*trees/s", "cores": 1, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "rows*trees/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args, rank, world, local):
    import torch

    from paper_1609_06119_b200 import _lib
    from paper_1609_06119_b200.datagen import CONFIGS, make_config
    from paper_1609_06119_b200.engine import fit_forest, fit_forest_device

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")

    spec = dict(CONFIGS[args.config])
    cfg = fit_kwargs(spec)
    X, y, w, _ = make_config(args.config)
    n, d = X.shape
    T = spec["trees"]
    Xd = torch.from_numpy(X).cuda()
    yd = torch.from_numpy(y.astype(np.int8)).cuda()
    wd = torch.from_numpy(w).cuda() if w is not None else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    def device_fit(profile):
        return fit_forest_device(Xd.data_ptr(), "float32", n, d, yd.data_ptr(),
                                 None if wd is None else wd.data_ptr(), cfg, profile=profile, device=local)

    for _ in range(args.warmup):
        device_fit(False)
    barrier()
    dev_ms, hist_ms, hist_launches, launches, mask_ms, wall = [], 0.0, 0, 0, [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f = device_fit(True)
            wall.append(time.perf_counter() - t0)
            tm = f.fit_info["timing_ms"]
            dev_ms.append(tm["device_total"])
            hist_ms += tm["hist_kernels"]
            hist_launches += f.fit_info["hist_launches"]
            launches += f.fit_info["kernel_launches"]
            mask_ms.append(tm["masks_host"])
        barrier()
    total_ms = sum(dev_ms)
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * n * T / (ms_per_step / 1e3)

    # roofline of the histogram kernel
    n_active = int(cfg.subsample * int((y > 0).sum())) + int(cfg.subsample * int((y <= 0).sum()))
    alg_bytes_fit = T * hist_algorithmic_bytes(n_active, d, spec["binning_levels"], spec["depth"])
    per_launch_bytes = alg_bytes_fit / (T * spec["depth"])
    avg_launch_ms = hist_ms / max(1, hist_launches)
    achieved = per_launch_bytes / (avg_launch_ms / 1e3) / 1e9 if avg_launch_ms > 0 else None
    peak, peak_kind = measured_peak()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"hist_traffic_{args.config}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # e2e through the public API from pinned host memory
    e2e = None
    if not args.no_e2e:
        Xp = torch.from_numpy(X).pin_memory().numpy()
        yp = torch.from_numpy(y.astype(np.int8)).pin_memory().numpy()
        wp = torch.from_numpy(w).pin_memory().numpy() if w is not None else None
        fit_forest(Xp, yp, wp, cfg)  # warm
        barrier()
        e2e_ms = []
        d2h = 0
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            f = fit_forest(Xp, yp, wp, cfg)
            e2e_ms.append(f.fit_info["timing_ms"]["device_total"])
            I, N = (1 << spec["depth"]) - 1, (1 << (spec["depth"] + 1)) - 1
            d2h = T * I * (4 + 4 + 1 + 8 + 8) + T * N * 16 + d * ((1 << spec["binning_levels"]) - 1) * 8 + 8 * n
        barrier()
        tot = sum(e2e_ms)
        if dist is not None:
            t = torch.tensor([tot], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot = float(t.item())
        e2e = {"value": world * n * T / (tot / args.steps / 1e3), "unit": "rows*trees/s",
               "h2d_bytes_per_step": int(X.nbytes + n + (0 if w is None else w.nbytes)),
               "d2h_bytes_per_step": int(d2h)}

    apply = None if args.no_apply else run_apply(args, rank, world, local, torch, dist)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        t_bin, t_tree = cpu_reference_step(X, y, w, spec)
        cpu = {"value": n * T / (t_bin + T * t_tree), "unit": "rows*trees/s", "cores": 1, "kind": "port",
               "sample": f"oracle port, binning ({t_bin:.2f} s) + 1 tree ({t_tree:.2f} s) over all {n} rows, "
                         f"extrapolated to {T} trees"}

    if rank == 0:
        line = {
            "metric": "fit rows*trees/s", "value": value, "unit": "rows*trees/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64", "data": "synthetic",
            "config": {"workload": f"{args.config} fit", "rows": n, "features": d, "trees": T,
                       "depth": spec["depth"], "bins": 1 << spec["binning_levels"], "subsample": spec["subsample"],
                       "parallelism": "single" if world == 1 else f"replicas{world}",
                       "l2": "flushed (256 MiB write) between steps"},
            "roofline": {"bound": "hbm", "kernel": "k_layer_hist", "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "alg_bytes_per_launch": per_launch_bytes, "avg_launch_ms": avg_launch_ms,
                         "hist_share_of_step": hist_ms / max(1e-9, total_ms)},
            "cpu_baseline": cpu,
            "apply": apply,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "breakdown_ms": {"mask_host_per_fit": statistics.mean(mask_ms), "wall_per_fit": 1e3 * statistics.mean(wall),
                             "device_per_fit": [round(x, 2) for x in dev_ms]},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world, local)


if __name__ == "__main__":
    main()
