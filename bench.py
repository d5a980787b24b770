"""Benchmark of the FastBDT B200 hot path (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl b200|reference]

A step is one complete fit (binning + every tree, including the exact
subsample-mask generation) of a BASELINE workload on seeded synthetic data
(datagen.py).  The headline is cfg3 (BASELINE.json configs[2], the largest
single-GPU fit config: 10M rows x 50 fp32 features, 400 depth-5 trees, 256
bins); the metric is fit rows*trees/s.

- value: inputs resident in HBM; device time from CUDA events recorded on
  the library's stream around each fit (bb_fit), summed over the K timed
  steps, max over ranks.  L2 is flushed (256 MiB write) between steps; the
  cfg3 inputs (2 GB) exceed L2 anyway.
- e2e: the same fit through the public API (engine.fit_forest) on PAGEABLE
  numpy arrays, as binboost_bridge users pass them: host wall clock around
  the call, which uploads X, y, w and downloads the fitted forest.
- roofline: the layer-histogram kernel (k_hist_list on this config).
  Algorithmic bytes per launch = A*(d*b + 9) +
  nodes*d*B*16 with A = active rows; achieved = that / the kernel's mean
  launch time from CUDA events on the library stream during the timed
  steps.  traffic: null (the ncu dram bytes per launch are in profiles/).
- cpu_baseline / --impl reference: the oracle port (oracle/, a numpy
  restatement bit-identical to the unmodified reference) on this host, one
  core (the reference fit is single-threaded by design), on a bounded sample
  (binning + 1 tree on a row slice), scaled linearly to the full rows and
  trees.  The reference itself is pure Python and cannot travel to the GPU
  box; measured in the build container on the same sample the port is 1.12x
  the reference's speed at cfg3 and 0.77x at cfg2 (PORT_SPEEDUP below).
- apply: cfg4 (BASELINE configs[3]: 100M rows x 40, the 1000-tree depth-3
  forest of seed 1 over 256-bin equal-frequency boundaries of all rows) with
  its own e2e and a host-cores CPU baseline.

Multi-GPU (N > 1): one row-sharded fit of the whole workload (strong
scaling): rank g holds its class-block shard of the rows (sharding.py), the
library exchanges binning histograms, class counts, layer histograms and
node sums over NCCL; value = all rows x trees / the
max over ranks of the fit time.  The apply leg runs one replica per rank.
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

# oracle port vs the unmodified reference on the same 250k-row sample in the
# build container (binning + per-tree cost, scaled to the config's trees;
# DESIGN.md §Measurement): port rows*trees/s / reference rows*trees/s
PORT_SPEEDUP = {"cfg3": 1.12, "cfg2": 0.77}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-apply", action="store_true")
    ap.add_argument("--apply-rows", type=int, default=100_000_000, help="cfg4 rows for the apply leg")
    ap.add_argument("--cpu-rows", type=int, default=250_000, help="row slice of the CPU-baseline sample")
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


def host_cpu():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def fit_config(spec):
    from paper_1609_06119_b200 import FitConfig

    return FitConfig(n_trees=spec["trees"], depth=spec["depth"], shrinkage=spec["shrinkage"],
                     subsample=spec["subsample"], binning_levels=spec["binning_levels"], seed=spec["seed"])


def workload_config(name, spec, n, d, world):
    """The `config` dict both arms print (identical keys and values)."""
    return {"workload": f"{name} fit", "rows": n, "features": d, "trees": spec["trees"], "depth": spec["depth"],
            "bins": 1 << spec["binning_levels"], "subsample": spec["subsample"], "shrinkage": spec["shrinkage"],
            "parallelism": "single" if world == 1 else f"rows{world}",
            "l2": "inputs exceed L2; 256 MiB L2 flush between device steps"}


def hist_algorithmic_bytes(n_active, d, levels, depth):
    """per layer A*(d*b + 9) + nodes*d*B*16 (b = code bytes)."""
    B = 1 << levels
    b = 1 if B <= 256 else 2
    return sum(n_active * (d * b + 9) + (1 << (layer - 1)) * d * B * 16 for layer in range(1, depth + 1))


def cpu_fit_sample(name, spec, rows):
    """Oracle port on a row slice of the workload: (binning s, 1-tree s)."""
    import oracle
    from paper_1609_06119_b200.datagen import make_config

    X, y, w, _ = make_config(name, n=rows)
    kw = dict(depth=spec["depth"], shrinkage=spec["shrinkage"], subsample=spec["subsample"],
              levels=spec["binning_levels"], seed=spec["seed"], hash_leaves=False)
    t0 = time.perf_counter()
    oracle.fit_forest(X, y, w, n_trees=0, **kw)
    t1 = time.perf_counter()
    oracle.fit_forest(X, y, w, n_trees=1, **kw)
    t2 = time.perf_counter()
    t_bin = t1 - t0
    return t_bin, max(1e-9, (t2 - t1) - t_bin)


def cpu_fit_value(name, spec, n, rows):
    """rows*trees/s of the port scaled from the sample: binning and trees are
    linear in rows (the reference's own acceptance criterion for trees,
    tests/test_acceptance.py:106-127; binning sorts, n log n, is treated as
    linear), trees linear in T."""
    t_bin, t_tree = cpu_fit_sample(name, spec, rows)
    scale = n / rows
    T = spec["trees"]
    t_full = scale * (t_bin + T * t_tree)
    sample = (f"oracle port, 1 core: binning ({t_bin:.2f} s) + 1 tree ({t_tree:.3f} s) on the first {rows} rows, "
              f"scaled x{scale:.1f} rows and x{T} trees")
    return n * T / t_full, t_bin + t_tree, sample


def run_reference(args, rank, world):
    """--impl reference: the CPU arm (oracle port of the reference, DESIGN.md
    §Reference install) on the same config, metric and unit."""
    from paper_1609_06119_b200.datagen import CONFIGS

    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    spec = dict(CONFIGS[args.config])
    n, d = spec["n"], spec["d"]
    vals, secs = [], []
    sample = ""
    for i in range(args.warmup + args.steps):
        v, s, sample = cpu_fit_value(args.config, spec, n, args.cpu_rows)
        if i >= args.warmup:
            vals.append(v)
            secs.append(s)
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": "fit rows*trees/s", "value": value, "unit": "rows*trees/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(secs), "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.config, spec, n, d, world),
        "cpu_baseline": {"value": value, "unit": "rows*trees/s", "cores": 1, "kind": "port", "sample": sample,
                         "host_cpu": host_cpu(), "port_speedup_vs_reference": PORT_SPEEDUP.get(args.config)},
        "e2e": {"value": value, "unit": "rows*trees/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_apply(args, rank, world, local, torch, dist):
    """cfg4 apply leg: rows/s of predict over the 1000-tree depth-3 forest
    (BASELINE.json configs[3]) on datagen's seed-1 N(0,1) rows; boundaries =
    256-bin equal-frequency boundaries of all rows (GPU binning)."""
    import ctypes as C

    import oracle
    from paper_1609_06119_b200 import _lib
    from paper_1609_06119_b200.datagen import make_apply_forest, make_config
    from paper_1609_06119_b200.engine import FeatureBinning, Forest, Tree, predict_batch, predict_batch_device

    n, T = args.apply_rows, 1000
    X, _, _, _ = make_config("cfg4", n=n)
    d = X.shape[1]
    bnd = np.zeros((d, 255))
    _lib.check(_lib.lib().bb_bin(_lib.context(local), _lib.ptr(X), _lib.BB_F32, n, d, 8, _lib.ptr(bnd), None))
    feat, cut, thr, nw = make_apply_forest(bnd, n_trees=T, depth=3, seed=1)
    trees = [Tree(depth=3, feature=feat[t], cut_bin=cut[t], threshold=thr[t], gain=np.zeros(7),
                  valid=np.ones(7, bool), node_weight=nw[t], node_purity=np.zeros(15)) for t in range(T)]
    forest = Forest(f0=0.0, trees=trees, binnings=[FeatureBinning(bnd[j], 8) for j in range(d)])
    Xd = torch.from_numpy(X).cuda()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(max(1, args.warmup)):
        predict_batch_device(forest, Xd.data_ptr(), "float32", n, d, out.data_ptr(), device=local)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        predict_batch_device(forest, Xd.data_ptr(), "float32", n, d, out.data_ptr(), device=local)
        e1.record(stream)  # bb_predict returns after its own stream synchronises
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    tot = sum(ms)
    if dist is not None:
        t = torch.tensor([tot], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t.item())
    step_s = tot / args.steps / 1e3
    value = world * n / step_s
    peak, kind = measured_peak()
    alg = n * (4 * d + 8)
    del Xd, out
    torch.cuda.empty_cache()
    # e2e through the public API from pageable host rows (a 10M-row slice)
    ne = min(n, 10_000_000)
    Xh = np.ascontiguousarray(X[:ne])
    predict_batch(forest, Xh[:min(ne, 1_000_000)])  # warm-up through the same staged path (pinned ring allocated once per context)
    e2e_s = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        predict_batch(forest, Xh)
        e2e_s.append(time.perf_counter() - t0)
    res = {"metric": "apply rows/s", "value": value, "unit": "rows/s", "ms_per_step": tot / args.steps,
           "config": {"workload": "cfg4 apply", "rows": n, "features": d, "trees": T, "depth": 3,
                      "data": "datagen cfg4: N(0,1) float32, seed 1 (2^20-row chunks of jumped PCG64 streams)"},
           "roofline": {"bound": "issue", "kernel": "k_apply_d", "achieved": alg / step_s / 1e9, "peak": peak,
                        "peak_kind": kind, "unit": "GB/s", "frac": alg / step_s / 1e9 / peak,
                        "alg_bytes_per_launch": alg, "node_visits_per_s": n * T * 3 / step_s},
           "e2e": {"value": ne / statistics.mean(e2e_s), "unit": "rows/s", "rows": ne,
                   "h2d_bytes_per_step": int(Xh.nbytes), "d2h_bytes_per_step": int(ne * 8),
                   "timing": "host wall clock around predict_batch (pageable numpy input)"}}
    if rank == 0 and world == 1 and not args.no_cpu:
        # the port's predict_batch(threads=T_host) (boosting.py:196-219) on a row slice
        threads = min(32, os.cpu_count() or 1)
        rows = 50_000
        of = oracle.binboost_np.OracleForest(
            f0=0.0, levels=8, depth=3, shrinkage=1.0, boundaries=bnd, feature=feat, cut_bin=cut, threshold=thr,
            gain=np.zeros((T, 7)), valid=np.ones((T, 7), bool), node_weight=nw, node_purity=np.zeros((T, 15)))
        t0 = time.perf_counter()
        oracle.predict(of, X[:rows], threads=threads)
        tt = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.predict(of, X[:rows // 10], threads=1)
        t1 = (time.perf_counter() - t0) * 10
        res["cpu_baseline"] = {"value": rows / tt, "unit": "rows/s", "cores": threads, "kind": "port",
                               "sample": f"oracle port predict(threads={threads}) on {rows} cfg4 rows x 1000 trees",
                               "value_1thread": rows / t1, "host_cpu": host_cpu()}
    return res


def run_b200(args, rank, world, local):
    import torch

    from paper_1609_06119_b200.datagen import CONFIGS, make_config
    from paper_1609_06119_b200.engine import fit_forest, fit_forest_device

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")

    spec = dict(CONFIGS[args.config])
    cfg = fit_config(spec)
    X, y, w, _ = make_config(args.config)
    n, d = X.shape  # the workload's (global) rows
    T = spec["trees"]
    ctx, f0 = None, float("nan")
    if world > 1:
        # row-sharded fit: this rank's class-block shard
        from paper_1609_06119_b200.distributed import comm_context, sharded_prior
        from paper_1609_06119_b200.sharding import shard_rows

        rows = shard_rows(y, rank, world)
        X, y, w = np.ascontiguousarray(X[rows]), y[rows], (None if w is None else w[rows])
        ctx = comm_context(local)
        f0 = sharded_prior(w, (y > 0).astype(np.int8))
    n_loc = X.shape[0]
    Xd = torch.from_numpy(X).cuda()
    yd = torch.from_numpy((y > 0).astype(np.int8)).cuda()
    wd = torch.from_numpy(w).cuda() if w is not None else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    def device_fit(profile):
        if ctx is None:
            return fit_forest_device(Xd.data_ptr(), "float32", n_loc, d, yd.data_ptr(),
                                     None if wd is None else wd.data_ptr(), cfg, profile=profile, device=local)
        import ctypes as C

        from paper_1609_06119_b200 import _lib
        from paper_1609_06119_b200.engine import _fit_native

        return _fit_native(C.c_void_p(Xd.data_ptr()), _lib.BB_F32, True, n_loc, d, C.c_void_p(yd.data_ptr()), True,
                           None if wd is None else C.c_void_p(wd.data_ptr()), True, cfg, profile=profile,
                           device=local, ctx=ctx, f0_override=f0)

    for _ in range(args.warmup):
        device_fit(False)
    barrier()
    dev_ms, hist_ms, hist_launches, launches, wall = [], 0.0, 0, 0, []
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
        barrier()
    total_ms = sum(dev_ms)
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = n * T / (ms_per_step / 1e3)  # all rows of the workload (sharded across ranks)

    # roofline of the layer-histogram kernel
    n_active = int(cfg.subsample * int((y > 0).sum())) + int(cfg.subsample * int((y <= 0).sum()))  # this rank's
    per_launch_bytes = hist_algorithmic_bytes(n_active, d, spec["binning_levels"], spec["depth"]) / spec["depth"]
    avg_launch_ms = hist_ms / max(1, hist_launches)
    achieved = per_launch_bytes / (avg_launch_ms / 1e3) / 1e9 if avg_launch_ms > 0 else None
    peak, peak_kind = measured_peak()
    B_ = 1 << spec["binning_levels"]
    hist_kernel = ("k_hist_list" if B_ <= 256 and d <= 64 else "k_hist_list16" if 256 < B_ <= 1024 else
                   "k_layer_hist_w/g")
    del Xd, yd, wd
    torch.cuda.empty_cache()

    # e2e through the public API from pageable numpy arrays (host wall clock)
    e2e = None
    if not args.no_e2e:
        if world > 1:
            from paper_1609_06119_b200.distributed import fit_forest_sharded

            def api_fit():
                return fit_forest_sharded(X, y, w, cfg, device=local)
        else:
            def api_fit():
                return fit_forest(X, y, w, cfg)
        api_fit()  # warm
        barrier()
        e2e_s = []
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            api_fit()
            e2e_s.append(time.perf_counter() - t0)
        barrier()
        tot = sum(e2e_s)
        if dist is not None:
            t = torch.tensor([tot], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot = float(t.item())
        I, N = (1 << spec["depth"]) - 1, (1 << (spec["depth"] + 1)) - 1
        d2h = T * I * (4 + 4 + 1 + 8 + 8) + T * N * 16 + d * ((1 << spec["binning_levels"]) - 1) * 8
        e2e = {"value": n * T / (tot / args.steps), "unit": "rows*trees/s",
               "h2d_bytes_per_step": int(X.nbytes + y.nbytes + (0 if w is None else w.nbytes)),
               "d2h_bytes_per_step": int(d2h),
               "timing": "host wall clock around engine.fit_forest (pageable numpy inputs)" if world == 1 else
                         "host wall clock around distributed.fit_forest_sharded per rank (pageable), max over ranks"}

    apply = None if args.no_apply else run_apply(args, rank, world, local, torch, dist)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, _, sample = cpu_fit_value(args.config, spec, n, args.cpu_rows)
        cpu = {"value": v, "unit": "rows*trees/s", "cores": 1, "kind": "port", "sample": sample,
               "host_cpu": host_cpu(), "port_speedup_vs_reference": PORT_SPEEDUP.get(args.config)}

    if rank == 0:
        line = {
            "metric": "fit rows*trees/s", "value": value, "unit": "rows*trees/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "int64+f64",
            "data": "synthetic", "config": workload_config(args.config, spec, n, d, world),
            "roofline": {"bound": "hbm", "kernel": hist_kernel, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": None,
                         "alg_bytes_per_launch": per_launch_bytes, "avg_launch_ms": avg_launch_ms,
                         "hist_share_of_step": hist_ms / max(1e-9, sum(dev_ms))},
            "cpu_baseline": cpu,
            "apply": apply,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "breakdown_ms": {"wall_per_fit": 1e3 * statistics.mean(wall),
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
