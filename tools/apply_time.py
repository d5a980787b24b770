"""Apply-leg timing only (bench.py's run_apply on cfg4): rows/s."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
a = argparse.Namespace(apply_rows=int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000, steps=3, warmup=2, no_e2e=True)
r = bench.run_apply(a, 0, 1, 0, torch, None)
print({k: r[k] for k in ("value", "ms_per_step")}, r["roofline"].get("node_visits_per_s"))
