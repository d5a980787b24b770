"""World-size-2 gloo test of the row-sharded fit's host logic (CPU).

Each rank takes its class-block shard (sharding.py), builds integer
fixed-point partial layer histograms over its rows with the oracle's exact
integer sums, and all-reduces them (int64 SUM); the result must equal the
single-process histogram bit-for-bit, so every rank takes the same cut —
the property the per-layer NCCL all-reduce relies on."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle.binboost_np import _exact_int_bincount
from paper_1609_06119_b200.sharding import slice_mask

N_SIG, N_BKG, D, L = 3001, 4999, 5, 4


def _data():
    rng = np.random.default_rng(17)
    codes_s = rng.integers(0, (1 << L) + 1, (N_SIG, D))
    codes_b = rng.integers(0, (1 << L) + 1, (N_BKG, D))
    q_s = rng.integers(0, 1 << 32, N_SIG)
    q_b = rng.integers(0, 1 << 32, N_BKG)
    node_s = rng.integers(3, 7, N_SIG)
    node_b = rng.integers(3, 7, N_BKG)
    rng2 = np.random.Generator(np.random.PCG64(5))
    ms, mb = oracle.subsample_masks(rng2, N_SIG, N_BKG, 0.5)
    return codes_s, codes_b, q_s, q_b, node_s, node_b, ms, mb


def _hist(codes, q, node, active, start=3, count=4):
    B1 = (1 << L) + 1
    out = np.zeros((count, D, B1), np.int64)
    sel = active & (node >= start)
    loc = node[sel] - start
    for j in range(D):
        out[:, j, :] = _exact_int_bincount(loc * B1 + codes[sel, j], q[sel], count * B1).reshape(count, B1)
    return out


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    codes_s, codes_b, q_s, q_b, node_s, node_b, ms, mb = _data()
    s0, s1 = N_SIG * rank // world, N_SIG * (rank + 1) // world
    b0, b1 = N_BKG * rank // world, N_BKG * (rank + 1) // world
    act = slice_mask(ms, mb, rank, world)
    n_s = s1 - s0
    hs = _hist(codes_s[s0:s1], q_s[s0:s1], node_s[s0:s1], act[:n_s])
    hb = _hist(codes_b[b0:b1], q_b[b0:b1], node_b[b0:b1], act[n_s:])
    t = torch.from_numpy(np.stack([hs, hb]))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    out_q.put((rank, t.numpy()))
    dist.destroy_process_group()


def test_sharded_histograms_allreduce_exact():
    codes_s, codes_b, q_s, q_b, node_s, node_b, ms, mb = _data()
    full = np.stack([_hist(codes_s, q_s, node_s, ms), _hist(codes_b, q_b, node_b, mb)])
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        np.testing.assert_array_equal(got[r], full)


def _prior_worker(rank, world, port, out_q):
    from paper_1609_06119_b200.distributed import _unique_id, sharded_prior
    from paper_1609_06119_b200.sharding import shard_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(4)
    y = (rng.random(10_001) < 0.3).astype(np.int8)
    w = rng.normal(1.0, 0.7, y.size)
    rows = shard_rows(y, rank, world)
    out_q.put((rank, sharded_prior(w[rows], y[rows]), _unique_id(dist, None)))
    dist.destroy_process_group()


def test_sharded_prior_and_unique_id_broadcast():
    """The sharded fit's host plumbing: the prior over the rank-ordered
    class blocks equals the single-process reference prior bit-for-bit, and
    every rank receives rank 0's 128-byte NCCL unique id."""
    import math

    rng = np.random.default_rng(4)
    y = (rng.random(10_001) < 0.3).astype(np.int8)
    w = rng.normal(1.0, 0.7, y.size)
    s, b = float(np.sum(w[y > 0])), float(np.sum(w[y <= 0]))
    want = 0.5 * math.log(s / b)  # boosting.py:76-83 over the global class blocks
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_prior_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        r, f0, uid = q.get(timeout=120)
        got[r] = (f0, uid)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0][0] == want and got[1][0] == want
    assert len(got[0][1]) == 128 and got[0][1] == got[1][1]


def _pairwise_worker(rank, world, port, sizes, out_q):
    from paper_1609_06119_b200.distributed import _agree, _global_pairwise

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = []
    for k, sz in enumerate(sizes):
        rng = np.random.default_rng(100 + k)
        full = rng.normal(size=sum(sz)) * 10.0 ** rng.integers(-3, 4, sum(sz))
        s0 = sum(sz[:rank])
        res.append(_global_pairwise(dist, None, full[s0:s0 + sz[rank]]))
    # a bad shard raises on EVERY rank (no rank left waiting in a collective)
    err = None
    try:
        _agree(dist, None, "weights shape (3,) does not match labels shape (4,)" if rank == 1 else None)
    except ValueError as e:
        err = str(e)
    out_q.put((rank, res, err))
    dist.destroy_process_group()


def test_global_pairwise_sum_and_rank_agreement():
    """The sharded prior's exchange: numpy's pairwise sum of the rank-ordered
    concatenation from per-rank leaf sums plus the <= 128-element heads and
    tails (leaves crossing shard boundaries, shards shorter than a leaf),
    bit-identical to np.sum; and argument errors agreed across ranks."""
    world = 3
    sizes = [(1000, 1000, 1000), (5, 300, 2), (127, 129, 1), (0, 4000, 77), (128, 128, 128), (3, 0, 0)]
    want = []
    for k, sz in enumerate(sizes):
        rng = np.random.default_rng(100 + k)
        full = rng.normal(size=sum(sz)) * 10.0 ** rng.integers(-3, 4, sum(sz))
        want.append(float(np.sum(full)))
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_pairwise_worker, args=(r, world, port, sizes, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        r, res, err = q.get(timeout=180)
        got[r] = (res, err)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert got[r][0] == want, r
        assert got[r][1] is not None and "does not match" in got[r][1]
