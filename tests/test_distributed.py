"""The N > 1 path on CPU: world_size-2 gloo processes run the event-sharded likelihood's
host logic (contiguous shards, all-gather of per-point Neumaier pairs, fixed rank-order
combine, global first-invalid index, extended term with the global N).  The per-rank
partial sums come from the oracle here (the GPU computes them on a B200); the exchange
and combine are the product's (paper_2003_12875_b200/distributed.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2003_12875_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 2048, 10_000_019):
        for world in (1, 2, 3, 8):
            spans = [D.shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_combine_is_fixed_order_and_compensated():
    rng = np.random.default_rng(0)
    pairs = np.zeros((4, 3, 2))
    pairs[:, :, 0] = rng.normal(1e7, 1e3, (4, 3))
    pairs[:, :, 1] = rng.normal(0, 1e-9, (4, 3))
    out = D.combine_pairs(pairs)
    import math
    for p in range(3):
        exact = math.fsum(list(pairs[:, p, 0]) + list(pairs[:, p, 1]))
        assert abs(out[p, 0] + out[p, 1] - exact) <= 1e-16 * abs(exact)
    assert np.array_equal(D.combine_pairs(pairs), out)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    from oracle.oracle import OracleModel
    from paper_2003_12875_b200 import configs

    w = configs.C4  # extended model: the extended term needs the global N
    o = OracleModel(w.text)
    n = 30_001
    cols, _ = o.sample(n, 7)
    pts = w.points(type("M", (), {"param_names": o.param_names, "theta": lambda self=None: o.theta.copy()}),
                   n_points=4)
    b, e = D.shard_bounds(n, world, rank)
    shard = [c[b:e] for c in cols]
    # local partial pairs: the oracle's Neumaier sum of this shard's events (no extended term)
    local = np.zeros((4, 2))
    bad = np.full(4, -1, dtype=np.int64)
    for p in range(4):
        _, comp, bi = o.nll(shard, pts[p])
        local[p] = (comp - o.extended_term(e - b, pts[p]), 0.0)
        bad[p] = bi
    t = torch.from_numpy(local)
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    tb = torch.from_numpy(bad)
    gb = [torch.zeros_like(tb) for _ in range(world)]
    dist.all_gather(gb, tb)
    offs = [D.shard_bounds(n, world, r)[0] for r in range(world)]
    combined = D.combine_pairs(np.stack([g.numpy() for g in gathered]))
    gbad = D.first_invalid_global(np.stack([g.numpy() for g in gb]), offs)
    ext = np.array([o.extended_term(n, pts[p]) for p in range(4)])
    vals = D.finalize(combined, gbad, ext)
    if rank == 0:
        full = np.array([o.nll(cols, pts[p])[1] for p in range(4)])
        q.put((vals, full))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_nll_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    vals, full = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.all(np.abs(vals - full) <= 1e-12 * np.abs(full))


def test_first_invalid_global_index():
    bad = np.array([[-1, 5], [3, -1]])
    assert list(D.first_invalid_global(bad, [0, 100])) == [103, 5]
    vals = D.finalize(np.zeros((2, 2)), np.array([-1, 7]), np.zeros(2))
    assert vals[0] == 0 and np.isinf(vals[1])
