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


def _spawn(target, world=2, timeout=300, args=()):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=timeout)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _oracle_partial(o, shard, n_local):
    """CPU stand-in for the GPU's per-rank launch: the oracle's Neumaier sum over this
    rank's events (no extended term) and its local first invalid event."""
    def partial(pts):
        pairs = np.zeros((len(pts), 2))
        bad = np.full(len(pts), -1, dtype=np.int64)
        for p, th in enumerate(pts):
            _, comp, bi = o.nll(shard, th)
            if bi >= 0:
                bad[p] = bi
            else:
                pairs[p] = (comp - o.extended_term(n_local, th), 0.0)
        return pairs, bad
    return partial


def _worker(rank, world, port, q, case):
    dist = _init(rank, world, port)
    import paper_2003_12875_b200 as fb
    from oracle.oracle import OracleModel
    from paper_2003_12875_b200 import configs

    w = configs.C4  # extended model: the extended term needs the global N
    m = fb.Model.from_string(w.text)
    o = OracleModel(w.text)
    n = 30_001
    cols, _ = o.sample(n, 7)
    if case == "invalid":
        cols[0][20_000] = np.nan  # non-finite data: invalid event (proj/src/eval.cpp:138-145)
        cols[0][25_000] = np.inf
    P = 600 if case == "many" else 4
    pts = w.points(m, n_points=P)
    b, e = D.shard_bounds(n, world, rank)
    shard = [c[b:e] for c in cols]
    snll = D.ShardedNll(m, None, n, b, dist, n_local=e - b, partial=_oracle_partial(o, shard, e - b))
    vals = snll.nll_points(pts)
    bad = snll.first_invalid.copy()
    if rank == 0:
        check = [0, P - 1] if P > 4 else list(range(P))
        full = [o.nll(cols, pts[p]) for p in check]
        q.put((vals[check], bad[check], np.array([f[1] for f in full]), np.array([f[2] for f in full]),
               snll.offsets))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["plain", "invalid", "many"])
def test_two_rank_gloo_sharded_nll_drives_the_product_class(case):
    """ShardedNll itself at world_size 2 over gloo: one all-gather of the packed
    [pairs | first-invalid] block per launch (600 points: two launches), rank-order combine,
    global first-invalid index, extended term with the global N -- equal to one process."""
    vals, bad, full, fbad, offsets = _spawn(_worker, args=(case,))
    assert offsets == [0, 15_000]
    assert np.array_equal(bad, fbad)
    if case == "invalid":
        assert np.all(bad == 20_000) and np.all(np.isinf(vals))
    else:
        assert np.all(bad == -1)
        assert np.all(np.abs(vals - full) <= 1e-12 * np.abs(full))


def _tiling_worker(rank, world, port, q):
    dist = _init(rank, world, port)
    import paper_2003_12875_b200 as fb
    from paper_2003_12875_b200 import configs
    m = fb.Model.from_string(configs.C1.text)
    try:
        D.ShardedNll(m, None, 100, 10 * rank, dist, n_local=10)  # rank 1 starts at 10, ends at 20: rows missing
        err = None
    except ValueError as e:
        err = str(e)
    if rank == 0:
        q.put(err)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_nll_checks_the_tiling_once():
    err = _spawn(_tiling_worker)
    assert err is not None and "n_total is 100" in err


def test_first_invalid_global_index():
    bad = np.array([[-1, 5], [3, -1]])
    assert list(D.first_invalid_global(bad, [0, 100])) == [103, 5]
    # the packed exchange block round trip (the C ABI's layout: pairs, then int64 indices)
    blocks = np.stack([D.pack(np.array([[1.0, 1e-17], [2.0, 0.0]]), np.array([-1, 5])),
                       D.pack(np.array([[3.0, 0.0], [4.0, 2e-17]]), np.array([3, -1]))])
    pairs, gbad = D.combine_packed(blocks, 2, 2, [0, 100])
    assert list(gbad) == [103, 5] and pairs[0, 0] == 4.0 and pairs[1, 1] == 2e-17
    vals = D.finalize(np.zeros((2, 2)), np.array([-1, 7]), np.zeros(2))
    assert vals[0] == 0 and np.isinf(vals[1])


def _c2_slots(o, names, coefs, cols_x, theta):
    """Numpy restatement of the gradient pass's slot sums for the C2 model (Gaussian m, s
    free; ArgusBG c free): slot 0 = sum -log p, A_c = sum leaf_c / p', B = sum coef dleaf / p,
    p' = p * 2^54 as on the device (the host finish applies 2^54-scaled coefficient
    derivatives)."""
    import math
    x = cols_x
    th = dict(zip(names, theta))
    g = np.exp(-(x - th["m"]) ** 2 / (2 * th["s"] ** 2))
    t = 1 - (x / th["m0"]) ** 2
    a = np.where(t > 0, x * np.sqrt(np.maximum(t, 0)) * np.exp(th["c"] * t), 0.0)
    p = coefs[0] * g + coefs[1] * a
    d = x - th["m"]
    rows = [
        -np.log(p),
        g / p / 2.0 ** 54,
        coefs[0] * g * d / th["s"] ** 2 / p,
        coefs[0] * g * d * d / th["s"] ** 3 / p,
        a / p / 2.0 ** 54,
        coefs[1] * a * np.where(t > 0, t, 0.0) / p,
    ]
    return np.array([[math.fsum(r), 0.0] for r in rows])


def _grad_worker(rank, world, port, q):
    dist = _init(rank, world, port)
    import paper_2003_12875_b200 as fb
    from oracle.oracle import OracleModel
    from paper_2003_12875_b200 import configs

    w = configs.C2
    m = fb.Model.from_string(w.text)
    o = OracleModel(w.text)
    n = 20_001
    cols, _ = o.sample(n, 3)
    th = w.points(m, n_points=2)[1]
    terms, _, _ = m.plan()
    coefs = m.point_constants(th)[[t["coff"] for t in terms]]
    assert fb.grad_slot_count(m) == 6
    b, e = D.shard_bounds(n, world, rank)

    def grad_partial(pts):  # CPU stand-in for the fused gradient pass on this shard
        return _c2_slots(o, m.param_names, coefs, cols[0][b:e], pts[0])[None], np.full(1, -1, dtype=np.int64)

    snll = D.ShardedNll(m, None, n, b, dist, n_local=e - b, grad_partial=grad_partial)
    vals, grads = snll.nll_grad(th[None])
    if rank == 0:
        q.put((vals, grads, th, cols[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_gradient():
    """Shard slot sums (numpy restatement), exchange over gloo, rank-order combine, the
    product's host finish with the global N: equal to the oracle NLL and its gradient."""
    import math

    from oracle.oracle import OracleModel
    from paper_2003_12875_b200 import configs
    vals, grads, th, x = _spawn(_grad_worker)
    o = OracleModel(configs.C2.text)
    _, comp, _ = o.nll([x], th)
    assert abs(vals[0] - comp) <= 1e-12 * abs(comp)
    import paper_2003_12875_b200 as fb
    names = fb.Model.from_string(configs.C2.text).param_names
    p0 = o.probabilities([x], th)
    for j, name in enumerate(names):
        if name in ("m0", "p"):
            assert grads[0, j] == 0.0
            continue
        h = 1e-4 * {"m": 0.09, "s": 0.009, "c": 99.0, "f": 1.0}[name]

        def P(dx):
            t = th.copy()
            t[j] += dx
            return o.probabilities([x], t)

        dl = (8 * (P(h) - P(-h)) - (P(2 * h) - P(-2 * h))) / (12 * h) / p0
        want = -math.fsum(dl)
        assert abs(grads[0, j] - want) <= 1e-8 * np.sum(np.abs(dl)), (name, grads[0, j], want)


def test_finalize_grad_marks_invalid_points():
    v, g = D.finalize_grad(np.array([1.0, 2.0]), np.ones((2, 3)), np.array([-1, 4]))
    assert v[0] == 1.0 and np.isinf(v[1])
    assert np.all(g[0] == 1.0) and np.all(np.isnan(g[1]))
