"""The event-sharded likelihood behind the C ABI (ffcu_shard_group_*, csrc/shard.hpp).

This build has one GPU, so the groups here have one rank; the NCCL all-gather, the packed
[pairs | first-invalid] exchange buffer, the rank-order combine kernel and the host finish
with the global event count all run, and a one-rank group must reproduce the single-device
path BIT FOR BIT (the combine of one rank is exact).  The multi-rank host logic is covered
by the 2-rank gloo tests (tests/test_distributed.py)."""
import numpy as np
import pytest

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs
from oracle.oracle import OracleModel

pytestmark = pytest.mark.gpu


def _data(w, n, seed=None):
    m = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(m, n, w.data_seed if seed is None else seed)
    return m, cols


@pytest.mark.parametrize("w", [configs.C2, configs.C4, configs.C3], ids=lambda w: w.name)
def test_one_rank_groups_match_the_single_device_path_bitwise(w):
    torch = pytest.importorskip("torch")  # noqa: F841  (one NCCL in the process: torch's)
    m, cols = _data(w, 150_001)
    ds = fb.DataSet.from_columns(cols)
    pts = w.points(m, n_points=24)
    want, wbad, _ = fb.nll_points(m, ds, pts)
    loc = fb.ShardGroup.local(m, cols, [0])
    assert loc.info() == {"world": 1, "local_devices": 1, "n_total": 150_001, "local_rows": 150_001,
                          "local_offset": 0}
    got, bad, launches = loc.nll_points(pts)
    assert np.array_equal(got, want) and np.array_equal(bad, wbad) and launches >= 2
    rank = fb.ShardGroup.for_rank(m, ds, 150_001, 0, 1, 0)
    got2, bad2, _ = rank.nll_points(pts)
    assert np.array_equal(got2, want) and np.array_equal(bad2, wbad)
    # one point (the streaming kernel) and more points than one launch holds
    one, _, _ = rank.nll_points(pts[:1])
    assert one[0] == fb.nll_points(m, ds, pts[:1])[0][0]
    many = np.repeat(pts, 23, axis=0)[:530]
    gm, _, _ = loc.nll_points(many)
    assert np.array_equal(gm, fb.nll_points(m, ds, many)[0])
    # oracle parity of the group's values (extended term with the global N included)
    o = OracleModel(w.text)
    xs = [cols[k] for k in m.observables]
    for p in (0, 23):
        _, comp, ob = o.nll(xs, pts[p])
        assert bad[p] == ob == -1
        assert abs(got[p] - comp) <= 1e-12 * abs(comp)


def test_device_variant_and_first_invalid():
    torch = pytest.importorskip("torch")
    w = configs.C2
    m, cols = _data(w, 70_003)
    x = cols["x"].copy()
    x[5000] = 5.2905  # beyond m0 for the Argus component only: still valid (Gaussian > 0)
    ds = fb.DataSet.from_columns({"x": x})
    grp = fb.ShardGroup.for_rank(m, ds, len(x), 0, 1, 0)
    pts = w.points(m, n_points=12)
    P = len(pts)
    dev = torch.device("cuda", 0)
    d_sc = torch.empty((P, 2), dtype=torch.float64, device=dev)
    d_bad = torch.empty(P, dtype=torch.int64, device=dev)
    s = torch.cuda.Stream(device=dev)
    grp.nll_points_device(pts, d_sc.data_ptr(), d_bad.data_ptr(), s.cuda_stream)
    s.synchronize()
    sc, bad = fb.nll_points_partial(m, ds, pts)
    assert np.array_equal(d_sc.cpu().numpy().reshape(-1), np.asarray(sc).reshape(-1))
    assert np.all(d_bad.cpu().numpy() == -1) and np.all(np.asarray(bad) == -1)
    # an Argus-only model: p = 0 beyond m0 -> first invalid, global index
    argus = """
observable x 5.2 5.3
parameter m0 5.291 5.0 5.4 const
parameter c -20 -100 -1
parameter p 0.5 0 1 const
pdf a ArgusBG(x, m0, c, p)
"""
    ma = fb.Model.from_string(argus)
    xa = np.linspace(5.2, 5.28, 9001)
    xa[7777] = 5.295
    xa[8000] = 5.299
    dsa = fb.DataSet.from_columns({"x": xa})
    ga = fb.ShardGroup.for_rank(ma, dsa, len(xa), 0, 1, 0)
    v, b, _ = ga.nll_points(np.tile(ma.theta(), (3, 1)))
    assert np.all(b == 7777) and np.all(np.isinf(v))


def test_gradient_and_fits_through_the_group_bitwise():
    torch = pytest.importorskip("torch")  # noqa: F841
    w = configs.C5
    m, cols = _data(w, 400_000)
    ds = fb.DataSet.from_columns(cols)
    grp = fb.ShardGroup.for_rank(m, ds, 400_000, 0, 1, 0)
    pts = w.points(m, n_points=3)
    v1, g1, b1, _ = grp.nll_grad(pts)
    v2, g2, b2, _ = fb.nll_grad(m, ds, pts)
    assert np.array_equal(v1, v2) and np.array_equal(g1, g2) and np.array_equal(b1, b2)
    start = w.points(m, n_points=1, seed=w.point_seed)[0]
    for analytic in (False, True):
        mg = fb.Model.from_string(w.text)
        ms = fb.Model.from_string(w.text)
        for mm in (mg, ms):
            for name, val in zip(mm.param_names, start):
                if not mm.is_constant(name):
                    mm.set(name, val)
        ref = fb.fit_gradient(ms, ds, tolerance=1e-12, max_iterations=60, analytic=analytic)
        g = fb.ShardGroup.for_rank(mg, ds, 400_000, 0, 1, 0)
        got = g.fit_gradient(tolerance=1e-12, max_iterations=60, analytic=analytic)
        assert got.converged == ref.converged and got.iterations == ref.iterations
        assert got.nll_min == ref.nll_min
        for a, b in zip(got.parameters, ref.parameters):
            assert a.name == b.name and a.value == b.value and a.uncertainty == b.uncertainty
        assert [mg.get(n) for n in mg.param_names] == [ms.get(n) for n in ms.param_names]


def test_rank_groups_check_the_tiling():
    torch = pytest.importorskip("torch")  # noqa: F841
    m = fb.Model.from_string(configs.C1.text)
    ds = fb.DataSet.from_columns({"x": np.linspace(-5, 5, 1000)})
    with pytest.raises(fb.FfitError) as e:
        fb.ShardGroup.for_rank(m, ds, 1000, 5, 1, 0)  # a gap before the only shard
    assert e.value.code == 1
    with pytest.raises(fb.FfitError) as e:
        fb.ShardGroup.for_rank(m, ds, 1500, 0, 1, 0)  # rows missing
    assert e.value.code == 1
    with pytest.raises(fb.FfitError):
        fb.ShardGroup.for_rank(m, ds, 1000, 0, 1, 0, nccl_id=b"short")
    assert fb.ShardGroup.nccl_version().count(".") == 2
