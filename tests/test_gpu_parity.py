"""GPU parity of the fused sm_100a path, through the C ABI, against the oracle and the
reference's own golden vectors.

Tolerances (BASELINE.json north_star): per-event PDF values within 1e-13 relative;
|dNLL|/|NLL| <= 1e-12 against the compensated (Neumaier) oracle sum.
"""
import math
import os

import numpy as np
import pytest

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs
from paper_2003_12875_b200 import distributed as D
from oracle.oracle import OracleModel
from tests.models import ARGUS_OURS, EXPR_MODELS, MIX, REF_MODELS

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PER_EVENT = 1e-13
NLL_TOL = 1e-12


def rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.abs(np.asarray(b)))


def setup(text, n, seed):
    m = fb.Model.from_string(text)
    cols, _ = fb.sample_host(m, n, seed)
    ds = fb.DataSet.from_columns(cols)
    return m, ds, [cols[k] for k in m.observables], OracleModel(text)


# ------------------------------------------------------------------ golden vectors

@pytest.mark.parametrize("name", list(REF_MODELS))
def test_golden_reference_models(name):
    """GPU vs the REFERENCE's own per-event values and compensated NLL (golden)."""
    text, _ = REF_MODELS[name]
    g = np.load(os.path.join(GOLD, "ref_models.npz"))
    x, p, sc = g[f"{name}/x"], g[f"{name}/p"], g[f"{name}/scalars"]
    m = fb.Model.from_string(text)
    ds = fb.DataSet.from_columns({"x": x})
    assert rel(fb.probabilities(m, ds), p) <= PER_EVENT
    v = fb.nll(m, ds)
    assert abs(v.value - sc[1]) <= NLL_TOL * abs(sc[1])
    assert abs(v.value - sc[0]) <= NLL_TOL * abs(sc[0])  # the reference's naive nll() too
    assert v.first_invalid == -1


@pytest.mark.parametrize("name", list(EXPR_MODELS))
def test_golden_expression_route(name):
    """Restated kinds vs the reference's Expression + Simpson route (golden)."""
    _, ours, _, col = EXPR_MODELS[name]
    g = np.load(os.path.join(GOLD, "expr_models.npz"))
    x, p, sc = g[f"{name}/x"], g[f"{name}/p"], g[f"{name}/scalars"]
    m = fb.Model.from_string(ours)
    ds = fb.DataSet.from_columns({col: x})
    assert rel(fb.probabilities(m, ds), p) <= PER_EVENT
    assert abs(fb.nll(m, ds).value - sc[0]) <= NLL_TOL * abs(sc[0])


# ------------------------------------------------------------------ oracle parity

ALL = {**{k: v[0] for k, v in REF_MODELS.items()}, **{k: v[1] for k, v in EXPR_MODELS.items()},
       **{w.name: w.text for w in configs.BY_INDEX[:4]}}


@pytest.mark.parametrize("name", list(ALL))
def test_oracle_parity_per_event_and_nll(name):
    m, ds, cols, o = setup(ALL[name], 100_003, 12345)
    assert rel(fb.probabilities(m, ds), o.probabilities(cols)) <= PER_EVENT
    v = fb.nll(m, ds)
    _, comp, bad = o.nll(cols)
    assert v.first_invalid == bad == -1
    assert abs(v.value - comp) <= NLL_TOL * abs(comp)


@pytest.mark.parametrize("w", configs.BY_INDEX[:4], ids=lambda w: w.name)
def test_multi_point_launch_parity(w):
    m, ds, cols, o = setup(w.text, 200_000, w.data_seed)
    pts = w.points(m, n_points=min(w.n_points, 24))
    vals, bad, launches = fb.nll_points(m, ds, pts)
    assert launches == 2  # one fused kernel + one fixed-order fold, independent of N and P
    for p in range(len(pts)):
        _, comp, ob = o.nll(cols, pts[p])
        assert bad[p] == ob == -1
        assert abs(vals[p] - comp) <= NLL_TOL * abs(comp), p


def test_points_are_independent_of_batching():
    """A point's value does not depend on the other points of the launch: bitwise within a
    kernel (the tile kernel over 40 points or over 9 of them), and to the last bit of the
    compensated cross-tile sum between kernels (one point: the streaming kernel)."""
    w = configs.C2
    m, ds, _, _ = setup(w.text, 300_001, 7)
    pts = w.points(m, n_points=40)
    full, _, _ = fb.nll_points(m, ds, pts)
    for p in (0, 13, 31):
        nine, _, _ = fb.nll_points(m, ds, pts[p:p + 9])
        assert np.array_equal(nine, full[p:p + 9])
        one, _, _ = fb.nll_points(m, ds, pts[p:p + 1])
        assert abs(one[0] - full[p]) <= 2.5e-16 * abs(full[p])
    again, _, _ = fb.nll_points(m, ds, pts)
    assert np.array_equal(again, full)  # deterministic run to run


def test_launch_constant_cache_is_bit_identical():
    """ArgusBG with m0 (and p = 1/2) fixed over a launch's points is served by the
    per-tile launch-constant cache; more points without a majority m0 turn the cache
    off for that launch.  The shared points' values are bitwise equal either way, and
    match the oracle."""
    w = configs.C2
    m, ds, cols, o = setup(w.text, 150_007, 21)
    pts = w.points(m, n_points=16)
    j = m.param_names.index("m0")
    assert np.all(pts[:, j] == pts[0, j])
    cached, bad, _ = fb.nll_points(m, ds, pts)
    assert fb.last_launch_cached(m) == 1
    other = np.repeat(pts[:1], 17, axis=0)  # 17 more points, each with its own m0: no majority
    other[:, j] = pts[0, j] * (1 + 1e-4 * np.arange(1, 18))
    plain, _, _ = fb.nll_points(m, ds, np.vstack([pts, other]))
    assert fb.last_launch_cached(m) == 0
    assert np.array_equal(cached, plain[:16])
    for p in (0, 7, 15):
        _, comp, ob = o.nll(cols, pts[p])
        assert bad[p] == ob == -1
        assert abs(cached[p] - comp) <= NLL_TOL * abs(comp)
    # a ragged last tile, events at the range edge and at / beyond m0 (t <= 0: the
    # Argus component is 0 there, the Gaussian keeps p > 0)
    x = np.concatenate([cols[0][:5000], [pts[0, j], 5.2905, 5.29, 5.2]])
    ds2 = fb.DataSet.from_columns({"x": x})
    v2, b2, _ = fb.nll_points(m, ds2, pts)
    assert fb.last_launch_cached(m) == 1
    for p in (0, 9):
        _, comp, ob = o.nll([x], pts[p])
        assert b2[p] == ob == -1
        assert abs(v2[p] - comp) <= NLL_TOL * abs(comp)
    # an Argus-only model: t <= 0 gives p = 0, the first such event is reported
    text = """
observable x 5.2 5.29
parameter m0 5.28 5.0 5.4 const
parameter c -20 -100 0
parameter p 0.5 0 3 const
pdf bkg ArgusBG(x, m0, c, p)
"""
    ma, oa = fb.Model.from_string(text), OracleModel(text)
    xa = np.random.default_rng(2).uniform(5.2, 5.279, 9000)
    xa[7000] = 5.285
    pa = np.array([[5.28, -20.0 * (1 + 0.01 * i), 0.5] for i in range(12)])
    va, ba, _ = fb.nll_points(ma, fb.DataSet.from_columns({"x": xa}), pa)
    assert fb.last_launch_cached(ma) == 1
    for p in (0, 11):
        _, comp, ob = oa.nll([xa], pa[p])
        assert ba[p] == ob == 7000 and va[p] == comp == math.inf
    xa[7000] = 5.25
    va, ba, _ = fb.nll_points(ma, fb.DataSet.from_columns({"x": xa}), pa)
    for p in (0, 11):
        _, comp, ob = oa.nll([xa], pa[p])
        assert ba[p] == ob == -1 and abs(va[p] - comp) <= NLL_TOL * abs(comp)


@pytest.mark.parametrize("name", ["c4_yields_only", "c3_cheb_fixed"])
def test_launch_constant_whole_leaves(name):
    """Leaves whose shape parameters are all fixed over a launch (a yield-only fit of the
    config-4 mixture; config 3 with the Chebychev coefficients fixed) are evaluated once per
    staged tile; each point reads them back.  Bitwise equal to the uncached launch (one more
    point that moves every shape parameter) and to the oracle."""
    w = configs.C4 if name.startswith("c4") else configs.C3
    m, ds, cols, o = setup(w.text, 60_007, 41)
    base = m.theta()
    names = m.param_names
    if name.startswith("c4"):
        vary = [k for k, n in enumerate(names) if n.startswith("n")]   # yields only
        expect = 6
    else:
        vary = [k for k, n in enumerate(names) if not n.startswith("a")]  # everything but a1..a3
        expect = 1
    pts = np.tile(base, (12, 1))
    for p in range(12):
        for k in vary:
            pts[p, k] = base[k] * (1.0 + 1e-3 * (p - 6)) if base[k] != 0 else 1e-3 * (p - 6)
    cached, bad, _ = fb.nll_points(m, ds, pts)
    assert fb.last_launch_cached(m) == expect
    other = pts[:1].copy()
    for k in range(len(names)):
        if k not in vary and not m.is_constant(names[k]):
            other[0, k] = base[k] * (1 + 1e-4) if base[k] != 0 else 1e-4
    plain, _, _ = fb.nll_points(m, ds, np.vstack([pts, other]))
    assert fb.last_launch_cached(m) == 0
    assert np.array_equal(cached, plain[:12])
    for p in (0, 11):
        _, comp, ob = o.nll(cols, pts[p])
        assert bad[p] == ob == -1
        assert abs(cached[p] - comp) <= NLL_TOL * abs(comp)  # the oracle includes the extended term


def test_more_than_512_points_split_launches():
    w = configs.C1
    m, ds, cols, o = setup(w.text, 20_000, 3)
    pts = w.points(m, n_points=1100)
    vals, bad, launches = fb.nll_points(m, ds, pts)
    assert launches == 6
    for p in (0, 511, 512, 1099):
        assert abs(vals[p] - o.nll(cols, pts[p])[1]) <= NLL_TOL * abs(vals[p])


@pytest.mark.parametrize("n", [1, 2, 3, 255, 2047, 2048, 2049, 4095, 4097, 10007])
def test_tile_boundaries_and_ragged_tails(n):
    m, ds, cols, o = setup(ARGUS_OURS, n, 11)
    assert rel(fb.probabilities(m, ds), o.probabilities(cols)) <= PER_EVENT
    v = fb.nll(m, ds)
    assert abs(v.value - o.nll(cols)[1]) <= NLL_TOL * abs(o.nll(cols)[1])


def test_misaligned_device_view_uses_cooperative_staging():
    """A slice starting at an odd index is 8- but not 16-byte aligned: no bulk copy."""
    m, ds, cols, o = setup(MIX, 50_001, 5)
    for b, e in ((1, 50_001), (3, 40_000), (2048 + 1, 2048 * 5 + 3)):
        sub = ds.slice(b, e)
        v = fb.nll(m, sub)
        _, comp, _ = o.nll([cols[0][b:e]])
        assert abs(v.value - comp) <= NLL_TOL * abs(comp)


def test_empty_dataset():
    m = fb.Model.from_string(MIX)
    ds = fb.DataSet.from_columns({"x": np.zeros(0)})
    v = fb.nll(m, ds)
    assert v.value == 0.0 and v.n_entries == 0  # proj/tests/test_eval.cpp:92-100
    ext = fb.Model.from_string(configs.C4.text)
    th = ext.theta()
    nu = sum(th[ext.param_names.index(k)] for k in ("n1", "n2", "n3", "n4", "n5", "nb"))
    assert fb.nll(ext, ds).value == pytest.approx(nu, rel=1e-15)


def test_invalid_events_report_first_index():
    # ArgusBG is zero for x >= m0: events at the top of the range are invalid
    text = EXPR_MODELS["argus_only"][1].replace("parameter m0 5.291 5.0 5.4 const",
                                                 "parameter m0 5.285 5.0 5.4 const")
    m = fb.Model.from_string(text)
    o = OracleModel(text)
    rng = np.random.default_rng(1)
    x = rng.uniform(5.20, 5.284, 30000)
    x[17011] = 5.2875  # beyond m0
    x[23000] = 5.289
    ds = fb.DataSet.from_columns({"x": x})
    v = fb.nll(m, ds)
    _, comp, bad = o.nll([x])
    assert math.isinf(v.value) and v.first_invalid == bad
    # NaN data are invalid too (proj/src/eval.cpp:138-145)
    x2 = rng.uniform(5.20, 5.28, 5000)
    x2[4321] = np.nan
    v = fb.nll(m, fb.DataSet.from_columns({"x": x2}))
    assert math.isinf(v.value) and v.first_invalid == 4321


@pytest.mark.parametrize("kind", ["Chebychev", "Polynomial"])
@pytest.mark.parametrize("order", [0, 1, 2, 3, 4, 5, 7])
def test_polynomial_orders(kind, order):
    """Compile-time orders 1-4 and the run-time loop (0, >4) agree with the oracle."""
    coefs = [0.13, -0.07, 0.05, -0.03, 0.02, -0.011, 0.006][:order]
    params = "".join(f"parameter a{i} {a} -1 1\n" for i, a in enumerate(coefs))
    args = "".join(f", a{i}" for i in range(order))
    text = f"observable z -1 1\n{params}pdf q {kind}(z{args})\n"
    m = fb.Model.from_string(text)
    o = OracleModel(text)
    z = np.random.default_rng(order).uniform(-1, 1, 30000)
    ds = fb.DataSet.from_columns({"z": z})
    assert rel(fb.probabilities(m, ds), o.probabilities([z])) <= PER_EVENT
    assert abs(fb.nll(m, ds).value - o.nll([z])[1]) <= NLL_TOL * abs(o.nll([z])[1])


@pytest.mark.parametrize("p,c", [(0.7, -20.0), (0.5, -800.0), (0.5, 3.0), (1.3, 750.0)])
def test_argus_general_path(p, c):
    """ArgusBG off the fast domain (p != 1/2 or |c| > 700) runs the full kernel build
    (pow, range-checked exp) and Simpson normalisation on the host."""
    text = f"""
observable x 5.2 5.29
parameter m0 5.291 5.0 5.4 const
parameter c {c} -1000 1000
parameter p {p} 0 3
pdf bkg ArgusBG(x, m0, c, p)
"""
    m = fb.Model.from_string(text)
    o = OracleModel(text)
    x = np.random.default_rng(4).uniform(5.2, 5.2905, 20000)
    ds = fb.DataSet.from_columns({"x": x})
    assert rel(fb.probabilities(m, ds), o.probabilities([x])) <= PER_EVENT
    assert abs(fb.nll(m, ds).value - o.nll([x])[1]) <= NLL_TOL * abs(o.nll([x])[1])


def test_non_finite_data_and_parameters():
    """Non-finite data make the event invalid (as the reference's arithmetic does);
    non-finite parameter values are rejected before any launch."""
    m = fb.Model.from_string(MIX)
    o = OracleModel(MIX)
    x = np.random.default_rng(9).uniform(-5, 5, 10000)
    for bad_value in (np.inf, -np.inf, np.nan):
        y = x.copy()
        y[777] = bad_value
        y[9000] = bad_value
        v = fb.nll(m, fb.DataSet.from_columns({"x": y}))
        _, comp, ob = o.nll([y])
        assert math.isinf(v.value) and v.first_invalid == ob == 777
        p = fb.probabilities(m, fb.DataSet.from_columns({"x": y}))
        assert math.isnan(p[777]) and np.all(np.isfinite(np.delete(p, [777, 9000])))
    pts = m.theta()[None, :].copy()
    pts[0, m.param_names.index("mu")] = np.nan
    with pytest.raises(fb.FfitError) as e:
        fb.nll_points(m, fb.DataSet.from_columns({"x": x}), pts)
    assert e.value.code == 3


def test_zero_density_chisquare_first_invalid():  # proj/tests/test_eval.cpp:205-217
    m = fb.Model.from_string("observable x 0 20\nparameter k 4 0.5 20\npdf c ChiSquare(x, k)\n")
    v = fb.nll(m, fb.DataSet.from_columns({"x": np.array([1.0, 0.0, 2.0])}))
    assert math.isinf(v.value) and v.first_invalid == 1


def test_single_entry_closed_form():  # proj/tests/test_eval.cpp:80-90
    m = fb.Model.from_string("observable x -10 10\nparameter mu 0 -5 5\nparameter sigma 1 0.1 5\n"
                             "pdf g Gaussian(x, mu, sigma)\n")
    v = fb.nll(m, fb.DataSet.from_columns({"x": np.array([0.0])}))
    assert v.value == pytest.approx(-math.log(1.0 / math.sqrt(2.0 * math.pi)), rel=1e-12)


def test_eval_batch_per_pdf():
    """PdfSpec::eval_batch of sub-pdfs (unnormalised; mixture components normalised)."""
    text = REF_MODELS["mix3_nested"][0]
    m, ds, cols, o = setup(text, 30_000, 4)
    names = m.pdf_names
    for node, name in enumerate(names):
        got = fb.eval_batch(m, name, ds)
        want = o.eval_batch(node, cols)
        assert rel(got, want) <= PER_EVENT, name


def test_sum_of_products_and_nested_sums():
    text = """
observable x -5 5
observable y 0 10
parameter m 0.2 -1 1
parameter s 1.1 0.1 3
parameter c -0.5 -2 0
parameter c2 -0.1 -2 0
parameter a1 0.1 -1 1
parameter f 0.3 0 1
parameter g 0.6 0 1
pdf gx Gaussian(x, m, s)
pdf ey Exponential(y, c)
pdf ex Exponential(x, c2)
pdf py Polynomial(y, a1)
pdf ey2 Exponential(y, c2)
pdf ymix AddPdf(py, g, ey2)
pdf sig ProdPdf(gx, ey)
pdf bkg ProdPdf(ex, ymix)
pdf model AddPdf(sig, f, bkg)
"""
    m = fb.Model.from_string(text)
    o = OracleModel(text)
    rng = np.random.default_rng(2)
    cols = [rng.uniform(-5, 5, 40_000), rng.uniform(0, 10, 40_000)]
    ds = fb.DataSet.from_columns({"x": cols[0], "y": cols[1]})
    assert rel(fb.probabilities(m, ds), o.probabilities(cols)) <= PER_EVENT
    assert abs(fb.nll(m, ds).value - o.nll(cols)[1]) <= NLL_TOL * abs(o.nll(cols)[1])


@pytest.mark.parametrize("ncols", [1, 2, 3, 4, 5])
def test_probabilities_and_eval_batch_over_one_to_five_columns(ncols):
    """probabilities / eval_batch: the per-kind-set kernel with the columns in registers (up to
    three columns) and the generic kernel (more) against the oracle, ragged sizes and non-finite
    data included (proj/src/eval.cpp:174-192, proj/src/pdfs.cpp:212-269)."""
    names = ["x", "y", "z", "u", "v"][:ncols]
    lines = [f"observable {n} -4 4" for n in names]
    lines += [f"parameter m{i} {0.1 * (i + 1)} -1 1\nparameter s{i} {0.8 + 0.1 * i} 0.2 3" for i in range(ncols)]
    lines += [f"pdf g{i} Gaussian({n}, m{i}, s{i})" for i, n in enumerate(names)]
    lines += ["pdf model ProdPdf(" + ", ".join(f"g{i}" for i in range(ncols)) + ")"] if ncols > 1 else []
    text = "\n".join(lines) + "\n"
    m = fb.Model.from_string(text)
    o = OracleModel(text)
    rng = np.random.default_rng(40 + ncols)
    for n in (1, 2047, 2049, 30_011):
        cols = [rng.uniform(-4, 4, n) for _ in names]
        ds = fb.DataSet.from_columns(dict(zip(names, cols)))
        assert rel(fb.probabilities(m, ds), o.probabilities(cols)) <= PER_EVENT
        got = fb.eval_batch(m, "g0", ds)  # a one-column sub-pdf of the same dataset
        assert rel(got, np.exp(-0.5 * ((cols[0] - 0.1) / 0.8) ** 2)) <= PER_EVENT
    cols = [rng.uniform(-4, 4, 5000) for _ in names]
    cols[-1][17] = np.nan
    cols[0][4021] = np.inf
    p = fb.probabilities(m, fb.DataSet.from_columns(dict(zip(names, cols))))
    assert np.isnan(p[17]) and np.isnan(p[4021]) and np.all(np.isfinite(np.delete(p, [17, 4021])))


def test_product_whose_first_factor_is_a_sum():
    """ProdPdf(AddPdf(a, f, b) on x, Gaussian on y, AddPdf on z): multi-term sums as the
    first and the last factor of a product."""
    text = """
observable x -5 5
observable y -3 3
observable z 0 4
parameter m 0.3 -1 1
parameter s 0.9 0.1 3
parameter c -0.4 -2 2
parameter f 0.35 0 1
parameter my 0.1 -1 1
parameter sy 1.2 0.1 3
parameter cz -0.7 -2 2
parameter a1 0.2 -1 1
parameter g 0.5 0 1
pdf gx Gaussian(x, m, s)
pdf ex Exponential(x, c)
pdf xmix AddPdf(gx, f, ex)
pdf gy Gaussian(y, my, sy)
pdf ez Exponential(z, cz)
pdf pz Polynomial(z, a1)
pdf zmix AddPdf(ez, g, pz)
pdf model ProdPdf(xmix, gy, zmix)
"""
    m = fb.Model.from_string(text)
    o = OracleModel(text)
    rng = np.random.default_rng(8)
    cols = [rng.uniform(-5, 5, 30000), rng.uniform(-3, 3, 30000), rng.uniform(0, 4, 30000)]
    ds = fb.DataSet.from_columns({"x": cols[0], "y": cols[1], "z": cols[2]})
    assert rel(fb.probabilities(m, ds), o.probabilities(cols)) <= PER_EVENT
    assert abs(fb.nll(m, ds).value - o.nll(cols)[1]) <= NLL_TOL * abs(o.nll(cols)[1])


def test_extended_model_parity():
    w = configs.C4
    m, ds, cols, o = setup(w.text, 150_000, 77)
    pts = w.points(m, n_points=6)
    vals, _, _ = fb.nll_points(m, ds, pts)
    for p in range(6):
        _, comp, _ = o.nll(cols, pts[p])
        assert abs(vals[p] - comp) <= NLL_TOL * abs(comp)


def test_launch_count_independent_of_n():  # proj/tests/test_eval.cpp:191-203
    m = fb.Model.from_string(MIX)
    small = fb.nll(m, fb.DataSet.from_columns({"x": np.full(100, 0.5)}))
    large = fb.nll(m, fb.DataSet.from_columns({"x": np.full(100000, 0.5)}))
    assert small.n_evaluations == large.n_evaluations == 2
    before = fb.kernel_launches()
    fb.nll(m, fb.DataSet.from_columns({"x": np.full(10, 0.5)}))
    assert fb.kernel_launches() - before == 2


def test_device_view_over_torch_tensors():
    import torch
    w = configs.C3
    m = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(m, 70_001, 5)
    tens = {k: torch.from_numpy(cols[k]).cuda() for k in m.observables}
    ds = fb.DataSet.from_device(tens, device=0)
    o = OracleModel(w.text)
    _, comp, _ = o.nll([cols[k] for k in m.observables])
    assert abs(fb.nll(m, ds).value - comp) <= NLL_TOL * abs(comp)


def test_c_abi_entry_points():
    m = fb.Model.from_string(MIX)
    ds, eff = fb.DataSet.sample(m, 20000, 314159)
    assert eff == -1.0 and ds.n_rows == 20000
    value, nev = fb.nll_c(m, ds, fb.EvalMode.Gpu)
    assert nev == 2
    v2, _ = fb.nll_c(m, ds, fb.EvalMode.BatchPrecise)
    assert v2 == value
    # Scalar == BatchPrecise bitwise in the reference (proj/tests/test_eval.cpp:113-157);
    # every mode returns the fused kernel's bits here, probabilities included
    for mode in (fb.EvalMode.Scalar, fb.EvalMode.BatchFast):
        assert fb.nll_c(m, ds, mode)[0] == value
        assert np.array_equal(fb.probabilities(m, ds, mode), fb.probabilities(m, ds, fb.EvalMode.Gpu))
    with pytest.raises(fb.FfitError) as e:
        fb.nll_c(m, ds, 7)
    assert e.value.code == 1
    o = OracleModel(MIX)
    x = ds.column("x")
    assert abs(value - o.nll([x])[1]) <= NLL_TOL * abs(value)
    m.set("sigma", 1.5)
    assert fb.nll_c(m, ds)[0] != value


@pytest.mark.parametrize("cell,ok", [("1.25", True), ("  1.25 \r", True), ("-3e-1", True), ("+1.25", False),
                                     ("0x1p0", False), ("\t1.25", False), ("1.25\t", False),
                                     ("1.25x", False), ("nan", True)])
def test_csv_cells_parse_as_the_reference(tmp_path, cell, ok):
    """proj/src/dataset.cpp:11-45: split on ',', trim trailing ' '/'\\r' and leading ' ',
    std::from_chars over the whole cell; anything else is FFIT_ERR_DATA 'unparsable numeric
    cell'.  (nan parses, then fails the range check and the row is dropped.)"""
    m = fb.Model.from_string(MIX)
    p = tmp_path / "c.csv"
    p.write_bytes(("x\n0.5\n" + cell + "\n").encode())
    if ok:
        ds, dropped = fb.DataSet.read_csv(m, str(p))
        assert ds.n_rows + dropped == 2
    else:
        with pytest.raises(fb.FfitError) as e:
            fb.DataSet.read_csv(m, str(p))
        assert e.value.code == 2 and "unparsable numeric cell at row 2, column 'x'" in e.value.message


def test_csv_round_trip(tmp_path):
    m = fb.Model.from_string(MIX)
    ds, _ = fb.DataSet.sample(m, 3000, 1)
    p = str(tmp_path / "d.csv")
    ds.write_csv(p)
    with open(p, "a") as fh:
        fh.write("7.5\n")  # outside [-5, 5]: dropped (proj/src/dataset.cpp:104-112)
    back, dropped = fb.DataSet.read_csv(m, p)
    assert dropped == 1 and np.array_equal(back.column("x"), ds.column("x"))


def test_combine_kernel_matches_host_combine():
    import torch
    rng = np.random.default_rng(3)
    pairs = np.zeros((3, 17, 2))
    pairs[..., 0] = rng.normal(-2e7, 1e4, (3, 17))
    pairs[..., 1] = rng.normal(0, 1e-8, (3, 17))
    d_in = torch.from_numpy(pairs).cuda()
    d_out = torch.zeros((17, 2), dtype=torch.float64, device="cuda")
    fb.ffit.combine_pairs_device(d_in.data_ptr(), 3, 17, d_out.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(d_out.cpu().numpy(), D.combine_pairs(pairs))


def test_sharded_single_rank_equals_direct():
    import torch.distributed as dist
    w = configs.C2
    m, ds, _, _ = setup(w.text, 100_000, 5)
    pts = w.points(m, n_points=5)
    sh = D.ShardedNll(m, ds, ds.n_rows, 0, dist, 0)
    vals = sh.nll_points(pts)
    direct, _, _ = fb.nll_points(m, ds, pts)
    assert np.array_equal(vals, direct)


def test_shard_sum_equals_whole():
    """Additivity over event shards (the multi-GPU decomposition), exact to 1e-12."""
    w = configs.C2
    m, ds, _, _ = setup(w.text, 1_000_003, 21)
    pts = w.points(m, n_points=3)
    whole, _, _ = fb.nll_points(m, ds, pts)
    parts = []
    for r in range(4):
        b, e = D.shard_bounds(ds.n_rows, 4, r)
        parts.append(fb.nll_points_partial(m, ds.slice(b, e), pts)[0])
    comb = D.combine_pairs(np.stack(parts))
    assert np.all(np.abs(comb.sum(axis=1) - whole) <= NLL_TOL * np.abs(whole))


# ------------------------------------------------------------------ full BASELINE sizes

@pytest.mark.slow
def test_c2_full_size_parity_and_properties():
    """configs[1] at 1e7 events: oracle parity at two points, shard additivity and
    permutation invariance at all sizes the oracle cannot afford."""
    w = configs.C2
    m, ds, cols, o = setup(w.text, w.n_events, w.data_seed)
    pts = w.points(m)
    vals, bad, _ = fb.nll_points(m, ds, pts)
    assert np.all(bad == -1) and np.all(np.isfinite(vals))
    for p in (0, 199):
        _, comp, _ = o.nll(cols, pts[p])
        assert abs(vals[p] - comp) <= NLL_TOL * abs(comp)
    perm = np.random.default_rng(0).permutation(w.n_events)
    shuffled = fb.DataSet.from_columns({"x": cols[0][perm]})
    sv, _, _ = fb.nll_points(m, shuffled, pts[:8])
    assert np.all(np.abs(sv - vals[:8]) <= NLL_TOL * np.abs(vals[:8]))


@pytest.mark.slow
def test_c3_full_size_three_columns():
    w = configs.C3
    m, ds, cols, o = setup(w.text, w.n_events, w.data_seed)
    pts = w.points(m, n_points=4)
    vals, bad, _ = fb.nll_points(m, ds, pts)
    assert np.all(bad == -1)
    half = w.n_events // 2
    a = fb.nll_points_partial(m, ds.slice(0, half), pts)[0]
    b = fb.nll_points_partial(m, ds.slice(half, w.n_events), pts)[0]
    comb = D.combine_pairs(np.stack([a, b])).sum(axis=1)
    assert np.all(np.abs(comb - vals) <= NLL_TOL * np.abs(vals))
    _, comp, _ = o.nll(cols, pts[0])
    assert abs(vals[0] - comp) <= NLL_TOL * abs(comp)


def test_streaming_and_tile_kernels_agree():
    """Launches of <= 8 points over aligned columns take the persistent streaming kernel,
    larger ones the tile-per-CTA kernel: same values to summation-order rounding."""
    w = configs.C2
    m, ds, cols, o = setup(w.text, 333_333, 21)
    pts = w.points(m, n_points=9)
    many, _, _ = fb.nll_points(m, ds, pts)           # tile kernel (P = 9)
    assert fb.last_launch(m)["nchunks"] > 0
    for p in range(9):
        one, _, _ = fb.nll_points(m, ds, pts[p])      # streaming kernel (P = 1)
        assert fb.last_launch(m)["nchunks"] == 0
        assert abs(one[0] - many[p]) <= 1e-13 * abs(many[p])
        _, comp, _ = o.nll(cols, pts[p])
        assert abs(one[0] - comp) <= NLL_TOL * abs(comp)
    few, _, _ = fb.nll_points(m, ds, pts[:8])         # streaming, several points
    assert np.all(np.abs(few - many[:8]) <= 1e-13 * np.abs(many[:8]))


@pytest.mark.parametrize("n", [1, 2, 3, 2047, 2048, 2049, 4097, 606_209])
def test_streaming_ragged_sizes(n):
    """Odd final elements (patched after the even-length bulk copy), fewer tiles than
    CTAs, and a tile count that is not a multiple of the grid."""
    m, ds, cols, o = setup(MIX, n, n)
    v = fb.nll(m, ds)
    _, comp, _ = o.nll(cols)
    assert abs(v.value - comp) <= NLL_TOL * abs(comp)
    assert v.first_invalid == -1


# ------------------------------------------------------------------ Expression pdfs (f4)

@pytest.mark.parametrize("name", list(EXPR_MODELS))
def test_expression_pdfs_run_the_reference_text_on_the_gpu(name):
    """The reference's OWN Expression model text (e.g. ArgusBG spelled as a formula) on the
    device interpreter vs the reference's per-event values and NLL (golden)."""
    ref_text, _, _, col = EXPR_MODELS[name]
    g = np.load(os.path.join(GOLD, "expr_models.npz"))
    x, p, sc = g[f"{name}/x"], g[f"{name}/p"], g[f"{name}/scalars"]
    m = fb.Model.from_string(ref_text)
    ds = fb.DataSet.from_columns({col: x})
    assert rel(fb.probabilities(m, ds), p) <= PER_EVENT
    assert abs(fb.nll(m, ds).value - sc[0]) <= NLL_TOL * abs(sc[0])
    many, _, _ = fb.nll_points(m, ds, np.repeat(m.theta()[None, :], 10, axis=0))  # tile kernel
    assert np.all(np.abs(many - sc[0]) <= NLL_TOL * abs(sc[0]))


def test_expression_config2_reference_text_matches_reference_engine():
    """BASELINE config 2 exactly as the reference spells it (configs.REFERENCE_TEXTS: the
    ArgusBG as an Expression) against the unmodified reference engine at several points."""
    from oracle.oracle import RefDataset, RefModel, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    w = configs.C2
    text = configs.REFERENCE_TEXTS[w.name]
    m = fb.Model.from_string(text)
    cols, _ = fb.sample_host(fb.Model.from_string(w.text), 30_011, 5)
    ds = fb.DataSet.from_columns(cols)
    r = RefModel(text)
    rds = RefDataset("x", cols["x"])
    pts = w.points(m, n_points=3)
    vals, _, _ = fb.nll_points(m, ds, pts)
    for p in range(3):
        for name, v in zip(m.param_names, pts[p]):
            if not m.is_constant(name):
                r.set(name, v)
        want = r.nll_compensated(rds)[0]
        assert abs(vals[p] - want) <= NLL_TOL * abs(want)


def test_expression_sub_pdf_eval_batch_and_invalid_events():
    """eval_batch of an Expression sub-pdf (its own uploaded program) against the host
    interpreter; a formula that is negative somewhere flags those events invalid."""
    text = EXPR_MODELS["argus_mix"][0]
    m = fb.Model.from_string(text)
    x = np.linspace(5.2, 5.29, 5001)
    ds = fb.DataSet.from_columns({"x": x})
    got = fb.eval_batch(m, "bkg", ds)
    want = fb.expr_eval("x*sqrt(1-(x/m0)^2)*exp(c*(1-(x/m0)^2))", ["x", "m0", "c"],
                        np.column_stack([x, np.full_like(x, 5.291), np.full_like(x, -20.0)]))
    assert rel(got, want) <= PER_EVENT
    bad = fb.Model.from_string("observable x -1 1\nparameter a 0.5 0 1\npdf e Expression(\"a + x\", x, a)\n")
    v = fb.nll(bad, fb.DataSet.from_columns({"x": np.array([0.1, 0.2, -0.7, 0.3])}))
    assert v.value == np.inf and v.first_invalid == 2


def test_expression_fit_analytic_and_automatic():
    """A gradient fit of the reference's Argus-as-formula model on analytic gradients
    (forward mode through the formula) reaches the minimum of the automatic choice, which
    for formula models is finite differences over the formula-specialised build."""
    text = EXPR_MODELS["argus_mix"][0]
    m = fb.Model.from_string(text)
    cols, _ = fb.sample_host(m, 20_000, 3)
    ds = fb.DataSet.from_columns(cols)
    r = fb.fit_gradient(m, ds, tolerance=1e-10, max_iterations=200, analytic=True)
    assert r.converged and r.analytic_gradient
    m2 = fb.Model.from_string(text)
    # the automatic choice: finite differences over the formula-specialised build
    r2 = fb.fit_gradient(m2, ds, tolerance=1e-10, max_iterations=200)
    assert r2.converged and not r2.analytic_gradient
    assert abs(r.nll_min - r2.nll_min) <= 1e-9 * abs(r2.nll_min)
    for a, b in zip(r.parameters, r2.parameters):
        assert abs(a.value - b.value) <= 1e-3 * max(b.uncertainty, 1e-12) + 1e-9 * abs(b.value)


@pytest.mark.parametrize("name", list(EXPR_MODELS))
def test_expression_analytic_gradient_matches_native_kind(name):
    """dNLL/dtheta of the Expression spelling (device forward mode through the formula,
    normalisation derivative by quadrature of the host forward mode) against the native
    kind's analytic gradient (pinned to the oracle in test_gpu_grad.py), same events."""
    text, ours, seed, col = EXPR_MODELS[name]
    me, mo = fb.Model.from_string(text), fb.Model.from_string(ours)
    cols, _ = fb.sample_host(mo, 30_000, seed)
    ds = fb.DataSet.from_columns({col: cols[col]})
    by = dict(zip(mo.param_names, mo.theta()))
    te = np.array([by[n] for n in me.param_names])
    ve, ge, be, _ = fb.nll_grad(me, ds, te)
    vo, go, bo, _ = fb.nll_grad(mo, ds, mo.theta())
    assert be[0] == bo[0] == -1
    assert abs(ve[0] - vo[0]) <= 1e-12 * abs(vo[0])
    gn = dict(zip(mo.param_names, go[0]))
    scale = max(1.0, np.max(np.abs(go[0])))
    for j, n in enumerate(me.param_names):
        if me.is_constant(n):
            continue
        assert abs(ge[0, j] - gn[n]) <= 1e-8 * scale, (n, ge[0, j], gn[n])


@pytest.mark.parametrize("name", list(EXPR_MODELS) + ["c2_reference_text"])
def test_expression_jit_matches_interpreter(name):
    """The formula-specialised (NVRTC) build against the device interpreter: same formulas in
    the same operation order; exp / log / sqrt take the table-driven forms (<= 2 ulp) in the
    specialised build, so the NLLs agree to 1e-13; both kernels (1 point: streaming; 10
    points: tile)."""
    if name == "c2_reference_text":
        text, col = configs.REFERENCE_TEXTS[configs.C2.name], "x"
        cols, _ = fb.sample_host(fb.Model.from_string(configs.C2.text), 50_000, 9)
        x = cols["x"]
    else:
        text, _, _, col = EXPR_MODELS[name]
        x = np.load(os.path.join(GOLD, "expr_models.npz"))[f"{name}/x"]
    m = fb.Model.from_string(text)
    ds = fb.DataSet.from_columns({col: x})
    pts = np.repeat(m.theta()[None, :], 10, axis=0)
    was = fb.expression_jit(True)
    try:
        one_j, _, _ = fb.nll_points(m, ds, pts[:1])
        assert fb.last_launch_jit(m), fb.expression_jit_status()
        many_j, _, _ = fb.nll_points(m, ds, pts)
        fb.expression_jit(False)
        one_i, _, _ = fb.nll_points(m, ds, pts[:1])
        assert not fb.last_launch_jit(m)
        many_i, _, _ = fb.nll_points(m, ds, pts)
    finally:
        fb.expression_jit(was)
    assert abs(one_j[0] - one_i[0]) <= 1e-13 * abs(one_i[0])
    assert np.all(np.abs(many_j - many_i) <= 1e-13 * np.abs(many_i))


def test_expression_launch_constant_subtrees_bit_identical():
    """The reference's config-2 text (ArgusBG as a formula): with m0 fixed over the launch,
    x*sqrt(1-(x/m0)^2) and 1-(x/m0)^2 are computed once per staged tile; one more point with
    another m0 leaves no launch-constant subtree, and the launch runs the plain formula
    build.  The shared points' values are bitwise equal either way and match the oracle on
    the native spelling."""
    w = configs.C2
    text = configs.REFERENCE_TEXTS[w.name]
    m = fb.Model.from_string(text)
    mo = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(mo, 120_013, 31)
    ds = fb.DataSet.from_columns(cols)
    by = [dict(zip(mo.param_names, r)) for r in w.points(mo, n_points=16)]
    pts = np.array([[d[n] for n in m.param_names] for d in by])
    was = fb.expression_jit(True)
    try:
        cached, bad, _ = fb.nll_points(m, ds, pts)
        assert fb.last_launch_jit(m) == 1 and fb.last_launch_cached(m) == 2, fb.expression_jit_status()
        other = pts[:1].copy()
        other[0, m.param_names.index("m0")] *= 1 + 1e-4
        plain, _, _ = fb.nll_points(m, ds, np.vstack([pts, other]))
        assert fb.last_launch_cached(m) == 0
    finally:
        fb.expression_jit(was)
    assert np.array_equal(cached, plain[:16])
    o = OracleModel(w.text)
    for p in (0, 15):
        _, comp, ob = o.nll([cols["x"]], np.array([by[p][n] for n in mo.param_names]))
        assert bad[p] == ob == -1
        assert abs(cached[p] - comp) <= NLL_TOL * abs(comp)


# ------------------------------------------------------------------ plan-specialised builds

def _spec_cases():
    from tests.test_gpu_grad import CASES
    return CASES


@pytest.mark.parametrize("name", list(_spec_cases()))
def test_plan_specialised_build_matches_static_build(name):
    """The tile kernel compiled around the launch's term list (jit.cpp plan_spec_source)
    against the static build on the same launch, and against the oracle."""
    from tests.test_gpu_grad import setup as grad_setup  # uniform events where no sampler exists
    text, n = _spec_cases()[name]
    m, ds, cols = grad_setup(text, n, 101)
    o = OracleModel(text)
    base = m.theta()
    free = [k for k, nm in enumerate(m.param_names) if not m.is_constant(nm)]
    pts = np.tile(base, (12, 1))
    for p in range(12):
        for k in free:
            pts[p, k] = base[k] * (1.0 + 2e-4 * (p - 6)) if base[k] != 0 else 1e-4 * (p - 6)
    old = fb.plan_spec_min_work(-1)
    try:
        static, sbad, _ = fb.nll_points(m, ds, pts)
        assert fb.last_launch_jit(m) == 0
        few, _, _ = fb.nll_points(m, ds, pts[:3])  # the streaming build where one exists
        fb.plan_spec_min_work(0)
        spec, bad, _ = fb.nll_points(m, ds, pts)
        assert fb.last_launch_jit(m) == 2, fb.expression_jit_status()
        few_spec, _, _ = fb.nll_points(m, ds, pts[:3])
        if len(m.observables) == 1:  # single-column single-sum: the specialised streaming kernel
            assert fb.last_launch_jit(m) == 2
    finally:
        fb.plan_spec_min_work(old)
    assert np.array_equal(bad, sbad)
    assert np.array_equal(spec, static), np.max(np.abs(spec - static) / np.abs(static))
    # few points: the specialised streaming kernel where one exists against the static build
    # (a different summation tree: equal to the last bit or two of the total)
    assert np.max(np.abs(few_spec - few) / np.abs(few)) <= 5e-16
    for p in (0, 11):
        _, comp, ob = o.nll(cols, pts[p])
        assert bad[p] == ob
        assert abs(spec[p] - comp) <= NLL_TOL * abs(comp)


@pytest.mark.parametrize("name", list(_spec_cases()))
def test_launch_constant_cache_every_leaf_kind(name):
    """Only one free parameter moves over the launch's points, so every leaf that does not
    read it is evaluated once per staged tile (the whole-leaf cache; every leaf kind and
    plan shape of the gradient-test models).  Bitwise equal to the same points in a launch
    where one more point moves every parameter (nothing cached), and to the oracle."""
    from tests.test_gpu_grad import setup as grad_setup
    text, n = _spec_cases()[name]
    m, ds, cols = grad_setup(text, n, 202)
    o = OracleModel(text)
    base = m.theta()
    free = [k for k, nm in enumerate(m.param_names) if not m.is_constant(nm)]
    j = free[-1]
    pts = np.tile(base, (12, 1))
    for p in range(12):
        pts[p, j] = base[j] * (1.0 + 2e-4 * (p - 6)) if base[j] != 0 else 1e-4 * (p - 6)
    cached, bad, _ = fb.nll_points(m, ds, pts)
    ncached = fb.last_launch_cached(m)
    # 13 more points moving every parameter (constant ones too: ArgusBG's m0 in config 2),
    # each to its own value: no launch-constant part and no majority m0 left
    other = np.repeat(base[None, :], 13, axis=0)
    for i in range(13):
        for k in range(len(base)):
            other[i, k] = base[k] * (1 + 1e-4 * (i + 1)) if base[k] != 0 else 1e-4 * (i + 1)
    plain, _, _ = fb.nll_points(m, ds, np.vstack([pts, other]))
    assert fb.last_launch_cached(m) == 0
    assert np.array_equal(cached, plain[:12]), (ncached, np.max(np.abs(cached - plain[:12]) / np.abs(plain[:12])))
    for p in (0, 11):
        _, comp, ob = o.nll(cols, pts[p])
        assert bad[p] == ob
        assert abs(cached[p] - comp) <= NLL_TOL * abs(comp)


@pytest.mark.parametrize("n", [1, 2047, 2049, 10007])
@pytest.mark.parametrize("shape", ["c4_yields_only", "c2_m0_fixed", "all_free"])
def test_cached_and_specialised_paths_edge_cases(n, shape):
    """The plan-specialised tile kernel with the launch-constant caches on ragged sizes,
    non-finite events (first invalid index) and an 8-byte-aligned device view."""
    w = configs.C4 if shape == "c4_yields_only" else configs.C2
    m = fb.Model.from_string(w.text)
    o = OracleModel(w.text)
    cols, _ = fb.sample_host(m, n + 1, 61)
    x = cols["x"]
    base = m.theta()
    names = m.param_names
    pts = np.tile(base, (12, 1))
    for p in range(12):
        for k, name in enumerate(names):
            moves = (name.startswith("n") if shape == "c4_yields_only"
                     else not m.is_constant(name))
            if moves:
                pts[p, k] = base[k] * (1.0 + 2e-4 * (p - 6))
    old = fb.plan_spec_min_work(0)
    try:
        for bad in (None, np.nan, np.inf):
            y = x.copy()
            if bad is not None and n > 3:
                y[n // 2] = bad
            full = fb.DataSet.from_columns({"x": y})
            view = full.slice(1, n + 1)  # starts 8 bytes into the column: cooperative staging
            for ds, xs in ((full, y), (view, y[1:n + 1])):
                vals, fi, _ = fb.nll_points(m, ds, pts)
                assert fb.last_launch_jit(m) == 2
                for p in (0, 11):
                    _, comp, ob = o.nll([xs], pts[p])
                    assert fi[p] == ob
                    if ob >= 0:
                        assert math.isinf(vals[p])
                    else:
                        assert abs(vals[p] - comp) <= NLL_TOL * abs(comp)
    finally:
        fb.plan_spec_min_work(old)


def test_few_point_calls_replay_a_cuda_graph():
    """A minimiser's single-point calls: the first call with a launch signature runs the
    plain sequence, the second captures it into a CUDA graph, later ones replay it (the
    kernel timer disables graphs: the plain path).  Same bits on every path, and the
    oracle's values at every point."""
    w = configs.C2
    m, ds, cols, o = setup(w.text, 100_003, 17)
    pts = w.points(m, n_points=6)
    fb.kernel_timer(True)
    plain = [fb.nll_points(m, ds, pts[p:p + 1])[0][0] for p in range(6)]
    fb.kernel_timer(False)
    fb.kernel_timer_read()
    launches0 = fb.kernel_launches()
    graphed = [fb.nll_points(m, ds, pts[p:p + 1])[0][0] for p in range(6)]
    again = [fb.nll_points(m, ds, pts[p:p + 1])[0][0] for p in range(6)]
    assert fb.kernel_launches() - launches0 == 2 * 12  # replays still count their kernels
    assert plain == graphed == again
    for p in (0, 5):
        _, comp, _ = o.nll(cols, pts[p])
        assert abs(graphed[p] - comp) <= NLL_TOL * abs(comp)
    # another dataset of the same size, then the first again: new signatures, same values
    ds2 = fb.DataSet.from_columns({"x": cols[0].copy()})
    v2 = [fb.nll_points(m, ds2, pts[:1])[0][0] for _ in range(3)]
    v1 = [fb.nll_points(m, ds, pts[:1])[0][0] for _ in range(3)]
    assert v2 == v1 == [plain[0]] * 3
    # a point leaving ArgusBG's fast domain changes the kernel build (new signature)
    bad = pts[:1].copy()
    bad[0, m.param_names.index("c")] = -750.0
    v3 = [fb.nll_points(m, ds, bad)[0][0] for _ in range(3)]
    _, comp3, _ = o.nll(cols, bad[0])
    assert v3[0] == v3[1] == v3[2] and abs(v3[0] - comp3) <= NLL_TOL * abs(comp3)


def test_distinct_models_on_distinct_threads():
    """SPEC.md: a model is single-owner, distinct models may run on distinct threads.  Four
    host threads, each with its own model (native and formula spellings), run single-point
    calls (CUDA-graph replay) and 16-point launches (run-time compiled builds) at once;
    every value equals the one-thread run bit for bit."""
    import threading
    w = configs.C2
    texts = [w.text, configs.REFERENCE_TEXTS[w.name], w.text, configs.REFERENCE_TEXTS[w.name]]
    mo = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(mo, 200_003, 23)
    ds = fb.DataSet.from_columns(cols)
    base = [dict(zip(mo.param_names, r)) for r in w.points(mo, n_points=16)]

    def work(text):
        m = fb.Model.from_string(text)
        pts = np.array([[d[n] for n in m.param_names] for d in base])
        out = [fb.nll_points(m, ds, pts[i:i + 1])[0][0] for i in range(4) for _ in range(3)]
        out += list(fb.nll_points(m, ds, pts)[0])
        return out

    want = [work(t) for t in texts]
    got = [None] * len(texts)
    errors = []

    def run(i):
        try:
            got[i] = work(texts[i])
        except Exception as e:  # reported below
            errors.append(e)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(texts))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert got == want


def test_launch_constant_cache_partly_shared_m0():
    """A finite-difference batch of the config-5 model (m0 free): 9 of 11 points share m0,
    so ArgusBG's data-only part is cached per tile for them (flagged rows) and the two m0
    steps evaluate the full leaf.  Bitwise equal to the same points in a launch without a
    majority m0 (nothing cached), and to the oracle."""
    w = configs.C5
    m, ds, cols, o = setup(w.text, 120_011, 29)
    th = m.theta()
    free = [k for k, n in enumerate(m.param_names) if not m.is_constant(n)]
    pts = [th.copy()]
    for k in free:
        for sgn in (1.0, -1.0):
            r = th.copy()
            r[k] += sgn * 1e-5 * max(abs(th[k]), 1.0)
            pts.append(r)
    pts = np.array(pts)
    assert len(pts) == 11
    hybrid, bad, _ = fb.nll_points(m, ds, pts)
    assert fb.last_launch_cached(m) == 1
    j = m.param_names.index("m0")
    extra = np.repeat(th[None, :], 14, axis=0)
    extra[:, j] = th[j] + 1e-4 * np.arange(1, 15)  # 14 distinct m0: no majority left
    plain, _, _ = fb.nll_points(m, ds, np.vstack([pts, extra]))
    assert fb.last_launch_cached(m) == 0
    assert np.array_equal(hybrid, plain[:11])
    for p in (0, 1, 2 * free.index(j) + 1, 10):
        _, comp, ob = o.nll(cols, pts[p])
        assert bad[p] == ob == -1
        assert abs(hybrid[p] - comp) <= NLL_TOL * abs(comp)


def test_more_points_than_one_launch():
    """P > 512 (the per-launch cap) is split into several launches; every chunk boundary
    point matches the oracle and is bit-identical to the same point evaluated in a launch
    of the same kernel shape."""
    m, ds, xs, o = setup(ARGUS_OURS, 30_001, 77)
    base = m.theta()
    P = 1100
    pts = np.tile(base, (P, 1))
    free = [k for k, nm in enumerate(m.param_names) if not m.is_constant(nm)]
    for p in range(P):
        for k in free:
            pts[p, k] = base[k] * (1.0 + 1e-4 * np.sin(p + k))
    vals, bad, _ = fb.nll_points(m, ds, pts)
    assert len(vals) == P and np.all(np.asarray(bad) == -1)
    for p in (0, 511, 512, 1023, 1024, P - 1):
        _, comp, ob = o.nll(xs, pts[p])
        assert ob == -1
        assert abs(vals[p] - comp) <= NLL_TOL * abs(comp), (p, vals[p], comp)
    # the second chunk alone (512 points: the same kernel shape as inside the big call)
    v2, _, _ = fb.nll_points(m, ds, pts[512:1024])
    assert np.array_equal(np.asarray(v2), np.asarray(vals[512:1024]))


def test_upload_stream_pipeline_is_bit_identical():
    """The double-buffered pipeline bench.py's e2e runs (ffcu_dataset_copy_from_host_async into
    the other of two datasets on a copy stream; ffcu_nll_points_device_upload copying the
    constant rows on that stream; the next step queued before the current one's results are
    read), with DIFFERENT events and points every step, interleaved with eval_batch_device on
    the model's own stream: every step's pairs equal ffcu_nll_points_partial on the same
    events and points, bit for bit (an ordering bug would mix rows or events of two steps)."""
    torch = pytest.importorskip("torch")
    w = configs.C2
    m = fb.Model.from_string(w.text)
    n, P, steps = 300_007, 12, 8
    data = [fb.sample_host(m, n, 5000 + i)[0]["x"] for i in range(steps)]
    pts = [w.points(m, n_points=P, seed=7000 + i) for i in range(steps)]
    dev = torch.device("cuda", 0)
    pinned = [torch.from_numpy(x).pin_memory() for x in data]
    bufs = [fb.DataSet.from_columns({"x": data[0]}), fb.DataSet.from_columns({"x": data[1]})]
    stream, copy_stream = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event() for _ in bufs]
    done = [torch.cuda.Event() for _ in bufs]
    d_sc = [torch.empty((P, 2), dtype=torch.float64, device=dev) for _ in range(steps)]
    d_bad = [torch.empty(P, dtype=torch.int64, device=dev) for _ in range(steps)]
    d_eval = torch.empty(n, dtype=torch.float64, device=dev)
    for i in range(steps):
        k = i % 2
        copy_stream.wait_event(done[k])
        bufs[k].copy_from_host_async({"x": pinned[i].numpy()}, copy_stream.cuda_stream)
        copied[k].record(copy_stream)
        stream.wait_event(copied[k])
        fb.nll_points_device(m, bufs[k], pts[i], d_sc[i].data_ptr(), d_bad[i].data_ptr(), stream.cuda_stream,
                             copy_stream.cuda_stream)
        if i % 3 == 1:  # a per-event evaluation on the model's own stream between steps
            fb.eval_batch_device(m, "sig", bufs[k], d_eval.data_ptr(), None)
        done[k].record(stream)
    torch.cuda.synchronize()
    for i in range(steps):
        want, wbad = fb.nll_points_partial(m, fb.DataSet.from_columns({"x": data[i]}), pts[i])
        got = d_sc[i].cpu().numpy()
        assert np.array_equal(got, want), i
        assert np.all(d_bad[i].cpu().numpy() == -1) and np.all(wbad == -1)


@pytest.mark.slow
def test_c4_full_size_parity_and_properties():
    """configs[3] at its full size, the bench's headline launch (1e8 events x 64 points,
    extended): oracle parity at four points (threaded oracle), shard additivity over four
    contiguous shards combined in rank order with the extended term on the global N, and
    permutation invariance."""
    w = configs.C4
    m, ds, cols, o = setup(w.text, w.n_events, w.data_seed)
    n = w.n_events
    pts = w.points(m)
    assert len(pts) == 64
    vals, bad, _ = fb.nll_points(m, ds, pts)
    assert np.all(bad == -1) and np.all(np.isfinite(vals))
    sel = [0, 21, 42, 63]
    comp = o.nll_points(cols, pts[sel], threads=4)
    assert np.all(np.abs(vals[sel] - comp) <= NLL_TOL * np.abs(comp)), (vals[sel] - comp) / comp
    parts = np.stack([fb.nll_points_partial(m, ds.slice(b, e), pts)[0]
                      for b, e in (D.shard_bounds(n, 4, r) for r in range(4))])
    comb = D.combine_pairs(parts).sum(axis=1) + m.extended_terms(pts, n)
    assert np.all(np.abs(comb - vals) <= NLL_TOL * np.abs(vals))
    perm = np.random.default_rng(0).permutation(n)
    shuffled = fb.DataSet.from_columns({"x": cols[0][perm]})
    del perm
    sv, _, _ = fb.nll_points(m, shuffled, pts[:8])
    assert np.all(np.abs(sv - vals[:8]) <= NLL_TOL * np.abs(vals[:8]))
