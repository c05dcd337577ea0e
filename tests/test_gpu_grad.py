"""The fused NLL + analytic-gradient pass against the oracle.

Reference gradient: dNLL/dtheta_j = -sum_i (dp_i/dtheta_j) / p_i with dp_i/dtheta_j a
4-point central difference of the ORACLE's per-event probabilities, step h = 1e-4 of
the parameter's range.  Per-event differences keep truncation and rounding near 1e-12
of each event's |d log p_i|; what remains is the rounding / quadrature noise of the
oracle's normalisation (closed forms ~1e-15, adaptive Simpson ~1e-12), which a
difference quotient amplifies by 1/h.  The bound is therefore
    1e-9 * sum_i |d log p_i / d theta_j|  +  |g_ref(h) - g_ref(2h)|
an L1 scale that stays meaningful where the gradient itself is near zero, plus the
reference's own step-to-step spread as its error estimate.  Extended models add
d(nu - N log nu)/dy = 1 - N/nu.
"""
import math
import zlib

import numpy as np
import pytest

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs
from oracle.oracle import OracleModel
from tests.models import EXPR_MODELS, MIX, REF_MODELS

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-9
NLL_TOL = 1e-12

SUM_OF_PRODUCTS = """
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

PROD_FIRST_SUM = """
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

ARGUS_ALL_FREE = configs.C5.text.replace("parameter p 0.5 0 1 const", "parameter p 0.5 0.1 1")

CASES = {
    "c1_gauss": (configs.C1.text, 30_000),
    "c2_gauss_argus": (configs.C2.text, 40_000),
    "c5_m0_free": (configs.C5.text, 40_000),
    "argus_p_free": (ARGUS_ALL_FREE, 40_000),
    "c3_product": (configs.C3.text, 30_000),
    "c4_extended": (configs.C4.text, 60_000),
    "johnson": (REF_MODELS["johnson"][0], 20_000),
    "chisq": (REF_MODELS["chisq"][0], 20_000),
    "mix": (MIX, 20_000),
    "mix3_nested": (REF_MODELS["mix3_nested"][0], 20_000),
    "mix_chisq": (REF_MODELS["mix_chisq"][0], 20_000),
    "cheb3_shifted": (EXPR_MODELS["cheb3_shifted"][1], 20_000),
    "poly2": (EXPR_MODELS["poly2"][1], 20_000),
    "sum_of_products": (SUM_OF_PRODUCTS, 20_000),
    "prod_first_sum": (PROD_FIRST_SUM, 20_000),
}


def param_table(text):
    """name -> (value, lo, hi, const) from the model text."""
    out = {}
    for line in text.splitlines():
        t = line.split()
        if t and t[0] == "parameter":
            out[t[1]] = (float(t[2]), float(t[3]), float(t[4]), len(t) > 5 and t[5] == "const")
    return out


def ref_gradient(text, cols, theta, names, n_events, extended_yields=()):
    """(gradient, L1 scale, error estimate) of the oracle NLL (module docstring)."""
    o = OracleModel(text)
    table = param_table(text)
    p0 = o.probabilities(cols, theta)
    g = np.zeros(len(theta))
    scale = np.zeros(len(theta))
    est = np.zeros(len(theta))
    for j, name in enumerate(names):
        _, lo, hi, const = table[name]
        if const:
            continue

        def P(d):
            t = np.array(theta, dtype=float)
            t[j] += d
            return o.probabilities(cols, t)

        def dlogp(h):
            return (8.0 * (P(h) - P(-h)) - (P(2 * h) - P(-2 * h))) / (12.0 * h) / p0

        h = 1e-4 * (hi - lo)
        t1, t2 = dlogp(h), dlogp(2 * h)
        g[j] = -math.fsum(t1)
        scale[j] = np.sum(np.abs(t1))
        est[j] = abs(math.fsum(t1) - math.fsum(t2))
    if extended_yields:
        nu = sum(theta[names.index(y)] for y in extended_yields)
        for y in extended_yields:
            k = names.index(y)
            g[k] += 1.0 - n_events / nu
            scale[k] += abs(n_events / nu) + 1.0
    return g, scale, est


def jittered(m, text, seed):
    """The model's values moved by a few per cent of each free parameter's range."""
    rng = np.random.default_rng(seed)
    table = param_table(text)
    th = m.theta().copy()
    for j, name in enumerate(m.param_names):
        v, lo, hi, const = table[name]
        if not const:
            th[j] = np.clip(v + 0.02 * (hi - lo) * rng.uniform(-1, 1), lo + 0.01 * (hi - lo),
                            hi - 0.01 * (hi - lo))
    return th


def setup(text, n, seed=5):
    m = fb.Model.from_string(text)
    if "ProdPdf(sig" in text.replace(" ", "") or "pdf sig ProdPdf" in text:
        # a sum of products has no toy generator (sampling needs 1-D factors): uniform
        # events over the observable ranges
        rng = np.random.default_rng(seed)
        cols = {}
        for line in text.splitlines():
            t = line.split()
            if t and t[0] == "observable":
                cols[t[1]] = rng.uniform(float(t[2]), float(t[3]), n)
    else:
        cols, _ = fb.sample_host(m, n, seed)
    ds = fb.DataSet.from_columns(cols)
    return m, ds, [cols[k] for k in m.observables]


def yields_of(text):
    for line in text.splitlines():
        t = line.split()
        if t and t[0] == "pdf" and t[2].startswith("AddPdf") and "model" == t[1]:
            args = line[line.index("(") + 1:line.rindex(")")].replace(",", " ").split()
            if len(args) % 2 == 0:  # extended: (c1, y1, ..., cn, yn)
                return tuple(args[1::2])
    return ()


@pytest.mark.parametrize("name", list(CASES))
def test_gradient_matches_oracle(name):
    text, n = CASES[name]
    m, ds, cols = setup(text, n)
    th = jittered(m, text, seed=zlib.crc32(name.encode()) % 1000)
    vals, grads, bad, launches = fb.nll_grad(m, ds, th)
    assert bad[0] == -1 and launches == 2
    # the value is the same NLL the likelihood pass computes
    want_v, _, _ = fb.nll_points(m, ds, th)
    assert abs(vals[0] - want_v[0]) <= NLL_TOL * abs(want_v[0])
    names = m.param_names
    g_ref, scale, est = ref_gradient(text, cols, th, names, n, yields_of(text))
    for j, pname in enumerate(names):
        if m.is_constant(pname):
            assert grads[0, j] == 0.0
            continue
        err = abs(grads[0, j] - g_ref[j])
        assert err <= GRAD_TOL * scale[j] + est[j], (pname, grads[0, j], g_ref[j], err / scale[j], est[j])


def test_multi_point_matches_single_points():
    text = configs.C2.text
    m, ds, _ = setup(text, 50_000)
    pts = configs.C2.points(m, n_points=5)
    vals, grads, _, launches = fb.nll_grad(m, ds, pts)
    assert launches == 2
    for p in range(5):
        # one point takes the plan-specialised pass, five the generic streaming pass: the
        # same sums in different groupings
        v1, g1, _, _ = fb.nll_grad(m, ds, pts[p])
        assert abs(v1[0] - vals[p]) <= 1e-13 * abs(vals[p])
        assert np.all(np.abs(g1[0] - grads[p]) <= 1e-9 * np.abs(grads[p]) + 1e-6)


@pytest.mark.parametrize("n", [1, 255, 1023, 1025, 4097])
def test_ragged_tiles(n):
    text = configs.C2.text
    m, ds, cols = setup(text, n, seed=n)
    th = jittered(m, text, seed=n)
    vals, grads, bad, _ = fb.nll_grad(m, ds, th)
    assert bad[0] == -1
    o = OracleModel(text)
    want = o.nll(cols, th)[1]
    assert abs(vals[0] - want) <= NLL_TOL * abs(want)
    g_ref, scale, est = ref_gradient(text, cols, th, m.param_names, n)
    free = [j for j, p in enumerate(m.param_names) if not m.is_constant(p)]
    assert np.all(np.abs(grads[0, free] - g_ref[free]) <= GRAD_TOL * scale[free] + est[free])


def test_invalid_event_gives_inf_and_nan_gradient():
    m = fb.Model.from_string(MIX)
    x = np.linspace(-4, 4, 5000)
    x[3210] = np.nan
    ds = fb.DataSet.from_columns({"x": x})
    vals, grads, bad, _ = fb.nll_grad(m, ds)
    assert vals[0] == np.inf and bad[0] == 3210
    assert np.all(np.isnan(grads[0]))


def test_empty_dataset():
    m = fb.Model.from_string(MIX)
    ds = fb.DataSet.from_columns({"x": np.zeros(0)})
    vals, grads, bad, _ = fb.nll_grad(m, ds)
    assert vals[0] == 0.0 and bad[0] == -1 and np.all(grads[0] == 0.0)
    w = configs.C4
    me = fb.Model.from_string(w.text)
    vals, grads, _, _ = fb.nll_grad(me, fb.DataSet.from_columns({"x": np.zeros(0)}))
    th = me.theta()
    names = me.param_names
    nu = sum(th[names.index(y)] for y in yields_of(w.text))
    assert vals[0] == pytest.approx(nu)
    for y in yields_of(w.text):
        assert grads[0, names.index(y)] == 1.0


def test_partial_and_finish_equal_the_one_call():
    """The multi-GPU split: per-shard slot pairs, combined, then the host finish with the
    global event count (what distributed.ShardedNll does for gradients)."""
    text = configs.C4.text
    m, ds, cols = setup(text, 40_000)
    th = jittered(m, text, seed=3)
    v_all, g_all, _, _ = fb.nll_grad(m, ds, th)
    half = 17_321
    shards = [fb.DataSet.from_columns({"x": cols[0][:half]}), fb.DataSet.from_columns({"x": cols[0][half:]})]
    sums = None
    for sh in shards:
        sc, bad = fb.nll_grad_partial(m, sh, th)
        assert bad[0] == -1
        s = sc[..., 0] + sc[..., 1]
        sums = s if sums is None else sums + s
    v, g = fb.nll_grad_finish(m, th, sums, 40_000)
    assert abs(v[0] - v_all[0]) <= NLL_TOL * abs(v_all[0])
    g_ref, scale, _ = ref_gradient(text, cols, th, m.param_names, 40_000, yields_of(text))
    assert np.all(np.abs(g[0] - g_all[0]) <= GRAD_TOL * scale)


def test_sharded_gradient_single_rank_equals_direct():
    """distributed.ShardedNll.nll_grad on one rank (no process group) reproduces nll_grad."""
    import torch
    import torch.distributed as dist

    from paper_2003_12875_b200 import distributed as D
    text = configs.C5.text
    m, ds, cols = setup(text, 70_001)
    th = jittered(m, text, seed=11)
    v0, g0, _, _ = fb.nll_grad(m, ds, th)
    sh = D.ShardedNll(m, ds, 70_001, 0, dist, torch.device("cuda:0"))
    v, g = sh.nll_grad(th)
    assert abs(v[0] - v0[0]) <= 1e-15 * abs(v0[0])
    assert np.allclose(g[0], g0[0], rtol=1e-14, atol=0)


@pytest.mark.parametrize("name", ["c2_gauss_argus", "c5_m0_free", "c4_extended", "c1_gauss", "c3_product",
                                  "sum_of_products", "prod_first_sum", "mix3_nested"])
def test_plan_specialised_gradient_pass(name, monkeypatch):
    """One-point gradients run the plan-specialised (NVRTC) pass -- single-column sums and
    products over up to three observables; it agrees with the generic pass and with the
    oracle-referenced gradient."""
    text, n = CASES[name]
    m, ds, cols = setup(text, n)
    th = jittered(m, text, seed=7)
    v_spec, g_spec, _, _ = fb.nll_grad(m, ds, th)
    assert fb.last_grad_jit(m)
    monkeypatch.setenv("FFB_NO_GRAD_SPEC", "1")
    v_gen, g_gen, _, _ = fb.nll_grad(m, ds, th)
    assert not fb.last_grad_jit(m)
    assert abs(v_spec[0] - v_gen[0]) <= 1e-13 * abs(v_gen[0])
    g_ref, scale, est = ref_gradient(text, cols, th, m.param_names, n, yields_of(text))
    for j, pname in enumerate(m.param_names):
        if m.is_constant(pname):
            assert g_spec[0, j] == 0.0
            continue
        assert abs(g_spec[0, j] - g_gen[0, j]) <= 1e-10 * scale[j]
        assert abs(g_spec[0, j] - g_ref[j]) <= GRAD_TOL * scale[j] + est[j]
