"""exp at the edges of its range on the GPU path, against the oracle (glibc semantics).

The reference evaluates every leaf with std::exp (proj/src/pdfs.cpp:15-33): between
exp(-745.13) and exp(-708.4) it returns SUBNORMAL values, so a density there is > 0 and
the event is valid (proj/src/eval.cpp:138-145); up to exp(709.78) it is finite.  The
device exp (csrc/fastmath.cuh exp_edge) must keep those semantics: a finite NLL where the
reference is finite, and the same first invalid event.

Every case runs through several launch shapes: one point (streaming kernel / graph
replay), 12 points (tile kernel), each in the static and the plan-specialised build.
"""
import math
import os

import numpy as np
import pytest

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs
from oracle.oracle import OracleModel
from tests.models import EXPO_EDGE, FAR_MIX, GAUSS_WIDE, edge_data, expo_edge_data, far_mix_data

pytestmark = pytest.mark.gpu

NLL_TOL = 1e-12
PER_EVENT = 1e-13
SMALLEST_NORMAL = 2.2250738585072014e-308
GOLD = os.path.join(os.path.dirname(__file__), "golden", "edge_models.npz")


def shapes(m, ds, base, moving, scale):
    """(P, spec, values, first_invalid) over the launch shapes; the points move the
    `moving` parameter by relative steps of `scale`."""
    k = m.param_names.index(moving)
    for P in (1, 12):
        pts = np.tile(base, (P, 1))
        pts[:, k] = base[k] * (1.0 + scale * np.arange(P))
        for spec in (False, True):
            old = fb.plan_spec_min_work(0 if spec else -1)
            try:
                vals, bad, _ = fb.nll_points(m, ds, pts)
            finally:
                fb.plan_spec_min_work(old)
            yield P, spec, pts, vals, bad


def check_against_oracle(text, cols, base, moving, scale, expect_bad=-1):
    m = fb.Model.from_string(text)
    o = OracleModel(text)
    ds = fb.DataSet.from_columns(dict(zip(m.observables, cols)))
    n_checked = 0
    for P, spec, pts, vals, bad in shapes(m, ds, base, moving, scale):
        for p in sorted({0, P - 1}):
            _, comp, ob = o.nll(cols, pts[p])
            assert ob == expect_bad, (P, spec, p, ob)
            assert bad[p] == ob, (P, spec, p, bad[p], ob)
            if ob < 0:
                assert math.isfinite(comp)
                assert abs(vals[p] - comp) <= NLL_TOL * abs(comp), (P, spec, p, vals[p], comp)
            else:
                assert vals[p] == math.inf
            n_checked += 1
    return m, o, ds, n_checked


def test_c1_gaussian_gradual_underflow():
    """C1's Gaussian at the sigma where the most distant event's exponent is -720:
    the reference's p there is subnormal (finite NLL); so must ours be."""
    w = configs.C1
    m = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(m, 20_011, w.data_seed)
    x = cols["x"]
    base = m.theta()
    mu = base[m.param_names.index("mean")]
    dmax = float(np.max(np.abs(x - mu)))
    sigma = dmax / math.sqrt(2.0 * 720.0)
    assert 0.1 < sigma < 10.0
    base[m.param_names.index("sigma")] = sigma
    o = OracleModel(w.text)
    p = o.probabilities([x], base)
    assert 0.0 < p.min() < SMALLEST_NORMAL  # the window the device used to flush to 0
    # sigma steps of 1e-5: exponents stay inside (-745, -707) for every point
    _, _, ds, n = check_against_oracle(w.text, [x], base, "sigma", 1e-5)
    assert n == 6  # P = 1: one point, P = 12: first and last; static and plan-specialised
    # per-event values: normal ones at the usual 1e-13, subnormal ones to their spacing
    got = fb.probabilities(m, ds, point=base)
    normal = p >= SMALLEST_NORMAL
    assert np.max(np.abs(got[normal] - p[normal]) / p[normal]) <= PER_EVENT
    sub = ~normal
    assert np.all(got[sub] > 0.0)
    assert np.all(np.abs(got[sub] - p[sub]) <= np.maximum(4 * 2.0 ** -1074, 1e-9 * p[sub]))


def test_c3_gaussian_factor_gradual_underflow():
    """C3's product with the x-Gaussian at sigma ~ 0.13 (exponent -720 at the edge)."""
    w = configs.C3
    m = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(m, 20_011, w.data_seed)
    base = m.theta()
    x = cols["x"]
    mu = base[m.param_names.index("mu")]
    sigma = float(np.max(np.abs(x - mu))) / math.sqrt(2.0 * 720.0)
    assert 0.1 < sigma < 5.0
    base[m.param_names.index("sigma")] = sigma
    xs = [cols[k] for k in m.observables]
    assert OracleModel(w.text).probabilities(xs, base).min() < SMALLEST_NORMAL
    check_against_oracle(w.text, xs, base, "sigma", 1e-5)


@pytest.mark.parametrize("name", sorted({k.split("/")[0] for k in np.load(GOLD).files}))
def test_exp_edges_against_reference_golden(name):
    """The reference's own values (tests/golden/make_edge_golden.py): first_invalid equal,
    NLL within 1e-12 of both its sums, per-event values within 1e-13 where normal and to a
    few subnormal spacings where the reference's p is subnormal."""
    g = np.load(GOLD)
    text = bytes(g[f"{name}/text"]).decode()
    x, p, sc = g[f"{name}/x"], g[f"{name}/p"], g[f"{name}/scalars"]
    m = fb.Model.from_string(text)
    ds = fb.DataSet.from_columns({"x": x})
    v = fb.nll(m, ds)
    assert v.first_invalid == int(sc[2])
    if sc[2] < 0:
        assert abs(v.value - sc[1]) <= NLL_TOL * abs(sc[1])
        assert abs(v.value - sc[0]) <= NLL_TOL * abs(sc[0])
    else:
        assert v.value == math.inf
    # the same point 12 times: the tile kernel, static and plan-specialised
    for spec in (False, True):
        old = fb.plan_spec_min_work(0 if spec else -1)
        try:
            vals, bad, _ = fb.nll_points(m, ds, np.tile(m.theta(), (12, 1)))
        finally:
            fb.plan_spec_min_work(old)
        assert np.all(bad == int(sc[2]))
        if sc[2] < 0:
            assert np.all(np.abs(vals - sc[1]) <= NLL_TOL * abs(sc[1])), (spec, vals[0], sc[1])
        else:
            assert np.all(vals == math.inf)
    got = fb.probabilities(m, ds)
    normal = p >= SMALLEST_NORMAL
    assert np.max(np.abs(got[normal] - p[normal]) / p[normal]) <= PER_EVENT
    sub = (p > 0) & ~normal
    assert np.all(got[sub] > 0.0)
    assert np.all(np.abs(got[sub] - p[sub]) <= np.maximum(4 * 2.0 ** -1074, 1e-9 * p[sub]))
    assert np.all(got[p == 0] == 0.0)


@pytest.mark.parametrize("sub_at,zero_at", [(3, 10), (10, 3)])
def test_first_invalid_across_the_underflow_window(sub_at, zero_at):
    """An event at exponent -720 is valid (subnormal p, as glibc); one at -800 is not.
    first_invalid is the first event whose p underflows to 0, wherever the subnormal one is,
    in every launch shape."""
    base = fb.Model.from_string(GAUSS_WIDE).theta()
    check_against_oracle(GAUSS_WIDE, [edge_data(sub_at, zero_at)], base, "sigma", 1e-6, expect_bad=zero_at)
    check_against_oracle(GAUSS_WIDE, [edge_data(sub_at, None)], base, "sigma", 1e-6)


def test_mixture_with_a_component_in_the_window():
    """A sum whose only non-zero component sits in the underflow window at some events."""
    x = far_mix_data()
    o = OracleModel(FAR_MIX)
    base = fb.Model.from_string(FAR_MIX).theta()
    p = o.probabilities([x], base)
    assert 0.0 < p[1234] < SMALLEST_NORMAL and 0.0 < p[17] < SMALLEST_NORMAL
    check_against_oracle(FAR_MIX, [x], base, "f", 1e-4)


def test_exponential_near_overflow():
    """exp(c x) with c x in (707, 709.78]: finite in the reference, finite here; c steps
    downward so c x stays below the overflow threshold at every point."""
    base = fb.Model.from_string(EXPO_EDGE).theta()
    check_against_oracle(EXPO_EDGE, [expo_edge_data()], base, "c", -1e-6)
