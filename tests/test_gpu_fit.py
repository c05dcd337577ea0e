"""Fit drivers on the GPU likelihood against the reference's own fits (golden values
from tests/golden/ref_fits.json, produced by the unmodified reference Nelder-Mead,
proj/src/fit.cpp:86-251).  Target (BASELINE north_star): fitted parameters within 1e-6,
read as |d theta| <= 1e-6 * max(1, |theta|): Nelder-Mead stops anywhere inside its NLL
tolerance, so two fits whose NLLs differ in the last bits (here ~1e-14 relative: libdevice
vs glibc exp/log, Expression vs closed-form ArgusBG) stop ~sqrt(2 tol) sigma apart.
"""
import json
import os

import numpy as np
import pytest

import paper_2003_12875_b200 as fb
from oracle.oracle import OracleModel
from tests.models import FIT_CASES

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_fits.json")))


def data_for(case):
    gen = fb.Model.from_string(case["ours_text"])
    for k, v in case.get("truth", {}).items():
        gen.set(k, v)
    cols, _ = fb.sample_host(gen, case["n"], case["seed"])
    return fb.DataSet.from_columns(cols), cols


def start_model(case):
    m = fb.Model.from_string(case["ours_text"])
    for k, v in case.get("start", {}).items():
        m.set(k, v)
    return m


@pytest.mark.parametrize("name", list(FIT_CASES))
def test_nelder_mead_matches_reference_fit(name):
    case, gold = FIT_CASES[name], GOLD[name]
    ds, _ = data_for(case)
    m = start_model(case)
    r = fb.fit_to(m, ds, tolerance=case["tol"])
    assert r.converged and gold["converged"]
    assert r.uncertainties_valid
    for p in r.parameters:
        want, unc = gold["params"][p.name]
        assert abs(p.value - want) <= 1e-6 * max(1.0, abs(want)), (p.name, p.value, want)
        assert p.uncertainty == pytest.approx(unc, rel=1e-3)
        assert m.get(p.name)[0] == p.value  # written back (proj/src/fit.cpp:228-246)
    assert abs(r.nll_min - gold["nll"]) <= 1e-12 * abs(gold["nll"]) + 1e-9
    assert r.n_launches < r.n_nll_calls  # independent points were batched


@pytest.mark.parametrize("analytic", [False, True], ids=["fd", "analytic"])
@pytest.mark.parametrize("name", list(FIT_CASES))
def test_gradient_fit_reaches_reference_minimum(name, analytic):
    case, gold = FIT_CASES[name], GOLD[name]
    ds, _ = data_for(case)
    m = start_model(case)
    r = fb.fit_gradient(m, ds, tolerance=1e-12, max_iterations=200, analytic=analytic)
    assert r.converged
    assert r.analytic_gradient == analytic
    # the achievable agreement: the reference's Nelder-Mead stops once its simplex's NLL
    # spread is below tol, i.e. anywhere with NLL - NLL_min <~ tol, up to sqrt(2 tol) sigma
    # from the minimum in any direction (x10 for a minimum outside the final simplex); the
    # gradient fit ends with a Newton step on the full Hessian, ~1e-6 sigma from it
    for p in r.parameters:
        want, unc = gold["params"][p.name]
        bound = 10.0 * np.sqrt(2.0 * case["tol"]) * unc + 1e-9 * max(1.0, abs(want))
        assert abs(p.value - want) <= bound, (p.name, p.value, want, bound)
    assert r.nll_min <= gold["nll"] + 1e-7
    assert r.uncertainties_valid
    for p in r.parameters:  # the reference's Hessian uncertainties
        assert p.uncertainty == pytest.approx(gold["params"][p.name][1], rel=1e-3)
    d = len(r.parameters)
    hess = 1 + 2 * d + 2 * d * (d - 1)  # the one Hessian launch
    L = r.n_launches
    if analytic:
        # the start launch (centre + 2d gradient points), one point per launch, the Hessian
        # from the gradients at u and u +- h e_i (2d+1 points, one launch), and the Newton
        # step (one point) if it was predicted to gain
        assert r.n_nll_calls in ((2 * d + 1) + (L - 3) + (2 * d + 1) + 1, (2 * d + 1) + (L - 2) + (2 * d + 1))
    else:
        # every iteration is one launch of 2d+1 points, the Hessian one launch, the Newton step
        assert r.n_nll_calls in ((L - 2) * (2 * d + 1) + hess + 1, (L - 1) * (2 * d + 1) + hess)


def test_fit_nll_matches_oracle_at_minimum():
    case = FIT_CASES["argus_mix"]
    ds, cols = data_for(case)
    m = start_model(case)
    r = fb.fit_to(m, ds, tolerance=case["tol"])
    o = OracleModel(case["ours_text"])
    th = m.theta()
    _, comp, _ = o.nll([cols["x"]], th)
    assert abs(r.nll_min - comp) <= 1e-12 * abs(comp)


def test_hessian_points_batched_into_one_launch():
    case = FIT_CASES["gauss_closure"]
    ds, _ = data_for(case)
    m = start_model(case)
    r = fb.fit_to(m, ds, tolerance=1e-8)
    gold = GOLD["gauss_closure"]
    for p in r.parameters:
        assert abs(p.value - gold["params"][p.name][0]) <= 5 * p.uncertainty * 1e-3 + 1e-6
    assert np.isfinite(r.nll_min)


C5_GOLD = os.path.join(os.path.dirname(__file__), "golden", "c5_cpu_fit.json")


@pytest.mark.slow
def test_c5_fit_matches_the_cpu_fit():
    """BASELINE config 5: the config-2 model at 2e8 events with 5 free parameters (m0 free),
    fitted on the GPU -- BFGS on central differences (2d+1 points per launch), on the fused
    analytic gradient, and through the event-sharded group (ffcu_shard_group_fit_gradient,
    one rank here) -- against the CPU fit (tests/golden/make_c5_fit.py: Newton on the
    oracle's NLL over all 2e8 events, converged to 1e-6 sigma): every fitted parameter
    within 1e-6 (absolute), the minimum NLL within 1e-12, the uncertainties within 1 %."""
    from paper_2003_12875_b200 import configs
    gold = json.load(open(C5_GOLD))
    w = configs.C5
    assert gold["workload"] == w.name and gold["n_events"] == w.n_events
    truth = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(truth, w.n_events, w.data_seed)
    ds = fb.DataSet.from_columns(cols)
    del cols
    for how in ("fd", "analytic", "sharded"):
        m = fb.Model.from_string(w.text)
        for k, v in gold["start"].items():
            m.set(k, v)
        if how == "sharded":
            pytest.importorskip("torch")
            r = fb.ShardGroup.for_rank(m, ds, w.n_events, 0, 1, 0).fit_gradient(tolerance=1e-12, max_iterations=100,
                                                                               analytic=False)
        else:
            r = fb.fit_gradient(m, ds, tolerance=1e-12, max_iterations=100, analytic=how == "analytic")
        assert r.converged, how
        assert set(p.name for p in r.parameters) == set(gold["parameters"])
        for p in r.parameters:
            want = gold["parameters"][p.name]
            assert abs(p.value - want) <= 1e-6, (how, p.name, p.value, want, p.value - want)
            assert p.uncertainty == pytest.approx(gold["sigma"][p.name], rel=1e-2), (how, p.name)
        assert abs(r.nll_min - gold["nll_min"]) <= 1e-12 * abs(gold["nll_min"]), (how, r.nll_min, gold["nll_min"])
