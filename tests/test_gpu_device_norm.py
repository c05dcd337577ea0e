"""Device-side numeric normalisation: the reference's adaptive Simpson
(integrate_adaptive_simpson, proj/src/eval.cpp:14-69) run on the GPU -- one warp per parameter
point, one lane per pre-panel -- against the host quadrature (bit-identical to the
reference's, tests/test_oracle.py) and, through the likelihood, against the oracle.

Tolerances: a normalisation within 1e-13 relative of the host's value (the two differ by the
device leaves' <= 2 ulp and, rarely, by a bisection decided the other way, both far below the
rule's own 1e-10 tolerance); NLL within the north_star's 1e-12.
"""
import numpy as np
import pytest

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs
from oracle.oracle import OracleModel
from tests.models import ARGUS_REF, EXPR_MODELS, REF_MODELS

pytestmark = pytest.mark.gpu

NORM_TOL = 1e-13
NLL_TOL = 1e-12

ARGUS_P = """
observable x 5.2 5.29
parameter m0 5.291 5.0 5.4 const
parameter c -20 -100 10
parameter p 0.7 0 2
pdf bkg ArgusBG(x, m0, c, p)
"""

# pdf name -> model text; every node named here has no closed-form normalisation
CASES = {
    "chisq": (REF_MODELS["chisq"][0], ["q"]),
    "johnson": (REF_MODELS["johnson"][0], ["j"]),
    "mix_chisq": (REF_MODELS["mix_chisq"][0], ["q", "m"]),  # a sum over a Simpson-normalised leaf
    "argus_ref_text": (ARGUS_REF, ["bkg", "model"]),        # BASELINE config 2 as the reference spells it
    "cheb3_expr": (EXPR_MODELS["cheb3"][0], ["ch"]),
    "poly2_expr": (EXPR_MODELS["poly2"][0], ["po"]),
    "argus_p07": (ARGUS_P, ["bkg"]),
}


def jitter(m, n_points, seed, text=None):
    """Points around the model's values: +-2 % of each free parameter's declared range (parsed
    from the model text), clipped to the range; constants stay.  Row 0 is the model's values."""
    rng = np.random.default_rng(seed)
    th = m.theta()
    ranges = {}
    for line in (text or "").splitlines():
        tok = line.split()
        if len(tok) >= 5 and tok[0] == "parameter":
            ranges[tok[1]] = (float(tok[3]), float(tok[4]))
    pts = np.repeat(th[None, :], n_points, axis=0)
    for j, name in enumerate(m.param_names):
        if m.is_constant(name):
            continue
        lo, hi = ranges.get(name, (th[j] - 1.0, th[j] + 1.0))
        span = 0.02 * (hi - lo)
        pts[1:, j] = np.clip(th[j] + span * (2.0 * rng.random(n_points - 1) - 1.0), lo, hi)
    return pts


@pytest.mark.parametrize("name", list(CASES))
def test_device_quadrature_matches_the_host_quadrature(name):
    text, pdfs = CASES[name]
    m = fb.Model.from_string(text)
    pts = jitter(m, 24, 11, text)
    for pdf in pdfs:
        before = fb.device_normalization_launches(m)
        got = fb.device_normalization(m, pdf, pts)
        assert fb.device_normalization_launches(m) > before
        want = np.array([fb.normalization(m, pdf, p) for p in pts])
        assert np.all(np.abs(got - want) <= NORM_TOL * np.abs(want)), (pdf, np.max(np.abs(got / want - 1)))
    # the current values (points = None)
    one = fb.device_normalization(m, pdfs[-1])
    assert abs(one[0] - fb.normalization(m, pdfs[-1])) <= NORM_TOL * abs(one[0])


def test_closed_forms_stay_closed_forms():
    m = fb.Model.from_string(REF_MODELS["mix"][0])
    pts = jitter(m, 5, 3, REF_MODELS["mix"][0])
    for pdf in ("s", "b", "m"):
        got = fb.device_normalization(m, pdf, pts)
        want = np.array([fb.normalization(m, pdf, p) for p in pts])
        assert np.array_equal(got, want)
    assert fb.device_normalization_launches(m) == 0


@pytest.mark.parametrize("name", ["mix_chisq", "argus_ref_text", "johnson"])
def test_likelihood_with_device_normalisation(name):
    """NLL, probabilities and eval_batch with the model's switch on: against the host-normalised
    values of the same library and against the oracle; the quadrature launches once per
    Simpson-normalised node, whatever the number of points."""
    text, pdfs = CASES[name]
    m = fb.Model.from_string(text)
    cols, _ = fb.sample_host(m, 20_011, 17)
    ds = fb.DataSet.from_columns(cols)
    pts = jitter(m, 12, 5, text)
    host_vals, host_bad, _ = fb.nll_points(m, ds, pts)
    host_p = fb.probabilities(m, ds)
    assert not fb.device_normalization_enabled(m)
    fb.set_device_normalization(m, True)
    assert fb.device_normalization_enabled(m)
    l0 = fb.device_normalization_launches(m)
    dev_vals, dev_bad, _ = fb.nll_points(m, ds, pts)
    assert fb.device_normalization_launches(m) - l0 == len(pdfs)
    l1 = fb.device_normalization_launches(m)
    fb.nll_points(m, ds, pts[:3])
    assert fb.device_normalization_launches(m) - l1 == len(pdfs)  # independent of P
    assert np.array_equal(dev_bad, host_bad)
    assert np.all(np.abs(dev_vals - host_vals) <= NORM_TOL * np.abs(host_vals))
    dev_p = fb.probabilities(m, ds)
    assert np.max(np.abs(dev_p - host_p) / host_p) <= NORM_TOL
    # the checker at a few points: the oracle (C restatement of the reference), or -- for the
    # formula model, which the oracle does not parse -- the reference engine itself
    x = cols[m.observables[0]]
    if "Expression" in text:
        from oracle.oracle import RefDataset, RefModel, ref_available
        if ref_available():
            r, rds = RefModel(text), RefDataset(m.observables[0], x)
            for p in (0, 5, 11):
                for pname, v in zip(m.param_names, pts[p]):
                    if not m.is_constant(pname):
                        r.set(pname, v)
                want = r.nll_compensated(rds)[0]
                assert abs(dev_vals[p] - want) <= NLL_TOL * abs(want)
    else:
        o = OracleModel(text)
        for p in (0, 5, 11):
            want = o.nll([x], theta=pts[p])[1]
            assert abs(dev_vals[p] - want) <= NLL_TOL * abs(want)
    fb.set_device_normalization(m, False)
    again, _, _ = fb.nll_points(m, ds, pts)
    assert np.array_equal(again, host_vals)


def test_reference_config2_text_full_launch():
    """BASELINE config 2 as the reference spells it (ArgusBG as a formula, Simpson-normalised)
    at the config's 200 points: device-normalised NLLs against the host-normalised ones."""
    w = configs.C2
    m = fb.Model.from_string(configs.REFERENCE_TEXTS[w.name])
    cols, _ = fb.sample_host(fb.Model.from_string(w.text), 50_021, 9)
    ds = fb.DataSet.from_columns(cols)
    pts = w.points(m, n_points=200)
    host_vals, _, _ = fb.nll_points(m, ds, pts)
    fb.set_device_normalization(m, True)
    dev_vals, _, _ = fb.nll_points(m, ds, pts)
    assert np.all(np.abs(dev_vals - host_vals) <= NORM_TOL * np.abs(host_vals))


def test_non_finite_integrand_is_a_numeric_error():
    """proj/src/eval.cpp:21-22,61-63: a non-finite integrand value is a Numeric error (x = 1 is a
    pre-panel boundary of [0, 2])."""
    m = fb.Model.from_string('observable x 0 2\nparameter a 1 0.5 2\npdf e Expression("a/(x-1)^2", x, a)\n')
    with pytest.raises(fb.FfitError) as host:
        fb.normalization(m, "e")
    with pytest.raises(fb.FfitError) as dev:
        fb.device_normalization(m, "e")
    assert dev.value.code == host.value.code
    out = np.full(2, -1.0)
    with pytest.raises(fb.FfitError):
        fb.device_normalization(m, "e", np.array([[1.0], [1.5]]))
    assert np.all(out == -1.0)


def test_degenerate_normalisation_is_rejected():
    """A formula that integrates to <= 0 is a degenerate PDF on both paths (proj/src/eval.cpp:79-84)."""
    m = fb.Model.from_string('observable x -1 1\nparameter a 1 0.5 2\npdf e Expression("a*x", x, a)\n')
    x = np.linspace(-0.9, 0.9, 101)
    ds = fb.DataSet.from_columns({"x": x})
    with pytest.raises(fb.FfitError) as host:
        fb.nll(m, ds)
    fb.set_device_normalization(m, True)
    with pytest.raises(fb.FfitError) as dev:
        fb.nll(m, ds)
    assert dev.value.code == host.value.code
