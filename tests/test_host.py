"""Host side of the product, no GPU needed: the C-ABI library loads and exports every
symbol include/ffit_b200.h declares; parser / error codes follow the reference; the
flattened plan, the per-point constants, the host normalisations and the seeded
generator agree with the oracle."""
import math
import os
import re

import numpy as np
import pytest

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs
from paper_2003_12875_b200._lib import LIB_PATH, SIGNATURES
from oracle.oracle import OracleModel
from tests.models import EXPR_MODELS, MIX, REF_MODELS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "ffit_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(ff(?:it|cu)_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    declared = header_symbols()
    assert declared, "no symbols parsed from the header"
    missing = declared - exported
    assert not missing, f"declared but not exported: {sorted(missing)}"
    assert declared == set(SIGNATURES), "ctypes signature table out of sync with the header"
    fb.lib()  # binds every symbol with its argtypes


def test_no_cpu_fallback_in_product():
    """The product never links or loads the oracle (the checker)."""
    import subprocess
    out = subprocess.run(["nm", "-D", LIB_PATH], capture_output=True, text=True).stdout
    syms = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    assert not any(s.startswith(("orc_", "ref_")) for s in syms)
    for fn in os.listdir(os.path.join(ROOT, "paper_2003_12875_b200")):
        if fn.endswith(".py"):
            src = open(os.path.join(ROOT, "paper_2003_12875_b200", fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn


def test_reference_models_parse_and_params():
    for name, (text, _) in REF_MODELS.items():
        m = fb.Model.from_string(text)
        o = OracleModel(text)
        assert m.param_names == o.param_names
        assert np.array_equal(m.theta(), o.theta)


def test_parse_errors_use_reference_codes():
    with pytest.raises(fb.FfitError) as e:
        fb.Model.from_string("observable x 0 1\npdf g Gaussian(x, mu, sigma)\n")
    assert e.value.code == 2 and "undeclared name: mu" in e.value.message  # proj/src/model.cpp:122-125
    with pytest.raises(fb.FfitError) as e:
        fb.Model.from_string("observable x 0 1\nparameter a 1 0 2\npdf g Bogus(x, a)\n")
    assert e.value.code == 2 and "unknown pdf kind" in e.value.message
    with pytest.raises(fb.FfitError) as e:
        fb.Model.from_string("observable x 0 1\nparameter a 5 0 2\n")
    assert e.value.code == 1  # value outside range: Graph::add_parameter, Usage
    with pytest.raises(fb.FfitError) as e:  # formula errors become model-file parse errors
        fb.Model.from_string('observable x 0 1\nparameter a 1 0 2\npdf e Expression("a*x+", x, a)\n')
    assert e.value.code == 2 and "syntax error at offset 4" in e.value.message
    with pytest.raises(fb.FfitError) as e:
        fb.Model.from_string("observable x 0 1\nparameter a 1 0 2\n")
    assert e.value.code == 2 and "no pdf" in e.value.message
    with pytest.raises(fb.FfitError) as e:  # ProdPdf needs independent observables
        fb.Model.from_string("observable x 0 1\nparameter a 1 0 2\npdf e Exponential(x, a)\n"
                             "pdf f Exponential(x, a)\npdf p ProdPdf(e, f)\n")
    assert e.value.code == 2 and "distinct observables" in e.value.message


def test_set_param_range_and_constant():
    m = fb.Model.from_string(configs.C2.text)
    m.set("m", 5.28)
    assert m.get("m")[0] == 5.28
    with pytest.raises(fb.FfitError) as e:
        m.set("m", 6.0)
    assert e.value.code == 3  # proj/src/graph.cpp:121-124
    with pytest.raises(fb.FfitError) as e:
        m.set("m0", 5.3)
    assert e.value.code == 1
    assert m.is_constant("m0") and not m.is_constant("m")


def test_plan_structure():
    # flags: 1 END_SUM, 2 END_PROD, 4 BEGIN_SUM, 8 BEGIN_PROD
    kinds = {"GAUSS": 0, "EXPO": 1, "ARGUS": 4, "CHEB": 5}
    t, nc, st = fb.Model.from_string(configs.C1.text).plan()
    assert [(x["kind"], x["flags"]) for x in t] == [(kinds["GAUSS"], 15)] and nc == 1 and st == 3
    t, nc, st = fb.Model.from_string(configs.C2.text).plan()
    assert [(x["kind"], x["flags"]) for x in t] == [(0, 4), (4, 11)] and nc == 1
    t, nc, st = fb.Model.from_string(configs.C3.text).plan()
    assert [(x["kind"], x["col"], x["flags"]) for x in t] == [(0, 0, 13), (1, 1, 5), (5, 2, 7)] and nc == 3
    assert t[2]["order"] == 3
    t, nc, st = fb.Model.from_string(configs.C4.text).plan()
    assert len(t) == 6 and t[-1]["flags"] == 11 and t[0]["flags"] == 4
    assert all(x["flags"] == 0 for x in t[1:-1])


def test_sum_of_products_plan():
    text = """
observable x -5 5
observable y 0 10
parameter m 0 -1 1
parameter s 1 0.1 3
parameter c -0.5 -2 0
parameter c2 -0.1 -2 0
parameter f 0.3 0 1
pdf gx Gaussian(x, m, s)
pdf ey Exponential(y, c)
pdf ex Exponential(x, c2)
pdf ey2 Exponential(y, c2)
pdf sig ProdPdf(gx, ey)
pdf bkg ProdPdf(ex, ey2)
pdf model AddPdf(sig, f, bkg)
"""
    m = fb.Model.from_string(text)
    t, nc, _ = m.plan()
    assert [x["flags"] for x in t] == [13, 7, 13, 7] and nc == 2
    o = OracleModel(text)
    assert fb.normalization(m) == o.normalization()


def test_point_constants_fold_normalisations():
    w = configs.C2
    m = fb.Model.from_string(w.text)
    o = OracleModel(w.text)
    row = m.point_constants()
    th = m.theta()
    names = m.param_names
    v = dict(zip(names, th))
    n_sig = o.normalization(node=0)
    n_bkg = o.normalization(node=1)
    n_mod = o.normalization()
    # [coef_g, mu, -1/(2s^2), coef_a, m0, c, p, 1/m0]
    assert row[1] == v["m"] and row[2] == -1.0 / (2.0 * v["s"] * v["s"])
    assert row[0] == pytest.approx((v["f"] / n_sig) / n_mod, rel=2e-16)
    assert row[3] == pytest.approx(((1 - v["f"]) / n_bkg) / n_mod, rel=2e-16)
    assert list(row[4:]) == [v["m0"], v["c"], v["p"], 1.0 / v["m0"], 0.0]  # + the launch-cache flag


@pytest.mark.parametrize("name", list(REF_MODELS) + list(EXPR_MODELS))
def test_host_normalisation_matches_oracle(name):
    text = REF_MODELS[name][0] if name in REF_MODELS else EXPR_MODELS[name][1]
    m = fb.Model.from_string(text)
    o = OracleModel(text)
    assert fb.normalization(m) == pytest.approx(o.normalization(), rel=1e-15)


@pytest.mark.parametrize("name", list(REF_MODELS) + list(EXPR_MODELS) + ["C2", "C3", "C4"])
def test_generator_bit_identical_to_oracle(name):
    if name in REF_MODELS:
        text, seed = REF_MODELS[name]
    elif name in EXPR_MODELS:
        text, seed = EXPR_MODELS[name][1], EXPR_MODELS[name][2]
    else:
        w = getattr(configs, name)
        text, seed = w.text, w.data_seed
    m = fb.Model.from_string(text)
    o = OracleModel(text)
    cols, eff = fb.sample_host(m, 5000, seed)
    ocols, oeff = o.sample(5000, seed)
    assert eff == oeff
    for k, oc in zip(m.observables, ocols):
        assert np.array_equal(cols[k], oc)


def test_reference_sampler_golden():
    """The generator reproduces the reference sampler's own output (golden)."""
    g = np.load(os.path.join(ROOT, "tests", "golden", "ref_models.npz"))
    for name, (text, seed) in REF_MODELS.items():
        m = fb.Model.from_string(text)
        x = g[f"{name}/x"]
        cols, _ = fb.sample_host(m, len(x), seed)
        assert np.array_equal(cols["x"], x), name


def test_workload_points_reproducible():
    m = fb.Model.from_string(configs.C2.text)
    a = configs.C2.points(m)
    b = configs.C2.points(m)
    assert a.shape == (200, len(m.param_names)) and np.array_equal(a, b)
    names = m.param_names
    base = m.theta()
    k = names.index("s")
    assert np.all(np.abs(a[:, k] / base[k] - 1) <= 0.1)
    assert np.all(a[:, names.index("m0")] == base[names.index("m0")])


def test_configs_rng_matches_reference_stream():
    from oracle.oracle import rng_uniform
    r = configs.Rng(2002)
    assert [r.uniform() for _ in range(50)] == list(rng_uniform(2002, 50))


def test_extended_terms_host():
    m = fb.Model.from_string(configs.C4.text)
    pts = configs.C4.points(m, n_points=3)
    ext = m.extended_terms(pts, 1e8)
    names = m.param_names
    for p in range(3):
        nu = sum(pts[p, names.index(n)] for n in ("n1", "n2", "n3", "n4", "n5", "nb"))
        assert ext[p] == pytest.approx(nu - 1e8 * math.log(nu), rel=1e-15)
    assert fb.Model.from_string(MIX).extended_terms(fb.Model.from_string(MIX).theta(), 10)[0] == 0.0


def test_gpu_calls_fail_loudly_without_device():
    """No CPU fallback: on a machine without a usable GPU the evaluation path errors."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(fb.FfitError) as e:
        fb.DataSet.from_columns({"x": np.zeros(10)})
    assert e.value.code == 3 and "CUDA" in e.value.message


def test_gradient_slot_layout():
    """Accumulators of the fused NLL + gradient pass (plan.hpp DevGradPlan): slot 0, then
    per term one A slot plus one B slot per FREE leaf parameter."""
    from paper_2003_12875_b200 import configs
    # C2: Gaussian (m, s free) + ArgusBG (m0, p const; c free)
    assert fb.grad_slot_count(fb.Model.from_string(configs.C2.text)) == 1 + 3 + 2
    # C5: m0 free too
    assert fb.grad_slot_count(fb.Model.from_string(configs.C5.text)) == 1 + 3 + 3
    # C4: 5 Gaussians (2 each) + Exponential (1)
    assert fb.grad_slot_count(fb.Model.from_string(configs.C4.text)) == 1 + 5 * 3 + 2
    # C3: Gaussian, Exponential, Chebychev-3
    assert fb.grad_slot_count(fb.Model.from_string(configs.C3.text)) == 1 + 3 + 2 + 4


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5", "johnson", "mix_chisq"])
def test_coefficient_derivatives(name):
    """d coef_c / d theta_j of the gradient pass's host side against 4-point differences
    of the constant builder at several steps (the closest one: the builder's own
    rounding bounds the difference quotients, not the analytic side)."""
    from paper_2003_12875_b200 import configs
    from tests.models import REF_MODELS
    text = {"c2": configs.C2.text, "c3": configs.C3.text, "c4": configs.C4.text, "c5": configs.C5.text,
            "johnson": REF_MODELS["johnson"][0], "mix_chisq": REF_MODELS["mix_chisq"][0]}[name]
    m = fb.Model.from_string(text)
    terms, _, _ = m.plan()
    coffs = [t["coff"] for t in terms]
    th = m.theta()
    spans = {}
    for line in text.splitlines():
        t = line.split()
        if t and t[0] == "parameter":
            spans[t[1]] = (float(t[4]) - float(t[3]), len(t) > 5)
    base = np.abs(m.point_constants(th)[coffs])
    for j, pn in enumerate(m.param_names):
        span, const = spans[pn]
        if const:
            continue
        d = m.coef_derivatives(j, th)
        ests = []
        for hr in (1e-6, 3e-6, 1e-5, 3e-5, 1e-4):
            h = hr * span

            def C(dx):
                t = th.copy()
                t[j] += dx
                return m.point_constants(t)[coffs]

            ests.append((8 * (C(h) - C(-h)) - (C(2 * h) - C(-2 * h))) / (12 * h))
        err = np.min(np.abs(np.array(ests) - d), axis=0)
        assert np.all(err <= 1e-9 * np.maximum(np.abs(d), base)), (pn, err)


@pytest.mark.parametrize("w", configs.BY_INDEX[:4], ids=lambda w: w.name)
def test_plan_specialised_source_compiles_with_nvrtc(w):
    """The plan-specialised likelihood (the tile kernel around the launch's term list,
    launch-constant rewrite included) compiles to sm_100a SASS with NVRTC, no GPU needed."""
    m = fb.Model.from_string(w.text)
    pts = w.points(m, n_points=16)
    src = fb.plan_spec_source(m, pts, compile=True)
    nterms = {"c1": 1, "c2": 2, "c3": 3, "c4": 6}[w.name[:2]]
    assert "struct PlanSpec" in src and f"nterms = {nterms};" in src
    if w.name.startswith("c2"):
        # ArgusBG with m0 fixed over the points: the cached kind (plan.hpp LK_ARGUS_CACHED = 8)
        assert "{8, 0, 1, " in src
    assert fb.plan_spec_source(m, compile=True)  # the plan without points: as built


def test_plan_spec_threshold_switch():
    old = fb.plan_spec_min_work(-2)
    try:
        assert fb.plan_spec_min_work(0) == old
        assert fb.plan_spec_min_work(-1) == 0
        assert fb.plan_spec_min_work(-2) == -1
    finally:
        fb.plan_spec_min_work(old)


def test_from_device_rejects_what_the_kernels_cannot_read():
    """DataSet.from_device checks dtype, device, contiguity and lengths before the view is
    made (the kernels read n fp64 values from each pointer)."""
    import torch
    good = torch.zeros(16, dtype=torch.float64)
    cases = {
        "float32": {"x": torch.zeros(16, dtype=torch.float32)},
        "host tensor": {"x": good},
        "no columns": {},
    }
    for what, cols in cases.items():
        with pytest.raises(fb.FfitError) as e:
            fb.DataSet.from_device(cols)
        assert e.value.code == fb.ffit.USAGE, what

    class FakeCuda:  # a CUDA tensor's surface, without a GPU
        def __init__(self, n, dtype="torch.float64", contiguous=True, index=0):
            self._n, self.dtype, self._c = n, dtype, contiguous
            self.device = type("D", (), {"type": "cuda", "index": index})()

        def numel(self):
            return self._n

        def is_contiguous(self):
            return self._c

        def data_ptr(self):
            return 256

    bad = {
        "strided": {"x": FakeCuda(16, contiguous=False)},
        "ragged": {"x": FakeCuda(16), "y": FakeCuda(15)},
        "two devices": {"x": FakeCuda(16), "y": FakeCuda(16, index=1)},
        "float32 cuda": {"x": FakeCuda(16, dtype="torch.float32")},
    }
    for what, cols in bad.items():
        with pytest.raises(fb.FfitError) as e:
            fb.DataSet.from_device(cols)
        assert e.value.code == fb.ffit.USAGE, what
    with pytest.raises(fb.FfitError):
        fb.DataSet.from_device({"x": FakeCuda(16, index=1)}, device=0)
