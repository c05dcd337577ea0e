"""The Expression formula language on the host, against the
reference's own compiler and scalar program (oracle/_ref, proj/src/expr.cpp): the same
values bit for bit and the same error messages, then Expression pdfs end to end on the
host side (normalisation by the reference's adaptive Simpson, the toy generator)."""
import numpy as np
import pytest

import paper_2003_12875_b200 as fb
from oracle.oracle import RefModel, ref_available, ref_expr_eval
from tests.models import EXPR_MODELS

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")

VARS = ["x", "m0", "c", "z", "a1", "a2", "k"]

FORMULAS = [
    "x*sqrt(1-(x/m0)^2)*exp(c*(1-(x/m0)^2))",  # ArgusBG as the reference spells it
    "1 + a1*z + a2*(2*z^2-1)",
    "-x^2", "(-x)^2", "-x^-2", "2^3^2", "2^-1", "x^0.5", "x^k",
    "pow(x, 3) + pow(x, 2.5) + pow(x, 4) - pow(2, 3)",
    "x^4 - x^3 + x^2", "(x*x)*(x*x) - x^4",
    "-(-x)", "- - x", "x - -x", "x/3/7", "x/(3/7)", "x*3/7",
    "exp(log(x)) * sin(x) / cos(x)", "abs(z) - sinh(z) + asinh(z)",
    "1.e-3*x + .25 - 1. + 2e2 + 1E-1", "((x))", "  x  +  1  ",
    "exp(-0.5*((x-m0)/k)^2)", "log(x) * k - 0.5*x", "sqrt(2)*x + 3*4 - 12",
    "exp(1000*x)", "log(z)", "sqrt(z)", "x/(z-z)",
]

BAD = ["x+", "x*(y)", "foo(x)", "pow(x)", "exp(x, 2)", "x $ 2", "(x", "x)", "", "1..2", "x^",
       "sin()", "2 3"]


def values(n, seed=1):
    rng = np.random.default_rng(seed)
    return np.column_stack([rng.uniform(0.1, 5.2, n), np.full(n, 5.291), rng.uniform(-30, 0, n),
                            rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n),
                            rng.uniform(0.5, 3, n)])


@pytest.mark.parametrize("formula", FORMULAS)
def test_values_bitwise_equal_to_reference(formula):
    v = values(500)
    ours = fb.expr_eval(formula, VARS, v)
    ref = ref_expr_eval(formula, VARS, v)
    assert np.array_equal(ours, ref, equal_nan=True)


@pytest.mark.parametrize("formula", BAD)
def test_errors_match_reference(formula):
    with pytest.raises(fb.FfitError) as ours:
        fb.expr_eval(formula, VARS, values(1))
    with pytest.raises(Exception) as ref:
        ref_expr_eval(formula, VARS, values(1))
    assert str(ours.value) == str(ref.value)
    assert ours.value.code == 1  # FFIT_ERR_USAGE


def test_documented_examples():
    """proj/docs/expression-grammar.md: -x^2 = -(x^2); 2^3^2 = 512; x^2..x^4 are products."""
    v = np.array([[3.0]])
    assert fb.expr_eval("-x^2", ["x"], v)[0] == -9.0
    assert fb.expr_eval("2^3^2", [], np.zeros((1, 0)))[0] == 512.0
    x = 1.1
    assert fb.expr_eval("x^3", ["x"], [[x]])[0] == x * x * x
    assert fb.expr_eval("x^4", ["x"], [[x]])[0] == (x * x) * (x * x)


@pytest.mark.parametrize("name", list(EXPR_MODELS))
def test_expression_models_normalisation_and_sampling_bitwise(name):
    """The reference's own Expression model texts: host normalisation (adaptive Simpson over
    the formula) and the toy generator (accept/reject) reproduce the reference bit for bit."""
    ref_text, _, seed, col = EXPR_MODELS[name]
    m = fb.Model.from_string(ref_text)
    r = RefModel(ref_text)
    assert fb.normalization(m) == r.normalization()
    cols, _ = fb.sample_host(m, 3000, seed)
    assert np.array_equal(cols[col], r.sample(3000, seed)[0])


def test_expression_parse_errors():
    with pytest.raises(fb.FfitError) as e:
        fb.Model.from_string("observable x 0 1\nparameter a 1 0 2\npdf e Expression(\"x*b\", x, a)\n")
    assert "unknown identifier: b" in str(e.value)
    with pytest.raises(fb.FfitError) as e:
        fb.Model.from_string("observable x 0 1\nobservable y 0 1\npdf e Expression(\"x*y\", x, y)\n")
    assert "one observable" in str(e.value)
    with pytest.raises(fb.FfitError) as e:
        fb.Model.from_string("observable x 0 1\npdf e Expression(\"x*q\", x, q)\n")
    assert "undeclared name: q" in str(e.value)


def test_expression_gradient_layout():
    """Expression leaves take part in the fused gradient pass (forward mode through the
    formula): one A slot per term, one B slot per free parameter of each leaf."""
    m = fb.Model.from_string(EXPR_MODELS["argus_mix"][0])
    free = sum(1 for n in m.param_names if not m.is_constant(n))
    assert fb.grad_slot_count(m) >= 1 + 2 + 1


def test_formula_specialised_source_compiles_with_nvrtc():
    """The generated straight-line formula code plus the fused kernels around it compile to
    sm_100a SASS with NVRTC (host-side: no GPU needed) for the reference's Argus spelling."""
    from paper_2003_12875_b200 import configs
    m = fb.Model.from_string(configs.REFERENCE_TEXTS[configs.C2.name])
    src = fb.expression_jit_source(m, compile=True)
    assert "ffb_expr_batch" in src and "ffb_vsqrt" in src
    # x / m0: a division by a point-uniform divisor takes the hoisted-reciprocal form
    assert "ffb_vdiv_uniform<E>(" in src.split("void ffb_expr_0")[1]
    # constants travel bit-exactly (hex bit patterns, not decimal text)
    assert "__longlong_as_double(0x3ff0000000000000ll)" in src


def test_formula_source_mirrors_the_program():
    m = fb.Model.from_string("observable x 0 2\nparameter a 0.5 0 1\n"
                             "pdf e Expression(\"1 + a*x^3 - x^2/4 + pow(x, 2.5)\", x, a)\n")
    src = fb.expression_jit_source(m)
    assert src.count("__dmul_rn") >= 4 and "ffb_pow" in src and "k[2]" in src


def test_formula_launch_constant_subtrees_compile_with_nvrtc():
    """With m0 fixed over a launch's points, the reference's Argus formula's m0-only subtrees
    (x*sqrt(1-(x/m0)^2), 1-(x/m0)^2) move to the per-tile cache; the source compiles."""
    from paper_2003_12875_b200 import configs
    w = configs.C2
    m = fb.Model.from_string(configs.REFERENCE_TEXTS[w.name])
    mo = fb.Model.from_string(w.text)
    by = [dict(zip(mo.param_names, r)) for r in w.points(mo, n_points=12)]
    pts = np.array([[d[n] for n in m.param_names] for d in by])
    src = fb.expression_jit_source(m, compile=True, points=pts)
    assert "FFB_EXPR_HOIST" in src and src.count("// column ") == 2
    pts[3, m.param_names.index("m0")] += 1e-4  # m0 no longer launch-constant: nothing cached
    assert "FFB_EXPR_HOIST" not in fb.expression_jit_source(m, points=pts)
