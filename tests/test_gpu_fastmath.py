"""Accuracy of the fused kernel's table-driven exp / log (csrc/fastmath.cuh) against
glibc (numpy's float64 exp/log are correctly rounded to within 1 ulp on these ranges;
mpmath spot checks pin the worst cases)."""
import math

import numpy as np
import pytest

import paper_2003_12875_b200 as fb

pytestmark = pytest.mark.gpu


def ulps(a, b):
    return np.abs(a - b) / np.spacing(np.abs(b))


def test_exp_accuracy_over_the_working_range():
    rng = np.random.default_rng(0)
    # the kernel's exp is exact-to-2-ulp on |x| <= 707 (the edges: test_exp_range_edges_match_glibc)
    x = np.concatenate([rng.uniform(-707.0, 707.0, 2_000_000), rng.uniform(-1, 1, 500_000),
                        rng.uniform(-40, 0, 500_000), np.array([0.0, -0.0, 1e-300, -1e-300, 1.0, -1.0])])
    got = fb.ffit.math_probe("exp", x)
    want = np.exp(x)
    assert np.max(ulps(got, want)) <= 2.0
    assert np.max(np.abs(got - want) / want) <= 4.5e-16


def test_exp_range_edges_match_glibc():
    """Past |x| = 707 the device exp takes its edge path (fastmath.cuh exp_edge): gradual
    underflow into the subnormals down to -745.13, +0 below; finite up to 709.78, +inf
    above; NaN / inf arguments as glibc.  Compared with glibc's exp (math.exp)."""
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.uniform(-745.2, -707.0, 200_000), rng.uniform(707.0, 709.78, 50_000),
                        np.array([-707.0, -707.5, -708.39, -708.4, -710.0, -720.0, -744.0, -745.0,
                                  -745.13, -745.14, -746.0, -800.0, -1e300, 707.5, 709.0, 709.78])])
    got = fb.ffit.math_probe("exp", x)

    def gexp(v):
        try:
            return math.exp(v)
        except OverflowError:
            return math.inf
    want = np.array([gexp(float(v)) for v in x])
    fin = want > 0
    # normal results: 2 ulp; subnormal ones: one rounding of a 2-ulp value
    tol = np.maximum(2.0 * np.spacing(want), 2.0 * 2.0 ** -1074)
    assert np.all(np.abs(got[fin] - want[fin]) <= tol[fin])
    assert np.all(got[~fin] == 0.0)
    sub = (want > 0) & (want < 2.2250738585072014e-308)
    assert sub.sum() > 50_000 and np.all(got[sub] > 0)
    edge = fb.ffit.math_probe("exp", np.array([709.79, 710.0, 800.0, 1e300, math.inf, -math.inf, math.nan]))
    assert np.all(np.isinf(edge[:5])) and np.all(edge[:5] > 0)
    assert edge[5] == 0.0 and math.isnan(edge[6])


def test_log_accuracy_absolute_and_relative():
    rng = np.random.default_rng(1)
    x = np.concatenate([10.0 ** rng.uniform(-300, 300, 2_000_000), rng.uniform(0.5, 2.0, 1_000_000),
                        np.array([1.0, 2.0, 0.5, 1e-310, 5e-324, 1.7976931348623157e308])])
    got = fb.ffit.math_probe("log", x)
    want = np.log(x)
    err = np.abs(got - want)
    assert np.all(err <= np.maximum(2.0 * np.spacing(np.abs(want)), 2.3e-16))
    assert got[-6] == 0.0  # log(1) exactly


def test_sqrt_unit_accuracy():
    """ArgusBG's branch-free sqrt on (0, 1]: within 1 ulp of the IEEE sqrt."""
    rng = np.random.default_rng(2)
    t = np.concatenate([rng.uniform(0, 1, 1_000_000), 10.0 ** rng.uniform(-16, 0, 1_000_000),
                        np.array([1.0, 0.25, 2.0 ** -52])])
    got = fb.ffit.math_probe("sqrt", t)
    assert np.max(ulps(got, np.sqrt(t))) <= 1.0
    seed = fb.ffit.math_probe("rsqrt_seed", t)
    rel = np.max(np.abs(seed * np.sqrt(t) - 1.0))
    print(f"MUFU rsqrt seed max relative error: {rel:.3e}")
    assert rel < 1e-4


def test_log_subnormals():
    x = np.array([1e-310, 2.2e-308, 4.9e-324, 1e-320])
    got = fb.ffit.math_probe("log", x)
    assert np.all(np.abs(got - np.log(x)) <= 2.0 * np.spacing(np.abs(np.log(x))))
