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
    # the kernel's exp is exact-to-2-ulp on |x| <= 707 and saturates beyond (fastmath.cuh)
    x = np.concatenate([rng.uniform(-707.0, 707.0, 2_000_000), rng.uniform(-1, 1, 500_000),
                        rng.uniform(-40, 0, 500_000), np.array([0.0, -0.0, 1e-300, -1e-300, 1.0, -1.0])])
    got = fb.ffit.math_probe("exp", x)
    want = np.exp(x)
    assert np.max(ulps(got, want)) <= 2.0
    assert np.max(np.abs(got - want) / want) <= 4.5e-16


def test_exp_saturation():
    """Beyond |x| = 707 the kernel's exp saturates (0 below, +inf above); NaN / inf
    arguments are never evaluated: events with non-finite data are flagged invalid by the
    kernels and non-finite parameters are rejected on the host."""
    x = np.array([-800.0, -746.0, -707.1, 707.1, 710.0, 800.0, 1e300, -1e300])
    got = fb.ffit.math_probe("exp", x)
    assert list(got[[0, 1, 2, 7]]) == [0.0, 0.0, 0.0, 0.0]
    assert np.all(np.isinf(got[[3, 4, 5, 6]]))


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
