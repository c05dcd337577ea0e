"""Model texts shared by the tests and the golden-fixture generator.

REF_MODELS use only the reference grammar (proj/docs/model-file.md), so the very same
text runs through the reference engine, the oracle and the GPU product.  The first five
are the acceptance-suite models (proj/tests/acceptance.cpp:38-80); `gauss_c1` is the
BASELINE config-1 shape.

EXPR_MODELS pair a restated kind (ArgusBG, Chebychev, Polynomial) with the reference's
Expression spelling of the same density.
"""

MIX = """
observable x -5 5
parameter mu 0.2 -2 2
parameter sigma 0.8 0.1 3
parameter c -0.35 -3 0
parameter f 0.4 0.05 0.95
pdf s Gaussian(x, mu, sigma)
pdf b Exponential(x, c)
pdf m WeightedSum(s, f, b)
"""

REF_MODELS = {
    "gauss": ("""
observable x -5 5
parameter mu 0.3 -2 2
parameter sigma 1.1 0.1 3
pdf g Gaussian(x, mu, sigma)
""", 8675309),
    "expo": ("""
observable x 0 8
parameter c -0.6 -3 0
pdf e Exponential(x, c)
""", 8675309),
    "chisq": ("""
observable x 0.1 15
parameter k 3.5 0.5 20
pdf q ChiSquare(x, k)
""", 8675309),
    "johnson": ("""
observable x -6 6
parameter mu 0.1 -2 2
parameter lambda 1.2 0.1 3
parameter gamma -0.3 -3 3
parameter delta 1.4 0.1 3
pdf j JohnsonSU(x, mu, lambda, gamma, delta)
""", 8675309),
    "mix": (MIX, 8675309),
    "gauss_c1": ("""
observable x -10 10
parameter mean 1.0 -5 5
parameter sigma 2.0 0.1 10
pdf g Gaussian(x, mean, sigma)
""", 1001),
    "mix3_nested": ("""
observable x -6 6
parameter m1 -2 -5 5
parameter s1 0.5 0.1 3
parameter m2 1.5 -5 5
parameter s2 0.9 0.1 3
parameter c -0.3 -3 3
parameter f1 0.3 0 1
parameter f2 0.25 0 1
parameter g 0.6 0 1
pdf a Gaussian(x, m1, s1)
pdf b Gaussian(x, m2, s2)
pdf e Exponential(x, c)
pdf ab WeightedSum(a, g, b)
pdf m WeightedSum(ab, f1, e, f2, a)
""", 77),
    "mix_chisq": ("""
observable x 0.1 12
parameter k 4.5 0.5 20
parameter mu 6 0 12
parameter sigma 1.0 0.1 3
parameter f 0.7 0 1
pdf q ChiSquare(x, k)
pdf g Gaussian(x, mu, sigma)
pdf m WeightedSum(q, f, g)
""", 5),
}

ARGUS_REF = """
observable x 5.2 5.29
parameter m 5.279 5.2 5.29
parameter s 0.003 0.001 0.01
parameter m0 5.291 5.0 5.4 const
parameter c -20 -100 10
parameter f 0.1 0 1
pdf sig Gaussian(x, m, s)
pdf bkg Expression("x*sqrt(1-(x/m0)^2)*exp(c*(1-(x/m0)^2))", x, m0, c)
pdf model WeightedSum(sig, f, bkg)
"""

ARGUS_OURS = """
observable x 5.2 5.29
parameter m 5.279 5.2 5.29
parameter s 0.003 0.001 0.01
parameter m0 5.291 5.0 5.4 const
parameter c -20 -100 10
parameter p 0.5 0 1 const
parameter f 0.1 0 1
pdf sig Gaussian(x, m, s)
pdf bkg ArgusBG(x, m0, c, p)
pdf model WeightedSum(sig, f, bkg)
"""

EXPR_MODELS = {
    "argus_mix": (ARGUS_REF, ARGUS_OURS, 1002, "x"),
    "argus_only": ("""
observable x 5.2 5.29
parameter m0 5.291 5.0 5.4 const
parameter c -20 -100 10
pdf bkg Expression("x*sqrt(1-(x/m0)^2)*exp(c*(1-(x/m0)^2))", x, m0, c)
""", """
observable x 5.2 5.29
parameter m0 5.291 5.0 5.4 const
parameter c -20 -100 10
parameter p 0.5 0 1 const
pdf bkg ArgusBG(x, m0, c, p)
""", 11, "x"),
    "cheb3": ("""
observable z -1 1
parameter a1 0.2 -1 1
parameter a2 -0.1 -1 1
parameter a3 0.05 -1 1
pdf ch Expression("1 + a1*z + a2*(2*z^2-1) + a3*(4*z^3-3*z)", z, a1, a2, a3)
""", """
observable z -1 1
parameter a1 0.2 -1 1
parameter a2 -0.1 -1 1
parameter a3 0.05 -1 1
pdf ch Chebychev(z, a1, a2, a3)
""", 1023, "z"),
    "cheb3_shifted": ("""
observable z 2 6
parameter a1 0.3 -1 1
parameter a2 0.1 -1 1
parameter a3 -0.05 -1 1
pdf ch Expression("1 + a1*((2*z-8)/4) + a2*(2*((2*z-8)/4)^2-1) + a3*(4*((2*z-8)/4)^3-3*((2*z-8)/4))", z, a1, a2, a3)
""", """
observable z 2 6
parameter a1 0.3 -1 1
parameter a2 0.1 -1 1
parameter a3 -0.05 -1 1
pdf ch Chebychev(z, a1, a2, a3)
""", 31, "z"),
    "poly2": ("""
observable x -1 2
parameter a1 0.2 -1 1
parameter a2 0.1 -1 1
pdf po Expression("1 + a1*x + a2*x^2", x, a1, a2)
""", """
observable x -1 2
parameter a1 0.2 -1 1
parameter a2 0.1 -1 1
pdf po Polynomial(x, a1, a2)
""", 13, "x"),
}

GAUSS_CLOSURE = """
observable x -6 6
parameter mu 0 -3 3
parameter sigma 1.2 0.1 4
pdf g Gaussian(x, mu, sigma)
"""

# Reference Nelder-Mead fits pinned as golden values (tests/golden/ref_fits.json).
# mix_acceptance: proj/tests/acceptance.cpp:122-135 (criterion 3 data);
# gauss_closure: proj/tests/acceptance.cpp:226-250 (criterion 8);
# argus_mix: the config-2 model (ArgusBG as the reference's Expression).
FIT_CASES = {
    "mix_acceptance": dict(ref_text=MIX, ours_text=MIX, n=20000, seed=314159, column="x", tol=1e-10,
                           free=["mu", "sigma", "c", "f"]),
    "gauss_closure": dict(ref_text=GAUSS_CLOSURE, ours_text=GAUSS_CLOSURE, n=50000, seed=424242, column="x",
                          tol=1e-10, truth={"mu": 0.5, "sigma": 1.0}, start={"mu": 0.0, "sigma": 1.2},
                          free=["mu", "sigma"]),
    "argus_mix": dict(ref_text=ARGUS_REF, ours_text=ARGUS_OURS, n=20000, seed=99, column="x", tol=1e-12,
                      data_from="oracle", start={"m": 5.2785, "s": 0.0032, "c": -18.0, "f": 0.12},
                      free=["m", "s", "c", "f"]),
}


# ---------------------------------------------------------------------------
# exp at the edges of its range (tests/golden/make_edge_golden.py):
# densities in glibc's gradual-underflow window (exp argument in (-745.13, -707]) are
# SUBNORMAL and valid in the reference, below it they are 0 and the event is invalid
# (proj/src/eval.cpp:138-145); exp(c x) stays finite up to c x = 709.78.

GAUSS_WIDE = """
observable x -50 50
parameter mu 0 -1 1
parameter sigma 1 0.5 2
pdf g Gaussian(x, mu, sigma)
"""

FAR_MIX = """
observable x -60 60
parameter m1 -5 -10 10
parameter s1 1 0.5 2
parameter m2 5 -10 10
parameter s2 1 0.5 2
parameter f 0.4 0 1
pdf a Gaussian(x, m1, s1)
pdf b Gaussian(x, m2, s2)
pdf model WeightedSum(a, f, b)
"""

EXPO_EDGE = """
observable x 700 709.7
parameter c 1.0 0.5 1.0
pdf e Exponential(x, c)
"""


def edge_data(sub_at, zero_at, n=4099):
    """Standard-normal events, one at exponent -720 (subnormal p), one at -800 (p = 0) and
    one more at -900 later on; zero_at = None leaves only the subnormal one."""
    import math

    import numpy as np
    x = np.random.default_rng(5).normal(0.0, 1.0, n)
    x[sub_at] = math.sqrt(2.0 * 720.0)
    if zero_at is not None:
        x[zero_at] = -math.sqrt(2.0 * 800.0)
        x[3000] = math.sqrt(2.0 * 900.0)
    return x


def far_mix_data():
    import math

    import numpy as np
    rng = np.random.default_rng(9)
    x = np.concatenate([rng.normal(-5, 1, 3000), rng.normal(5, 1, 3000)])
    x[17] = -5 - math.sqrt(2 * 722.0)   # component a at -722, b far below -745
    x[1234] = 5 + math.sqrt(2 * 710.0)  # component b at -710 (subnormal), a 0
    return x


def expo_edge_data():
    import numpy as np
    x = np.random.default_rng(11).uniform(700.0, 709.7, 30_011)
    x[:4] = [709.7, 709.65, 707.01, 708.2]
    return x


def c1_sigma720_text(x):
    """The C1 model with sigma set so that the most distant event's exponent is -720."""
    import math

    import numpy as np
    sigma = float(np.max(np.abs(x - 1.0))) / math.sqrt(2.0 * 720.0)
    return f"""
observable x -10 10
parameter mean 1.0 -5 5
parameter sigma {sigma!r} 0.1 10
pdf g Gaussian(x, mean, sigma)
"""


EXPR_GAUSS_WIDE = """
observable x -50 50
parameter mu 0 -1 1
parameter sigma 1 0.5 2
pdf g Expression("exp(-0.5*((x-mu)/sigma)^2)", x, mu, sigma)
"""

# name -> (text, events) ; c1_sigma720 is built from the reference sampler's C1 events
EDGE_CASES = {
    "gauss_sub_then_zero": lambda: (GAUSS_WIDE, edge_data(3, 10)),
    "gauss_zero_then_sub": lambda: (GAUSS_WIDE, edge_data(10, 3)),
    "gauss_sub_only": lambda: (GAUSS_WIDE, edge_data(3, None)),
    "far_mix": lambda: (FAR_MIX, far_mix_data()),
    "expo_overflow_edge": lambda: (EXPO_EDGE, expo_edge_data()),
    # the reference's Expression + adaptive-Simpson route (the formula-specialised build)
    "expr_sub_then_zero": lambda: (EXPR_GAUSS_WIDE, edge_data(3, 10)),
    "expr_sub_only": lambda: (EXPR_GAUSS_WIDE, edge_data(3, None)),
}
