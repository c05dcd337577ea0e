"""Generate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Runs in the build container only (needs /root/reference, via oracle/_ref/libffit_ref.so
compiled from the reference's own sources by oracle/Makefile).  The GPU box never
runs this; it only reads the committed fixtures.

    python tests/golden/make_golden.py

Fixtures (all float64, bit-exact from the reference build):
  rng.npz            reference Rng streams: uniform / gauss for several seeds
                     (proj/src/sampling.cpp:9-54)
  ref_models.npz     for each model in MODELS: sampled events (reference sampler,
                     proj/src/sampling.cpp:172-197), per-event probabilities
                     (BatchPrecise == Scalar bitwise, proj/src/eval.cpp:174-192),
                     naive nll() (proj/src/eval.cpp:119-163), Neumaier NLL, norm,
                     n_evaluations
  expr_models.npz    restated kinds through the reference's Expression + adaptive
                     Simpson route (ArgusBG, Chebychev, Polynomial; proj/src/expr.cpp,
                     proj/src/eval.cpp:40-86) -- cross-check, not bitwise
  argus_mp.json      ArgusBG (p = 1/2) normalisation integrals by mpmath quadrature
                     at 50 digits (closed-form pin)
  ref_fits.json      reference Nelder-Mead fits (proj/src/fit.cpp:86-251, tolerance
                     1e-10) on seeded data: fitted values, uncertainties, NLL minimum
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import RefDataset, RefModel, build, ref_rng_gauss, ref_rng_uniform  # noqa: E402
from tests.models import EXPR_MODELS, FIT_CASES, REF_MODELS  # noqa: E402

N_EVENTS = 4096


def main():
    build()
    rng = {}
    for seed in (0, 1, 42, 8675309, 2**63 + 5):
        rng[f"uniform_{seed}"] = ref_rng_uniform(seed, 257)
        rng[f"gauss_{seed}"] = ref_rng_gauss(seed, 257)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **rng)

    out = {}
    for name, (text, seed) in REF_MODELS.items():
        m = RefModel(text)
        xs, eff = m.sample(N_EVENTS, seed)
        ds = RefDataset("x", xs)
        p = m.probabilities(ds, RefModel.PRECISE)
        ps = m.probabilities(ds, RefModel.SCALAR)
        assert np.array_equal(p, ps), name
        nll, nev, bad = m.nll(ds, RefModel.PRECISE)
        comp, _ = m.nll_compensated(ds, RefModel.PRECISE)
        out[f"{name}/x"] = xs
        out[f"{name}/p"] = p
        out[f"{name}/scalars"] = np.array([nll, comp, m.normalization(), nev, bad, eff, seed])
    np.savez_compressed(os.path.join(HERE, "ref_models.npz"), **out)

    out = {}
    for name, (ref_text, _ours, seed, col) in EXPR_MODELS.items():
        m = RefModel(ref_text)
        rs = np.random.default_rng(seed)
        lo, hi = _range(ref_text)
        xs = rs.uniform(lo, hi, 2048)
        xs.sort()
        ds = RefDataset(col, xs)
        p = m.probabilities(ds, RefModel.PRECISE)
        comp, bad = m.nll_compensated(ds, RefModel.PRECISE)
        out[f"{name}/x"] = xs
        out[f"{name}/p"] = p
        out[f"{name}/scalars"] = np.array([comp, m.normalization(), bad])
    np.savez_compressed(os.path.join(HERE, "expr_models.npz"), **out)

    import mpmath as mp
    mp.mp.dps = 50
    cases = []
    for (m0, c, lo, hi) in [(5.291, -20.0, 5.20, 5.29), (5.291, -5.0, 5.20, 5.29),
                            (5.291, -100.0, 5.20, 5.29), (5.291, 0.0, 5.20, 5.29),
                            (5.291, 2.5, 5.20, 5.29), (5.3, -20.0, 5.0, 5.3),
                            (1.0, -60.0, 0.0, 1.0), (1.0, -0.01, 0.5, 0.99)]:
        mm0 = mp.mpf(m0)
        f = lambda x: x * mp.sqrt(1 - (x / mm0) ** 2) * mp.exp(mp.mpf(c) * (1 - (x / mm0) ** 2))
        val = mp.quad(f, [mp.mpf(lo), min(mp.mpf(hi), mm0)])
        cases.append(dict(m0=m0, c=c, lo=lo, hi=hi, integral=float(val)))
    with open(os.path.join(HERE, "argus_mp.json"), "w") as fh:
        json.dump(cases, fh, indent=1)
    fits = {}
    for name, case in FIT_CASES.items():
        gen = RefModel(case["ref_text"])
        for k, v in case.get("truth", {}).items():
            gen.set(k, v)
        if case.get("data_from") == "oracle":
            from oracle.oracle import OracleModel
            o = OracleModel(case["ours_text"])
            for k, v in case.get("truth", {}).items():
                o.set(k, v)
            (xs,), _ = o.sample(case["n"], case["seed"])
        else:
            xs, _ = gen.sample(case["n"], case["seed"])
        ds = RefDataset(case["column"], xs)
        fit = RefModel(case["ref_text"])
        for k, v in case.get("start", {}).items():
            fit.set(k, v)
        r = fit.fit(ds, RefModel.PRECISE, tol=case["tol"])
        r["params"] = {k: list(fit.get(k)) for k in case["free"]}
        fits[name] = r
        print("fit", name, r)
    with open(os.path.join(HERE, "ref_fits.json"), "w") as fh:
        json.dump(fits, fh, indent=1)
    print("golden fixtures written to", HERE)


def _range(text):
    for line in text.splitlines():
        t = line.split()
        if t and t[0] == "observable":
            return float(t[2]), float(t[3])
    raise ValueError


if __name__ == "__main__":
    main()
