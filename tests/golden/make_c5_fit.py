"""The CPU fit of BASELINE config 5 (2e8 events, 5 free parameters): the golden the GPU fits
are compared with (tests/test_gpu_fit.py::test_c5_fit_matches_the_cpu_fit, bench.py --fit).

Build container only, run once (minutes on 8 host threads):

    python tests/golden/make_c5_fit.py

Data: the config's seeded events (configs.C5: seed 1005; the oracle's generator reproduces
the reference Rng and is bit-identical to the library's, tests/test_host.py).  Likelihood:
the oracle (oracle/ffit_oracle.c, pinned to the reference: tests/test_oracle.py) -- the
compensated NLL over all 2e8 events, one point per host thread.  Minimiser: Newton's method
in parameter space on central-difference gradients and Hessians (the 1 + 2d + 2d(d-1) point
stencil of proj/src/fit.cpp:200-225, in theta instead of u), steps h_i = 0.05 sigma_i once
sigma is known, a halving line search, until every Newton step is below 1e-6 sigma_i.  The
result is the minimum itself to ~1e-6 sigma (the NLL's rounding, ~1 ulp of 5e8, allows
that), so any converged minimiser -- the GPU's BFGS, Nelder-Mead -- can be held to it.

Writes tests/golden/c5_cpu_fit.json.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import OracleModel, build  # noqa: E402
from paper_2003_12875_b200 import configs  # noqa: E402


def main():
    build()
    w = configs.C5
    threads = os.cpu_count() or 1
    o = OracleModel(w.text)
    t0 = time.time()
    cols, _ = o.sample(w.n_events, w.data_seed)
    print(f"sampled {w.n_events} events in {time.time() - t0:.1f} s", flush=True)
    names = o.param_names

    class M:
        param_names = names

        @staticmethod
        def theta():
            return o.theta.copy()

    start = w.points(M, n_points=1, seed=w.point_seed)[0]
    free = [k for k, p in enumerate(o.pm.params) if not p[4]]  # (name, value, lo, hi, const)
    lo = np.array([o.pm.params[k][2] for k in free])
    hi = np.array([o.pm.params[k][3] for k in free])
    d = len(free)

    def rows_of(thetas_free):
        out = np.tile(start, (len(thetas_free), 1))
        out[:, free] = thetas_free
        return out

    def nll(thetas_free):
        return o.nll_points(cols, rows_of(np.atleast_2d(thetas_free)), threads=threads)

    x = start[free].copy()
    h = 1e-4 * (hi - lo)
    log = []
    f_x = float(nll(x[None])[0])
    for it in range(30):
        pts = [x.copy()]
        for i in range(d):
            for sgn in (1, -1):
                p = x.copy()
                p[i] += sgn * h[i]
                pts.append(p)
            for j in range(i + 1, d):
                for si, sj in ((1, 1), (1, -1), (-1, -1), (-1, 1)):
                    p = x.copy()
                    p[i] += si * h[i]
                    p[j] += sj * h[j]
                    pts.append(p)
        t1 = time.time()
        v = nll(np.array(pts))
        f0 = v[0]
        g = np.zeros(d)
        H = np.zeros((d, d))
        k = 1
        for i in range(d):
            fp, fm = v[k], v[k + 1]
            k += 2
            g[i] = (fp - fm) / (2 * h[i])
            H[i, i] = (fp - 2 * f0 + fm) / (h[i] * h[i])
            for j in range(i + 1, d):
                fpp, fpm, fmm, fmp = v[k:k + 4]
                k += 4
                H[i, j] = H[j, i] = (fpp - fpm - fmp + fmm) / (4 * h[i] * h[j])
        cov = np.linalg.inv(H)
        sigma = np.sqrt(np.diag(cov))
        step = -cov @ g
        lam = 1.0
        while True:
            xn = np.clip(x + lam * step, lo + 1e-12 * (hi - lo), hi - 1e-12 * (hi - lo))
            fn = float(nll(xn[None])[0])
            if fn <= f0 or lam < 1e-3:
                break
            lam *= 0.5
        rel = np.max(np.abs(lam * step) / sigma)
        log.append({"iteration": it, "nll": f0, "step_over_sigma": float(rel), "lambda": lam,
                    "seconds": time.time() - t1})
        print(json.dumps(log[-1]), flush=True)
        if fn <= f0:
            x, f_x = xn, fn
        h = 0.05 * sigma
        if rel < 1e-6 and it >= 2:
            break
    out = {
        "workload": w.name, "n_events": w.n_events, "data_seed": w.data_seed, "point_seed": w.point_seed,
        "start": {names[k]: float(start[k]) for k in free},
        "parameters": {names[k]: float(x[i]) for i, k in enumerate(free)},
        "sigma": {names[k]: float(sigma[i]) for i, k in enumerate(free)},
        "nll_min": f_x,
        "method": "Newton in parameter space on central-difference gradients / Hessians of the oracle's "
                  "compensated NLL over all events (tests/golden/make_c5_fit.py); converged when every "
                  "Newton step < 1e-6 sigma",
        "iterations": log,
        "host_threads": threads,
    }
    with open(os.path.join(HERE, "c5_cpu_fit.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", os.path.join(HERE, "c5_cpu_fit.json"))


if __name__ == "__main__":
    main()
