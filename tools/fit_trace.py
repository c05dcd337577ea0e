"""Fit-convergence diagnostic: the C5 model fitted with finite-difference and with
analytic gradients; prints each mode's NLL trace relative to the final minimum."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
w = configs.C5
truth = fb.Model.from_string(w.text)
cols, _ = fb.sample_host(truth, n, w.data_seed)
ds = fb.DataSet.from_columns(cols)
for analytic in (False, True):
    m = fb.Model.from_string(w.text)
    start = w.points(m, n_points=1, seed=w.point_seed)[0]
    for name, v in zip(m.param_names, start):
        if not m.is_constant(name):
            m.set(name, v)
    r = fb.fit_gradient(m, ds, tolerance=1e-12, max_iterations=60, analytic=analytic)
    tr = np.array(r.trace)
    print(f"analytic={analytic} converged={r.converged} iters={r.iterations} launches={r.n_launches} "
          f"wall={r.wall_seconds:.3f}s nll_min={r.nll_min!r}")
    print("  trace - min:", " ".join(f"{v:.3g}" for v in tr - r.nll_min))
    print("  params:", {p.name: (p.value, p.uncertainty) for p in r.parameters})
