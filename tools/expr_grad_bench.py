"""Expression models (the reference config-2 text with m0 free): the analytic gradient pass (device
interpreter forward mode) against 2d+1-point finite differences (formula-specialised NLL), per call and
per fit."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs
w = configs.C2
text = configs.REFERENCE_TEXTS[w.name].replace("parameter m0 5.291 5.0 5.4 const", "parameter m0 5.291 5.2901 5.30")
m = fb.Model.from_string(text)
mo = fb.Model.from_string(w.text)
n = 10_000_000
cols, _ = fb.sample_host(mo, n, w.data_seed)
ds = fb.DataSet.from_columns(cols)
th = m.theta()
d = sum(1 for nm in m.param_names if not m.is_constant(nm))
pts = np.repeat(th[None, :], 2 * d + 1, axis=0)
for k, nm in enumerate([nm for nm in m.param_names]):
    pass
free = [k for k, nm in enumerate(m.param_names) if not m.is_constant(nm)]
for i, k in enumerate(free):
    pts[1 + 2 * i, k] += 1e-6; pts[2 + 2 * i, k] -= 1e-6
for f, name in ((lambda: fb.nll_grad(m, ds, th), "analytic grad"), (lambda: fb.nll_points(m, ds, pts), f"FD {len(pts)} pts")):
    f(); print(name, "spec build:", fb.last_grad_jit(m), "status:", fb.expression_jit_status()[:300])
    for _ in range(3): f()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(10): f()
    torch.cuda.synchronize(); print(name, "%.3f ms" % ((time.perf_counter() - t) / 10 * 1e3))
t = time.perf_counter(); r = fb.fit_gradient(m, ds, tolerance=1e-10, max_iterations=100, analytic=True); print("fit analytic", r.analytic_gradient, "%.3f s" % (time.perf_counter() - t), r.iterations)
m2 = fb.Model.from_string(text)
t = time.perf_counter(); r = fb.fit_gradient(m2, ds, tolerance=1e-10, max_iterations=100, analytic=False); print("fit FD", "%.3f s" % (time.perf_counter() - t), r.iterations)
