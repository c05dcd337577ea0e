"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): the tile kernel (multi-point, one and several columns, ragged sizes), the
streaming kernel, the gradient passes (streaming and tile), eval / probabilities, the
combine kernel, the Expression interpreter and the formula-specialised build."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs
from tests.models import EXPR_MODELS

for w, n in ((configs.C2, 10_001), (configs.C3, 5_003)):
    m = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(m, n, 3)
    ds = fb.DataSet.from_columns(cols)
    pts = w.points(m, n_points=12)
    fb.nll_points(m, ds, pts)          # tile kernel
    fb.nll_points(m, ds, pts[:3])      # streaming kernel (one column) / tile (three columns)
    fb.probabilities(m, ds)
    fb.nll_grad(m, ds, pts[:2])        # gradient pass, streaming
    fb.nll_grad(m, ds, pts)            # gradient pass, tile (P > 8)
text = EXPR_MODELS["argus_mix"][0]
m = fb.Model.from_string(text)
cols, _ = fb.sample_host(m, 4_097, 5)
ds = fb.DataSet.from_columns(cols)
for jit in (False, True):
    fb.expression_jit(jit)
    fb.nll_points(m, ds, m.theta())
    fb.nll_points(m, ds, np.repeat(m.theta()[None, :], 10, axis=0))

# the run-time compiled builds at small sizes (threshold 0): plan-specialised tile and
# streaming kernels (one and three columns), the launch-constant caches (ArgusBG pair,
# whole leaves), formula subtrees cached per tile, the formula gradient pass, and the
# CUDA-graph replay of single-point calls
fb.plan_spec_min_work(0)
for w, n in ((configs.C2, 10_001), (configs.C3, 5_003), (configs.C4, 7_001)):
    m = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(m, n, 3)
    ds = fb.DataSet.from_columns(cols)
    pts = w.points(m, n_points=12)
    if w is configs.C4:  # yields only: every leaf cached per tile
        base = m.theta()
        for k, name in enumerate(m.param_names):
            if not name.startswith("n"):
                pts[:, k] = base[k]
    fb.nll_points(m, ds, pts)
    fb.nll_points(m, ds, pts[:2])
    for _ in range(3):
        fb.nll_points(m, ds, pts[:1])  # plain, capture, replay
    fb.nll_grad(m, ds, pts[0])
ref = configs.REFERENCE_TEXTS[configs.C2.name]
m = fb.Model.from_string(ref)
mo = fb.Model.from_string(configs.C2.text)
cols, _ = fb.sample_host(mo, 9_001, 4)
ds = fb.DataSet.from_columns(cols)
by = [dict(zip(mo.param_names, r)) for r in configs.C2.points(mo, n_points=12)]
pts = np.array([[d[k] for k in m.param_names] for d in by])
fb.nll_points(m, ds, pts)            # formula build with cached subtrees
mf = fb.Model.from_string(ref.replace("parameter m0 5.291 5.0 5.4 const", "parameter m0 5.291 5.2901 5.30"))
fb.nll_grad(mf, ds, mf.theta())      # plan-specialised gradient pass with formula tangents

# round 2: the one-column eval_fast_kernel builds (eval_batch per node, probabilities), the
# device-side adaptive Simpson (simpson_kernel) on the reference's Simpson-normalised text, the
# parallel reduce_kernel over many tiles, the event-sharded group (send block, NCCL all-gather
# at world 1, combine kernel; NLL and gradients), exp at glibc's range edges, and both fit drivers
fb.plan_spec_min_work(-2.0)
m = fb.Model.from_string(configs.C4.text)
cols, _ = fb.sample_host(m, 300_007, 3)
ds = fb.DataSet.from_columns(cols)
pts = configs.C4.points(m, n_points=16)
for name in m.pdf_names:
    fb.eval_batch(m, name, ds)
fb.probabilities(m, ds)
fb.nll_points(m, ds, pts)            # 147 tiles x 16 points through reduce_kernel
if os.environ.get("SANITIZE_NCCL", "1") == "1":
    import torch  # noqa: F401  (one NCCL in the process: torch's)
    grp = fb.ShardGroup.for_rank(m, ds, ds.n_rows, 0, 1, 0)
    grp.nll_points(pts)
    grp.nll_grad(pts[:2])
me = fb.Model.from_string(ref)
fb.set_device_normalization(me, True)
pts_ref = np.array([[d[k] for k in me.param_names] for d in by])
fb.nll_points(me, fb.DataSet.from_columns(fb.sample_host(mo, 9_001, 4)[0]), pts_ref)
fb.device_normalization(me, None, pts_ref)
gw = fb.Model.from_string("observable x -50 50\nparameter mu 0 -1 1\nparameter sigma 1 0.5 2\n"
                          "pdf g Gaussian(x, mu, sigma)\n")
fb.nll(gw, fb.DataSet.from_columns({"x": np.array([0.1, -0.3, float(np.sqrt(1440.0)), 1.2, 40.0])}))
mf2 = fb.Model.from_string(configs.C1.text)
c1, _ = fb.sample_host(mf2, 20_011, 9)
d1 = fb.DataSet.from_columns(c1)
fb.fit_to(mf2, d1)
fb.fit_gradient(mf2, d1, analytic=True)
fb.fit_gradient(mf2, d1, analytic=False)
print("sanitize smoke done")
