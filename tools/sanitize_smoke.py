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
print("sanitize smoke done")
