"""One shape for profiling the few-point streaming kernel under ncu: C5 model, 5e7 events,
single-point NLL launches (what a Nelder-Mead or Minuit caller issues)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs

w = configs.C5
m = fb.Model.from_string(w.text)
cols, _ = fb.sample_host(m, 50_000_000, w.data_seed)
ds = fb.DataSet.from_columns(cols)
th = m.theta()
for _ in range(5):
    v, _, _ = fb.nll_points(m, ds, th[None, :])
print(v[0], fb.last_launch_jit(m))
