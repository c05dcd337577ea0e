"""One shape for profiling the generic gradient pass under ncu: the config-3 product
(three columns, general plan), 5e7 events, single-point gradient launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs

w = configs.C3
m = fb.Model.from_string(w.text)
cols, _ = fb.sample_host(m, 50_000_000, w.data_seed)
ds = fb.DataSet.from_columns(cols)
th = m.theta()
for _ in range(5):
    v, g, _, _ = fb.nll_grad(m, ds, th)
print(v[0], g[0])
