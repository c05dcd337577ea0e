"""Yield-only fit shape (the config-4 mixture with its shape parameters fixed over the
launch: RooFit's constant-term case): fused-kernel event-points/s for 64 points over 1e8
events, launch-constant whole-leaf cache on (default) and off (FFB_NO_CONST_CACHE=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs

w = configs.C4
n = int(sys.argv[1]) if len(sys.argv) > 1 else w.n_events
m = fb.Model.from_string(w.text)
cols, _ = fb.sample_host(m, n, w.data_seed)
ds = fb.DataSet.from_columns(cols)
pts = w.points(m, n_points=64)
base = m.theta()
for k, name in enumerate(m.param_names):
    if not name.startswith("n"):
        pts[:, k] = base[k]  # shapes fixed: only the yields move
for _ in range(3):
    fb.nll_points(m, ds, pts)
torch.cuda.synchronize()
fb.kernel_timer(True)
fb.kernel_timer_read()
K = 10
for _ in range(K):
    vals, _, _ = fb.nll_points(m, ds, pts)
ms, c = fb.kernel_timer_read()
tag = "off" if os.environ.get("FFB_NO_CONST_CACHE") else "on"
print(f"c4 yields-only cache={tag} cached_terms={fb.last_launch_cached(m)} kernel {ms / c:.3f} ms "
      f"-> {n * len(pts) / (ms / c / 1e3):.3e} event-points/s")
