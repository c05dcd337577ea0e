"""Per-call latency (FFB_NO_GRAPHS=1: without the CUDA-graph replay) of a single-point NLL (what a Minuit / Nelder-Mead caller pays per
function evaluation) on small datasets: wall time per ffcu_nll_points call from Python,
fused-kernel time, and the reference Nelder-Mead fit (ffit_fit) wall time per NLL call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs

w = configs.C1
for n in (10_000, 100_000, 1_000_000):
    m = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(m, n, w.data_seed)
    ds = fb.DataSet.from_columns(cols)
    th = m.theta()[None, :]
    for _ in range(20):
        fb.nll_points(m, ds, th)
    torch.cuda.synchronize()
    K = 200
    t0 = time.perf_counter()
    for _ in range(K):  # (no kernel timer here: it turns the CUDA-graph replay off)
        fb.nll_points(m, ds, th)
    wall = (time.perf_counter() - t0) / K
    fb.kernel_timer(True)
    fb.kernel_timer_read()
    for _ in range(K):
        fb.nll_points(m, ds, th)
    kms, c = fb.kernel_timer_read()
    fb.kernel_timer(False)
    start = w.points(m, n_points=1, seed=7)[0]
    for name, v in zip(m.param_names, start):
        m.set(name, v)
    t0 = time.perf_counter()
    r = fb.fit_to(m, ds, tolerance=1e-8)
    fw = time.perf_counter() - t0
    print(f"n={n}: nll call wall {wall * 1e6:.1f} us, kernel {kms / c * 1e3:.1f} us | "
          f"fit_to: {r.n_nll_calls} calls in {r.n_launches} launches, {fw * 1e3:.1f} ms ({fw / r.n_launches * 1e6:.1f} us per launch)", flush=True)
