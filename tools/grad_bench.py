"""Timing of the fused NLL + gradient pass against one NLL point and the 2d+1-point
finite-difference batch it replaces (C2, C5, C4, C3 shapes; CUDA events on the
launching stream via the library kernel timer)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, torch
import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs
for w in (configs.C2, configs.C5, configs.C4, configs.C3):
    n = min(w.n_events, 50_000_000)
    m = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(m, n, w.data_seed)
    ds = fb.DataSet.from_columns(cols)
    th = m.theta()
    for _ in range(3): fb.nll_grad(m, ds, th); fb.nll_points(m, ds, th[None,:])
    torch.cuda.synchronize()
    fb.kernel_timer(True); fb.kernel_timer_read()
    K=20
    t=time.perf_counter()
    for _ in range(K): fb.nll_grad(m, ds, th)
    wall_g=(time.perf_counter()-t)/K
    kg, c = fb.kernel_timer_read()
    t=time.perf_counter()
    for _ in range(K): fb.nll_points(m, ds, th[None,:])
    wall_n=(time.perf_counter()-t)/K
    kn, c2 = fb.kernel_timer_read()
    d = sum(1 for p in m.param_names if not m.is_constant(p))
    P = 2*d+1
    pts = np.repeat(th[None,:], P, axis=0)
    for _ in range(2): fb.nll_points(m, ds, pts)
    fb.kernel_timer_read()
    t=time.perf_counter()
    for _ in range(K): fb.nll_points(m, ds, pts)
    wall_fd=(time.perf_counter()-t)/K
    kfd, _ = fb.kernel_timer_read()
    print(f"{w.name}: n={n} d={d} grad kernel {kg/K:.3f} ms (wall {wall_g*1e3:.3f}) | nll 1pt kernel {kn/K:.3f} ms (wall {wall_n*1e3:.3f}) | fd {P} pts kernel {kfd/K:.3f} ms (wall {wall_fd*1e3:.3f})", flush=True)
