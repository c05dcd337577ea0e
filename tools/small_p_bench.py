"""Few-point NLL launches (what a Minuit-style caller issues): fused-kernel time per
launch for P = 1, 2, 4, 8, 16 points on the C1 / C2 / C5 shapes (CUDA events on the
launching stream via the library kernel timer).  FFB_NO_STREAM=1 forces the
tile-per-CTA kernel for the A/B."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs

tag = "tile" if os.environ.get("FFB_NO_STREAM") else "stream"
for w, n in ((configs.C1, 1_000_000), (configs.C2, 10_000_000), (configs.C5, 50_000_000), (configs.C3, 50_000_000)):
    m = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(m, n, w.data_seed)
    ds = fb.DataSet.from_columns(cols)
    allpts = w.points(m, n_points=16)
    row = []
    for P in (1, 2, 4, 8, 16):
        pts = allpts[:P]
        for _ in range(3):
            fb.nll_points(m, ds, pts)
        torch.cuda.synchronize()
        fb.kernel_timer(True)
        fb.kernel_timer_read()
        K = 30
        for _ in range(K):
            fb.nll_points(m, ds, pts)
        ms, cnt = fb.kernel_timer_read()
        fb.kernel_timer(False)
        per = ms / cnt
        row.append(f"P={P}: {per:.4f} ms ({n * P / (per * 1e-3):.3e} ev-pt/s)")
    print(f"[{tag}] {w.name} n={n}: " + " | ".join(row), flush=True)
