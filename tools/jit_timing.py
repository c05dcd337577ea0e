"""First-call (NVRTC compile + module load) vs steady-state cost of the run-time builds:
the plan-specialised gradient pass (C5 model) and the formula-specialised Expression
likelihood (the reference's config-2 text)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs

w = configs.C5
m = fb.Model.from_string(w.text)
cols, _ = fb.sample_host(m, 1_000_000, 1)
ds = fb.DataSet.from_columns(cols)
th = m.theta()
fb.nll_points(m, ds, th)  # CUDA context and static kernels outside the timing
for i in range(3):
    t = time.perf_counter()
    fb.nll_grad(m, ds, th)
    print(f"gradient call {i}: {1e3 * (time.perf_counter() - t):.1f} ms, specialised={fb.last_grad_jit(m)}")
me = fb.Model.from_string(configs.REFERENCE_TEXTS[configs.C2.name])
for i in range(3):
    t = time.perf_counter()
    fb.nll_points(me, ds, me.theta())
    print(f"Expression likelihood call {i}: {1e3 * (time.perf_counter() - t):.1f} ms, jit={fb.last_launch_jit(me)}")
print(fb.expression_jit_status())
