"""Host vs device numeric normalisation on BASELINE config 2 as the reference spells it (ArgusBG as
an Expression pdf inside a WeightedSum: two Simpson-normalised nodes per point), 200 points:
  * the normalisations alone: host loop (ffcu_normalization, one thread) vs ffcu_device_normalization;
  * a whole synchronous likelihood call (rows + launch + read-back) on a small dataset, where the
    rows dominate, and on 1e7 events."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2003_12875_b200 as fb  # noqa: E402
from paper_2003_12875_b200 import configs  # noqa: E402


def best(f, reps=7):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return min(ts)


w = configs.C2
m = fb.Model.from_string(configs.REFERENCE_TEXTS[w.name])
pts = w.points(m, n_points=200)
out = {"points": 200, "model": "c2 reference text (Expression ArgusBG in a WeightedSum)"}
fb.device_normalization(m, "model", pts)  # warm-up (sub-plans, buffers)
out["norms_host_one_thread_ms"] = 1e3 * best(lambda: [fb.normalization(m, "model", p) for p in pts], 3)
out["norms_device_ms"] = 1e3 * best(lambda: fb.device_normalization(m, "model", pts))
for n in (20_000, 10_000_000):
    cols, _ = fb.sample_host(fb.Model.from_string(w.text), n, 1002)
    ds = fb.DataSet.from_columns(cols)
    for on in (False, True):
        fb.set_device_normalization(m, on)
        fb.nll_points(m, ds, pts)
        fb.nll_points(m, ds, pts)
        out[f"nll_call_{n}_events_{'device' if on else 'host'}_norm_ms"] = 1e3 * best(lambda: fb.nll_points(m, ds, pts))
print(json.dumps(out, indent=1))
