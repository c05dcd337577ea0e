"""The HBM-bound kernel of the path: eval_kernel (PdfSpec::eval_batch / probabilities: one read
and one write of 8 B per event and column) on resident columns, device output, CUDA events on
the launching stream; achieved GB/s against MEASURED_PEAKS.json's copy bandwidth."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2003_12875_b200 as fb  # noqa: E402
from paper_2003_12875_b200 import configs  # noqa: E402

peaks = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
out = {"hbm_peak_gbs": peaks.get("hbm_gbs"), "rows": []}
stream = torch.cuda.Stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for w, n in ((configs.C1, 100_000_000), (configs.C4, 100_000_000), (configs.C3, 50_000_000)):
    m = fb.Model.from_string(w.text)
    cols, _ = fb.sample_host(m, 1_000_000, 7)
    big = {k: np.tile(v, n // len(v)) for k, v in cols.items()}
    ds = fb.DataSet.from_columns(big)
    d_out = torch.empty(n, dtype=torch.float64, device="cuda")
    top = m.pdf_names[-1] if hasattr(m, "pdf_names") else None
    times = []
    for it in range(8):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fb.eval_batch_device(m, top, ds, d_out.data_ptr(), stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        if it >= 3:
            times.append(a.elapsed_time(b))
    ms = float(np.median(times))
    ncols = len(cols)
    bytes_ = n * 8 * (ncols + 1)
    out["rows"].append({"model": w.name, "events": n, "columns": ncols, "ms": ms, "algorithmic_bytes": bytes_,
                        "achieved_gbs": bytes_ / ms / 1e6, "frac_of_hbm_peak": bytes_ / ms / 1e6 / (peaks.get("hbm_gbs") or 1),
                        "events_per_s": n / ms * 1e3, "finite": bool(torch.isfinite(d_out[:1000]).all())})
    del ds, d_out
print(json.dumps(out, indent=1))
