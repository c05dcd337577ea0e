"""Dataset ingestion: .ffsoa load (pinned, chunked, overlapped H2D)
vs the reference's CSV format (ffit_dataset_read_csv, proj/src/dataset.cpp:61-121) and
vs a pageable host-array upload, on C4-sized data (1e8 rows).  Files go to /tmp; the
first load after writing is served from the page cache (the file was just written)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
rng = np.random.default_rng(1)
x = rng.uniform(-6, 6, n)
path = "/tmp/ffb_bench.ffsoa"
fb.DataSet.from_columns({"x": x[:10]})  # CUDA context outside the timings
t = time.perf_counter()
fb.write_soa(path, {"x": x})
t_write = time.perf_counter() - t
for rep in range(3):
    ds, sec = fb.DataSet.load_soa(path)
    print(f"ffsoa load {n} rows: {sec:.3f} s = {n * 8 / sec / 1e9:.2f} GB/s (rep {rep})", flush=True)
    del ds
t = time.perf_counter()
ds = fb.DataSet.from_columns({"x": x})
t_up = time.perf_counter() - t
print(f"pageable host-array upload: {t_up:.3f} s = {n * 8 / t_up / 1e9:.2f} GB/s; ffsoa write {t_write:.2f} s")
m = fb.Model.from_string(configs.C4.text)
nc = min(n, 5_000_000)
csv = "/tmp/ffb_bench.csv"
with open(csv, "w") as fh:
    fh.write("x\n")
    np.savetxt(fh, x[:nc], fmt="%.17g")
t = time.perf_counter()
d2 = fb.DataSet.read_csv(m, csv)
t_csv = time.perf_counter() - t
print(f"CSV read {nc} rows: {t_csv:.3f} s = {nc / t_csv / 1e6:.2f} M rows/s "
      f"(-> {n / (nc / t_csv):.1f} s for {n} rows)")
os.remove(path)
os.remove(csv)
