"""Diagnostics of the end-to-end (host buffers) step: the bench's double-buffered pipeline
timed with and without its pieces (C2 shape by default; argv[1] = workload)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs

w = {c.name[:2]: c for c in configs.BY_INDEX[:4]}[sys.argv[1] if len(sys.argv) > 1 else "c2"]
m = fb.Model.from_string(w.text)
cols, _ = fb.sample_host(m, w.n_events, w.data_seed)
names = m.observables
pts = w.points(m, n_points=w.n_points)
P = len(pts)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
copy_stream = torch.cuda.Stream(device=dev)
d_sc = torch.zeros((P, 2), dtype=torch.float64, device=dev)
d_bad = torch.zeros(P, dtype=torch.int64, device=dev)
pinned = {k: torch.from_numpy(cols[k]).pin_memory() for k in names}
hp = {k: pinned[k].numpy() for k in names}
bufs = [fb.DataSet.from_columns(cols), fb.DataSet.from_columns(cols)]
res_host = torch.empty((P, 2), dtype=torch.float64).pin_memory()
nbytes = sum(c.nbytes for c in cols.values())


def t(f, K=20):
    f(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(K):
        f(i)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / K * 1e3


def compute(i):
    with torch.cuda.stream(stream):
        fb.nll_points_device(m, bufs[i % 2], pts, d_sc.data_ptr(), d_bad.data_ptr(), stream.cuda_stream)


def copy(i):
    bufs[i % 2].copy_from_host_async(hp, copy_stream.cuda_stream)


def both(i):  # the copy of the other buffer on the copy stream, compute on the compute stream
    copy(i + 1)
    compute(i)


def compute_sync(i):
    compute(i)
    with torch.cuda.stream(stream):
        res_host.copy_(d_sc, non_blocking=True)
    stream.synchronize()


print(f"{w.name}: {nbytes / 1e6:.0f} MB of columns, P={P}")
print(f"  compute only          {t(compute):8.3f} ms/step")
print(f"  copy only             {t(copy):8.3f} ms/step  ({nbytes / t(copy) / 1e6:.1f} GB/s)")
print(f"  copy || compute       {t(both):8.3f} ms/step")
print(f"  compute + D2H + sync  {t(compute_sync):8.3f} ms/step")

# the bench's pipelined loop (bench.py run_ours), timed as there
copied = [torch.cuda.Event() for _ in bufs]
done = [torch.cuda.Event() for _ in bufs]
steps = 20


def upload(i):
    b = i % 2
    copy_stream.wait_event(done[b])
    bufs[b].copy_from_host_async(hp, copy_stream.cuda_stream)
    copied[b].record(copy_stream)


def e2e_step(i):
    b = i % 2
    with torch.cuda.stream(stream):
        stream.wait_event(copied[b])
        fb.nll_points_device(m, bufs[b], pts, d_sc.data_ptr(), d_bad.data_ptr(), stream.cuda_stream)
        done[b].record(stream)
        res_host.copy_(d_sc, non_blocking=True)
    if i + 1 < steps:
        upload(i + 1)
    stream.synchronize()


for i in range(2):
    upload(i)
    e2e_step(i)
torch.cuda.synchronize()
t0 = time.perf_counter()
upload(0)
for i in range(steps):
    e2e_step(i)
torch.cuda.synchronize()
print(f"  bench pipeline        {(time.perf_counter() - t0) / steps * 1e3:8.3f} ms/step")

# depth-2: step i+1 queued before the host reads step i's results
res_ready = [torch.cuda.Event() for _ in bufs]
res2 = [torch.empty((P, 2), dtype=torch.float64).pin_memory() for _ in bufs]


def enqueue(i):
    b = i % 2
    with torch.cuda.stream(stream):
        stream.wait_event(copied[b])
        fb.nll_points_device(m, bufs[b], pts, d_sc.data_ptr(), d_bad.data_ptr(), stream.cuda_stream)
        done[b].record(stream)
        res2[b].copy_(d_sc, non_blocking=True)
        res_ready[b].record(stream)


def run(steps, read=True):
    upload(0)
    for i in range(steps):
        enqueue(i)
        if i + 1 < steps:
            upload(i + 1)
        if i >= 1 and read:
            res_ready[(i - 1) % 2].synchronize()
    res_ready[(steps - 1) % 2].synchronize()


for read in (True, False):
    run(3, read)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(steps, read)
    torch.cuda.synchronize()
    print(f"  depth-2 pipeline read={read}  {(time.perf_counter() - t0) / steps * 1e3:8.3f} ms/step")
