#!/usr/bin/env python
"""Benchmark of the hot path: batched PDF-graph evaluation + unbinned NLL over
SoA fp64 event columns, P parameter points per launch (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

One step = one multi-point launch of the workload's P parameter points over the
rank's HBM-resident shard (weak scaling: every rank owns a full config-sized
shard), plus, for N > 1, the one exchange step of the path: an NCCL all-gather of
the per-point Neumaier pairs and a fixed-rank-order combine kernel.  The default
workload is BASELINE configs[1] (Gauss + ArgusBG, 1e7 events, 200 points).

Rank 0 prints one JSON line.  `--impl reference` times the reference's own CPU
implementation (oracle/_ref: the unmodified reference engine compiled from its
sources; the C restatement when that library is absent) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NLL events/sec (fp64) at 1/2/4/8 B200; % of HBM/FP64 roofline vs host CPU"
UNIT = "event-points/s"


def env_int(k, d):
    return int(os.environ.get(k, d))


# The JSON line goes to the ORIGINAL stdout; everything else that writes to fd 1
# (NCCL's version banner, library chatter) is redirected to stderr, so rank 0's
# stdout carries exactly one line.
_JSON_OUT = None


def _claim_stdout():
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line):
    _claim_stdout()
    _JSON_OUT.write(json.dumps(line) + "\n")
    _JSON_OUT.flush()


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)

class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index, out_path=None):
        self.gpu_index = gpu_index
        self.rows = []
        self.proc = None
        self.out_path = out_path

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu_index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, ValueError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        if self.out_path:
            with open(self.out_path, "w") as fh:
                fh.write(self.QUERY + "\n")
                for r in self.rows:
                    fh.write(",".join(r) + "\n")
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------

def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def profiled(workload, key):
    """A figure of the committed ncu --set full capture (profiles/ncu_summary.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            d = json.load(fh)
        return d.get(workload, {}).get(key)
    except (OSError, ValueError):
        return None


def profiled_traffic(workload):
    """dram bytes per fused-kernel launch from the committed ncu --set full capture."""
    return profiled(workload, "dram_bytes_per_launch")


def shard_seed(w, rank):
    return w.data_seed if rank == 0 else w.data_seed + 100003 * rank


def cpu_baseline_port(w, cols_list, pts, n):
    """The C restatement (oracle port) on the host cores, bounded sample."""
    from oracle.oracle import OracleModel
    threads = os.cpu_count() or 1
    o = OracleModel(w.text)
    # batches of one point per thread until ~12 s of CPU work (threads x wall), all points,
    # or 20 s wall -- whichever comes first
    step = max(8, threads)
    Pc, dt = 0, 0.0
    while Pc < len(pts) and dt * threads < 12.0 and dt < 20.0:
        k = min(step, len(pts) - Pc)
        t0 = time.perf_counter()
        o.nll_points(cols_list, pts[Pc:Pc + k], threads=threads)
        dt += time.perf_counter() - t0
        Pc += k
    return {"value": n * Pc / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{Pc} of the {len(pts)} points x all {n} events, oracle/ffit_oracle.c, "
                      f"{threads} threads, {dt:.2f} s wall (~{dt * threads:.0f} s of CPU work)"}


# ---------------------------------------------------------------------------

def run_ours(args, w):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2003_12875_b200 as fb

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # the exchange step (NCCL all-gather + fixed-order combine) runs whenever there is
    # more than one rank; --force-collective runs it at N = 1 too (exercises the path)
    coll = world > 1 or args.force_collective
    if coll:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=dev)

    model = fb.Model.from_string(w.text)
    n = args.events or w.n_events
    load_s = None
    if args.inputs:
        # tools/make_inputs.py output: the same seeded events, from disk through the
        # pinned overlapped .ffsoa upload (its time reported as config.inputs_load_s)
        import json as _json
        stem = os.path.join(args.inputs, w.name + (f".r{rank}" if rank else ""))
        man = _json.load(open(stem + ".json"))
        if man["seed"] != shard_seed(w, rank) or (args.events and man["n"] != n):
            raise SystemExit(f"{stem}.json does not match this run (seed/events)")
        n = man["n"]
        ds_disk, load_s = fb.DataSet.load_soa(stem + ".ffsoa")
        cols = {k: ds_disk.column(k) for k in man["columns"]}
        del ds_disk
    else:
        cols, _ = fb.sample_host(model, n, shard_seed(w, rank))
    if args.spelling == "reference":
        # the reference's own model text (C2: ArgusBG as an Expression pdf) through the
        # device Expression interpreter, on the same events
        from paper_2003_12875_b200 import configs as _cfg
        model = fb.Model.from_string(_cfg.REFERENCE_TEXTS[w.name])
    names = model.observables
    ds = fb.DataSet.from_columns(cols)
    pts = w.points(model, n_points=args.points)
    P = len(pts)

    stream = torch.cuda.Stream(device=dev)
    d_sc = torch.zeros((P, 2), dtype=torch.float64, device=dev)
    d_bad = torch.zeros(P, dtype=torch.int64, device=dev)
    gathered = torch.zeros((world, P, 2), dtype=torch.float64, device=dev)
    final = torch.zeros((P, 2), dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step():
        with torch.cuda.stream(stream):
            fb.nll_points_device(model, ds, pts, d_sc.data_ptr(), d_bad.data_ptr(), stream.cuda_stream)
            if coll:
                dist.all_gather_into_tensor(gathered.view(world * P, 2), d_sc)
                fb.ffit.combine_pairs_device(gathered.data_ptr(), world, P, final.data_ptr(),
                                             stream.cuda_stream)

    peak_fma, _ = fb.fp64_peak()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local, os.path.join(ROOT, "gpurun_out", "clocks.csv")
                          if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else None)
    clocks.start()
    time.sleep(0.3)
    fb.kernel_timer(True)
    fb.kernel_timer_read()
    launches0 = fb.kernel_launches()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if coll:
        dist.barrier()
    torch.cuda.synchronize()
    for a, b in evs:
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush between timed steps, outside the step's events
        a.record(stream)
        step()
        b.record(stream)
    torch.cuda.synchronize()
    if coll:
        dist.barrier()
    launches = fb.kernel_launches() - launches0
    build = {0: "static build", 1: "formula-specialised NVRTC build",
             2: "plan-specialised NVRTC build"}.get(fb.last_launch_jit(model), "?")
    cached_terms = fb.last_launch_cached(model)
    kms, kcount = fb.kernel_timer_read()
    fb.kernel_timer(False)
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if coll:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = world * n * P * args.steps / (total_ms / 1e3)

    # sanity of the result (finite, no invalid event)
    res = (final if coll else d_sc).cpu().numpy()
    ok = bool(np.all(np.isfinite(res)) and int((d_bad.cpu().numpy() != -1).sum()) == 0)

    # --- end-to-end through the C ABI with host buffers (H2D + launch + D2H per step).
    # A double-buffered pipeline: step i+1's events are copied from pinned host memory into
    # the other device dataset on a copy stream while step i computes (a buffer is refilled
    # only after the step that read it has finished: events); step i+1 is queued -- its
    # constant rows copied on the same copy stream, so no H2D waits behind step i's kernel --
    # before the host reads step i's P results, and every step's results come back.
    pinned = {k: torch.from_numpy(cols[k]).pin_memory() for k in names}
    host_ptr_cols = {k: pinned[k].numpy() for k in names}
    e2e_steps = max(3, min(args.steps, 20))
    bufs = [ds, fb.DataSet.from_columns(cols)]
    copy_stream = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event() for _ in bufs]
    done = [torch.cuda.Event() for _ in bufs]
    res_ready = [torch.cuda.Event() for _ in bufs]
    res_host = [torch.empty((P, 2), dtype=torch.float64).pin_memory() for _ in bufs]

    def upload(i):
        b = i % 2
        copy_stream.wait_event(done[b])  # the step that last read this buffer has finished
        bufs[b].copy_from_host_async(host_ptr_cols, copy_stream.cuda_stream)
        copied[b].record(copy_stream)

    def enqueue(i):
        b = i % 2
        with torch.cuda.stream(stream):
            stream.wait_event(copied[b])
            fb.nll_points_device(model, bufs[b], pts, d_sc.data_ptr(), d_bad.data_ptr(), stream.cuda_stream,
                                 copy_stream.cuda_stream)
            out = d_sc
            if coll:
                dist.all_gather_into_tensor(gathered.view(world * P, 2), d_sc)
                fb.ffit.combine_pairs_device(gathered.data_ptr(), world, P, final.data_ptr(), stream.cuda_stream)
                out = final
            done[b].record(stream)
            res_host[b].copy_(out, non_blocking=True)
            res_ready[b].record(stream)

    def run_e2e(steps):
        results = []
        upload(0)
        for i in range(steps):
            enqueue(i)
            if i + 1 < steps:
                upload(i + 1)  # overlaps step i's compute
            if i >= 1:  # step i is queued: read step i-1's results
                res_ready[(i - 1) % 2].synchronize()
                results.append(res_host[(i - 1) % 2].numpy().copy())
        res_ready[(steps - 1) % 2].synchronize()
        results.append(res_host[(steps - 1) % 2].numpy().copy())
        return results

    run_e2e(3)  # warm the pipeline's streams and events
    if coll:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_results = run_e2e(e2e_steps)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    host_res = torch.from_numpy(e2e_results[-1])
    assert len(e2e_results) == e2e_steps and np.isfinite(e2e_results[-1]).all()
    t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if coll:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    e2e = {"value": world * n * P * e2e_steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(n * 8 * len(names) + P * model.plan()[2] * 8),
           "d2h_bytes_per_step": int(host_res.numel() * 8),
           "path": "ffcu_dataset_copy_from_host_async (pinned, double-buffered: step i+1's copy overlaps step i) "
                   "+ ffcu_nll_points_device_upload (constant rows on the copy stream; step i+1 queued before "
                   "step i's results are read)" + (" + NCCL all_gather + combine" if coll else "")
                   + " + D2H of the P results every step"}

    avg_kernel_ms = kms / max(kcount, 1)
    instr = w.fp64_instr_per_event_point * n * P
    achieved = instr / (avg_kernel_ms / 1e3) / 1e12
    peak = peak_fma / 1e12
    info = fb.last_launch(model)
    roofline = {
        "bound": "fp64", "unit": "T fp64-instr/s",
        "achieved": achieved, "peak": peak, "frac": achieved / peak,
        "peak_source": "measured live: DFMA-chain microbenchmark (ffcu_fp64_peak); MEASURED_PEAKS.json has no FP64 figure",
        "work_per_event_point": w.fp64_instr_per_event_point,
        "kernel": f"nll_kernel<256,8> ({build}"
                  + (f", {cached_terms} launch-constant cached term(s)" if cached_terms else "") + ")",
        "kernel_ms_avg": avg_kernel_ms, "kernel_launches_timed": kcount,
        "kernel_share_of_step": avg_kernel_ms / (total_ms / args.steps),
        "hbm_algorithmic_bytes_per_launch": n * w.bytes_per_event,
        "hbm_achieved_gbs": n * w.bytes_per_event * info["nchunks"] / (avg_kernel_ms / 1e3) / 1e9,
        "hbm_peak_gbs": peaks().get("hbm_gbs"),
        "traffic": profiled_traffic(w.name),
        # the same kernel's measured FP64-pipe busy fraction (ncu), beside the work-model frac
        "ncu_fp64_pipe_active": profiled(w.name, "fp64_pipe_active"),
        "ncu_source": profiled(w.name, "source"),
        "frac_note": "achieved counts the SURVEY 8(d) algorithmic work (libdevice-weighted ops of the "
                     "reference's per-event algorithm); the kernel executes fewer (table-driven exp/log, "
                     "launch-constant caches), so frac can exceed 1 -- the executed bound is "
                     "ncu_fp64_pipe_active (DESIGN.md, 'Why frac exceeds 1.0')",
    }

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, reference Rng)",
        "config": {"workload": w.name, "description": w.description, "events_per_gpu": n, "points_per_launch": P,
                   "l2": "flushed between timed steps (512 MiB write)",
                   "parallelism": f"event shards x{world}" + (", NCCL all_gather of 2P doubles" if coll else ""),
                   "launch": info, "spelling": args.spelling,
                   "inputs": args.inputs or "generated in-process (seeded)", "inputs_load_s": load_s},
        "roofline": roofline, "e2e": e2e, "clocks": clk, "gpu_launches": int(launches),
        "result_finite": ok,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_port(w, [cols[k] for k in names], pts, n)
    if rank == 0:
        emit(line)
    if coll:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation on the host cores

def run_reference(args, w):
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    if rank != 0:
        return
    import numpy as np

    from oracle import oracle as orc
    from paper_2003_12875_b200 import configs

    threads = os.cpu_count() or 1
    n_full = args.events or w.n_events
    o = orc.OracleModel(w.text)
    # inputs: the same seeded columns the GPU arm reads (C restatement of the generator,
    # bit-identical to the library's); the timed code never touches the product
    pts_all = _points_for_reference(w, o, args.points)
    cols, _ = o.sample(n_full, w.data_seed)
    ref_text = configs.REFERENCE_TEXTS.get(w.name)
    use_ref = orc.ref_available() and ref_text is not None
    budget = max(2.0, 150.0 / (args.steps + args.warmup))
    Pc = min(len(pts_all), threads)
    names = [nm for nm in o.param_names if nm in _ref_param_names(ref_text)] if use_ref else o.param_names
    idx = [o.param_names.index(nm) for nm in names]
    pts = pts_all[:Pc][:, idx] if use_ref else pts_all[:Pc]

    def run(nsub):
        sub = [c[:nsub] for c in cols]
        if use_ref:
            ds = orc.RefDataset(o.obs[0][0], sub[0])
            t0 = time.perf_counter()
            orc.ref_nll_points_threaded(ref_text, ds, names, pts, threads)
            return time.perf_counter() - t0
        t0 = time.perf_counter()
        o.nll_points(sub, pts, threads=threads)
        return time.perf_counter() - t0

    probe_n = min(n_full, 100_000)
    tp = run(probe_n)
    per_event = max(tp, 1e-6) / probe_n
    nsub = int(min(n_full, max(probe_n, budget / per_event)))
    for _ in range(args.warmup):
        run(nsub)
    times = [run(nsub) for _ in range(args.steps)]
    total = sum(times)
    value = nsub * Pc * args.steps / total
    kind = "reference" if use_ref else "port"
    sample = (f"{Pc} of the {len(pts_all)} points x first {nsub} of {n_full} events per step, "
              + ("oracle/_ref (unmodified reference engine, " + configs.REFERENCE_NOTES.get(w.name, "") + ")"
                 if use_ref else "oracle/ffit_oracle.c restatement")
              + f", {threads} threads, BatchPrecise")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, reference Rng)",
        "config": {"workload": w.name, "description": w.description, "events_per_gpu": n_full,
                   "points_per_launch": len(pts_all)},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def run_fit(args, w):
    """BASELINE configs[4]: the Minuit-style fit loop (BFGS on central differences,
    2d+1 points per launch, Hessian points in one launch) on one GPU; value = event-points/s
    through the whole fit, plus NLL evaluations/s, fit wall time and the fitted parameters."""
    import numpy as np
    import torch

    import paper_2003_12875_b200 as fb

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if rank != 0:
        return
    torch.cuda.set_device(local)
    n = args.events or w.n_events
    truth = fb.Model.from_string(w.text)
    t0 = time.perf_counter()
    cols, _ = fb.sample_host(truth, n, w.data_seed)
    t_gen = time.perf_counter() - t0
    ds = fb.DataSet.from_columns(cols)
    model = fb.Model.from_string(w.text)
    start = w.points(model, n_points=1, seed=w.point_seed)[0]
    for name, v in zip(model.param_names, start):
        if not model.is_constant(name):
            model.set(name, v)
    fb.nll_points(model, ds, start[None, :])  # warm-up (module load, first launch)
    jit_s = None
    if args.gradient == "fd":
        # one-time run-time compile of the plan-specialised likelihood build the fit's
        # (2d+1)-point launches take (NVRTC), outside the timed fit, reported beside it
        free = [k for k, name in enumerate(model.param_names) if not model.is_constant(name)]
        rows = [start]
        for k in free:
            for sgn in (1.0, -1.0):
                r_ = start.copy()
                r_[k] += sgn * 1e-6 * max(abs(start[k]), 1.0)
                rows.append(r_)
        t0 = time.perf_counter()
        fb.nll_points(model, ds, np.array(rows))
        jit_s = time.perf_counter() - t0
    if args.gradient == "analytic":
        # one-time run-time compile of the plan-specialised gradient pass (NVRTC), outside
        # the timed fit and reported beside it
        t0 = time.perf_counter()
        fb.nll_grad(model, ds, start)
        jit_s = time.perf_counter() - t0
    torch.cuda.synchronize()
    fb.kernel_timer(True)
    fb.kernel_timer_read()
    launches0 = fb.kernel_launches()
    analytic = args.gradient == "analytic"
    r = fb.fit_gradient(model, ds, tolerance=1e-12, max_iterations=args.iterations, analytic=analytic)
    torch.cuda.synchronize()
    kms, kcount = fb.kernel_timer_read()
    launches = fb.kernel_launches() - launches0
    d = sum(1 for p in model.param_names if not model.is_constant(p))
    line = {
        "metric": METRIC, "value": r.n_nll_calls * n / r.wall_seconds, "unit": UNIT, "n_gpus": 1,
        "steps": r.iterations, "warmup": 1, "ms_per_step": 1e3 * r.wall_seconds / max(r.n_launches, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, reference Rng)",
        "config": {"workload": w.name, "description": w.description, "events_per_gpu": n,
                   "gradient": "analytic (fused NLL + gradient pass, one point per launch)" if r.analytic_gradient
                   else "central differences (2d+1 points per launch)",
                   "points_per_launch": 1 if r.analytic_gradient else 2 * d + 1, "free_parameters": d},
        "fit": {"converged": r.converged, "iterations": r.iterations, "launches": r.n_launches,
                "nll_evaluations": r.n_nll_calls, "nll_evaluations_per_s": r.n_nll_calls / r.wall_seconds,
                "wall_seconds": r.wall_seconds, "kernel_ms_total": kms, "kernel_launches_timed": kcount,
                "nll_min": r.nll_min, "analytic_gradient": r.analytic_gradient,
                "first_call_s": jit_s,
                "first_call": "the one-time NVRTC build of the launch shape the fit uses (plan-specialised "
                              "likelihood for FD, gradient pass for analytic), outside the timed fit",
                "kernel_ms_per_launch": kms / max(kcount, 1),
                "parameters": {p.name: [p.value, p.uncertainty] for p in r.parameters},
                "truth": dict(zip(truth.param_names, [float(v) for v in truth.theta()])),
                "data_generation_s": t_gen},
        "gpu_launches": int(launches),
    }
    emit(line)


def _ref_param_names(text):
    out = []
    for line in (text or "").splitlines():
        t = line.split()
        if t and t[0] == "parameter" and not (len(t) == 6 and t[5] == "const"):
            out.append(t[1])
    return out


def _points_for_reference(w, o, n_points):
    """Same points as the GPU arm (configs.Workload.points over the oracle's parameter table)."""
    class _M:
        param_names = o.param_names

        @staticmethod
        def theta():
            return o.theta.copy()
    return w.points(_M, n_points=n_points)


def main():
    _claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", help="c1..c5 or a configs.WORKLOADS name")
    ap.add_argument("--events", type=int, default=0, help="override events per GPU")
    ap.add_argument("--points", type=int, default=None, help="override points per launch")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fit", action="store_true", help="time the Minuit-style fit loop (config 5 style)")
    ap.add_argument("--force-collective", action="store_true",
                    help="run the NCCL all-gather + combine exchange even at N = 1")
    ap.add_argument("--iterations", type=int, default=50, help="fit iterations (--fit / c5)")
    ap.add_argument("--inputs", default="", help="directory of tools/make_inputs.py files (.ffsoa + manifest)")
    ap.add_argument("--spelling", default="ours", choices=["ours", "reference"],
                    help="model text: ours (ArgusBG kind) or the reference's (Expression pdf)")
    ap.add_argument("--gradient", default="fd", choices=["fd", "analytic"],
                    help="c5 fit gradients: central differences (the config's 2d+1 points per launch) "
                         "or the fused NLL + gradient pass")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    from paper_2003_12875_b200 import configs
    if args.workload in configs.WORKLOADS:
        w = configs.WORKLOADS[args.workload]
    else:
        w = configs.BY_INDEX[int(args.workload.lstrip("c")) - 1]
    if args.impl == "reference":
        run_reference(args, w)
    elif args.fit or w is configs.C5:
        run_fit(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
