#!/usr/bin/env python
"""Benchmark of the hot path: batched PDF-graph evaluation + unbinned NLL over SoA fp64
event columns, P parameter points per launch (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4] [--impl ours|reference]

Default workload: BASELINE configs[3] (C4: extended AddPdf of 5 Gaussians + Exponential,
1e8 events, 64 points), the config the metric's "1/2/4/8 B200" is quoted on.  Strong
scaling: the config's events are split into N contiguous shards (one per rank, resident in
its HBM); one step = one launch of all P points on every shard plus, for N > 1, the path's
one exchange step -- ONE NCCL all-gather of each rank's [P Neumaier pairs | P first-invalid
indices] and a rank-order combine kernel, inside the library (ffcu_shard_group_*).

Rank 0 prints one JSON line.  `--impl reference` times the reference's own CPU engine
(oracle/_ref: the unmodified reference compiled from its sources) on the host cores, on the
same workload as configs.REF_ARMS spells it for the reference's grammar.
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
L2_NOTE = "GPU arm: L2 flushed between timed steps (512 MiB write); inputs >= 80 MB"


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
    """A figure of the committed ncu captures (profiles/ncu_summary.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            d = json.load(fh)
        return d.get(workload, {}).get(key)
    except (OSError, ValueError):
        return None


def shard_bounds(n, world, rank):
    return (n * rank) // world, (n * (rank + 1)) // world


def config_for(w, n_total, world, P):
    """The workload as both arms report it (identical dicts: the driver compares them)."""
    return {"workload": w.name, "description": w.description, "events_total": n_total,
            "events_per_gpu": -(-n_total // world), "points_per_launch": P,
            "parallelism": f"event shards x{world}" + (" + one NCCL all-gather of 3P words per launch"
                                                      if world > 1 else ""),
            "scaling_rule": "strong: the config's events split into N contiguous shards",
            "l2": L2_NOTE}


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        gxx = subprocess.run(["g++", "--version"], capture_output=True, text=True).stdout.splitlines()[0]
    except (OSError, IndexError):
        gxx = None
    try:
        affinity = len(os.sched_getaffinity(0))
    except AttributeError:
        affinity = os.cpu_count()
    return {"nproc": affinity, "cpu_model": model, "compiler": gxx}


# ---------------------------------------------------------------------------
# the reference's own CPU engine (oracle/_ref) on the host cores -- the CPU baseline and
# the reference arm.  Test infrastructure: the one place bench.py executes oracle/.

class RefRunner:
    """The workload through the unmodified reference engine as configs.REF_ARMS spells it:
    each part one reference model over its column; ref_nll_points_threaded runs T host
    threads, each with its own Model over the shared immutable DataSet."""

    MODES = {0: "Scalar", 1: "BatchPrecise", 2: "BatchFast"}

    def __init__(self, w, cols_by_name, pts):
        from oracle import oracle as orc
        from paper_2003_12875_b200 import configs
        self.orc = orc
        self.arm = configs.REF_ARMS[w.name]
        self.cols = cols_by_name
        self.pts = pts
        self.n_full = len(next(iter(cols_by_name.values())))
        self._ds = {}

    def available(self, variant=None):
        return self.orc.ref_available(variant)

    def _column(self, variant, name, nsub):
        """The reference DataSet of the first nsub events of a column, made once (outside the
        timed calls: the reference's DataSet owns a copy of its columns)."""
        key = (variant, name, nsub)
        if key not in self._ds:
            if len(self._ds) > 8:
                self._ds.clear()
            self._ds[key] = self.orc.RefColumn(variant, name, self.cols[name][:nsub])
        return self._ds[key]

    def call(self, nsub, pts, threads, variant=None, mode=1):
        """Wall seconds of one reference evaluation of `pts` over the first nsub events."""
        cols = [self._column(variant, part.column, nsub) for part in self.arm.parts]
        rows = [part.rows(pts) for part in self.arm.parts]
        t0 = time.perf_counter()
        vals = 0.0
        for part, c, r in zip(self.arm.parts, cols, rows):
            vals = vals + c.nll_points(part.text, part.names, r, threads, mode)
        if self.arm.extended is not None:
            vals = vals + self.arm.extended(pts, nsub)
        return time.perf_counter() - t0, vals

    def sample_size(self, target_s, threads=1, variant=None, mode=1):
        """Events per call so that one call of one point per thread takes ~target_s."""
        probe = min(self.n_full, 100_000)
        pts = self.pts[:threads]
        dt, _ = self.call(probe, pts, threads, variant, mode)
        per = max(dt, 1e-6) / probe
        return int(min(self.n_full, max(probe, target_s / per)))

    def matrix(self, scalar=False):
        """{Release build, the -march build the host supports} x
        {BatchPrecise, BatchFast (, Scalar)} x {1 core, all cores}; median of 7 calls
        (proj/tools/ffit_main.cpp:59-73) on a bounded sample."""
        info = host_info()
        T = info["nproc"] or 1
        levels = self.orc.host_isa_levels()
        best = levels[-1] if levels and self.available(levels[-1]) else None
        builds = [(None, "-std=c++20 -O3 -DNDEBUG (the reference's Release flags)")]
        if best:
            builds.append((best, f"-std=c++20 -O3 -DNDEBUG -march=x86-64-{best} (the -march=native stand-in: "
                                 f"highest ISA level this host reports)"))
        modes = [1, 2] + ([0] if scalar else [])
        cells = []
        for variant, flags in builds:
            for mode in modes:
                for threads in (1, T):
                    nsub = self.sample_size(0.12, 1, variant, mode)
                    pts = self.pts[:threads] if len(self.pts) >= threads else \
                        self.pts[[i % len(self.pts) for i in range(threads)]]
                    times = sorted(self.call(nsub, pts, threads, variant, mode)[0] for _ in range(7))
                    med = times[3]
                    cells.append({"build": variant or "release", "mode": self.MODES[mode], "threads": threads,
                                  "value": nsub * len(pts) / med, "unit": UNIT, "events": nsub, "points": len(pts),
                                  "median_s": med, "flags": flags})
        return {"cells": cells, "method": "median of 7 calls (proj/tools/ffit_main.cpp:59-73); 1 core = one "
                                          "point per call, all cores = one point per thread per call",
                "spelling": self.arm.note, **info}


# ---------------------------------------------------------------------------

def generate_shard(fb, model, w, n_total, b, e, inputs, rank):
    """The rank's rows [b, e) of the config's seeded events (every rank draws the same
    stream: the generator is sequential), or from tools/make_inputs.py files."""
    if inputs:
        stem = os.path.join(inputs, w.name)
        man = json.load(open(stem + ".json"))
        if man["seed"] != w.data_seed or man["n"] != n_total:
            raise SystemExit(f"{stem}.json does not match this run (seed/events)")
        ds_disk, load_s = fb.DataSet.load_soa(stem + ".ffsoa")
        cols = {k: ds_disk.column(k)[b:e].copy() for k in man["columns"]}
        return cols, load_s
    full, _ = fb.sample_host(model, n_total, w.data_seed)
    return {k: v[b:e].copy() for k, v in full.items()}, None


def run_ours(args, w):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2003_12875_b200 as fb

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    coll = world > 1 or args.force_collective
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)

    model = fb.Model.from_string(w.text)
    n_total = args.events or w.n_events
    b, e = shard_bounds(n_total, world, rank)
    n = e - b
    t0 = time.perf_counter()
    cols, load_s = generate_shard(fb, model, w, n_total, b, e, args.inputs, rank)
    gen_s = time.perf_counter() - t0
    names = model.observables
    ds = fb.DataSet.from_columns(cols)
    pts = w.points(model, n_points=args.points)
    P = len(pts)

    def broadcast(obj):
        if world == 1:
            return obj
        box = [obj]
        dist.broadcast_object_list(box, src=0)
        return box[0]

    group = fb.ShardGroup.for_rank(model, ds, n_total, b, world, rank, broadcast) if coll else None

    stream = torch.cuda.Stream(device=dev)
    d_sc = torch.zeros((P, 2), dtype=torch.float64, device=dev)
    d_bad = torch.zeros(P, dtype=torch.int64, device=dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step(dset=ds, grp=group, upload_stream=None):
        with torch.cuda.stream(stream):
            if grp is not None:
                grp.nll_points_device(pts, d_sc.data_ptr(), d_bad.data_ptr(), stream.cuda_stream, upload_stream)
            else:
                fb.nll_points_device(model, dset, pts, d_sc.data_ptr(), d_bad.data_ptr(), stream.cuda_stream,
                                     upload_stream)

    def timed(nsteps, warm):
        for _ in range(warm):
            step()
        torch.cuda.synchronize()
        fb.kernel_timer(True)
        fb.kernel_timer_read()
        launches0 = fb.kernel_launches()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nsteps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for a, bb in evs:
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush between timed steps, outside the step's events
            a.record(stream)
            step()
            bb.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches = fb.kernel_launches() - launches0
        kms, kcount = fb.kernel_timer_read()
        fb.kernel_timer(False)
        total_ms = sum(a.elapsed_time(bb) for a, bb in evs)
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), kms / max(kcount, 1), kcount, launches

    peak_fma, _ = fb.fp64_peak()
    clocks = ClockSampler(local, os.path.join(ROOT, "gpurun_out", "clocks.csv")
                          if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else None)
    clocks.start()
    time.sleep(0.3)
    total_ms, avg_kernel_ms, kcount, launches = timed(args.steps, args.warmup)
    clk = clocks.stop()
    value = n_total * P * args.steps / (total_ms / 1e3)
    build = {0: "static build", 1: "formula-specialised NVRTC build",
             2: "plan-specialised NVRTC build"}.get(fb.last_launch_jit(model), "?")
    cached_terms = fb.last_launch_cached(model)
    info = fb.last_launch(model)
    res = d_sc.cpu().numpy()
    ok = bool(np.all(np.isfinite(res)) and int((d_bad.cpu().numpy() != -1).sum()) == 0)
    if world > 1:
        okt = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)  # every rank's results, not only rank 0's
        ok = bool(okt.item())

    # --- end to end through the C ABI with host buffers (H2D + launch + D2H per step).
    # A double-buffered pipeline: step i+1's shard is copied from pinned host memory into the
    # other device dataset on a copy stream while step i computes (a buffer is refilled only
    # after the step that read it has finished: events); step i+1 is queued -- its constant
    # rows copied on the same copy stream -- before the host reads step i's P results.  For
    # N > 1 each buffer has its own shard group (its own NCCL communicator).
    pinned = {k: torch.from_numpy(cols[k]).pin_memory() for k in names}
    host_ptr_cols = {k: pinned[k].numpy() for k in names}
    e2e_steps = max(3, min(args.steps, 20))
    bufs = [ds, fb.DataSet.from_columns(cols)]
    groups = [group, fb.ShardGroup.for_rank(model, bufs[1], n_total, b, world, rank, broadcast)] if coll else [None, None]
    copy_stream = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event() for _ in bufs]
    done = [torch.cuda.Event() for _ in bufs]
    res_ready = [torch.cuda.Event() for _ in bufs]
    res_host = [torch.empty((P, 2), dtype=torch.float64).pin_memory() for _ in bufs]

    def upload(i):
        k = i % 2
        copy_stream.wait_event(done[k])  # the step that last read this buffer has finished
        bufs[k].copy_from_host_async(host_ptr_cols, copy_stream.cuda_stream)
        copied[k].record(copy_stream)

    def enqueue(i):
        k = i % 2
        with torch.cuda.stream(stream):
            stream.wait_event(copied[k])
            step(bufs[k], groups[k], copy_stream.cuda_stream)
            done[k].record(stream)
            res_host[k].copy_(d_sc, non_blocking=True)
            res_ready[k].record(stream)

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
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_results = run_e2e(e2e_steps)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    assert len(e2e_results) == e2e_steps and np.isfinite(e2e_results[-1]).all()
    t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    e2e = {"value": n_total * P * e2e_steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(n * 8 * len(names) + P * model.plan()[2] * 8),
           "d2h_bytes_per_step": int(P * 2 * 8),
           "path": "ffcu_dataset_copy_from_host_async (pinned, double-buffered: step i+1's copy overlaps step i) + "
                   + ("ffcu_shard_group_nll_points_device (launch + NCCL all-gather + combine)" if coll else
                      "ffcu_nll_points_device_upload (constant rows on the copy stream)")
                   + "; step i+1 queued before step i's results are read; D2H of the P results every step"}

    # --- the per-event-log variant: the grouped log (one table log per 8 events' product,
    # an algebraic rewrite) replaced by one log per event (NVRTC build with
    # -DFFB_LOG_PER_EVENT; build caches are keyed by the options)
    variants = {}
    if not args.no_variants:
        os.environ["FFB_JIT_OPTS"] = (os.environ.get("FFB_JIT_OPTS", "") + " -DFFB_LOG_PER_EVENT").strip()
        old = fb.plan_spec_min_work(0)
        try:
            v_ms, v_kms, _, _ = timed(max(3, args.steps // 2), 3)
        finally:
            fb.plan_spec_min_work(old)
            os.environ["FFB_JIT_OPTS"] = os.environ["FFB_JIT_OPTS"].replace("-DFFB_LOG_PER_EVENT", "").strip()
        variants["per_event_log"] = {
            "value": n_total * P * max(3, args.steps // 2) / (v_ms / 1e3), "unit": UNIT, "kernel_ms_avg": v_kms,
            "note": "one table log per event instead of one per product of 8 events (the headline's grouped "
                    "log is an algebraic rewrite of -sum log p)"}

    # --- roofline of the fused kernel: FP64 pipe (no contraction, and at
    # P >= 2 the event columns are read once per launch -- HBM is < 1 % busy)
    instr_alg = w.fp64_instr_per_event_point * n * P
    executed = profiled(w.name, "fp64_thread_instr_per_event_point")
    peak = peak_fma / 1e12
    ach_alg = instr_alg / (avg_kernel_ms / 1e3) / 1e12
    roofline = {
        "bound": "fp64", "unit": "T fp64-instr/s", "peak": peak,
        "peak_source": "measured live: DFMA-chain microbenchmark (ffcu_fp64_peak; MEASURED_PEAKS.json has no "
                       "FP64 figure; nominal 148 SMs x 64 lanes x 1.965 GHz = 18.6 T)",
        "kernel": f"nll_kernel<256,8> ({build}" + (f", {cached_terms} launch-constant cached term(s)" if cached_terms
                                                    else "") + ")",
        "kernel_ms_avg": avg_kernel_ms, "kernel_launches_timed": kcount,
        "kernel_share_of_step": avg_kernel_ms / (total_ms / args.steps),
        "hbm_algorithmic_bytes_per_launch": n * w.bytes_per_event,
        "hbm_achieved_gbs": n * w.bytes_per_event * info["nchunks"] / (avg_kernel_ms / 1e3) / 1e9,
        "hbm_peak_gbs": peaks().get("hbm_gbs"),
        "traffic": profiled(w.name, "dram_bytes_per_launch"),
        "ncu_fp64_pipe_active": profiled(w.name, "fp64_pipe_active"),
        "ncu_source": profiled(w.name, "source"),
        # the algorithmic work of SURVEY.md §8(d) (libdevice-weighted ops of the reference's
        # per-event formula) over the same time: > 1 where the kernel's own math is cheaper
        "algorithmic_work_per_event_point": w.fp64_instr_per_event_point,
        "algorithmic_achieved": ach_alg, "algorithmic_frac": ach_alg / peak,
    }
    if executed:
        ach = executed * n * P / (avg_kernel_ms / 1e3) / 1e12
        roofline.update({"achieved": ach, "frac": ach / peak, "executed_frac": ach / peak,
                         "executed_fp64_instr_per_event_point": executed,
                         "frac_note": "achieved = FP64-pipe thread instructions the kernel executes per event-point "
                                      "(ncu, profiles/ncu_summary.json) x event-points / kernel time; frac is the "
                                      "FP64 pipe's share of its measured peak"})
        # the SM's issue limit for this instruction mix: the DFMA rate of a
        # synthetic stream with the kernel's ratio of non-FP64 instructions (integer multiply-adds),
        # measured live at the two neighbouring ratios and interpolated
        total = profiled(w.name, "thread_instr_per_event_point")
        if total and total > executed:
            k8 = 8.0 * (total - executed) / executed
            grid = [0, 2, 4, 5, 6, 8, 16]
            lo = max(g for g in grid if g <= min(k8, 16))
            hi = min(g for g in grid if g >= min(k8, 16))
            r_lo = max(fb.fp64_issue_probe(lo) for _ in range(2)) / 1e12
            r_hi = r_lo if hi == lo else max(fb.fp64_issue_probe(hi) for _ in range(2)) / 1e12
            ceil = r_lo if hi == lo else r_lo + (r_hi - r_lo) * (min(k8, 16) - lo) / (hi - lo)
            roofline["issue_mix"] = {
                "other_instr_per_8_fp64": k8, "probe_dfma_rate": ceil, "unit": "T fp64-instr/s",
                "achieved_over_probe": ach / ceil,
                "note": "DFMA rate of dfma_mix_kernel (8 DFMA chains + K independent IMADs per round) at the "
                        "kernel's K: what the SM issues at this FP64 : other ratio with nothing else in the way"}
    else:
        roofline.update({"achieved": ach_alg, "frac": ach_alg / peak, "executed_frac": None,
                         "frac_note": "no executed-instruction count profiled for this workload: achieved is the "
                                      "algorithmic count (SURVEY.md §8(d))"})

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, reference Rng)",
        "config": config_for(w, n_total, world, P),
        "run": {"events_this_rank": n, "launch": info, "inputs": args.inputs or "generated in-process (seeded)",
                "inputs_s": load_s if load_s is not None else gen_s, "nccl": fb.ShardGroup.nccl_version() if coll else None},
        "roofline": roofline, "e2e": e2e, "variants": variants, "clocks": clk, "gpu_launches": int(launches),
        "result_finite": ok,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, cols, pts)
    if rank == 0:
        emit(line)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(w, cols, pts):
    """The reference engine itself (oracle/_ref) on the box's host cores, bounded samples."""
    from paper_2003_12875_b200 import configs
    if w.name not in configs.REF_ARMS:
        return None
    r = RefRunner(w, cols, pts)
    if not r.available():
        return {"value": None, "kind": "reference", "unavailable": "oracle/_ref not built"}
    mat = r.matrix(scalar=w.name == configs.C1.name)
    head = next(c for c in mat["cells"] if c["build"] == "release" and c["mode"] == "BatchPrecise"
                and c["threads"] == mat["nproc"])
    out = {"value": head["value"], "unit": UNIT, "cores": mat["nproc"], "kind": "reference",
           "sample": f"{head['points']} points (one per thread) x the first {head['events']} of this rank's events "
                     f"per call, median of 7; oracle/_ref = the unmodified reference engine, Release flags, "
                     f"BatchPrecise, {r.arm.note}",
           "matrix": mat}
    out["port"] = cpu_port(w, cols, pts, mat["nproc"] or 1)
    return out


def cpu_port(w, cols, pts, threads):
    """the restated oracle (oracle/ffit_oracle.c, the workload's NATIVE kinds --
    ArgusBG, Chebychev, ProdPdf, the extended term -- in one model, one point per thread) timed
    beside the reference engine's spelling: 1 thread and all threads, median of 5 on a bounded
    sample."""
    import numpy as np

    from oracle import oracle as orc
    o = orc.OracleModel(w.text)
    xs = [np.ascontiguousarray(cols[name]) for (name, _, _) in o.obs]
    n_full = len(xs[0])

    def call(nsub, npts, nthreads):
        sub = [x[:nsub] for x in xs]
        th = np.ascontiguousarray(pts[[i % len(pts) for i in range(npts)]])
        t0 = time.perf_counter()
        o.nll_points(sub, th, nthreads)
        return time.perf_counter() - t0

    cells = []
    for nthreads in sorted({1, threads}):
        probe = min(n_full, 100_000)
        per = max(call(probe, nthreads, nthreads), 1e-6) / probe
        nsub = int(min(n_full, max(probe, 0.12 / per)))
        med = sorted(call(nsub, nthreads, nthreads) for _ in range(5))[2]
        cells.append({"threads": nthreads, "value": nsub * nthreads / med, "unit": UNIT, "events": nsub,
                      "points": nthreads, "median_s": med})
    return {"kind": "port", "what": "oracle/ffit_oracle.c (C restatement, -O2, scalar per event; native kinds)",
            "cells": cells}


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation on the host cores

def run_reference(args, w):
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    if rank != 0:
        return
    import numpy as np

    from oracle import oracle as orc
    from paper_2003_12875_b200 import configs

    n_total = args.events or w.n_events
    o = orc.OracleModel(w.text)
    pts_all = _points_for_reference(w, o, args.points)
    # inputs: the same seeded columns the GPU arm reads (C restatement of the generator,
    # bit-identical to the library's); the timed code is the reference engine alone
    cols, _ = o.sample(n_total, w.data_seed)
    by = {name: c for (name, _, _), c in zip(o.obs, cols)}
    info = host_info()
    T = info["nproc"] or 1
    r = RefRunner(w, by, pts_all)
    if not r.available():
        emit({"impl": "reference", "unavailable": "oracle/_ref (the reference compiled from its sources) is missing"})
        return
    budget = max(0.2, 120.0 / (args.steps + args.warmup))  # seconds per step, whole run ~2 min
    nsub = r.sample_size(budget, T)
    P = len(pts_all)

    def step(i):
        sel = [(i * T + j) % P for j in range(T)]  # T distinct points, one per thread
        return r.call(nsub, pts_all[sel], T)[0]

    for i in range(args.warmup):
        step(i)
    times = [step(args.warmup + i) for i in range(args.steps)]
    total = sum(times)
    value = nsub * T * args.steps / total
    sample = (f"{T} of the {P} points per step (one per thread) x the first {nsub} of {n_total} events, "
              f"oracle/_ref (the unmodified reference engine, Release flags), BatchPrecise, {r.arm.note}")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, reference Rng)",
        "config": config_for(w, n_total, world, P),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": T, "kind": "reference", "sample": sample, **info},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    del np


def run_fit(args, w):
    """BASELINE configs[4]: the Minuit-style fit loop (BFGS on central differences, 2d+1
    points per launch, Hessian points in one launch), event-sharded over the ranks (one
    NCCL all-gather per launch, ffcu_shard_group_fit_gradient); value = event-points/s
    through the whole fit, plus NLL evaluations/s, fit wall time and the fitted parameters."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2003_12875_b200 as fb

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    n_total = args.events or w.n_events
    b, e = shard_bounds(n_total, world, rank)
    truth = fb.Model.from_string(w.text)
    t0 = time.perf_counter()
    cols, _ = generate_shard(fb, truth, w, n_total, b, e, args.inputs, rank)
    t_gen = time.perf_counter() - t0
    ds = fb.DataSet.from_columns(cols)
    model = fb.Model.from_string(w.text)
    start = w.points(model, n_points=1, seed=w.point_seed)[0]
    for name, v in zip(model.param_names, start):
        if not model.is_constant(name):
            model.set(name, v)

    def broadcast(obj):
        if world == 1:
            return obj
        box = [obj]
        dist.broadcast_object_list(box, src=0)
        return box[0]

    group = fb.ShardGroup.for_rank(model, ds, n_total, b, world, rank, broadcast)
    analytic = args.gradient == "analytic"
    free = [k for k, name in enumerate(model.param_names) if not model.is_constant(name)]
    # one untimed fit from the same start first: the run-time compiles (NVRTC) of every launch
    # shape the fit issues (the 2d+1-point steps, the batched Hessian, the one-point Newton
    # step) happen there, once per process; reported as first_call_s
    t0 = time.perf_counter()
    group.fit_gradient(tolerance=1e-12, max_iterations=args.iterations, analytic=analytic)
    jit_s = time.perf_counter() - t0
    for name, v in zip(model.param_names, start):
        if not model.is_constant(name):
            model.set(name, v)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    fb.kernel_timer(True)
    fb.kernel_timer_read()
    launches0 = fb.kernel_launches()
    r = group.fit_gradient(tolerance=1e-12, max_iterations=args.iterations, analytic=analytic)
    torch.cuda.synchronize()
    kms, kcount = fb.kernel_timer_read()
    launches = fb.kernel_launches() - launches0
    wall = torch.tensor([r.wall_seconds], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(wall, op=dist.ReduceOp.MAX)
    wall_s = float(wall.item())
    d = len(free)
    golden = _fit_golden(w.name, n_total)
    line = {
        "metric": METRIC, "value": r.n_nll_calls * n_total / wall_s, "unit": UNIT, "n_gpus": world,
        "steps": r.iterations, "warmup": 1, "ms_per_step": 1e3 * wall_s / max(r.n_launches, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, reference Rng)",
        "config": {**config_for(w, n_total, world, 1 if r.analytic_gradient else 2 * d + 1),
                   "gradient": "analytic (fused NLL + gradient pass, one point per launch)" if r.analytic_gradient
                   else "central differences (2d+1 points per launch)", "free_parameters": d},
        "fit": {"converged": r.converged, "iterations": r.iterations, "launches": r.n_launches,
                "nll_evaluations": r.n_nll_calls, "nll_evaluations_per_s": r.n_nll_calls / wall_s,
                "wall_seconds": wall_s, "kernel_ms_total_rank0": kms, "kernel_launches_timed_rank0": kcount,
                "nll_min": r.nll_min, "analytic_gradient": r.analytic_gradient, "first_call_s": jit_s,
                "first_call": "an untimed fit from the same start before the timed one: the one-time NVRTC "
                              "builds of every launch shape the fit uses",
                "parameters": {p.name: [p.value, p.uncertainty] for p in r.parameters},
                "truth": dict(zip(truth.param_names, [float(v) for v in truth.theta()])),
                "data_generation_s": t_gen},
        "gpu_launches": int(launches),
    }
    if golden:
        diffs = {p.name: abs(p.value - golden["parameters"][p.name]) for p in r.parameters
                 if p.name in golden["parameters"]}
        line["fit"]["vs_cpu_fit"] = {"max_abs_param_diff": max(diffs.values()) if diffs else None,
                                     "per_param": diffs, "golden": "tests/golden/c5_cpu_fit.json",
                                     "cpu_nll_min": golden.get("nll_min")}
    if rank == 0:
        emit(line)
    if world > 1:
        dist.destroy_process_group()


def _fit_golden(name, n_total):
    try:
        with open(os.path.join(ROOT, "tests", "golden", "c5_cpu_fit.json")) as fh:
            g = json.load(fh)
        return g if g.get("workload") == name and g.get("n_events") == n_total else None
    except (OSError, ValueError):
        return None


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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", help="c1..c5 or a configs.WORKLOADS name")
    ap.add_argument("--events", type=int, default=0, help="override the config's total events")
    ap.add_argument("--points", type=int, default=None, help="override points per launch")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the per-event-log variant line")
    ap.add_argument("--fit", action="store_true", help="time the Minuit-style fit loop (config 5 style)")
    ap.add_argument("--force-collective", action="store_true",
                    help="run the sharded path (NCCL all-gather + combine) even at N = 1")
    ap.add_argument("--iterations", type=int, default=50, help="fit iterations (--fit / c5)")
    ap.add_argument("--inputs", default="", help="directory of tools/make_inputs.py files (.ffsoa + manifest)")
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
