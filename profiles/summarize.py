"""Summarise ncu outputs brought back in gpurun_out/ into committed text under profiles/.

    python profiles/summarize.py launches gpurun_out/launches.csv  > profiles/rNN_launches_<tag>.txt
    python profiles/summarize.py full gpurun_out/prof.ncu-rep [kernel-regex] > profiles/rNN_ncu_<tag>.txt
"""
import collections
import csv
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.per_cycle_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[r[ki][:90]][0] += 1
        agg[r[ki][:90]][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none ({path})")
    print(f"# {'launches':>8} {'total ms':>10} {'share':>7}  kernel")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {c:8d} {v / 1e6:10.3f} {100 * v / tot:6.2f}%  {k}  (avg {v / c / 1e3:.1f} us)")


def full(path, kernel=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, zip(units, vals)))
        name = d.get("Kernel Name", ("", ""))[1]
        if kernel and not re.search(kernel, name):
            continue
        print(f"# ncu --set full ({path}) kernel: {name}")
        for k in KEYS:
            if k in d:
                print(f"{k:70s} {d[k][1]:>20s} {d[k][0]}")
        stalls = {k: float(v[1]) for k, v in d.items()
                  if re.fullmatch(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+", k) and not k.endswith("not_issued")
                  and v[1] not in ("", "n/a")}
        tot = sum(stalls.values()) or 1.0
        print("# warp-state samples (share)")
        for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:10]:
            print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * v / tot:6.2f}%")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
