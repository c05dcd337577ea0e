"""Fold one profiling run (tools/bench_r02.sh PROFILE=...) into profiles/ncu_summary.json, which
bench.py reads for the roofline's executed-instruction count and DRAM traffic.

    python profiles/update_summary.py <tag-dir under profiles/> c4 [c1 c2 c3]

For each workload: ncu_<w>.txt (profiles/summarize.py full) gives the fused kernel's DRAM bytes
per launch and its FP64-pipe share; src_<w>.csv.gz (the source page) gives the executed op mix
(profiles/opmix.py): DFMA + DMUL + DADD + DSETP thread instructions per event-point.
"""
import csv
import gzip
import json
import os
import re
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from paper_2003_12875_b200 import configs  # noqa: E402

FP64_OPS = ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX")


def opmix(path, evpt):
    rows = list(csv.reader(gzip.open(path, "rt")))
    hdr = rows[1]
    ia, ie = hdr.index("Source"), hdr.index("Instructions Executed")
    mix = {}
    for r in rows[2:]:
        if len(r) <= ie:
            continue
        try:
            n = int(r[ie])
        except ValueError:
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", r[ia].strip())
        base = (m.group(2) if m else r[ia].strip()).split(".")[0]
        mix[base] = mix.get(base, 0) + n
    return {k: v * 32.0 / evpt for k, v in mix.items()}


def main():
    tag, names = sys.argv[1], sys.argv[2:]
    d = os.path.join(HERE, tag)
    path = os.path.join(HERE, "ncu_summary.json")
    summary = json.load(open(path))
    for short in names:
        w = configs.BY_INDEX[int(short.lstrip("c")) - 1]
        evpt = w.n_events * w.n_points
        txt = open(os.path.join(d, f"ncu_{short}.txt")).read()
        rd = float(re.search(r"dram__bytes_read.sum\s+([\d.]+) (\w+)", txt).group(1))
        unit_r = re.search(r"dram__bytes_read.sum\s+[\d.]+ (\w+)", txt).group(1)
        wr = re.search(r"dram__bytes_write.sum\s+([\d.]+) (\w+)", txt)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        dram = rd * scale[unit_r] + (float(wr.group(1)) * scale[wr.group(2)] if wr else 0.0)
        pipe = float(re.search(r"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active\s+([\d.]+)", txt).group(1))
        kernel = re.search(r"kernel: (.*)", txt).group(1)[:90]
        mix = opmix(os.path.join(d, f"src_{short}.csv.gz"), evpt)
        fp64 = sum(mix.get(k, 0.0) for k in FP64_OPS)
        with open(os.path.join(d, f"opmix_{short}.txt"), "w") as fh:
            fh.write(f"total instr per ev*pt: {sum(mix.values()):.2f}\n")
            for k, v in sorted(mix.items(), key=lambda x: -x[1])[:40]:
                fh.write(f"{k:10s} {v:6.2f}\n")
        summary[w.name] = {
            "dram_bytes_per_launch": int(dram),
            "fp64_pipe_active": round(pipe / 100.0, 4),
            "fp64_thread_instr_per_event_point": round(fp64, 2),
            "thread_instr_per_event_point": round(sum(mix.values()), 2),
            "fp64_thread_instr_source": f"profiles/{tag}/opmix_{short}.txt ("
                                        + " + ".join(f"{k} {mix.get(k, 0.0):.2f}" for k in FP64_OPS if mix.get(k))
                                        + " thread instructions per event-point)",
            "source": f"profiles/{tag}/ncu_{short}.txt ({kernel}, bench.py --workload {short}: "
                      f"dram__bytes_read.sum + dram__bytes_write.sum per launch, "
                      f"sm__pipe_fp64_cycles_active {pipe:.1f} %)",
        }
        print(short, summary[w.name])
    json.dump(summary, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
