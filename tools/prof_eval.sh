# ncu --set full of eval_fast_kernel (probabilities of the C1 Gaussian over 1e8 events): the
# HBM-bound kernel of the path.  TAG=.. bash tools/prof_eval.sh
TAG=${TAG:-r02_eval}; O=gpurun_out/$TAG; mkdir -p $O
python tools/eval_bench.py > $O/plain_eval.json 2>$O/plain_eval.err &&
ncu --set full --clock-control none --import-source on -k regex:eval_fast_kernel -s 2 -c 1 -o $O/prof_eval python tools/eval_bench.py > $O/ncu_eval.log 2>&1
ncu -i $O/prof_eval.ncu-rep --page raw --csv 2>/dev/null > $O/raw_eval.csv
python - <<PY
import csv
rows = list(csv.reader(open("$O/raw_eval.csv")))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, zip(units, vals)))
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]
with open("$O/ncu_eval.txt", "w") as fh:
    fh.write("# ncu --set full of eval_fast_kernel (tools/prof_eval.sh: probabilities of a Gaussian over 1e8 events)\n")
    for k in keys:
        if k in d:
            fh.write(f"{k:70s} {d[k][1]:>24s} {d[k][0]}\n")
print(open("$O/ncu_eval.txt").read())
PY
rm -f $O/prof_eval.ncu-rep $O/raw_eval.csv
