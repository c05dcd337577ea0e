# round-2 bench validation: TAG=... bash tools/bench_r02.sh
TAG=${TAG:-r02b}
O=gpurun_out/$TAG
mkdir -p $O
lscpu > $O/lscpu.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 900 python bench.py ${BENCH_ARGS} > $O/bench_default.json 2> $O/bench_default.err; echo "rc $?" >> $O/bench_default.err
timeout 900 python bench.py --impl reference ${BENCH_ARGS} > $O/bench_reference.json 2> $O/bench_reference.err; echo "rc $?" >> $O/bench_reference.err
for w in $EXTRA; do timeout 900 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
if [ -n "$PROFILE" ]; then
  for w in $PROFILE; do
    C="python bench.py --workload $w --no-cpu-baseline --no-variants --steps 1 --warmup 3"
    $C > $O/plain_$w.log 2>&1 &&
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 1 -c 1 -o $O/prof_$w $C > $O/ncu_$w.log 2>&1
    python profiles/summarize.py full $O/prof_$w.ncu-rep > $O/ncu_$w.txt 2>&1
    ncu -i $O/prof_$w.ncu-rep --page source --csv 2>/dev/null | gzip > $O/src_$w.csv.gz
    [ "$w" = "${KEEP_REP:-none}" ] || rm -f $O/prof_$w.ncu-rep
  done
  C="python bench.py --no-cpu-baseline --no-variants --steps 2 --warmup 3"
  $C > $O/plain_launch.log 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $C > $O/ncu_launch.log 2>&1
  python profiles/summarize.py launches $O/launches.csv > $O/launches.txt 2>&1
fi
tail -3 $O/*.err
python - <<PY
import json
for f in ["bench_default", "bench_reference"]:
    try:
        d = json.load(open("$O/" + f + ".json"))
        print(f, "%.4e" % d["value"], "e2e %.4e" % d["e2e"]["value"], d.get("roofline", {}).get("frac"), d.get("variants"))
    except Exception as e:
        print(f, "ERR", e)
PY
