# ncu evidence for the bench workloads: the launch list of the default bench and one
# --set full capture of the fused NLL kernel per workload (each after a plain run of the
# same command line has exited 0).  Usage: TAG=v16 WORKLOADS="c2 c1" bash tools/profile.sh
TAG=${TAG:-v16}
WORKLOADS=${WORKLOADS:-c2}
O=gpurun_out/$TAG
mkdir -p $O
if [ -n "$RUN_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
fi
CMD="python bench.py --no-cpu-baseline --steps 2 --warmup 3"
$CMD > $O/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv $CMD > $O/ncu_launch.log 2>&1
for w in $WORKLOADS; do
  C="python bench.py --workload $w --no-cpu-baseline --steps 1 --warmup 3"
  $C > $O/plain_$w.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 1 -c 1 -o $O/prof_$w $C > $O/ncu_$w.log 2>&1
  # summaries on the box (gpurun brings back <= 64 MiB): raw metrics, the source page
  python profiles/summarize.py full $O/prof_$w.ncu-rep > $O/ncu_$w.txt 2>&1
  ncu -i $O/prof_$w.ncu-rep --page source --csv 2>/dev/null | gzip > $O/src_$w.csv.gz
  [ "$w" = "${KEEP_REP:-c2}" ] || rm -f $O/prof_$w.ncu-rep
done
python profiles/summarize.py launches $O/launches_c2.csv > $O/launches_c2.txt 2>&1
ls -la $O
