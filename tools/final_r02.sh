# Final validation of the round: GPU suite, smoke, every bench line, the reference arm, the
# C5 fits, the one-rank collective path, ncu (launch list + --set full per workload), and the
# side benches.  TAG=r02_v12 bash tools/final_r02.sh
set -x
TAG=${TAG:-r02_v12}; O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
lscpu > $O/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
FFB_RANDOM_SEEDS=16:120 timeout 1500 python -m pytest tests/test_gpu_random_models.py -m gpu -q > $O/pytest_random_sweep.log 2>&1; echo "pytest rc $?" >> $O/pytest_random_sweep.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for w in c1 c2 c3; do timeout 900 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 900 python bench.py --workload c5 > $O/bench_c5_fd.json 2> $O/bench_c5_fd.err
timeout 900 python bench.py --workload c5 --gradient analytic > $O/bench_c5_an.json 2> $O/bench_c5_an.err
timeout 900 python bench.py --force-collective --no-cpu-baseline > $O/bench_forcecoll.json 2> $O/bench_forcecoll.err
python tools/eval_bench.py > $O/eval_bench.json 2> $O/eval_bench.err
python tools/device_norm_bench.py > $O/device_norm_bench.json 2> $O/device_norm_bench.err
python tools/issue_probe.py > $O/issue_probe.json 2> $O/issue_probe.err
CMD="python bench.py --no-cpu-baseline --steps 2 --warmup 3"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv $CMD > $O/ncu_launch.log 2>&1
python profiles/summarize.py launches $O/launches_c4.csv > $O/launches_c4.txt 2>&1
for w in c4 c1 c2 c3; do
  C="python bench.py --workload $w --no-cpu-baseline --no-variants --steps 1 --warmup 3"
  $C > $O/plain_$w.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 1 -c 1 -o $O/prof_$w $C > $O/ncu_$w.log 2>&1
  python profiles/summarize.py full $O/prof_$w.ncu-rep > $O/ncu_$w.txt 2>&1
  ncu -i $O/prof_$w.ncu-rep --page source --csv 2>/dev/null | gzip > $O/src_$w.csv.gz
  rm -f $O/prof_$w.ncu-rep
done
tail -n 3 $O/pytest_gpu.log; tail -n 3 $O/smoke.log
