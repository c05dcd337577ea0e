# the bench's other modes on one GPU: TAG=.. bash tools/bench_modes.sh
TAG=${TAG:-r02m}; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python bench.py --force-collective --no-cpu-baseline --no-variants --steps 10 > $O/bench_forcecoll.json 2> $O/bench_forcecoll.err; echo "rc $?" >> $O/bench_forcecoll.err
timeout 900 python bench.py --workload c5 > $O/bench_c5_fd.json 2> $O/bench_c5_fd.err; echo "rc $?" >> $O/bench_c5_fd.err
timeout 900 python bench.py --workload c5 --gradient analytic > $O/bench_c5_an.json 2> $O/bench_c5_an.err; echo "rc $?" >> $O/bench_c5_an.err
for w in c1 c2 c3; do
  timeout 900 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; echo "rc $?" >> $O/bench_$w.err
  timeout 900 python bench.py --workload $w --impl reference --steps 5 --warmup 1 > $O/ref_$w.json 2> $O/ref_$w.err; echo "rc $?" >> $O/ref_$w.err
done
tail -n 2 $O/*.err
