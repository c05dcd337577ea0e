# C5 fit (FD and analytic gradients), few-point launches, and the default bench line
TAG=${TAG:-vX}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python bench.py --workload c5 --no-cpu-baseline > $O/c5_fd.json 2> $O/c5_fd.err
timeout 600 python bench.py --workload c5 --gradient analytic --no-cpu-baseline > $O/c5_analytic.json 2> $O/c5_analytic.err
timeout 600 python tools/small_p_bench.py > $O/small_p.txt 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for f in $O/c5_fd.json $O/c5_analytic.json; do python -c "import json;d=json.load(open('$f'));print('$f', '%.3e'%d['value'], d['fit']['iterations'], d['fit']['wall_seconds'], d['fit']['converged'])"; done
cat $O/small_p.txt
python -c "import json;d=json.load(open('$O/bench_default.json'));print('default', '%.3e'%d['value'], d['e2e']['value'], d['cpu_baseline'])"
