# Quick validation of the tree in one GPU call: GPU suite, smoke, default bench, reference arm.
# TAG=r02_v16 bash tools/quick_check.sh
set -x
TAG=${TAG:-r02_quick}; O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for w in c1 c2 c3; do timeout 900 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
tail -n 3 $O/pytest_gpu.log; tail -n 3 $O/smoke.log
