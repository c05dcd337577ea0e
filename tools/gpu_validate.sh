set -x
TAG=${TAG:-v12}
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$TAG/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/$TAG/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/$TAG/smoke.log
timeout 600 python bench.py > gpurun_out/$TAG/bench_default.json 2> gpurun_out/$TAG/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/$TAG/bench_reference.json 2> gpurun_out/$TAG/bench_reference.err
for w in c1 c3 c4 c5; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/$TAG/bench_$w.json 2> gpurun_out/$TAG/bench_$w.err; done
tail -3 gpurun_out/$TAG/pytest_gpu.log
