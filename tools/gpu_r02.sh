# round-2 GPU validation: TAG=... bash tools/gpu_r02.sh [tests...]
TAG=${TAG:-r02}
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$TAG/smi.txt
if [ -n "$TESTS" ]; then
  timeout 1200 python -m pytest $TESTS -q -x > gpurun_out/$TAG/pytest_sel.log 2>&1; echo "rc $?" >> gpurun_out/$TAG/pytest_sel.log
fi
if [ -n "$FULL" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/$TAG/pytest_gpu.log
fi
for w in $BENCH; do timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 20 > gpurun_out/$TAG/bench_$w.json 2> gpurun_out/$TAG/bench_$w.err; done
tail -2 gpurun_out/$TAG/*.log
for w in $BENCH; do python -c "import json;d=json.load(open('gpurun_out/$TAG/bench_$w.json'));print('$w', '%.4e'%d['value'], d['roofline']['kernel_ms_avg'])"; done
