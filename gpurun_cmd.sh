python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in c2 c1 c4 c3; do
for v in 0 1; do
  FFB_NLL_VARIANT=$v python bench.py --workload $w --no-cpu-baseline --steps 20 > gpurun_out/sweep_${w}_v$v.json 2>> gpurun_out/bench_err.log
done
done
echo done
