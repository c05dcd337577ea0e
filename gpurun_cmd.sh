python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in c2 c1 c4 c3; do
for v in 0 1 2 3; do
  FFB_NLL_VARIANT=$v python bench.py --workload $w --no-cpu-baseline --steps 5 > gpurun_out/sweep_${w}_v$v.json 2>> gpurun_out/sweep_err.log
done
done
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --points 50 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 3 -c 1 -o gpurun_out/prof_c2_v4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --points 50 > gpurun_out/ncu_full.log 2>&1
echo done
