python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in c2 c1 c4 c3; do
  python bench.py --workload $w --no-cpu-baseline --steps 20 > gpurun_out/sweep_${w}_v0.json 2>> gpurun_out/bench_err.log
done
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --points 50 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 3 -c 1 -o gpurun_out/prof_c2_v8 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --points 50 > gpurun_out/ncu_full.log 2>&1
echo done
