python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
mkdir -p gpurun_out/v10
for w in c2 c1 c3 c4; do
  python bench.py --workload $w --steps 20 > gpurun_out/v10/bench_$w.json 2>> gpurun_out/v10/err.log
done
python bench.py --workload c5 --gradient fd > gpurun_out/v10/bench_c5_fd.json 2>> gpurun_out/v10/err.log
python bench.py --workload c5 --gradient analytic > gpurun_out/v10/bench_c5_analytic.json 2>> gpurun_out/v10/err.log
python tools/small_p_bench.py > gpurun_out/v10/small_p.txt 2>&1
python tools/grad_bench.py > gpurun_out/v10/grad_bench.txt 2>&1
python bench.py > gpurun_out/v10/bench_default.json 2>> gpurun_out/v10/err.log
cat gpurun_out/pytest_gpu.log
