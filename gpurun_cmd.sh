python bench.py --workload c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo "c5 rc=$?"
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "default rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo done
