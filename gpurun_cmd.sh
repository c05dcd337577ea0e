set -x
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo "bench rc=$?"
python bench.py --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2>>gpurun_out/bench_c2.err
python bench.py --workload c3 --no-cpu-baseline --steps 10 > gpurun_out/bench_c3.json 2>>gpurun_out/bench_c2.err
python bench.py --workload c4 --no-cpu-baseline --steps 10 > gpurun_out/bench_c4.json 2>>gpurun_out/bench_c2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>>gpurun_out/bench_c2.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --points 50 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --points 50 > gpurun_out/ncu_full.log 2>&1
echo done
