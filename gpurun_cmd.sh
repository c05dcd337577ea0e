python bench.py --workload c2 --spelling reference --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/pre.json 2>gpurun_out/pre.err && \
ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 5 -c 1 -o gpurun_out/prof_jit2 python bench.py --workload c2 --spelling reference --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/ncu_full.log 2>&1
echo rc=$?
