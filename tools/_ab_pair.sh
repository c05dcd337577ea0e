set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "argus or c2 or cache or golden or hybrid or random" > gpurun_out/r02_pair_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r02_pair_pytest.log
TAG=r02_pair WS="c2" REPS=3 STEPS=20 VARIANTS="pair: nopair:-DFFB_NO_ARGUS_PAIR" bash tools/ab_jit.sh
timeout 600 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/r02_pair/bench_c5_fd.json 2> gpurun_out/r02_pair/bench_c5_fd.err
tail -n 3 gpurun_out/r02_pair_pytest.log
