# GPU suite, then every workload's bench line (regression / A-B check)
TAG=${TAG:-vX}
mkdir -p gpurun_out/$TAG
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/$TAG/pytest_gpu.log
tail -4 gpurun_out/$TAG/pytest_gpu.log
TAG=$TAG bash tools/bench_all.sh
