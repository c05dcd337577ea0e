# a sequence of round-2 jobs in one gpurun call: JOBS="ab prof" TAG=... bash tools/gpu_job.sh
for j in $JOBS; do
  case $j in
    ab) TAG=$TAG W=${AB_W:-c4} B="$AB_B" bash tools/ab_r02.sh ;;
    prof) TAG=$TAG PROFILE="${PROF_W:-c4}" KEEP_REP=${KEEP_REP:-none} BENCH_ARGS="--no-cpu-baseline" bash tools/bench_r02.sh ;;
    tests) mkdir -p gpurun_out/$TAG; timeout 1800 python -m pytest ${TESTS:-tests} -m gpu -q -x > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/$TAG/pytest_gpu.log; tail -3 gpurun_out/$TAG/pytest_gpu.log ;;
  esac
done
