set -x
TAG=${TAG:-r02_pre1}; O=gpurun_out/$TAG; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
tail -4 $O/pytest_gpu.log
TAG=$TAG REPS=2 WS="c4 c1 c2 c3" VARIANTS="${VARIANTS:-base: nopre:-DFFB_EXP_NO_PRESCALE addr2:-DFFB_EXP_ADDR2}" bash tools/ab_jit.sh
sort $O/ab.txt
