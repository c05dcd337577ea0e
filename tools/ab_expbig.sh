# A/B of the 3211-entry exp table builds (FFB_EXP_BIG=1) against the default on C4/C1/C2/C3, then the
# parity suites on the BIG builds
set -x
TAG=${TAG:-r02_big1}; O=gpurun_out/$TAG; mkdir -p $O
TAG=$TAG REPS=2 WS="c4 c1 c2 c3" VARIANTS="base: big:env=FFB_EXP_BIG=1" bash tools/ab_jit.sh
FFB_EXP_BIG=1 FFB_PLAN_SPEC_MIN=0 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exp_edges.py tests/test_gpu_random_models.py -m gpu -q -x > $O/pytest_big.log 2>&1; echo "rc $?" >> $O/pytest_big.log
tail -5 $O/pytest_big.log
cat $O/ab.txt
