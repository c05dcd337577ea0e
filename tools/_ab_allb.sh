set -x
TAG=r02_allb WS="c4 c1 c3" REPS=2 STEPS=20 VARIANTS="allb: noallb:-DFFB_NO_ALL_BOUNDED" bash tools/ab_jit.sh
timeout 900 python -m pytest tests -m gpu -q -x -k "edge or parity or golden or underflow or chunk or random" > gpurun_out/r02_allb/pytest.log 2>&1; echo "rc $?" >> gpurun_out/r02_allb/pytest.log
tail -n 3 gpurun_out/r02_allb/pytest.log
