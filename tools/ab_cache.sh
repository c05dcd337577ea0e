# A/B of the launch-constant branch cache on the headline workload (and the GPU suite)
TAG=${TAG:-v13}
mkdir -p gpurun_out/$TAG
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/$TAG/pytest_gpu.log
for rep in 1 2; do
  FFB_NO_CONST_CACHE=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/$TAG/c2_nocache_$rep.json 2>/dev/null
  timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/$TAG/c2_cache_$rep.json 2>/dev/null
done
for f in gpurun_out/$TAG/c2_*.json; do python -c "import json;d=json.load(open('$f'));print('$f', '%.4e'%d['value'], d['roofline']['frac'])"; done
tail -3 gpurun_out/$TAG/pytest_gpu.log
