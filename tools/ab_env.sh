# A/B of one environment setting on the bench workloads: AB_ENV="FFB_JIT_OPTS=-DFFB_CONST_BANK" bash tools/ab_env.sh
TAG=${TAG:-ab}
O=gpurun_out/$TAG
mkdir -p $O
for rep in 1 2; do
  for w in ${WORKLOADS:-c1 c2 c3 c4}; do
    timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 20 > $O/${w}_A_$rep.json 2>/dev/null
    env $AB_ENV timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 20 > $O/${w}_B_$rep.json 2>/dev/null
    python -c "import json;a=json.load(open('$O/${w}_A_$rep.json'))['value'];b=json.load(open('$O/${w}_B_$rep.json'))['value'];print('$w rep$rep A %.4e B %.4e B/A %.3f'%(a,b,b/a))"
  done
done
