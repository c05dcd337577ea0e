# grid waves A/B (FFB_NLL_WAVES) on the bench workloads
O=gpurun_out/${TAG:-waves}
mkdir -p $O
for w in ${WORKLOADS:-c1 c2}; do
  for v in 2 3 4 6 8 12; do
    FFB_NLL_WAVES=$v timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 20 > $O/${w}_$v.json 2>/dev/null
    python -c "import json;d=json.load(open('$O/${w}_$v.json'));print('$w waves=$v %.4e'%d['value'], d['config']['launch'])"
  done
done
