python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for rep in 1 2; do
for tag in base gv1; do
  if [ $tag = base ]; then unset FFB_LIB_VARIANT; else export FFB_LIB_VARIANT=$tag; fi
  python bench.py --workload c3 --no-cpu-baseline --steps 20 > gpurun_out/ab.json 2>> gpurun_out/ab_err.log
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('c3 $tag', '%.4e'%d['value'])"
done
done
