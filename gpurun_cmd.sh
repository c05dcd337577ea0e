python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for w in c3 c2; do
  python bench.py --workload $w --no-cpu-baseline --steps 20 > gpurun_out/ab.json 2>> gpurun_out/ab_err.log
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$w', '%.4e'%d['value'])"
done
