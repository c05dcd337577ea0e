set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for w in c2 c1 c4 c3; do
  python bench.py --workload $w --no-cpu-baseline --steps 20 > gpurun_out/b_${w}.json 2>> gpurun_out/b_err.log
  python -c "import json;d=json.load(open('gpurun_out/b_${w}.json'));print('$w', '%.4e'%d['value'], d['roofline']['frac'], d['e2e']['value'])"
done
python tools/small_p_bench.py
