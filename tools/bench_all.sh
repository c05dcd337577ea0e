# every workload's bench line (no CPU baseline): quick regression check
TAG=${TAG:-v14}
mkdir -p gpurun_out/$TAG
for w in c1 c2 c3 c4; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 20 > gpurun_out/$TAG/$w.json 2>gpurun_out/$TAG/$w.err
  python -c "import json;d=json.load(open('gpurun_out/$TAG/$w.json'));print('$w', '%.4e'%d['value'], d['roofline']['frac'])"
done
FFB_NO_CONST_CACHE=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/$TAG/c2_nocache.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/$TAG/c2_nocache.json'));print('c2 nocache', '%.4e'%d['value'])"
