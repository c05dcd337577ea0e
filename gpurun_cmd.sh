for w in c1 c2 c4; do for wv in 8 2 4 16; do
  FFB_NLL_WAVES=$wv python bench.py --workload $w --no-cpu-baseline --steps 20 > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$w waves=$wv', '%.4e'%d['value'], d['config']['launch']['grid'])"
done; done
