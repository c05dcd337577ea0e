for rep in 1 2; do for tag in base spec; do
  if [ $tag = base ]; then unset FFB_LIB_VARIANT; else export FFB_LIB_VARIANT=$tag; fi
  python bench.py --workload c2 --no-cpu-baseline --steps 20 > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('c2 $tag', '%.4e'%d['value'])"
done; done
