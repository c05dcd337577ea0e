# A/B of two library builds on one workload: TAG=.. W=c4 B="onecopy:-DFFB_EXP_LANES=1" bash tools/ab_r02.sh
TAG=${TAG:-r02ab}; W=${W:-c4}
O=gpurun_out/$TAG; mkdir -p $O
tag=${B%%:*}; opts=${B#*:}
for rep in 1 2 3; do
  for v in base $tag; do
    if [ $v = base ]; then
      python bench.py --workload $W --no-cpu-baseline --no-variants --steps 10 > $O/ab_${v}_$rep.json 2>/dev/null
    else
      FFB_LIB_VARIANT=$tag FFB_JIT_OPTS="$opts" python bench.py --workload $W --no-cpu-baseline --no-variants --steps 10 > $O/ab_${v}_$rep.json 2>/dev/null
    fi
    python -c "import json;d=json.load(open('$O/ab_${v}_$rep.json'));print('$W $v $rep', '%.4e'%d['value'], '%.3f'%d['roofline']['kernel_ms_avg'])" | tee -a $O/ab.txt
  done
done
