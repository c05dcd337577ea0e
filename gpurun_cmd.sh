for w in c2 c1 c4 c3; do
for tag in base cbank base cbank; do
  if [ $tag = base ]; then unset FFB_LIB_VARIANT; else export FFB_LIB_VARIANT=$tag; fi
  python bench.py --workload $w --no-cpu-baseline --steps 20 > gpurun_out/ab_${w}_${tag}_$RANDOM.json 2>> gpurun_out/ab_err.log
done
unset FFB_LIB_VARIANT
done
echo done
