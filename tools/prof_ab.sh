# ncu --set full of the fused kernel under env variants: TAG=.. WS="c4" VARS="base: nopre:FFB_JIT_OPTS=-DFFB_EXP_NO_PRESCALE" bash tools/prof_ab.sh
TAG=${TAG:-r02_prof}; O=gpurun_out/$TAG; mkdir -p $O
for w in ${WS:-c4}; do
  for v in $VARS; do
    name=${v%%:*}; envs=$(echo ${v#*:} | tr '+' ' ')
    C="python bench.py --workload $w --no-cpu-baseline --no-variants --steps 1 --warmup 3"
    env $envs FFB_PLAN_SPEC_MIN=0 $C > $O/plain_${w}_$name.log 2>&1 &&
    env $envs FFB_PLAN_SPEC_MIN=0 ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 1 -c 1 -o $O/prof_${w}_$name $C > $O/ncu_${w}_$name.log 2>&1
    python profiles/summarize.py full $O/prof_${w}_$name.ncu-rep > $O/ncu_${w}_$name.txt 2>&1
    ncu -i $O/prof_${w}_$name.ncu-rep --page source --csv 2>/dev/null | gzip > $O/src_${w}_$name.csv.gz
    ncu -i $O/prof_${w}_$name.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/raw_${w}_$name.csv.gz
    rm -f $O/prof_${w}_$name.ncu-rep
  done
done
ls -la $O
