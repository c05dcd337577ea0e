# A/B of NVRTC build options (plan-specialised builds, FFB_JIT_OPTS) and env knobs on several
# workloads:  TAG=.. WS="c4 c1" VARIANTS="base: tree:-DFFB_LOG_TREE waves8:env=FFB_NLL_WAVES=8" bash tools/ab_jit.sh
# (a variant's tokens are '+'-separated: -D... go to FFB_JIT_OPTS, env=K=V is exported,
#  lib=<tag> loads lib/ab/libffit_b200_<tag>.so)
TAG=${TAG:-r02jit}; O=gpurun_out/$TAG; mkdir -p $O
for rep in $(seq 1 ${REPS:-2}); do
  for w in ${WS:-c4}; do
    for v in $VARIANTS; do
      name=${v%%:*}; toks=$(echo ${v#*:} | tr '+' ' ')
      opts=""; lib=""; envs=""
      for t in $toks; do
        case $t in lib=*) lib=${t#lib=};; env=*) envs="$envs ${t#env=}";; *) opts="$opts $t";; esac
      done
      env $envs FFB_LIB_VARIANT=$lib FFB_JIT_OPTS="$opts" FFB_PLAN_SPEC_MIN=0 python bench.py --workload $w --no-cpu-baseline --no-variants --steps ${STEPS:-10} > $O/${w}_${name}_$rep.json 2>$O/${w}_${name}_$rep.err
      python -c "import json;d=json.load(open('$O/${w}_${name}_$rep.json'));print('$w $name $rep', '%.4e'%d['value'], '%.4f'%d['roofline']['kernel_ms_avg'], d['run']['launch'])" | tee -a $O/ab.txt
    done
  done
done
