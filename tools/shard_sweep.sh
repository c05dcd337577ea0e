# What ONE rank does at N = 1, 2, 4, 8 of BASELINE config 4's strong-scaled split: its shard of
# 1e8 / N events through the library's sharded step (launch + NCCL all-gather at world 1 + the
# combine kernel).  A projection input for DESIGN.md "Multi-GPU", not a multi-GPU measurement.
TAG=${TAG:-r02_sweep}; O=gpurun_out/$TAG; mkdir -p $O
for N in 1 2 4 8; do
  python bench.py --events $((100000000 / N)) --force-collective --no-cpu-baseline --no-variants > $O/shard_1of$N.json 2> $O/shard_1of$N.err
  python -c "
import json;d=json.load(open('$O/shard_1of$N.json'))
print('N=$N events/rank', d['config']['events_per_gpu'], 'step ms %.4f' % d['ms_per_step'], 'kernel ms %.4f' % d['roofline']['kernel_ms_avg'], 'rate %.4e' % d['value'], 'e2e %.4e' % d['e2e']['value'])" | tee -a $O/sweep.txt
done
