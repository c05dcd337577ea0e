# compute-sanitizer over tools/sanitize_smoke.py (every kernel family at small sizes):
# memcheck, racecheck, synccheck, initcheck.  TAG=r02_san bash tools/sanitize.sh
# (This round's GPU pool refuses compute-sanitizer -- "closed on this pool", rc 86 -- so only the
# plain run of the smoke set is recorded, gpurun_out/r02_san/plain.log; the script is for a pool that allows it.)
# The NCCL leg is left out under racecheck / initcheck (NCCL's own kernels are not ours to check
# and slow the tools down); memcheck and synccheck run it.
set -x
TAG=${TAG:-r02_san}; O=gpurun_out/$TAG; mkdir -p $O
python tools/sanitize_smoke.py > $O/plain.log 2>&1 || { echo "plain run failed"; tail -20 $O/plain.log; exit 1; }
for t in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 20 python tools/sanitize_smoke.py > $O/$t.log 2>&1
  echo "$t rc $?" >> $O/$t.log
done
for t in racecheck initcheck; do
  SANITIZE_NCCL=0 timeout 1800 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 20 python tools/sanitize_smoke.py > $O/$t.log 2>&1
  echo "$t rc $?" >> $O/$t.log
done
grep -H "ERROR SUMMARY\|rc \|sanitize smoke done" $O/*.log
