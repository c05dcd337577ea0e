for tag in base wt gb3 both; do
  if [ $tag = base ]; then unset FFB_LIB_VARIANT; else export FFB_LIB_VARIANT=$tag; fi
  echo "== $tag"; python tools/grad_bench.py 2>&1 | cut -c1-80
done
