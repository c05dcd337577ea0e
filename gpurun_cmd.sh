for tag in base ge8 ge2; do
  if [ $tag = base ]; then unset FFB_LIB_VARIANT; else export FFB_LIB_VARIANT=$tag; fi
  echo "== $tag"; python tools/grad_bench.py 2>&1 | cut -c1-80
done
