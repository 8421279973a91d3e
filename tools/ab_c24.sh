for v in default pk2 pk4; do
  if [ "$v" = default ]; then unset FCW_LIB_VARIANT; else export FCW_LIB_VARIANT=$v; fi
  for c in c2 c4; do python bench.py --config $c --no-cpu --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', {k: round(v,4) for k,v in d['kernels_ms'].items()}, round(d['value']))"; done
done
