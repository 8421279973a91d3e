#!/bin/bash
# A/B of library variants on configs: CONFIGS="c4" VARIANTS="default x" bash tools/ab_cfg.sh
for c in ${CONFIGS:-c5}; do
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then unset FCW_LIB_VARIANT; else export FCW_LIB_VARIANT=$v; fi
  for r in 1 2; do
    python bench.py --config $c --no-cpu --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$v', {k: round(v,4) for k,v in d['kernels_ms'].items()}, round(d['value']))"
  done
done
done
