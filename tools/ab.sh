#!/bin/bash
# A/B of library variants (build.py --variant NAME ...) on C5: kernel ms per variant
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then unset FCW_LIB_VARIANT; else export FCW_LIB_VARIANT=$v; fi
  for r in 1 2; do
    python bench.py --no-cpu --no-e2e --units 512 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', {k: round(v,3) for k,v in d['kernels_ms'].items()}, round(d['value']))"
  done
done
