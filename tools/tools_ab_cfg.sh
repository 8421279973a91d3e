#!/bin/bash
# A/B of library variants on one config: CFG=c2 VARIANTS="default x" bash tools/tools_ab_cfg.sh
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then unset FCW_LIB_VARIANT; else export FCW_LIB_VARIANT=$v; fi
  python bench.py --config ${CFG:-c5} --no-cpu --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '${CFG:-c5}', {k: round(v,3) for k,v in d['kernels_ms'].items()}, round(d['value']))"
done
