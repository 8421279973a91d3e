#!/bin/bash
# Quick A/B on the GPU box: parity subset + C5 device-path bench (+ optional extra configs).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -3
for c in ${CONFIGS:-c5}; do
  timeout 300 python bench.py --config $c --no-cpu --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), {k: round(v,3) for k,v in d['kernels_ms'].items()}, 'hbm', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])"
done
