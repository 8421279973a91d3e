#!/bin/bash
mkdir -p gpurun_out
for c in c4 c2 c1; do
  python bench.py --config $c --no-cpu --e2e-steps 2 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  tail -1 gpurun_out/bench_$c.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value']), d['kernels_ms'], round(d['roofline']['txrx_frac'],4), 'e2e', round(d['e2e']['value']))"
done
