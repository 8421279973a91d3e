#!/bin/bash
# schedule A/B on C5: dynamic run lengths vs static ranges
run() { python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', {k: round(v,3) for k,v in d['kernels_ms'].items()}, round(d['value']))"; }
run default
FCW_SCHED=static run static
FCW_CHUNK_TX=56 FCW_CHUNK_RX=32 run c56_32
FCW_CHUNK_TX=140 FCW_CHUNK_RX=56 run c140_56
FCW_CHUNK_TX=14 FCW_CHUNK_RX=8 run c14_8
run default
