run() { python bench.py --no-cpu --no-e2e --units 64 --steps 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', {k: round(v,4) for k,v in d['kernels_ms'].items()}, round(d['value']))"; }
run static
for c in 4 7 14; do FCW_CHUNK_RX=$c run rx$c; done
for c in 14 20 28 35; do FCW_CHUNK_TX=$c run tx$c; done
