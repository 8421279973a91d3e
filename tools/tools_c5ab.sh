# C5 device-path A/B: 512 units (dynamic schedule) x2 and 64 units (static) x1
for u in 512 512 64; do python bench.py --no-cpu --no-e2e --units $u 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print($u, round(d['value']), {k: round(v,3) for k,v in d['kernels_ms'].items()}, d['clocks']['sm_mhz'])"; done
