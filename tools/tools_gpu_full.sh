mkdir -p gpurun_out
python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
for c in c5 c4 c2 c1 c3; do
  python bench.py --config $c --no-cpu --e2e-steps 2 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  tail -1 gpurun_out/bench_$c.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value']), {k: round(v,3) for k,v in d['kernels_ms'].items()}, round(d['roofline']['txrx_frac'],4), 'e2e', round(d['e2e']['value']))"
done
