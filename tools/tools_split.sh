for s in 0 1 2 3; do FCW_DEBUG_SKIP=$s python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('skip',$s, d['kernels_ms'])"; done
