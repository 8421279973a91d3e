# Stage cost breakdown via FCW_DEBUG_SKIP bits (1: TX/RX short stage, 2: long stage; dev only)
for sk in ${SKIPS:-0 1 2 3}; do FCW_DEBUG_SKIP=$sk python bench.py --no-cpu --no-e2e --units 512 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('skip=$sk', {k: round(v,3) for k,v in d['kernels_ms'].items()})"; done
