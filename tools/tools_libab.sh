# A/B two prebuilt libraries (abtmp/old.so, abtmp/new.so) with and without FCW_DEBUG_SKIP
L=paper_2008_00672_b200/lib/libfcwave_b200.so
for v in old new; do for sk in 0 1; do cp abtmp/$v.so $L; FCW_DEBUG_SKIP=$sk python bench.py --no-cpu --no-e2e --units 512 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v skip=$sk', {k: round(v,3) for k,v in d['kernels_ms'].items()})"; done; done
