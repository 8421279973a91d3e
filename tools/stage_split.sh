#!/bin/bash
# Stage cost breakdown (dev only): builds the `dev` library variant with the
# FCW_DEBUG_SKIP knob compiled in (bit 1: TX/RX short stage, bit 2: long
# transform) and times C5 with each bit set.  The release library has no knob.
[ -f paper_2008_00672_b200/lib/libfcwave_b200_dev.so ] || python -m paper_2008_00672_b200.build --variant dev FCW_DEV_KNOBS=1 fcw_launch.cu,fcw_k_n4096z.cu > /dev/null
export FCW_LIB_VARIANT=dev
for sk in ${SKIPS:-0 1 2 3}; do FCW_DEBUG_SKIP=$sk python bench.py --no-cpu --no-e2e --units 512 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('skip=$sk', {k: round(v,3) for k,v in d['kernels_ms'].items()})"; done
