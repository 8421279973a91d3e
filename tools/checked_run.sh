#!/bin/bash
# Bounds-checked run (stands in for compute-sanitizer, which the GPU pool does
# not allow): every .cu of the library rebuilt with -DFCW_CHECK=1 (a trap on
# any out-of-range SMEM / global index on the hot path, fcw_device.cuh
# FCW_ASSERT) as the `check` variant, then the whole GPU suite on it — every
# config, every work schedule (FCW_CHUNK=1/7, static) and both RX paths.
# Build it where nvcc is (here or on the box):
#   python -m paper_2008_00672_b200.build --variant check FCW_CHECK=1 ALL
mkdir -p gpurun_out
[ -f paper_2008_00672_b200/lib/libfcwave_b200_check.so ] || \
  python -m paper_2008_00672_b200.build --variant check FCW_CHECK=1 ALL > /dev/null
FCW_LIB_VARIANT=check timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider \
  > gpurun_out/checked_run.txt 2>&1
echo "checked run rc=$?"; tail -3 gpurun_out/checked_run.txt
