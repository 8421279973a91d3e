#!/bin/bash
# One gpurun call of round evidence (run from the repo root on the GPU box):
#   STAGE=tests   pytest -m gpu + smoke
#   STAGE=bench   C5 bench (e2e + cpu_baseline), reference arm, C1-C4 lines
#   STAGE=ncu     launch list + one --set full capture of both C5 kernels (each after a clean run)
#   STAGE=fp32    FP32 issue ceiling (tools/ubench_fp32.cu) -> gpurun_out/fp32_peak.json
# Default: all stages.  Logs go to gpurun_out/.
mkdir -p gpurun_out
want() { [ -z "$STAGE" ] || [[ " $STAGE " == *" $1 "* ]]; }
if want tests; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
fi
if want fp32; then
  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubench_fp32 tools/ubench_fp32.cu && /tmp/ubench_fp32 > gpurun_out/fp32_peak.txt 2>&1
  echo "fp32 rc=$?"; tail -2 gpurun_out/fp32_peak.txt
fi
if want bench; then
  timeout 600 python bench.py > gpurun_out/bench_c5.log 2>&1; echo "bench c5 rc=$?"; tail -1 gpurun_out/bench_c5.log | cut -c1-400
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
  for c in ${CONFIGS:-c1 c2 c3 c4}; do
    timeout 600 python bench.py --config $c --no-cpu --e2e-steps 2 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  done
fi
if want ncu; then
  SMALL="python bench.py --units 64 --steps 2 --warmup 1 --no-e2e --no-cpu"
  $SMALL > gpurun_out/plain_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  $SMALL > gpurun_out/plain_small2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"tx_kernel|rx_kernel" -s 2 -c 2 \
      -o gpurun_out/prof -f $SMALL > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
