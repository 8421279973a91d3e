#!/bin/bash
# ncu full capture of both kernels on a small C5 run (plain run first)
mkdir -p gpurun_out
SMALL="python bench.py --units 64 --steps 2 --warmup 1 --no-e2e --no-cpu"
$SMALL > gpurun_out/plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"tx_kernel|rx_kernel" -s 2 -c 2 -o gpurun_out/prof -f $SMALL > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
