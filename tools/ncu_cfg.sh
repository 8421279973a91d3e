#!/bin/bash
# ncu --set full of one config's TX/RX kernels (after a clean run of the same command)
# CFG=c4 [UNITS=..] bash tools/ncu_cfg.sh   -> gpurun_out/prof_$CFG.ncu-rep
mkdir -p gpurun_out
CMD="python bench.py --config $CFG ${UNITS:+--units $UNITS} --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"tx_kernel|rx_kernel" -s ${SKIP:-2} -c ${COUNT:-2} \
    -o gpurun_out/prof_$CFG -f $CMD > gpurun_out/ncu_$CFG.log 2>&1; echo "ncu $CFG rc=$?"
