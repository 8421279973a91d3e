mkdir -p gpurun_out
SMALL="python bench.py --units 64 --steps 2 --warmup 1 --no-e2e --no-cpu"
$SMALL > gpurun_out/plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
$SMALL > gpurun_out/plain_small2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"tx_kernel|rx_kernel" -s 2 -c 2 -o gpurun_out/prof -f $SMALL > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
