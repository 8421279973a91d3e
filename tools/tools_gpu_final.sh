#!/bin/bash
# Round evidence: default bench (C5, e2e + cpu_baseline), reference arm, all configs,
# launch list and one full ncu capture of both kernels (each after a clean run).
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c5.log 2>&1; echo "bench c5 rc=$?"; tail -1 gpurun_out/bench_c5.log | cut -c1-300
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
for c in c1 c2 c3 c4; do
  python bench.py --config $c --no-cpu --e2e-steps 2 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
done
SMALL="python bench.py --units 64 --steps 2 --warmup 1 --no-e2e --no-cpu"
$SMALL > gpurun_out/plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
$SMALL > gpurun_out/plain_small2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"tx_kernel|rx_kernel" -s 2 -c 2 -o gpurun_out/prof -f $SMALL > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python tools/bench_rows.py --units 64 > gpurun_out/rows.jsonl 2>&1; echo "rows rc=$?"
