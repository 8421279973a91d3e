#!/bin/bash
# tests + bench (no ncu)
mkdir -p gpurun_out
python -m pytest tests/ -q -m gpu -x 2>&1 | tail -15
python bench.py --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-1500
