#!/bin/bash
# compute-sanitizer racecheck / memcheck / synccheck of the hot kernels on small
# BASELINE cases, including the TX carry recompute at every run start
# (FCW_CHUNK=1 / 7).  Logs: gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
CS="compute-sanitizer --error-exitcode 9"
run() {  # tool tag env... -- args
  local tool=$1 tag=$2; shift 2
  env "$@" timeout 1500 $CS --tool $tool python tools/sanitize_case.py $CASE > gpurun_out/sanitize_${tool}_${tag}.txt 2>&1
  echo "$tool $tag rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_${tool}_${tag}.txt | tail -1)"
}
CASE="c5 2 20"
run racecheck c5_chunk1 FCW_CHUNK=1
run racecheck c5_chunk7 FCW_CHUNK=7
run racecheck c5_static FCW_SCHED=static
run memcheck c5_chunk7 FCW_CHUNK=7
run synccheck c5_chunk7 FCW_CHUNK=7
CASE="c4 1 16"; run racecheck c4_chunk3 FCW_CHUNK=3; run memcheck c4 X=1
CASE="c2 2"; run racecheck c2 X=1; run memcheck c2 X=1
CASE="c1 8"; run racecheck c1 X=1; run memcheck c1 X=1
CASE="c3 1"; run racecheck c3 X=1; run memcheck c3 X=1
