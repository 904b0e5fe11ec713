#!/bin/bash
# Plan tie-break by gather-row length (CYC_PLAN_TIE=0 disables): layout/shard parity, then C3 with and without.
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_shard_engine.py -x -q > gpurun_out/tie_tests.log 2>&1; echo TIE_TESTS=$?; tail -2 gpurun_out/tie_tests.log
for T in 0 1; do
  echo "== tie $T"
  CYC_PLAN_TIE=$T CYC_DEBUG_TIMING=1 TRACE=64 timeout 600 python scripts/c3_probe.py 3 0 auto > gpurun_out/c3_tie$T.log 2>&1; echo C3=$?
  grep -v "^\[cyc build\]" gpurun_out/c3_tie$T.log | grep -v "^\[cyc" | sed -n '3p;5,12p'; grep "plan\|place\|sell" gpurun_out/c3_tie$T.log | head -8
done
