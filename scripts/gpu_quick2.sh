#!/bin/bash
# Quick loop: core parity files, then the C3/C2/C5 perf check.
cd "$(dirname "$0")/.."
for f in tests/test_gpu_layout.py tests/test_gpu_shard_engine.py tests/test_gpu_parity.py; do
  timeout ${TMO:-600} python -m pytest $f -x -q > gpurun_out/t.log 2>&1; echo "$f rc=$? $(tail -1 gpurun_out/t.log)"
done
bash scripts/gpu_perf_check.sh
