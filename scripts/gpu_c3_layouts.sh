#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_layout.py -x -q > gpurun_out/layout_tests.log 2>&1; echo LAYOUT_TESTS=$?
tail -3 gpurun_out/layout_tests.log
for L in ${LAYOUTS:-2 1}; do
  CYC_LAYOUT=$L CYC_DEBUG_TIMING=1 TRACE=64 timeout 600 python scripts/c3_probe.py 3 0 auto > gpurun_out/c3_layout$L.log 2>&1; echo C3_L$L=$?
  grep -v "^\[cyc build\]" gpurun_out/c3_layout$L.log | tail -${TAILN:-20}
done
