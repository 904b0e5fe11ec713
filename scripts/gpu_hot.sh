#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_layout.py -x -q > gpurun_out/layout_tests.log 2>&1; echo LAYOUT_TESTS=$?
tail -3 gpurun_out/layout_tests.log
for H in ${HOTS:-0 524288}; do
  CYC_HOT_POS=$H CYC_LAYOUT=2 TRACE=64 timeout 600 python scripts/c3_probe.py 3 0 auto > gpurun_out/c3_hot$H.log 2>&1; echo C3_HOT$H=$?
  grep -v "^\[cyc" gpurun_out/c3_hot$H.log | tail -${TAILN:-9}
done
