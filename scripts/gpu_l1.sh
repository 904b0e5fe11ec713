#!/bin/bash
cd "$(dirname "$0")/.."
for v in base na; do for H in 4294967295 131072 65536 32768 16384; do
  CYC_LIB_PATH=paper_0912_2555_b200/_lib/variants/$v.so CYC_L1_HOT=$H TRACE=64 timeout 300 python scripts/c3_probe.py 3 0 auto > gpurun_out/l1.log 2>&1
  echo "== $v L1_HOT=$H: $(grep loop_ms gpurun_out/l1.log | tail -1 | sed 's/.*loop_ms.: \([0-9.]*\).*/\1/') | $(grep 'step   2\|step   4' gpurun_out/l1.log | tail -2 | awk '{print $11, $13}' | tr '\n' ' ')"
done; done
