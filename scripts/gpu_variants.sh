#!/bin/bash
# C3 steady-state loop per library variant (paper_0912_2555_b200/_lib/variants/*.so)
cd "$(dirname "$0")/.."
for v in ${VARIANTS:-$(ls paper_0912_2555_b200/_lib/variants/*.so)}; do
  CYC_LIB_PATH=$v CYC_LAYOUT=${LAYOUT:-0} CFG=${CFG:-3} TRACE=64 timeout 600 python scripts/c3_probe.py 3 0 auto > gpurun_out/var.log 2>&1
  echo "== $v rc=$? loop $(grep loop_ms gpurun_out/var.log | tail -1 | sed 's/.*loop_ms.: \([0-9.]*\).*/\1/') | step ends: $(grep '^mode' gpurun_out/var.log | awk '{print $NF-0}' | tr '\n' ' ' | head -c 120)"
done
