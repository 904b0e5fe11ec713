#!/bin/bash
# C3 steady-state loop per library variant (paper_0912_2555_b200/_lib/variants/*.so)
cd "$(dirname "$0")/.."
for v in ${VARIANTS:-$(ls paper_0912_2555_b200/_lib/variants/*.so)}; do
  CYC_LIB_PATH=$v CYC_LAYOUT=${LAYOUT:-2} TRACE=64 timeout 600 python scripts/c3_probe.py 3 0 auto > gpurun_out/var.log 2>&1; echo "== $v rc=$?"
  grep -v "^\[cyc" gpurun_out/var.log | sed -n '3p;6,9p'
done
