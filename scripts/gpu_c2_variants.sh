#!/bin/bash
cd "$(dirname "$0")/.."
for v in $(ls paper_0912_2555_b200/_lib/variants/*.so); do
  CYC_LIB_PATH=$v CFG=${CFG:-2} timeout 300 python scripts/c3_probe.py 3 1 auto > gpurun_out/var.log 2>&1; echo "== $v rc=$?"; tail -1 gpurun_out/var.log | cut -c1-200
done
