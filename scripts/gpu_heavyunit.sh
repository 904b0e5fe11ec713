#!/bin/bash
# Dynamic heavy-chunk claims (pull_heavy_slab): parity with the default build, C3 per unit size.
cd "$(dirname "$0")/.."
for f in tests/test_gpu_layout.py tests/test_gpu_shard_engine.py tests/test_gpu_full_parity.py; do
  timeout 600 python -m pytest $f -x -q > gpurun_out/t.log 2>&1; echo "$f rc=$? $(tail -1 gpurun_out/t.log)"
done
for V in default hu16 hu32 hu128; do
  echo "== $V"
  L=""; [ $V != default ] && L="CYC_LIB_PATH=paper_0912_2555_b200/_lib/variants/$V.so"
  env $L TRACE=64 timeout 600 python scripts/c3_probe.py 3 0 auto > gpurun_out/c3_$V.log 2>&1; echo C3=$?
  grep -v "^\[cyc" gpurun_out/c3_$V.log | sed -n '3,8p'
done
