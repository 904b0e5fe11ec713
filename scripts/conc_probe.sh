#!/bin/bash
# Repeats the multi-context test (30 runs, no process-wide lock) and the C++
# drop-in test (10 runs); keeps the log of the first hang.
cd "$(dirname "$0")/.."
ok=0
for i in $(seq 1 ${RUNS:-30}); do
  if timeout 60 python -m pytest tests/test_gpu_concurrency.py -q -s -p no:cacheprovider > gpurun_out/conc.log 2>&1; then
    ok=$((ok+1))
  else
    echo "hang/fail at run $i"; cp gpurun_out/conc.log gpurun_out/conc_hang.log; break
  fi
done
echo "concurrency ok=$ok"
ok=0
for i in $(seq 1 10); do timeout 60 ./oracle/_ref/dropin_test 150 > gpurun_out/dropin.out 2>&1 && ok=$((ok+1)); done
echo "dropin ok=$ok/10"
