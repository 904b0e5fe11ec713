#!/bin/bash
# Regression round: GPU tests file by file under timeouts (default layout, then
# degree layout forced with L2=1), then config 3/2/5 timings.
cd "$(dirname "$0")/.."
for f in tests/test_gpu_shard_engine.py tests/test_gpu_layout.py tests/test_gpu_parity.py tests/test_gpu_full_parity.py \
         tests/test_gpu_dropin.py tests/test_gpu_concurrency.py tests/test_gpu_sharded.py; do
  timeout ${TMO:-600} python -m pytest $f -x -q > gpurun_out/t.log 2>&1; echo "$f rc=$? $(tail -1 gpurun_out/t.log)"
done
if [ -n "$L2" ]; then CYC_LAYOUT=2 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_l2.log 2>&1; echo GPU_TESTS_L2=$?; tail -1 gpurun_out/gpu_tests_l2.log; fi
bash scripts/gpu_perf_check.sh
