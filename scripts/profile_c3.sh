#!/bin/bash
# Round-2 evidence: GPU tests (both layouts), bench launch list, ncu --set full of k_map_run on config 3.
cd "$(dirname "$0")/.."
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo GPU_TESTS=$?; tail -2 gpurun_out/gpu_tests.log
CYC_LAYOUT=2 timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_l2.log 2>&1; echo GPU_TESTS_L2=$?; tail -2 gpurun_out/gpu_tests_l2.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo LAUNCH_EXIT=$?
CMD2="python scripts/c3_probe.py 2 0 auto"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_map_run -s 1 -c 1 \
      -o gpurun_out/r02_c3_map_run $CMD2 > gpurun_out/ncu_full.log 2>&1; echo FULL_EXIT=$?
