#!/bin/bash
# Round-2 evidence: bench line (N=1), reference arm, sharded N=1 line, launch
# list and ncu --set full of k_map_run on config 3 (outputs in gpurun_out/).
cd "$(dirname "$0")/.."
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo BENCH=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_c3.log 2>&1; echo REF=$?
timeout 900 python bench.py --sharded --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_shard1.log 2>&1; echo SHARD=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo LAUNCH_EXIT=$?
CMD2="python scripts/c3_probe.py 2 0 auto"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_map_run -s 1 -c 1 \
      -o gpurun_out/r02_c3_map_run $CMD2 > gpurun_out/ncu_full.log 2>&1; echo FULL_EXIT=$?
