#!/bin/bash
# C3 baseline probe: timings, per-step trace, launch list, ncu --set full of k_map_run on C3.
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c3_smi.txt
timeout 600 python scripts/run_config.py 3 0 > gpurun_out/c3_cfg_r0.log 2>&1; echo CFG0=$?
timeout 600 python scripts/run_config.py 3 1 > gpurun_out/c3_cfg_r1.log 2>&1; echo CFG1=$?
TRACE=256 timeout 600 python scripts/c3_probe.py 2 0 auto > gpurun_out/c3_trace_auto.log 2>&1; echo TRA=$?
TRACE=256 timeout 600 python scripts/c3_probe.py 2 0 pull > gpurun_out/c3_trace_pull.log 2>&1; echo TRP=$?
timeout 600 python scripts/c3_probe.py 2 0 auto > gpurun_out/c3_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_map_run -s 1 -c 1 \
   -o gpurun_out/c3_map_run python scripts/c3_probe.py 2 0 auto > gpurun_out/c3_ncu.log 2>&1; echo NCU=$?
tail -3 gpurun_out/c3_ncu.log
