#!/bin/bash
# Quick perf regression check: C3 steady-state loop (degree layout) and C2 bench-style run_map.
cd "$(dirname "$0")/.."
TRACE=64 timeout 600 python scripts/c3_probe.py 3 0 auto > gpurun_out/c3_perf.log 2>&1; echo C3=$?
grep -v "^\[cyc" gpurun_out/c3_perf.log | sed -n '3p;5,9p'
CFG=2 timeout 600 python scripts/c3_probe.py 4 1 auto > gpurun_out/c2_perf.log 2>&1; echo C2=$?; tail -2 gpurun_out/c2_perf.log
CFG=5 timeout 600 python scripts/c3_probe.py 3 1 auto > gpurun_out/c5_perf.log 2>&1; echo C5=$?; tail -1 gpurun_out/c5_perf.log
