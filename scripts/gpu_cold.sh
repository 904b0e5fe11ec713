#!/bin/bash
# Cold first call with and without the background pool reserve (bench.py, config 3).
cd "$(dirname "$0")/.."
for R in "" "--no-reserve"; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline $R > gpurun_out/cold$R.log 2>&1; echo "rc=$? $R"
  tail -1 gpurun_out/cold$R.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['time_to_verdict_ms']; print(d['value'], t['e2e_host'], t['cold_first_call_e2e_host'], t['cold_reserve']['wait_ms'])"
done
