#!/bin/bash
# One GPU call: the bench line, the reference arm, the launch list and one
# ncu --set full capture of the persistent MAP kernel (outputs in gpurun_out/).
make -C paper_0912_2555_b200/csrc -j8 >/dev/null && make -C oracle >/dev/null || exit 1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo BENCH_EXIT=$?
tail -1 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo REF_EXIT=$?
tail -1 gpurun_out/bench_ref.log
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo LAUNCH_EXIT=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_map_run -s 3 -c 1 \
      -o gpurun_out/map_run $CMD > gpurun_out/ncu_full.log 2>&1; echo FULL_EXIT=$?
ls -la gpurun_out/ | head -30
