# Repeats the multi-context test (30 runs); keeps the log of the first hang.
make -C paper_0912_2555_b200/csrc -j8 >/dev/null 2>&1
ok=0
for i in $(seq 1 30); do
  if CYC_TRACE_CALLS=1 timeout 40 python -m pytest tests/test_gpu_concurrency.py -q -s -p no:cacheprovider > gpurun_out/conc.log 2>&1; then
    ok=$((ok+1))
  else
    echo "hang/fail at run $i"; cp gpurun_out/conc.log gpurun_out/conc_hang2.log; break
  fi
done
echo "ok=$ok"
