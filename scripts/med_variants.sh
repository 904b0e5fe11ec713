set -e
F=paper_0912_2555_b200/csrc/build.cu
for t in 256 512 1024; do
  sed -i "s/constexpr int kMedThreads = [0-9]*;/constexpr int kMedThreads = $t;/" $F
  make -C paper_0912_2555_b200/csrc -j8 >/dev/null 2>&1
  echo "== kMedThreads $t"
  CYC_DEBUG_TIMING=1 timeout 300 python scripts/build_only.py 3 3 2>&1 | grep -E "row_sort|^build" | tail -6
done
