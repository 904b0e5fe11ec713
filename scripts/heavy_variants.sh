set -e
H=paper_0912_2555_b200/csrc/build.cuh
for cfg in "64 128" "32 128" "64 256" "32 256" "128 128"; do
  set -- $cfg
  sed -i "s/constexpr uint32_t kHeavyDeg = [0-9]*;/constexpr uint32_t kHeavyDeg = $1;/; s/constexpr uint32_t kHeavyChunk = [0-9]*;/constexpr uint32_t kHeavyChunk = $2;/" $H
  make -C paper_0912_2555_b200/csrc -j8 >/dev/null 2>&1
  echo "== heavy $1 chunk $2"
  timeout 300 python scripts/run_config.py 3 0 pull | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 pull8', d['loop_ms'])"
  timeout 300 python scripts/run_config.py 3 0 auto | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 auto8', d['loop_ms'])"
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', d['ms_per_step'])"
done
