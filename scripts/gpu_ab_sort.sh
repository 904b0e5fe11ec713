#!/bin/bash
# A/B of sorted heavy rows (CYC_SORT_HEAVY=1) on config 3, alternating, 3 runs x 3 reps each.
cd "$(dirname "$0")/.."
for k in 1 2 3; do
  for S in 0 1; do
    CYC_SORT_HEAVY=$S timeout 300 python scripts/c3_probe.py 4 0 auto 2>&1 | grep loop_ms | tail -2 | python -c "
import sys,ast; v=[ast.literal_eval(l)['loop_ms'] for l in sys.stdin]; print('sort $S', ' '.join('%.3f'%x for x in v))"
  done
done
