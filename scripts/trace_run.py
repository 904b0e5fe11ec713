"""Per-step timing trace of the device loop (diagnostics for the push/pull
heuristic): python scripts/trace_run.py [config] [mode] [alpha]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0912_2555_b200 as eng  # noqa: E402
from paper_0912_2555_b200 import _abi  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["auto", "pull", "push"]
alpha = int(sys.argv[3]) if len(sys.argv) > 3 else 0
p = eng.preset(cfg)
ctx = eng.default_context()
e = np.zeros((p.m, 2), np.uint32)
a = np.zeros((p.n + 63) // 64, np.uint64)
_abi.check(_abi.lib().cyc_gen_fill(ctx.handle, _abi.C.byref(p), _abi.ptr(e), _abi.ptr(a)))
s = eng.build_snapshot((p.n, e, eng.Bitset.from_words(a, p.n)))
print(f"config {cfg}: n={s.n} m={s.m}")
for mode in modes:
    opt = eng.MapOptions(mode=mode, push_alpha=alpha, trace_cap=1 << 16)
    for _ in range(2):
        v, st = eng.run_map(s, s.accepting, opt)
    tr = eng.map_trace(s)
    clk = tr[:, 4]
    dt = np.diff(clk) / 1.965e3  # us at max SM clock
    kind, ef = tr[1:, 0], tr[1:, 2]
    print(f"-- {mode}: loop {st.device['loop_ms']:.2f} ms, steps {len(tr)}, verdict {v}, "
          f"calls {st.kernel_calls}")
    for k, name in ((1, "pull"), (2, "push")):
        sel = kind == k
        if not sel.any():
            continue
        print(f"   {name}: n={sel.sum()} mean {dt[sel].mean():.2f} us  p50 {np.median(dt[sel]):.2f}  "
              f"p90 {np.percentile(dt[sel], 90):.2f}  total {dt[sel].sum()/1e3:.2f} ms")
        if k == 2:
            bins = [0, 1e3, 1e4, 1e5, 3e5, 1e6, 3e6, 1e9]
            for lo, hi in zip(bins[:-1], bins[1:]):
                m = sel & (ef >= lo) & (ef < hi)
                if m.any():
                    print(f"      Ef in [{lo:.0e},{hi:.0e}): n={m.sum():5d} mean {dt[m].mean():7.2f} us "
                          f"({dt[m].mean() * 1e3 / max(ef[m].mean(), 1):.3f} ns/edge)")
