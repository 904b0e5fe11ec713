"""Per-step timing trace of the device loop (diagnostics for the push/pull
heuristic and the per-phase critical path):
    python scripts/trace_run.py [config] [modes] [alpha]"""
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
    opt = eng.MapOptions(mode=mode, push_alpha=alpha, trace_cap=1 << 14)
    for _ in range(2):
        v, st = eng.run_map(s, s.accepting, opt)
    tr = eng.map_trace(s)
    kind, ef = tr[:, 0], tr[:, 2]
    if os.environ.get("TRACE_DUMP"):
        lo = int(os.environ["TRACE_DUMP"])
        for r in tr[lo:lo + 24]:
            print("      mode %d step %4d Ef %9d raised %8d chunks %6d | ph0 %6.2f ph1 %6.2f fl %6.2f end %6.2f" % (
                r[0], r[1], r[2], r[3], r[9], (r[5]-r[4])/1e3, (r[6]-r[4])/1e3, (r[7]-r[4])/1e3, (r[8]-r[4])/1e3))
    t0, p0, p1, fl, t1 = (tr[:, k].astype(np.float64) for k in range(4, 9))
    dur = (t1 - t0) / 1e3
    print(f"-- {mode}: loop {st.device['loop_ms']:.2f} ms, steps {len(tr)}, {v}, calls {st.kernel_calls}")
    for k, name in ((1, "pull"), (2, "push")):
        sel = kind == k
        if not sel.any():
            continue
        ph = lambda x: np.median((x[sel] - t0[sel]) / 1e3)
        print(f"   {name}: n={sel.sum()} mean {dur[sel].mean():.2f} us p50 {np.median(dur[sel]):.2f} "
              f"total {dur[sel].sum()/1e3:.2f} ms | p50 phase0 {ph(p0):.2f} phase1 {ph(p1):.2f} "
              f"flags {ph(fl):.2f} end {ph(t1):.2f} us")
        if k == 2:
            bins = [0, 1e3, 1e4, 1e5, 3e5, 1e6, 3e6, 1e9]
            for lo, hi in zip(bins[:-1], bins[1:]):
                m = sel & (ef >= lo) & (ef < hi)
                if m.any():
                    q = lambda x: np.median((x[m] - t0[m]) / 1e3)
                    print(f"      Ef in [{lo:.0e},{hi:.0e}): n={m.sum():5d} mean {dur[m].mean():7.2f} us "
                          f"| phase0 {q(p0):6.2f} phase1 {q(p1):6.2f} flags {q(fl):6.2f} end {q(t1):6.2f}")
    if os.environ.get("TRACE_RAISED"):
        raised = tr[:, 3]
        for k, name in ((1, "pull"), (2, "push")):
            sel = kind == k
            if sel.any():
                qs = np.percentile(raised[sel], [5, 25, 50, 75, 95])
                print(f"   {name} raised per step: p5/25/50/75/95 = {qs.astype(int).tolist()} (n={s.n})")
        # raised vs step-in-fixpoint for the first few fixpoints
        print("   step-in-fixpoint raised (first fixpoint):", [int(r) for r in tr[:70, 3]])
    if os.environ.get("TRACE_GAPS"):
        t_start, t_end = tr[:, 4].astype(np.float64), tr[:, 8].astype(np.float64)
        gap = (t_start[1:] - t_end[:-1]) / 1e3
        per = (t_start[1:] - t_start[:-1]) / 1e3
        print(f"   step period p50 {np.median(per):.2f} us, gap end->next start p50 {np.median(gap):.2f} us")
