"""The explorer's on-the-fly detector (explore.cpp:71-124, 184-209) on the
device: the log of a config grows in rounds; each round the detector takes
the snapshot of the current prefix and runs MAP (early exit). Compares an
incremental snapshot (cyc_graph_extend: only the new edges sorted, merged
into the previous round's CSRs) with the per-round full rebuild the
reference does. python scripts/detector_demo.py [config] [rounds] [map 0|1]
(config 4 unrestricted is MAP's worst case — 49 K dense steps — so its demo
skips MAP by default)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0912_2555_b200 as eng  # noqa: E402
from paper_0912_2555_b200 import _abi  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 8
do_map = (int(sys.argv[3]) if len(sys.argv) > 3 else int(cfg != 4)) != 0
p = eng.preset(cfg)
eng.prepare(p)
ctx = eng.default_context()
L, C = _abi.lib(), _abi.C
de, da = C.c_void_p(), C.c_void_p()
_abi.check(L.cyc_device_alloc(ctx.handle, p.m * 8, C.byref(de)))
_abi.check(L.cyc_device_alloc(ctx.handle, ((p.n + 63) // 64) * 8, C.byref(da)))
_abi.check(L.cyc_gen_fill(ctx.handle, C.byref(p), de, da))
# vertex prefix of each round: the largest endpoint so far (ids are BFS discovery order for config 4)
host = np.zeros((p.m, 2), np.uint32)
_abi.check(L.cyc_memcpy(ctx.handle, _abi.ptr(host), de, p.m * 8))
cuts = [int(p.m * (r + 1) / rounds) for r in range(rounds)]
maxend = np.maximum.accumulate(host.max(axis=1))
E = lambda off: C.cast(C.c_void_p(de.value + off * 8), C.POINTER(C.c_uint32))  # noqa: E731
A = C.cast(da, C.POINTER(C.c_uint64))
prev, prev_m, out = None, 0, []
for r, m in enumerate(cuts):
    n = int(maxend[m - 1]) + 1
    t0 = time.perf_counter()
    h = C.c_void_p()
    if prev is None:
        _abi.check(L.cyc_graph_build(ctx.handle, E(0), m, n, A, 1, C.byref(h)))
    else:
        _abi.check(L.cyc_graph_extend(ctx.handle, prev, E(prev_m), m - prev_m, n, A, C.byref(h)))
    t1 = time.perf_counter()
    hf = C.c_void_p()
    _abi.check(L.cyc_graph_build(ctx.handle, E(0), m, n, A, 1, C.byref(hf)))
    t2 = time.perf_counter()
    s = eng.CsrSnapshot(h, ctx)
    if do_map:
        v, st = eng.run_map(s, None)
    t3 = time.perf_counter()
    L.cyc_graph_destroy(hf)
    out.append({"round": r, "m_log": m, "n": n, "snapshot_ms": round((t1 - t0) * 1e3, 1),
                "rebuild_ms": round((t2 - t1) * 1e3, 1),
                **({"map_ms": round((t3 - t2) * 1e3, 1), "cycle": v.cycle_found(), "steps": st.kernel_calls}
                   if do_map else {})})
    if prev is not None:
        L.cyc_graph_destroy(prev)
    prev, prev_m = h, m
    s._h = None  # ownership stays with `prev`
for o in out:
    print(json.dumps(o))
