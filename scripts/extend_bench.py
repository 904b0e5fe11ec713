"""Incremental snapshot vs full rebuild on a BASELINE config (the explorer's
per-round detector rebuild, explore.cpp:71-124): build the snapshot of the
first `frac` of the log, then extend it by the rest, against building the
whole prefix. python scripts/extend_bench.py <config> [frac]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0912_2555_b200 as eng  # noqa: E402
from paper_0912_2555_b200 import _abi  # noqa: E402

cfg = int(sys.argv[1])
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
p = eng.preset(cfg)
eng.prepare(p)
ctx = eng.default_context()
L, C = _abi.lib(), _abi.C
de, da = C.c_void_p(), C.c_void_p()
_abi.check(L.cyc_device_alloc(ctx.handle, p.m * 8, C.byref(de)))
_abi.check(L.cyc_device_alloc(ctx.handle, ((p.n + 63) // 64) * 8, C.byref(da)))
_abi.check(L.cyc_gen_fill(ctx.handle, C.byref(p), de, da))
m0 = int(p.m * frac)
E = lambda off: C.cast(C.c_void_p(de.value + off * 8), C.POINTER(C.c_uint32))
A = C.cast(da, C.POINTER(C.c_uint64))
res = {}
for rep in range(3):
    h0, h1, hf = C.c_void_p(), C.c_void_p(), C.c_void_p()
    _abi.check(L.cyc_graph_build(ctx.handle, E(0), m0, p.n, A, 1, C.byref(h0)))
    t0 = time.perf_counter()
    _abi.check(L.cyc_graph_extend(ctx.handle, h0, E(m0), p.m - m0, p.n, A, C.byref(h1)))
    t1 = time.perf_counter()
    _abi.check(L.cyc_graph_build(ctx.handle, E(0), p.m, p.n, A, 1, C.byref(hf)))
    t2 = time.perf_counter()
    s1, sf = eng.CsrSnapshot(h1, ctx), eng.CsrSnapshot(hf, ctx)
    res = {"config": cfg, "m_log": int(p.m), "m_new": int(p.m - m0), "extend_ms": round((t1 - t0) * 1e3, 2),
           "rebuild_ms": round((t2 - t1) * 1e3, 2), "m": sf.m, "same_m": s1.m == sf.m}
    L.cyc_graph_destroy(h0)
print(json.dumps(res))
