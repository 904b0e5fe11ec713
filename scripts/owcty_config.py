"""Full-size verdict cross-check on a BASELINE config: device OWCTY (forward
snapshot, as cycheck_main.cpp:98-106), device SCC verdict and MAP, with
timings. python scripts/owcty_config.py <config> [k=v overrides ...]
  env OWCTY_ORIENT=0|1 (default both), OWCTY_REPS (default 2), OWCTY_MAP=0 skips MAP"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0912_2555_b200 as eng  # noqa: E402
from paper_0912_2555_b200 import _abi  # noqa: E402

cfg = int(sys.argv[1])
p = eng.preset(cfg)
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    setattr(p, k, int(v))
eng.prepare(p)
ctx = eng.default_context()
L = _abi.lib()
C = _abi.C
de, da = C.c_void_p(), C.c_void_p()
_abi.check(L.cyc_device_alloc(ctx.handle, p.m * 8, C.byref(de)))
_abi.check(L.cyc_device_alloc(ctx.handle, ((p.n + 63) // 64) * 8, C.byref(da)))
_abi.check(L.cyc_gen_fill(ctx.handle, C.byref(p), de, da))
orients = [int(os.environ["OWCTY_ORIENT"])] if "OWCTY_ORIENT" in os.environ else [0, 1]
reps = int(os.environ.get("OWCTY_REPS", "2"))
for orient in orients:
    h = C.c_void_p()
    t0 = time.perf_counter()
    _abi.check(L.cyc_graph_build(ctx.handle, C.cast(de, C.POINTER(C.c_uint32)), p.m, p.n,
                                 C.cast(da, C.POINTER(C.c_uint64)), orient, C.byref(h)))
    build_ms = (time.perf_counter() - t0) * 1e3
    s = eng.CsrSnapshot(h, ctx)
    out = {"config": cfg, "orientation": ["forward", "transposed"][orient], "n": s.n, "m": s.m,
           "build_ms": round(build_ms, 1)}
    for rep in range(reps):
        t0 = time.perf_counter()
        v, st = eng.run_owcty(s)
        out["owcty_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
    out.update(owcty_cycle=v.cycle_found(), owcty_witness=v.witness, outer=st.outer_iterations,
               final_size=st.final_size, reach_ms=round(st.reach_ms, 2), elim_ms=round(st.elim_ms, 2))
    for rep in range(reps):
        t0 = time.perf_counter()
        ov = eng.scc_verdict(s)
        out.update(scc_ms=round((time.perf_counter() - t0) * 1e3, 2), scc_cycle=ov.verdict.cycle_found(),
                   scc_witness=ov.verdict.witness)
    if os.environ.get("OWCTY_MAP", "1") != "0":
        t0 = time.perf_counter()
        mv, ms = eng.run_map(s, s.accepting)
        out.update(map_ms=round((time.perf_counter() - t0) * 1e3, 2), map_cycle=mv.cycle_found())
    print(json.dumps(out), flush=True)
