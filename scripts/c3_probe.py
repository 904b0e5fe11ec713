"""Config-3 probe: device-generated R-MAT 2^26 x 16, transposed snapshot,
run_map with early_exit off (steady-state dense steps) REPS times; prints the
per-run loop time and MapStats. Used as the ncu target for k_map_run on C3:
    python scripts/c3_probe.py [reps] [early] [mode]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0912_2555_b200 as eng  # noqa: E402
from paper_0912_2555_b200 import _abi  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
early = len(sys.argv) > 2 and sys.argv[2] == "1"
mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
C = _abi.C
L = _abi.lib()
p = eng.prepare(eng.preset(int(os.environ.get("CFG", "3"))))
ctx = eng.default_context()
de, da = C.c_void_p(), C.c_void_p()
_abi.check(L.cyc_device_alloc(ctx.handle, p.m * 8, C.byref(de)))
_abi.check(L.cyc_device_alloc(ctx.handle, ((p.n + 63) // 64) * 8, C.byref(da)))
_abi.check(L.cyc_gen_fill(ctx.handle, C.byref(p), de, da))
g = C.c_void_p()
_abi.check(L.cyc_graph_build(ctx.handle, C.cast(de, C.POINTER(C.c_uint32)), p.m, p.n,
                             C.cast(da, C.POINTER(C.c_uint64)), 1, C.byref(g)))
L.cyc_device_free(ctx.handle, de)
opt = eng.MapOptions(early_exit=early, mode=mode, trace_cap=int(os.environ.get("TRACE", "0"))).to_c(
    0, int(os.environ.get("MAXSTEPS", "0")))
for r in range(reps):
    st = _abi.MapStatsC()
    _abi.check(L.cyc_flush_l2(ctx.handle, 512 << 20))
    _abi.check(L.cyc_map_run(ctx.handle, g, None, C.byref(opt), C.byref(st), None, None, None, 0))
    d = eng.api.stats_dict(st)
    print({k: d[k] for k in ("cycle_found", "witness", "iterations", "kernel_calls", "pull_steps",
                             "push_steps", "loop_ms", "edges_touched")}, flush=True)
if opt.trace_cap:
    import numpy as np
    tr = eng.map_trace(eng.CsrSnapshot(g, ctx))
    for r in tr[:64]:
        print("mode %d step %3d Ef %11d raised %9d | ph0 %8.1f ph1 %8.1f flags %8.1f end %8.1f us" % (
            r[0], r[1], r[2], r[3], (r[5] - r[4]) / 1e3, (r[6] - r[4]) / 1e3, (r[7] - r[4]) / 1e3,
            (r[8] - r[4]) / 1e3))
