"""Builds config <c> from a device-generated log (for build profiling)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0912_2555_b200 as eng
from paper_0912_2555_b200 import _abi
cfg = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = eng.preset(cfg); eng.prepare(p)
ctx = eng.default_context(); L = _abi.lib(); C = _abi.C
de, da = C.c_void_p(), C.c_void_p()
_abi.check(L.cyc_device_alloc(ctx.handle, p.m * 8, C.byref(de)))
_abi.check(L.cyc_device_alloc(ctx.handle, ((p.n + 63) // 64) * 8, C.byref(da)))
_abi.check(L.cyc_gen_fill(ctx.handle, C.byref(p), de, da))
for r in range(reps):
    g = C.c_void_p()
    t0 = time.perf_counter()
    _abi.check(L.cyc_graph_build(ctx.handle, C.cast(de, C.POINTER(C.c_uint32)), p.m, p.n,
                                 C.cast(da, C.POINTER(C.c_uint64)), 1, C.byref(g)))
    print(f"build {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
    L.cyc_graph_destroy(g)
