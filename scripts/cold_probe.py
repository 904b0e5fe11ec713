"""Cold-call probe: time of the first cyc_check of a process (config 3, pinned host log), then warm calls."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
t0 = time.perf_counter()
import paper_0912_2555_b200 as eng  # noqa: E402
from paper_0912_2555_b200 import _abi  # noqa: E402

L = _abi.lib()
ctx = eng.Context(0)
t_ctx = time.perf_counter() - t0
p = eng.prepare(eng.preset(int(os.environ.get("CFG", "3"))))
n, m = int(p.n), int(p.m)
d_e, d_a, h_e, h_a = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
_abi.check(L.cyc_device_alloc(ctx.handle, m * 8, C.byref(d_e)))
_abi.check(L.cyc_device_alloc(ctx.handle, ((n + 63) // 64) * 8, C.byref(d_a)))
_abi.check(L.cyc_gen_fill(ctx.handle, C.byref(p), d_e, d_a))
_abi.check(L.cyc_host_alloc(m * 8, C.byref(h_e)))
_abi.check(L.cyc_host_alloc(((n + 63) // 64) * 8, C.byref(h_a)))
_abi.check(L.cyc_memcpy(ctx.handle, h_e, d_e, m * 8))
_abi.check(L.cyc_memcpy(ctx.handle, h_a, d_a, ((n + 63) // 64) * 8))
L.cyc_device_free(ctx.handle, d_e)
L.cyc_device_free(ctx.handle, d_a)
opt = eng.MapOptions(early_exit=True).to_c()
out = []
for i in range(4):
    st, ms = _abi.MapStatsC(), (C.c_double * 4)()
    t = time.perf_counter()
    _abi.check(L.cyc_check(ctx.handle, C.cast(h_e, C.POINTER(C.c_uint32)), m, n,
                           C.cast(h_a, C.POINTER(C.c_uint64)), 1, 0, C.byref(opt), C.byref(st), ms))
    out.append((round((time.perf_counter() - t) * 1e3, 1), [round(x, 1) for x in ms], round(st.plan_ms, 1)))
print({"ctx_s": round(t_ctx, 2), "calls_ms_phases_plan": out}, flush=True)
