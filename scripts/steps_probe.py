"""Runs a bounded number of MAP steps on a config (profiling aid):
python scripts/steps_probe.py <config> <max_steps> [mode]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0912_2555_b200 as eng  # noqa: E402
from paper_0912_2555_b200 import _abi  # noqa: E402

cfg, k = int(sys.argv[1]), int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
p = eng.preset(cfg)
eng.prepare(p)
ctx = eng.default_context()
L, C = _abi.lib(), _abi.C
de, da = C.c_void_p(), C.c_void_p()
_abi.check(L.cyc_device_alloc(ctx.handle, p.m * 8, C.byref(de)))
_abi.check(L.cyc_device_alloc(ctx.handle, ((p.n + 63) // 64) * 8, C.byref(da)))
_abi.check(L.cyc_gen_fill(ctx.handle, C.byref(p), de, da))
h = C.c_void_p()
_abi.check(L.cyc_graph_build(ctx.handle, C.cast(de, C.POINTER(C.c_uint32)), p.m, p.n,
                             C.cast(da, C.POINTER(C.c_uint64)), 1, C.byref(h)))
s = eng.CsrSnapshot(h, ctx)
opt = eng.MapOptions(mode=mode).to_c(max_steps=k)
for rep in range(2):
    st = _abi.MapStatsC()
    _abi.check(L.cyc_map_run(ctx.handle, h, None, C.byref(opt), C.byref(st), None, None, None, 0))
    print(f"config {cfg} {mode}: {st.kernel_calls} steps, loop {st.loop_ms:.2f} ms, "
          f"{st.loop_ms / max(st.kernel_calls, 1):.3f} ms/step, pull {st.pull_steps} push {st.push_steps}")
