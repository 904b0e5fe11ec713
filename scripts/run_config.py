"""Runs a BASELINE config at full size through the one-call pipeline and
reports phase timings: python scripts/run_config.py <config> [restrict] [mode] [overrides k=v ...]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0912_2555_b200 as eng  # noqa: E402
from paper_0912_2555_b200 import _abi  # noqa: E402

cfg = int(sys.argv[1])
restrict = len(sys.argv) > 2 and sys.argv[2] == "1"
mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
p = eng.preset(cfg)
for kv in sys.argv[4:]:
    k, v = kv.split("=")
    setattr(p, k, int(v))
eng.prepare(p)
ctx = eng.default_context()
L = _abi.lib()
C = _abi.C
de, da = C.c_void_p(), C.c_void_p()
_abi.check(L.cyc_device_alloc(ctx.handle, p.m * 8, C.byref(de)))
_abi.check(L.cyc_device_alloc(ctx.handle, ((p.n + 63) // 64) * 8, C.byref(da)))
t0 = time.perf_counter()
_abi.check(L.cyc_gen_fill(ctx.handle, C.byref(p), de, da))
print(f"config {cfg}: n={p.n} m_log={p.m} generated in {time.perf_counter()-t0:.2f}s", flush=True)
for early in (True, False):
    opt = eng.MapOptions(early_exit=early, mode=mode, push_alpha=int(os.environ.get("ALPHA", "0"))).to_c()
    for rep in range(int(os.environ.get("REPS", "2"))):
        st = _abi.MapStatsC()
        ms = (C.c_double * 4)()
        t0 = time.perf_counter()
        _abi.check(L.cyc_check(ctx.handle, C.cast(de, C.POINTER(C.c_uint32)), p.m, p.n,
                               C.cast(da, C.POINTER(C.c_uint64)), 1, int(restrict), C.byref(opt),
                               C.byref(st), ms))
        wall = (time.perf_counter() - t0) * 1e3
        d = eng.api.stats_dict(st)
        if rep == int(os.environ.get("REPS", "2")) - 1 or os.environ.get("ALL_REPS"):
            print(json.dumps({"early_exit": early, "restrict": restrict, "wall_ms": round(wall, 2),
                              "phase_ms": [round(x, 2) for x in ms], "cycle": d["cycle_found"],
                              "witness": d["witness"], "iterations": d["iterations"],
                              "kernel_calls": d["kernel_calls"], "pull": d["pull_steps"],
                              "push": d["push_steps"], "loop_ms": round(d["loop_ms"], 3)}), flush=True)
