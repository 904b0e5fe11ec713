#!/usr/bin/env python3
"""MAP propagation GTEPS and time-to-verdict on B200 (BASELINE.json metric).

Workload (N=1 headline): BASELINE config 3 — R-MAT (Graph500 .57/.19/.19)
scale 26, edgefactor 16 (2^30 logged edges, 1.06 G snapshot edges after
dedup), 1 % accepting, seeded vertex permutation (include/cyc_gen.h),
transposed snapshot, no restriction:

* value (steady state): run_map with early_exit off on the device-resident
  snapshot — the reference's `MaxPropagation::step` loop to fixpoint
  (map_engine.cpp:94-121, 8 Jacobi steps on this graph). One bench step = one
  run_map; GTEPS = m x kernel_calls / device time of the loop kernel.
* e2e: the same metric through the C ABI from a pinned HOST edge log
  (cyc_check: H2D + both CSRs + run_map in id order + stats D2H).
* time_to_verdict_ms: early_exit on (the `cycheck graph` default), device-
  resident and from host memory, plus the first (cold) call of the process.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--sharded]
  N>1 under torchrun: ONE graph row-sharded over the ranks (strong scaling,
  csrc/shard.cu); --sharded runs that path at N=1 too.

The reference arm (--impl reference) never loads the engine: it times the
reference's own MaxPropagation::step with WorkerPool(nproc) on the same graph
(built for it by a parallel setup builder equal to build_snapshot) and prints
the same metric/config; see run_reference_arm.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MAP propagation GTEPS and time-to-verdict at 1/2/4/8 B200 vs CPU ref"
L2_FLUSH_BYTES = 512 << 20
REF_TTV_FILE = os.path.join(ROOT, "profiles", "r02_ref_ttv_c3.json")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world, local, backend):
    if world <= 1:
        return None
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend == "nccl":
        import torch

        torch.cuda.set_device(local)
    dist.init_process_group(backend=backend)
    return dist


def max_over_ranks(dist, x: float, device=None) -> float:
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist, device=None):
    if dist is not None:
        if device is not None:
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() in ("active", "1"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def gen_params(args, reference: bool = False):
    """Generator parameters of include/cyc_gen.h: the engine's presets for the
    B200 arm, the oracle's own mirror for the reference arm (which must never
    load the engine library). Both come from the same header."""
    if reference:
        import oracle

        src = oracle.Restatement()
    else:
        import paper_0912_2555_b200 as src
    p = src.preset(args.config)
    for k in ("L", "W", "S", "scale", "edgefactor"):
        v = getattr(args, k, None)
        if v:
            setattr(p, k, v)
    return src.prepare(p)


WORKLOADS = {
    1: "config1: uniform random digraph 2^16 x 4, 5% accepting",
    2: "config2: layered DAG of SCCs 2^22 (L=64 W=4096 S=16), accepting connectors",
    3: "config3: R-MAT scale 26 edgefactor 16 (a,b,c=.57,.19,.19), 1% accepting",
    4: "config4: product graph 2^13 x 2^13 torus x 4-state Buchi, 2^28 states",
    5: "config5: chain of SCCs 2^24 (L=64 W=512 S=512), sink accepting",
}


def bench_config(args, p):
    """The `config` dict, identical in both arms (a function of the arguments only)."""
    return {"workload": WORKLOADS.get(args.config, f"config{args.config}"), "n": int(p.n), "m_log": int(p.m),
            "orientation": "transposed", "early_exit": False, "scc_restriction": False,
            "step": "one run_map to fixpoint (MaxPropagation::step loop)", "gteps": "m x kernel_calls / time"}


def load_traffic():
    """dram bytes per k_map_run launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_map_run_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("traffic_bytes_per_launch"), d.get("source")
    except Exception:
        return None, None


def recorded_ref_ttv():
    try:
        with open(REF_TTV_FILE) as f:
            return json.load(f)
    except Exception:
        return None


# ------------------------------------------------------------- reference arm
_REF_SNAP = {}


def cpu_reference_sample(params, seconds: float, workers: int):
    """The reference's own MaxPropagation (gather-index build, map_engine.cpp:
    9-19, then Jacobi steps from all-NIL, map_engine.cpp:21-79) with a
    WorkerPool of `workers` threads on the same seeded graph, bounded to
    `seconds` of steps. The CsrSnapshot it runs on comes from the parallel
    setup builder (oracle ref_snapshot_gen_fast, equal to build_snapshot by
    tests/test_oracle.py) — setup, not timed. Returns (gteps, steps, step_s, m, info)."""
    import oracle

    key = bytes(params)
    if key not in _REF_SNAP:
        ref = oracle.Reference()
        t0 = time.perf_counter()
        _REF_SNAP[key] = (ref.snapshot_gen_fast(params, True), time.perf_counter() - t0)
    snap, t_snap = _REF_SNAP[key]
    gather_s, steps_s, k = snap.time_steps(workers, 1 << 40, seconds)
    gteps = snap.m * k / steps_s / 1e9 if steps_s > 0 else 0.0
    return gteps, k, steps_s, snap.m, {"gather_build_s": round(gather_s, 3),
                                       "setup_snapshot_s": round(t_snap, 3)}


def ref_live(params, args, workers, samples):
    """The reference's CPU numbers measured in THIS run on this host: the W=1
    step rate (one bounded sample), the spread of the W=nproc samples, and
    its run_map part of the time to verdict (gather-index build + the early-
    exit step count at the measured step time) beside the recorded one."""
    g1, k1, s1, _, _ = cpu_reference_sample(params, max(1.0, args.ref_seconds / 2), 1)
    rates = [v[0] for v in samples]
    step_s = statistics.median(v[2] / max(v[1], 1) for v in samples)
    out = {"w1_gteps": round(g1, 5), "w1_steps": k1, "wn_gteps_min": round(min(rates), 5),
           "wn_gteps_max": round(max(rates), 5), "wn_samples": len(rates), "wn_step_s": round(step_s, 4)}
    rec = recorded_ref_ttv()
    if rec and rec.get("config") == args.config and (rec.get("n"), rec.get("m_log")) == (int(params.n), int(params.m)):
        kc = rec["stats"][str(workers)][3] if str(workers) in rec["stats"] else rec["stats"]["1"][3]
        out["run_map_s_live_estimate"] = round(samples[0][3] + kc * step_s, 3)
        out["ttv_s_live_estimate"] = round(rec["build_snapshot_s"] + out["run_map_s_live_estimate"], 3)
    return out


def ref_ttv_summary(args, params):
    """CPU time to verdict (early exit) of the reference, phase by phase
    (cycheck_main.cpp:88-97: csr = build_snapshot, kernel = run_map incl. its
    gather-index build) at W=1 and W=nproc. A full config-3 run takes ~10
    minutes of host time, too long for every bench call, so it is RECORDED by
    scripts/ref_ttv.py on a GPU box host (same oracle/_ref build) and quoted
    from profiles/r02_ref_ttv_c3.json; None for other configs."""
    rec = recorded_ref_ttv()
    if not rec or rec.get("config") != args.config or (rec.get("n"), rec.get("m_log")) != (int(params.n), int(params.m)):
        return None
    return {"recorded": os.path.relpath(REF_TTV_FILE, ROOT), "cpu_model": rec.get("cpu_model"),
            "nproc": rec.get("nproc"), "build_snapshot_s": rec.get("build_snapshot_s"),
            "log_fill_s": rec.get("log_fill_s"), "run_map_s_by_workers": rec.get("run_map_s"),
            "ttv_s_by_workers": {w: round(rec["build_snapshot_s"] + t, 3) for w, t in rec["run_map_s"].items()},
            "verdict_by_workers": rec.get("stats")}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    import oracle

    params = gen_params(args, reference=True)
    workers = os.cpu_count() or 1
    vals = []
    info = None
    m = 0
    for i in range(args.warmup + args.steps):
        g, k, secs, m, info = cpu_reference_sample(params, args.ref_seconds, workers)
        if i >= args.warmup:
            vals.append((g, k, secs, info["gather_build_s"]))
    gteps = statistics.median(v[0] for v in vals)
    live = ref_live(params, args, workers, vals)
    sample = (f"{WORKLOADS.get(args.config)}: reference MaxPropagation::step with WorkerPool({workers}), "
              f"Jacobi steps of the first fixpoint from all-NIL (restarted at the fixpoint), "
              f"~{args.ref_seconds}s per bench step ({vals[0][1]} steps)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gteps, 5), "unit": "GTEPS",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * statistics.median(v[2] for v in vals), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded include/cyc_gen.h)",
        "config": bench_config(args, params),
        "cpu_baseline": {"value": round(gteps, 5), "unit": "GTEPS", "cores": workers, "kind": "reference",
                         "sample": sample, "cpu_model": cpu_model(), "nproc": os.cpu_count(), **(info or {}),
                         "live": live, "time_to_verdict": ref_ttv_summary(args, params)},
        "e2e": {"value": round(gteps, 5), "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    # the reference arm must not have mapped the engine library
    assert "paper_0912_2555_b200" not in sys.modules
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------- B200 arm
def run_b200(args, rank, world, local):
    import paper_0912_2555_b200 as eng
    from paper_0912_2555_b200 import _abi

    dist = init_dist(world, local, "nccl")
    device = None
    if dist is not None:
        import torch

        device = torch.device("cuda", local)
    ctx = eng.Context(local)
    L = _abi.lib()
    params = gen_params(args)
    n, m_log = int(params.n), int(params.m)
    nw64 = (n + 63) // 64
    # map the build's pool memory on a library thread while the log is
    # generated and staged (cyc_ctx_reserve); the wait left is timed below
    if not args.no_reserve:
        ctx.reserve(m_log, n, background=True)
    # device-resident input (value, TTV) and a pinned host copy (e2e)
    d_edges, d_acc = C.c_void_p(), C.c_void_p()
    _abi.check(L.cyc_device_alloc(ctx.handle, m_log * 8, C.byref(d_edges)))
    _abi.check(L.cyc_device_alloc(ctx.handle, nw64 * 8, C.byref(d_acc)))
    _abi.check(L.cyc_gen_fill(ctx.handle, C.byref(params), d_edges, d_acc))
    h_edges, h_acc = C.c_void_p(), C.c_void_p()
    _abi.check(L.cyc_host_alloc(m_log * 8, C.byref(h_edges)))
    _abi.check(L.cyc_host_alloc(nw64 * 8, C.byref(h_acc)))
    _abi.check(L.cyc_memcpy(ctx.handle, h_edges, d_edges, m_log * 8))
    _abi.check(L.cyc_memcpy(ctx.handle, h_acc, d_acc, nw64 * 8))
    _abi.check(L.cyc_ctx_synchronize(ctx.handle))
    u32p, u64p = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
    orient = _abi.CYC_TRANSPOSED
    ttv_opt = eng.MapOptions(early_exit=True, mode=args.mode).to_c()
    full_opt = eng.MapOptions(early_exit=False, mode=args.mode).to_c()

    def check_call(edges, acc, opt):
        st, ms = _abi.MapStatsC(), (C.c_double * 4)()
        _abi.check(L.cyc_flush_l2(ctx.handle, L2_FLUSH_BYTES))
        _abi.check(L.cyc_ctx_synchronize(ctx.handle))
        t0 = time.perf_counter()
        _abi.check(L.cyc_check(ctx.handle, C.cast(edges, u32p), m_log, n, C.cast(acc, u64p), orient, 0,
                               C.byref(opt), C.byref(st), ms))
        return (time.perf_counter() - t0) * 1e3, list(ms), st

    # the first call of the process (cold TTV): whatever the background
    # reserve has not finished yet, then the call's own first touches
    t0 = time.perf_counter()
    ctx.reserve(0, 0, background=False)  # joins the reserve thread
    reserve_wait_ms = (time.perf_counter() - t0) * 1e3
    cold_ms, cold_phases, cold_st = check_call(h_edges, h_acc, ttv_opt)

    g = C.c_void_p()
    _abi.check(L.cyc_graph_build(ctx.handle, C.cast(d_edges, u32p), m_log, n, C.cast(d_acc, u64p), orient,
                                 C.byref(g)))
    snap = eng.CsrSnapshot(g, ctx)
    m = snap.m
    st = _abi.MapStatsC()

    def one_run():
        _abi.check(L.cyc_flush_l2(ctx.handle, L2_FLUSH_BYTES))
        _abi.check(L.cyc_map_run(ctx.handle, g, None, C.byref(full_opt), C.byref(st), None, None, None, 0))
        return float(st.loop_ms)

    one_run()  # auto layout: a graph's first loop runs in id order ...
    one_run()  # ... and the second builds the storage plan (cached on the snapshot)
    plan_ms = float(st.plan_ms)
    for _ in range(args.warmup):
        one_run()
    barrier(dist, device)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = eng.launch_count()
    loop_ms = [one_run() for _ in range(args.steps)]
    _abi.check(L.cyc_ctx_synchronize(ctx.handle))
    launches = eng.launch_count() - launches0
    barrier(dist, device)
    stats = _abi.MapStatsC.from_buffer_copy(st)
    total_ms = max_over_ranks(dist, sum(loop_ms), device)
    ms_per_step = total_ms / args.steps
    kernel_calls = int(stats.kernel_calls)
    value = world * m * kernel_calls / (ms_per_step * 1e-3) / 1e9

    reps = max(1, min(args.steps, 5))
    # time to verdict (early exit): device-resident log and pinned host log
    ttv_dev = [check_call(d_edges, d_acc, ttv_opt) for _ in range(reps)]
    ttv_host = [check_call(h_edges, h_acc, ttv_opt) for _ in range(reps)]
    # e2e of the headline metric: host log -> steady-state verdict through the C ABI
    e2e = [check_call(h_edges, h_acc, full_opt) for _ in range(reps)]
    clk = clocks.stop()
    for _, _, s3 in e2e:
        assert (s3.cycle_found, s3.kernel_calls) == (stats.cycle_found, stats.kernel_calls)
    e2e_ms = max_over_ranks(dist, statistics.median(x[0] for x in e2e), device)
    e2e_value = world * m * kernel_calls / (e2e_ms * 1e-3) / 1e9
    ttv_st = ttv_dev[0][2]

    peak, peak_src = peaks()
    loop_s = statistics.median(loop_ms) * 1e-3
    achieved = stats.algorithmic_bytes / loop_s / 1e9 if loop_s > 0 else 0.0
    traffic, traffic_src = load_traffic()
    med = lambda xs: round(statistics.median(xs), 3)  # noqa: E731
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded include/cyc_gen.h, generated on device)",
        "config": bench_config(args, params),
        "setup": {"m": m, "mode": args.mode, "layout": "degree" if stats.layout == 2 else "identity",
                  "parallelism": f"replicas{world}" if world > 1 else "single",
                  "l2": f"flushed ({L2_FLUSH_BYTES >> 20} MiB write) before every timed call",
                  "grid": [int(stats.grid_blocks), int(stats.block_threads)]},
        "verdict": {"cycle_found": bool(stats.cycle_found), "witness": int(stats.witness),
                    "iterations": int(stats.iterations), "kernel_calls": kernel_calls,
                    "demoted_total": int(stats.demoted_total)},
        "time_to_verdict_ms": {
            "early_exit": True, "cycle_found": bool(ttv_st.cycle_found), "witness": int(ttv_st.witness),
            "kernel_calls": int(ttv_st.kernel_calls),
            "device_resident": med([x[0] for x in ttv_dev]),
            "device_resident_phases": {"build": med([x[1][0] for x in ttv_dev]),
                                       "plan_plus_loop": med([x[1][2] for x in ttv_dev])},
            "e2e_host": med([x[0] for x in ttv_host]),
            "cold_first_call_e2e_host": round(cold_ms, 3),
            "cold_reserve": {"used": not args.no_reserve, "wait_ms": round(reserve_wait_ms, 3),
                             "what": "build memory allocated by cyc_ctx_reserve on a library thread from context "
                                     "creation on, overlapping log generation and staging; wait_ms = what was "
                                     "left when the first call started (cold TTV = wait_ms + the call)"},
            "steady_state_plan_build_ms": round(plan_ms, 3)},
        "steps_detail": {"pull_steps": int(stats.pull_steps), "push_steps": int(stats.push_steps),
                         "edges_touched": int(stats.edges_touched), "rows_touched": int(stats.rows_touched)},
        "e2e": {"value": round(e2e_value, 3), "unit": "GTEPS", "ms": round(e2e_ms, 3),
                "h2d_bytes_per_step": m_log * 8 + nw64 * 8, "d2h_bytes_per_step": C.sizeof(_abi.MapStatsC),
                "what": "cyc_check from a pinned host edge log: H2D + both CSRs + run_map (early_exit off; "
                        "a one-shot call runs its loop in id order, auto layout) + stats D2H"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "k_map_run (persistent, one launch per run_map)",
                     "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": int(stats.algorithmic_bytes),
                     "bytes_model": "sum over steps of 8*E_s + 12*V_s (pull: E=m, V=n; push: touched)",
                     "traffic": traffic, "traffic_source": traffic_src},
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            workers = os.cpu_count() or 1
            rp = gen_params(args, reference=True)
            g_cpu, k, secs, m_ref, info = cpu_reference_sample(rp, args.ref_seconds, workers)
            assert m_ref == m
            live = ref_live(rp, args, workers, [(g_cpu, k, secs, info["gather_build_s"])])
            line["cpu_baseline"] = {
                "value": round(g_cpu, 5), "unit": "GTEPS", "cores": workers, "kind": "reference",
                "cpu_model": cpu_model(),
                "sample": f"reference MaxPropagation::step, WorkerPool({workers}), {k} Jacobi steps of the "
                          f"first fixpoint of the same graph in {secs:.1f}s", **info, "live": live,
                "time_to_verdict": ref_ttv_summary(args, rp)}
        except Exception as ex:  # reference build missing on this box
            line["cpu_baseline"] = {"value": None, "unit": "GTEPS", "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"unavailable: {ex}"}
    if rank == 0:
        print(json.dumps(line))
    snap.close()
    for p in (d_edges, d_acc):
        L.cyc_device_free(ctx.handle, p)
    for p in (h_edges, h_acc):
        L.cyc_host_free(p)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def run_b200_sharded(args, rank, world, local):
    """One graph, rows sharded over the ranks (csrc/shard.cu, cyc_shard_*): every
    rank generates the log on its device, keeps only its own rows (~1/N of the
    edges) and runs ONE persistent kernel that stores the rows it changes into
    every peer's replicated vector over NVLink peer memory and meets the other
    ranks at a system-scope barrier per step (no collective per step).
    torch.distributed only carries the IPC handle blobs and the timings."""
    import torch
    import torch.distributed as dist

    import paper_0912_2555_b200 as eng
    from paper_0912_2555_b200 import _abi
    from paper_0912_2555_b200.sharded import MapShard, exchange_handles

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    ddist = None
    gloo = None
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=device)
        gloo = dist.new_group(backend="gloo")
        ddist = dist
    ctx = eng.Context(local)
    L = _abi.lib()
    params = gen_params(args)
    n, m_log = int(params.n), int(params.m)
    nw64 = (n + 63) // 64
    d_edges, d_acc = C.c_void_p(), C.c_void_p()
    _abi.check(L.cyc_device_alloc(ctx.handle, m_log * 8, C.byref(d_edges)))
    _abi.check(L.cyc_device_alloc(ctx.handle, nw64 * 8, C.byref(d_acc)))
    _abi.check(L.cyc_gen_fill(ctx.handle, C.byref(params), d_edges, d_acc))
    _abi.check(L.cyc_ctx_synchronize(ctx.handle))

    def build(edges, acc):
        t0 = time.perf_counter()
        sh = MapShard(ctx, edges.value, m_log, n, acc.value, world, rank, layout="auto")
        blob = exchange_handles(ddist, sh.handle(), world, gloo) if world > 1 else sh.handle()
        sh.connect(blob)
        _abi.check(L.cyc_ctx_synchronize(ctx.handle))
        ms = (time.perf_counter() - t0) * 1e3
        if world > 1:
            dist.barrier(group=gloo)  # every rank connected before anyone runs
        return sh, ms

    def close(sh):  # peers may have our buffers mapped: everyone done before anyone frees
        if world > 1:
            dist.barrier(group=gloo)
        sh.close()
        if world > 1:
            dist.barrier(group=gloo)

    def run(sh, early):
        _abi.check(L.cyc_flush_l2(ctx.handle, L2_FLUSH_BYTES))
        _abi.check(L.cyc_ctx_synchronize(ctx.handle))
        if world > 1:
            dist.barrier(group=gloo)
        r = MapShard.run_map([sh], early_exit=early, mode=args.mode, want_values=False, hash_cap=0)
        return r, float(r.stats.device["loop_ms"])

    sh, build_ms = build(d_edges, d_acc)
    info = sh.info()
    for _ in range(args.warmup):
        run(sh, False)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = eng.launch_count()
    loop_ms = []
    for _ in range(args.steps):
        res, ms = run(sh, False)
        loop_ms.append(ms)
    launches = eng.launch_count() - launches0
    total_ms = max_over_ranks(ddist, sum(loop_ms), device)
    ms_per_step = total_ms / args.steps
    st = res.stats.device
    m = int(sum_over_ranks(ddist, info["local_edges"], device))
    kernel_calls = int(st["kernel_calls"])
    value = m * kernel_calls / (ms_per_step * 1e-3) / 1e9
    # time to verdict (early exit), device-resident log: shard build + run
    ttv = []
    for _ in range(max(1, min(args.steps, 3))):
        close(sh)
        sh, bms = build(d_edges, d_acc)
        r2, ms2 = run(sh, True)
        ttv.append((bms + ms2, bms, ms2, r2))
    ttv_ms = max_over_ranks(ddist, statistics.median(x[0] for x in ttv), device)
    # e2e: pinned host log -> shard build (H2D inside) -> steady-state verdict
    h_edges, h_acc = C.c_void_p(), C.c_void_p()
    _abi.check(L.cyc_host_alloc(m_log * 8, C.byref(h_edges)))
    _abi.check(L.cyc_host_alloc(nw64 * 8, C.byref(h_acc)))
    _abi.check(L.cyc_memcpy(ctx.handle, h_edges, d_edges, m_log * 8))
    _abi.check(L.cyc_memcpy(ctx.handle, h_acc, d_acc, nw64 * 8))
    _abi.check(L.cyc_ctx_synchronize(ctx.handle))
    close(sh)
    for p in (d_edges, d_acc):
        L.cyc_device_free(ctx.handle, p)
    e2e = []
    for _ in range(max(1, min(args.steps, 3))):
        if world > 1:
            dist.barrier(group=gloo)
        t0 = time.perf_counter()
        sh, _ = build(h_edges, h_acc)
        r3, _ = run(sh, False)
        e2e.append((time.perf_counter() - t0) * 1e3)
        assert int(r3.stats.kernel_calls) == kernel_calls
        close(sh)
    clk = clocks.stop()
    e2e_ms = max_over_ranks(ddist, statistics.median(e2e), device)
    # NVLink: every changed row goes to each peer (4 B word) with its frontier word (1/32 of a word)
    exch_rows = int(st.get("exchanged_rows", 0))
    nvl_bytes = exch_rows * (world - 1) * (4 + 4 / 32)
    peak, peak_src = peaks()
    loop_s = statistics.median(loop_ms) * 1e-3
    alg = int(st["algorithmic_bytes"])
    achieved = alg / world / loop_s / 1e9 if loop_s > 0 else 0.0
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded include/cyc_gen.h, generated on every rank's device)",
        "config": bench_config(args, params),
        "setup": {"m": m, "mode": args.mode, "layout": "degree" if st.get("layout") == 2 else "identity",
                  "parallelism": f"rowshard{world}",
                  "exchange": "fused: each rank's persistent kernel stores its changed rows into every peer's "
                              "replicated vector (NVLink peer memory) + system-scope barrier per step",
                  "rank0_rows": [info["row_lo"], info["row_hi"]],
                  "per_rank_edges_max": int(max_over_ranks(ddist, info["local_edges"], device)),
                  "per_rank_graph_bytes_max": int(max_over_ranks(ddist, info["device_bytes"], device)),
                  "l2": f"flushed ({L2_FLUSH_BYTES >> 20} MiB write) before every timed call"},
        "verdict": {"cycle_found": bool(res.verdict.cycle_found()), "witness": res.verdict.witness,
                    "iterations": int(st["iterations"]), "kernel_calls": kernel_calls,
                    "demoted_total": int(st["demoted_total"])},
        "time_to_verdict_ms": {"early_exit": True, "device_resident": round(ttv_ms, 3),
                               "shard_build_ms": round(statistics.median(x[1] for x in ttv), 3),
                               "run_ms": round(statistics.median(x[2] for x in ttv), 3),
                               "kernel_calls": int(ttv[0][3].stats.kernel_calls)},
        "e2e": {"value": round(m * kernel_calls / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GTEPS",
                "ms": round(e2e_ms, 3), "h2d_bytes_per_step": m_log * 8 + nw64 * 8,
                "d2h_bytes_per_step": C.sizeof(_abi.MapStatsC),
                "what": "per rank: cyc_shard_build from a pinned host log (H2D inside) + handle exchange + "
                        "cyc_shard_run_map (early_exit off); max over ranks"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "k_map_run<*, sharded> (persistent, one launch per rank per run_map)",
                     "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": alg // world,
                     "bytes_model": "whole-graph 8*E_s + 12*V_s per step divided by the ranks", "traffic": None},
        "nvlink": {"bytes_per_rank_per_run": int(nvl_bytes), "per_step": int(nvl_bytes / max(kernel_calls, 1)),
                   "time_at_770GBps_ms": round(nvl_bytes / 770e9 * 1e3, 4),
                   "frac_of_run": round(nvl_bytes / 770e9 / loop_s, 4) if loop_s > 0 else None,
                   "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction"},
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line))
    for p in (h_edges, h_acc):
        L.cyc_host_free(p)
    if world > 1:
        dist.destroy_process_group()
    return 0


def sum_over_ranks(dist, x: float, device=None) -> float:
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--mode", default="auto", choices=["auto", "pull", "push"])
    ap.add_argument("--L", type=int, default=0)
    ap.add_argument("--W", type=int, default=0)
    ap.add_argument("--S", type=int, default=0)
    ap.add_argument("--scale", type=int, default=0)
    ap.add_argument("--edgefactor", type=int, default=0)
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-reserve", action="store_true",
                    help="do not pre-map the build's pool memory at context creation (cold-call comparison)")
    ap.add_argument("--sharded", action="store_true",
                    help="run the row-sharded engine even at N=1 (N>1 always shards one graph over the ranks)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent replicas of the single-GPU engine instead of one sharded graph")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)
    if args.sharded or (world > 1 and not args.replicas):
        return run_b200_sharded(args, rank, world, local)
    return run_b200(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
