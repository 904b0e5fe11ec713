#!/usr/bin/env python3
"""MAP propagation GTEPS and time-to-verdict on B200 (BASELINE.json metric).

Workload (N=1 headline): config 2 of BASELINE.json — the 2^22-vertex layered
DAG of SCCs (L=64 layers, W=4096 rings of S=16 per layer, accepting
connectors; include/cyc_gen.h) run through run_map with early_exit, no SCC
restriction (restriction keeps 0 vertices on this family). It
forces L+1 = 65 MAP iterations and (L+1)^2 = 4225 propagation steps.

One bench "step" = one full run_map to verdict over the device-resident
snapshot (value) / one cyc_check call from a pinned host edge log through
H2D + CSR build + run_map (e2e). GTEPS = m x kernel_calls / time.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  N>1 under torchrun: independent replicas.
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


def make_params(eng, args):
    p = eng.preset(args.config)
    for k in ("L", "W", "S", "scale", "edgefactor"):
        v = getattr(args, k, None)
        if v:
            setattr(p, k, v)
    if args.n_override:
        p.n = args.n_override
    return eng.prepare(p)


def load_traffic():
    """dram bytes per k_map_run launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_map_run_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("traffic_bytes_per_launch"), d.get("source")
    except Exception:
        return None, None


# ------------------------------------------------------------- reference arm
_REF_SNAP = {}


def cpu_reference_sample(params, seconds: float, workers: int):
    """Times the reference's own MaxPropagation::step (WorkerPool of `workers`
    threads) on the same seeded graph: first Jacobi steps of MAP iteration 1,
    bounded to `seconds`. Returns (gteps, steps, step_seconds, m, info)."""
    import oracle

    key = bytes(params)
    if key not in _REF_SNAP:
        ref = oracle.Reference()
        t0 = time.perf_counter()
        _REF_SNAP[key] = (ref.snapshot_gen(params, True), time.perf_counter() - t0)
    snap, t_snap = _REF_SNAP[key]
    gather_s, steps_s, k = snap.time_steps(workers, 1 << 40, seconds)
    gteps = snap.m * k / steps_s / 1e9 if steps_s > 0 else 0.0
    return gteps, k, steps_s, snap.m, {"gather_build_s": round(gather_s, 3),
                                       "log_fill_plus_build_snapshot_s": round(t_snap, 3)}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    import paper_0912_2555_b200 as eng

    params = make_params(eng, args)
    import oracle

    workers = os.cpu_count() or 1
    vals = []
    info = None
    m = 0
    # each bench step is one bounded sample of propagation steps
    for i in range(args.warmup + args.steps):
        g, k, secs, m, info = cpu_reference_sample(params, args.ref_seconds, workers)
        if i >= args.warmup:
            vals.append((g, k, secs))
    gteps = statistics.median(v[0] for v in vals)
    sample = (f"config {args.config}: first {vals[0][1]} Jacobi steps of MAP iteration 1 "
              f"(MaxPropagation::step, WorkerPool({workers})) per step, ~{args.ref_seconds}s each")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gteps, 5), "unit": "GTEPS",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * statistics.median(v[2] for v in vals), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded include/cyc_gen.h)",
        "config": {"workload": f"config{args.config}", "n": int(params.n), "m_log": int(params.m),
                   "m": int(m), "parallelism": "cpu-threads"},
        "cpu_baseline": {"value": round(gteps, 5), "unit": "GTEPS", "cores": workers,
                         "kind": "reference", "sample": sample, **(info or {})},
        "e2e": {"value": round(gteps, 5), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------- B200 arm
def run_b200(args, rank, world, local):
    import numpy as np

    import paper_0912_2555_b200 as eng
    from paper_0912_2555_b200 import _abi

    dist = init_dist(world, local, "nccl")
    device = None
    if dist is not None:
        import torch

        device = torch.device("cuda", local)
    ctx = eng.Context(local)
    L = _abi.lib()
    params = make_params(eng, args)
    n, m_log = int(params.n), int(params.m)
    # device-resident input (value) and pinned host input (e2e)
    d_edges, d_acc = C.c_void_p(), C.c_void_p()
    _abi.check(L.cyc_device_alloc(ctx.handle, m_log * 8, C.byref(d_edges)))
    _abi.check(L.cyc_device_alloc(ctx.handle, ((n + 63) // 64) * 8, C.byref(d_acc)))
    _abi.check(L.cyc_gen_fill(ctx.handle, C.byref(params), d_edges, d_acc))
    h_edges, h_acc = C.c_void_p(), C.c_void_p()
    _abi.check(L.cyc_host_alloc(m_log * 8, C.byref(h_edges)))
    _abi.check(L.cyc_host_alloc(((n + 63) // 64) * 8, C.byref(h_acc)))
    _abi.check(L.cyc_memcpy(ctx.handle, h_edges, d_edges, m_log * 8))
    _abi.check(L.cyc_memcpy(ctx.handle, h_acc, d_acc, ((n + 63) // 64) * 8))

    orient = _abi.CYC_TRANSPOSED
    g = C.c_void_p()
    t0 = time.perf_counter()
    _abi.check(L.cyc_graph_build(ctx.handle, C.cast(d_edges, C.POINTER(C.c_uint32)), m_log, n,
                                 C.cast(d_acc, C.POINTER(C.c_uint64)), orient, C.byref(g)))
    build_ms_first = (time.perf_counter() - t0) * 1e3
    snap = eng.CsrSnapshot(g, ctx)
    m = snap.m
    opt = eng.MapOptions(early_exit=True, mode=args.mode).to_c()
    st = _abi.MapStatsC()

    def one_run():
        _abi.check(L.cyc_flush_l2(ctx.handle, L2_FLUSH_BYTES))
        _abi.check(L.cyc_map_run(ctx.handle, g, None, C.byref(opt), C.byref(st), None, None, None, 0))
        return float(st.loop_ms)

    for _ in range(args.warmup):
        one_run()
    barrier(dist, device)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = eng.launch_count()
    loop_ms = []
    for _ in range(args.steps):
        loop_ms.append(one_run())
    _abi.check(L.cyc_ctx_synchronize(ctx.handle))
    launches = eng.launch_count() - launches0
    barrier(dist, device)
    stats = _abi.MapStatsC.from_buffer_copy(st)
    total_ms = max_over_ranks(dist, sum(loop_ms), device)
    ms_per_step = total_ms / args.steps
    kernel_calls = int(stats.kernel_calls)
    value = world * m * kernel_calls / (ms_per_step * 1e-3) / 1e9

    # device-resident time to verdict: CSR build from the resident log + run_map
    ttv = []
    for _ in range(max(1, min(args.steps, 5))):
        _abi.check(L.cyc_flush_l2(ctx.handle, L2_FLUSH_BYTES))
        _abi.check(L.cyc_ctx_synchronize(ctx.handle))
        ms = (C.c_double * 4)()
        s2 = _abi.MapStatsC()
        _abi.check(L.cyc_check(ctx.handle, C.cast(d_edges, C.POINTER(C.c_uint32)), m_log, n,
                               C.cast(d_acc, C.POINTER(C.c_uint64)), orient, 0, C.byref(opt),
                               C.byref(s2), ms))
        ttv.append(list(ms))
    # e2e: pinned host log -> verdict through the C ABI (H2D inside)
    e2e = []
    for _ in range(max(1, min(args.steps, 5))):
        _abi.check(L.cyc_flush_l2(ctx.handle, L2_FLUSH_BYTES))
        _abi.check(L.cyc_ctx_synchronize(ctx.handle))
        ms = (C.c_double * 4)()
        s3 = _abi.MapStatsC()
        t0 = time.perf_counter()
        _abi.check(L.cyc_check(ctx.handle, C.cast(h_edges, C.POINTER(C.c_uint32)), m_log, n,
                               C.cast(h_acc, C.POINTER(C.c_uint64)), orient, 0, C.byref(opt),
                               C.byref(s3), ms))
        e2e.append((time.perf_counter() - t0) * 1e3)
        assert (s3.cycle_found, s3.kernel_calls) == (stats.cycle_found, stats.kernel_calls)
    clk = clocks.stop()
    e2e_ms = max_over_ranks(dist, statistics.median(e2e), device)
    ttv_ms = max_over_ranks(dist, statistics.median(t[3] for t in ttv), device)
    e2e_value = world * m * kernel_calls / (e2e_ms * 1e-3) / 1e9

    peak, peak_src = peaks()
    loop_s = statistics.median(loop_ms) * 1e-3
    achieved = stats.algorithmic_bytes / loop_s / 1e9 if loop_s > 0 else 0.0
    traffic, traffic_src = load_traffic()
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded include/cyc_gen.h, generated on device)",
        "config": {"workload": f"config{args.config}: layered DAG of SCCs, L={params.L} W={params.W} "
                               f"S={params.S}" if args.config in (2, 5) else f"config{args.config}",
                   "n": n, "m_log": m_log, "m": m, "orientation": "transposed",
                   "early_exit": True, "scc_restriction": False, "mode": args.mode,
                   "parallelism": f"replicas{world}" if world > 1 else "single",
                   "l2": f"flushed ({L2_FLUSH_BYTES >> 20} MiB write) before every timed step"},
        "verdict": {"cycle_found": bool(stats.cycle_found), "iterations": int(stats.iterations),
                    "kernel_calls": kernel_calls, "demoted_total": int(stats.demoted_total)},
        "time_to_verdict_ms": {"device_resident": round(ttv_ms, 3), "e2e_host": round(e2e_ms, 3),
                               "build_ms": round(statistics.median(t[0] for t in ttv), 3),
                               "loop_ms": round(statistics.median(loop_ms), 3)},
        "steps_detail": {"pull_steps": int(stats.pull_steps), "push_steps": int(stats.push_steps),
                         "edges_touched": int(stats.edges_touched), "rows_touched": int(stats.rows_touched),
                         "grid": [int(stats.grid_blocks), int(stats.block_threads)]},
        "e2e": {"value": round(e2e_value, 3), "unit": "GTEPS", "h2d_bytes_per_step": m_log * 8 + ((n + 63) // 64) * 8,
                "d2h_bytes_per_step": C.sizeof(_abi.MapStatsC)},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "k_map_run (persistent, one launch per run_map)",
                     "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": int(stats.algorithmic_bytes),
                     "traffic": traffic, "traffic_source": traffic_src},
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            g_cpu, k, secs, m_ref, info = cpu_reference_sample(params, args.ref_seconds, os.cpu_count() or 1)
            line["cpu_baseline"] = {"value": round(g_cpu, 5), "unit": "GTEPS", "cores": os.cpu_count(),
                                    "kind": "reference",
                                    "sample": f"first {k} Jacobi steps of MAP iteration 1 of the same "
                                              f"graph, reference MaxPropagation::step with "
                                              f"WorkerPool({os.cpu_count()}), {secs:.1f}s", **info}
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
    """One graph, rows sharded over the ranks (paper_0912_2555_b200/sharded.py)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_0912_2555_b200 as eng
    from paper_0912_2555_b200 import _abi, sharded

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", rank=rank, world_size=world)
    ctx = eng.Context(local)
    params = make_params(eng, args)
    n, m_log = int(params.n), int(params.m)
    e = np.zeros((m_log, 2), np.uint32)
    a = np.zeros((n + 63) // 64, np.uint64)
    _abi.check(_abi.lib().cyc_gen_fill(ctx.handle, C.byref(params), _abi.ptr(e), _abi.ptr(a)))
    snap = eng.build_snapshot((n, e, eng.Bitset.from_words(a, n)), ctx=ctx)
    off, _ = snap.gather_index()
    bounds = sharded.plan(off, world)
    words = snap.accepting.words().copy()
    if args.fused:  # exchange fused into the step kernel over peer memory
        fs = sharded.FusedShard(snap, dist, rank, world, bounds)
        run = lambda: fs.run(words, True)  # noqa: E731
    else:
        be = sharded.CudaShardBackend(snap, device)
        run = lambda: sharded.run_map_sharded(be, dist, rank, world, bounds, words, True,  # noqa: E731
                                              exchange=args.exchange)
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        _abi.check(_abi.lib().cyc_flush_l2(ctx.handle, L2_FLUSH_BYTES))
        dist.barrier(device_ids=[local])
        torch.cuda.synchronize(device)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        res = run()
        t1.record()
        torch.cuda.synchronize(device)
        times.append(t0.elapsed_time(t1))
    ms = max_over_ranks(dist, sum(times) / len(times), device)
    m = snap.m
    value = m * res.stats.kernel_calls / (ms * 1e-3) / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": round(value, 3), "unit": "GTEPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded include/cyc_gen.h)",
            "config": {"workload": f"config{args.config}", "n": n, "m": m,
                       "parallelism": f"rowshard{world}",
                       "exchange": ("fused: peer-memory stores in the step kernel + system-scope barrier"
                                    if args.fused else f"nccl ({args.exchange}): allgather + allreduce per step")},
            "verdict": {"cycle_found": res.verdict.cycle_found(), "iterations": res.stats.iterations,
                        "kernel_calls": res.stats.kernel_calls}}))
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--mode", default="auto", choices=["auto", "pull", "push"])
    ap.add_argument("--L", type=int, default=0)
    ap.add_argument("--W", type=int, default=0)
    ap.add_argument("--S", type=int, default=0)
    ap.add_argument("--scale", type=int, default=0)
    ap.add_argument("--edgefactor", type=int, default=0)
    ap.add_argument("--n-override", type=int, default=0)
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fused", action="store_true",
                    help="with --sharded: exchange fused into the step kernel (peer memory) instead of NCCL")
    ap.add_argument("--exchange", default="dense", choices=["dense", "sparse", "auto"],
                    help="with --sharded (NCCL): dense slices, changed-only pairs, or auto")
    ap.add_argument("--sharded", action="store_true",
                    help="N>1: row-shard one graph over the ranks (NCCL exchange per step) "
                         "instead of independent replicas")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)
    if args.sharded:
        return run_b200_sharded(args, rank, world, local)
    return run_b200(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
