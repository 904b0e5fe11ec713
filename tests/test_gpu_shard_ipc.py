"""GPU: the multi-process plumbing of the row-sharded engine (the bench's
N>1 path) — two processes each build their rank of one graph on the same
GPU, exchange cyc_shard_handle() blobs and connect through CUDA IPC. They do
NOT run: ranks that wait on each other must not share one GPU
(B200_PROFILING.md); the kernel-level exchange is covered by the emulated
ranks of test_gpu_shard_engine.py. Checked here: every rank opens every
peer's buffers, the ranks agree on the graph's edge count, and their rows
split the graph."""
import multiprocessing as mp
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rank(rank, world, conn):
    sys.path.insert(0, ROOT)
    import ctypes as C

    import numpy as np

    import paper_0912_2555_b200 as eng
    from paper_0912_2555_b200.sharded import MapShard

    p = eng.preset(3)
    p.scale = 14
    eng.prepare(p)
    n, m = int(p.n), int(p.m)
    e = np.zeros((m, 2), np.uint32)
    a = np.zeros((n + 63) // 64, np.uint64)
    ctx = eng.default_context()
    eng._abi.check(eng._abi.lib().cyc_gen_fill(ctx.handle, C.byref(p), eng._abi.ptr(e), eng._abi.ptr(a)))
    sh = MapShard(ctx, e, m, n, a, world, rank)
    conn.send(sh.handle())
    blob = conn.recv()
    sh.connect(blob)
    info = sh.info()
    conn.send(info)
    conn.recv()  # every rank connected and reported before anyone frees its buffers
    sh.close()
    conn.close()


def test_two_processes_connect_by_ipc(eng, R):
    world = 2
    ctx = mp.get_context("spawn")
    pipes, procs = [], []
    for r in range(world):
        a, b = ctx.Pipe()
        pr = ctx.Process(target=_rank, args=(r, world, b))
        pr.start()
        pipes.append(a)
        procs.append(pr)
    try:
        handles = [c.recv() for c in pipes]
        assert all(len(h) == eng._abi.SHARD_HANDLE_BYTES for h in handles)
        blob = b"".join(handles)
        for c in pipes:
            c.send(blob)
        infos = [c.recv() for c in pipes]
        for c in pipes:
            c.send(True)
        p = R.preset(3)
        p.scale = 14
        R.prepare(p)
        n, e, _ = R.generate(p)
        m = R.build_snapshot(n, e, True).m
        assert sum(i["local_edges"] for i in infos) == m
        assert infos[0]["row_lo"] == 0 and infos[0]["row_hi"] == infos[1]["row_lo"]
    finally:
        for pr in procs:
            pr.join(timeout=120)
            if pr.is_alive():
                pr.kill()
    assert all(pr.exitcode == 0 for pr in procs)
