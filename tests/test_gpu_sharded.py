"""GPU: the sharded protocol's CUDA backend (row-range step kernel + device
demotion through the C ABI, NCCL collectives, library ordered on torch's
stream) on one rank reproduces run_map exactly; rows are split into several
ranges within the rank to exercise the range kernel."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl():
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_port())
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


def test_cuda_shard_backend_matches_run_map(eng, R, nccl):
    import torch

    from paper_0912_2555_b200 import sharded

    torch.cuda.set_device(0)
    rng = np.random.default_rng(21)
    # the config-2 family: the case that exposed unsynchronised streams
    p = eng.preset(2)
    p.L, p.W, p.S = 8, 64, 8
    eng.prepare(p)
    gn, ge, ga = R.generate(p)
    gsnap = eng.build_snapshot((gn, ge, eng.Bitset.from_words(ga, gn)))
    gbe = sharded.CudaShardBackend(gsnap, torch.device("cuda", 0))
    res = sharded.run_map_sharded(gbe, nccl, 0, 1, [0, gn], ga, True)
    assert (res.stats.iterations, res.stats.kernel_calls, res.stats.demoted_total) == (9, 81, 8)
    gbe.release()
    for t in range(4):
        n = int(rng.integers(500, 20000))
        e = rng.integers(0, n, size=(n * 3, 2)).astype(np.uint32)
        acc = rng.random(n) < [0.01, 0.2][t % 2]
        snap = eng.build_snapshot((n, e, acc))
        words = snap.accepting.words().copy()
        be = sharded.CudaShardBackend(snap, torch.device("cuda", 0))
        off, _ = snap.gather_index()
        for early in (True, False):
            # eager launches and captured CUDA-graph batches, dense / sparse
            # (capacity 7: overflow and dense completion) / auto exchange
            exchange, cap = [("auto", None), ("sparse", None), ("dense", None), ("sparse", 7)][(2 * t + early) % 4]
            res = sharded.run_map_sharded(be, nccl, 0, 1, [0, n], words, early, graphs=bool(t % 2),
                                          exchange=exchange, sparse_cap=cap)
            ref = R.run_map(R.transpose(R.build_snapshot(n, e, True)), words, early)
            got = (res.verdict.cycle_found(), res.verdict.witness, res.stats.iterations,
                   res.stats.kernel_calls, res.stats.demoted_total)
            assert got == (ref.cycle, ref.witness, ref.iterations, ref.kernel_calls, ref.demoted_total)
            assert np.array_equal(res.final_values.cpu().numpy().view(np.uint32), ref.final_x)
        # the row-range kernel over an edge-balanced split equals the full step
        b = sharded.plan(off, 3)
        x = torch.from_numpy(rng.integers(0, n + 1, size=n).astype(np.int32)).cuda()
        accd = be.acc_tensor(words)
        outs, recs = [], []
        for r in range(3):
            o = be.zeros(int(b[r + 1] - b[r]))
            rec = be.zeros(2, torch.int64)
            be.step(x, accd, int(b[r]), int(b[r + 1]), o, rec)
            outs.append(o[: int(b[r + 1] - b[r])].cpu().numpy())
            recs.append(rec.cpu().numpy())
        full, ch, wit = R.step(R.transpose(R.build_snapshot(n, e, True)), x.cpu().numpy().view(np.uint32), words)
        assert np.array_equal(np.concatenate(outs).view(np.uint32), full)
        red = np.max(np.stack(recs), axis=0)
        assert bool(red[0]) == bool(ch)
        assert (0xFFFFFFFF - int(red[1])) == (0xFFFFFFFF if wit is None else wit)
        # a decided fixpoint turns the step into a no-op
        done = be.zeros(4, torch.int64)
        done[0] = 1
        o = be.zeros(n)
        o.fill_(-1)
        be.step(x, accd, 0, n, o, rec, done)
        assert bool((o == -1).all())
        be.release()


def test_fused_shard_matches_run_map(eng, R, nccl):
    """The fused peer-memory exchange path (cyc_fused_*), world 1: the
    persistent kernel with system-scope barriers and IPC-exported buffers
    reproduces run_map (verdict, witness, MapStats, final vector)."""
    from paper_0912_2555_b200 import sharded

    rng = np.random.default_rng(77)
    p = eng.preset(2)
    p.L, p.W, p.S = 8, 64, 8
    eng.prepare(p)
    gn, ge, ga = R.generate(p)
    s = eng.build_snapshot((gn, ge, eng.Bitset.from_words(ga, gn)))
    f = sharded.FusedShard(s, nccl, 0, 1, [0, gn])
    res = f.run(ga, True)
    assert (res.stats.iterations, res.stats.kernel_calls, res.stats.demoted_total) == (9, 81, 8)
    f.close()
    for t in range(4):
        n = int(rng.integers(500, 20000))
        e = rng.integers(0, n, size=(n * 3, 2)).astype(np.uint32)
        acc = rng.random(n) < [0.01, 0.2][t % 2]
        snap = eng.build_snapshot((n, e, acc))
        words = snap.accepting.words().copy()
        f = sharded.FusedShard(snap, nccl, 0, 1, [0, n])
        for early in (True, False):
            for rep in range(2):  # barrier counters carry over between runs
                res = f.run(words, early)
                ref = R.run_map(R.transpose(R.build_snapshot(n, e, True)), words, early)
                got = (res.verdict.cycle_found(), res.verdict.witness, res.stats.iterations,
                       res.stats.kernel_calls, res.stats.demoted_total)
                assert got == (ref.cycle, ref.witness, ref.iterations, ref.kernel_calls, ref.demoted_total)
                assert np.array_equal(res.final_values, ref.final_x)
        f.close()
