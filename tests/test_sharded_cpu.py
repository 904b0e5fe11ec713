"""CPU (gloo, world_size 2 and 3): the row-sharded MAP protocol
(paper_0912_2555_b200/sharded.py) reproduces the single-device run_map —
verdict, witness, MapStats and the final vector — with a host backend doing
each rank's row-range step (oracle restatement, test-only)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class HostShardBackend:
    """Row-range Jacobi step on the host (oracle restatement): test backend
    with the same step / post / demote contract as CudaShardBackend."""

    NONE = 0xFFFFFFFF

    def __init__(self, R, gather, n, snap=None):
        self.torch = torch
        self.R = R
        self.gather = gather
        self.snap = snap if snap is not None else R.transpose(gather)  # push side rows
        self.n = n
        self.bounds = None
        self.raised = []

    def zeros(self, k, dtype=None):
        return torch.zeros(max(k, 1), dtype=dtype or torch.int32)

    def acc_tensor(self, words):
        return torch.from_numpy(words.view(np.int64).copy())

    def prepare(self, bounds):
        self.bounds = [int(b) for b in bounds]

    def step(self, x, acc, lo, hi, out, rec, state=None, first_only=False):
        rec.zero_()
        if state is not None and (int(state[0]) or int(state[4]) or (first_only and int(state[1]))):
            return
        xv = x.numpy().view(np.uint32)[: self.n]
        words = acc.numpy().view(np.uint64)
        full, _, _ = self.R.step(self.gather, xv, words)
        sl = full[lo:hi]
        out[: hi - lo] = torch.from_numpy(sl.view(np.int32).copy())
        accb = np.unpackbits(words.view(np.uint8), bitorder="little")[: self.n].astype(bool)
        ids = np.arange(lo, hi, dtype=np.int64)
        w = ids[(sl.astype(np.int64) == ids + 1) & accb[lo:hi]]
        rec[0] = int(np.any(sl != xv[lo:hi]))
        rec[1] = (self.NONE - int(w.min())) if len(w) else 0

    def post(self, rec, state, x_pad, world, maxrows, x):
        for r in range(world):
            k = self.bounds[r + 1] - self.bounds[r]
            x[self.bounds[r]: self.bounds[r + 1]] = x_pad[r * maxrows: r * maxrows + k]
        if not int(state[0]):
            wit = self.NONE - int(rec[1])
            state[1] += 1
            if (int(state[3]) and wit != self.NONE) or not int(rec[0]):
                state[0] = 1
                state[2] = wit

    def push(self, sp_all, world, cap, acc, lo, hi, out, rbits, rlist, rcnt, state):
        self.raised = []
        if int(state[0]) or int(state[4]) or int(state[1]) == 0:
            return
        words = acc.numpy().view(np.uint64)
        a = sp_all.numpy().reshape(world, cap + 1, 2)
        o = out.numpy()
        seen = set()
        for r in range(world):
            c = int(a[r, 0, 0]) & 0xFFFFFFFF
            for i in range(c):
                u, val = int(a[r, 1 + i, 0]), int(a[r, 1 + i, 1])
                if (int(words[u >> 6]) >> (u & 63)) & 1:
                    val = max(val, u + 1)
                for t in self.snap.col[self.snap.off[u]: self.snap.off[u + 1]].tolist():
                    if lo <= t < hi and val > int(o[t - lo]):
                        o[t - lo] = val
                        if t not in seen:
                            seen.add(t)
                            self.raised.append(t - lo)

    def collect(self, lo, hi, x, out, cap, sp, state, lists=None):
        sp.zero_()
        if int(state[0]) or int(state[4]):
            return
        if lists is not None and int(state[1]) != 0:
            rec = lists[4]
            words = lists[3].numpy().view(np.uint64)
            o = out.numpy()
            sp[0] = len(self.raised)
            wit = None
            for i, t in enumerate(self.raised):
                v, val = lo + t, int(o[t])
                if i < cap:
                    sp[2 + 2 * i] = v
                    sp[3 + 2 * i] = val
                if val == v + 1 and (int(words[v >> 6]) >> (v & 63)) & 1:
                    wit = v if wit is None else min(wit, v)
            if self.raised:
                rec[0] = max(int(rec[0]), 1)
            if wit is not None:
                rec[1] = max(int(rec[1]), self.NONE - wit)
            return
        xv = x.numpy()[lo:hi]
        ov = out.numpy()[: hi - lo]
        idx = np.flatnonzero(ov != xv)
        sp[0] = len(idx)
        k = min(len(idx), cap)
        pairs = np.stack([idx[:k] + lo, ov[idx[:k]].astype(np.int64)], 1).astype(np.int64)
        sp[2: 2 + 2 * k] = torch.from_numpy(pairs.reshape(-1).astype(np.int32))

    def post_sparse(self, rec, state, sp_all, world, cap, x):
        a = sp_all.numpy().reshape(world, cap + 1, 2)
        counts = a[:, 0, 0].astype(np.int64) & 0xFFFFFFFF
        over = counts.max() > cap
        if not over:
            for r in range(world):
                c = int(counts[r])
                if c:
                    x[torch.from_numpy(a[r, 1:1 + c, 0].astype(np.int64))] = torch.from_numpy(a[r, 1:1 + c, 1].copy())
        if not (int(state[0]) or int(state[4])):
            state[5] = max(int(state[5]), int(counts.max()))
            if over:
                state[4] = 1
                state[6] = rec[0]
                state[7] = rec[1]
            else:
                wit = self.NONE - int(rec[1])
                state[1] += 1
                if (int(state[3]) and wit != self.NONE) or not int(rec[0]):
                    state[0] = 1
                    state[2] = wit

    def demote(self, x, acc):
        rem, dem = self.R.demote(x.numpy().view(np.uint32)[: self.n], acc.numpy().view(np.uint64))
        fsize = int(np.unpackbits(rem.view(np.uint8)).sum())
        return torch.from_numpy(rem.view(np.int64).copy()), len(dem), fsize


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_0912_2555_b200 import sharded

    R = oracle.Restatement()
    out = []
    for t, (n, edges, accw, early) in enumerate(cases):
        gat = R.transpose(R.build_snapshot(n, edges, True))
        bounds = sharded.shard_bounds(gat.off, world)
        be = HostShardBackend(R, gat, n, R.build_snapshot(n, edges, True))
        # dense, sparse with overflow fallbacks (tiny capacity) and auto
        exchange, cap = [("dense", None), ("sparse", 3), ("auto", None), ("sparse", None), ("auto", 1)][t % 5]
        res = sharded.run_map_sharded(be, dist, rank, world, bounds, accw, early, exchange=exchange,
                                      sparse_cap=cap)
        out.append((res.verdict.cycle_found(), res.verdict.witness, res.stats.iterations,
                    res.stats.kernel_calls, res.stats.demoted_total,
                    res.final_values.numpy().view(np.uint32).copy()))
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def _cases():
    import oracle

    R = oracle.Restatement()
    rng = np.random.default_rng(88)
    cases = []
    for t in range(10):
        n = int(rng.integers(20, 400))
        e = rng.integers(0, n, size=(int(n * rng.choice([1, 2, 3])), 2)).astype(np.uint32)
        acc = rng.random(n) < [0.05, 0.3][t % 2]
        w = np.zeros((n + 63) // 64, np.uint64)
        idx = np.flatnonzero(acc)
        np.bitwise_or.at(w, idx >> 6, np.uint64(1) << (idx & 63).astype(np.uint64))
        cases.append((n, e, w, bool(t % 3)))
    p = R.preset(2)  # the config-2 family (closed form: (L+1) iterations, (L+1)^2 steps)
    p.L, p.W, p.S = 6, 8, 4
    R.prepare(p)
    n, e, w = R.generate(p)
    cases.append((n, e, w, True))
    return R, cases


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_protocol_matches_single_device(world):
    R, cases = _cases()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (n, e, w, early), g in zip(cases, got):
        ref = R.run_map(R.transpose(R.build_snapshot(n, e, True)), w, early)
        assert g[:5] == (ref.cycle, ref.witness, ref.iterations, ref.kernel_calls, ref.demoted_total)
        assert np.array_equal(g[5], ref.final_x)


def _handles_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_0912_2555_b200 import sharded

    mine = bytes([rank]) * 64
    blob = sharded.exchange_handles(dist, mine, world)
    if rank == 0:
        q.put(blob)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_handle_exchange(world):
    """The fused path's host protocol: every rank ends up with all ranks'
    IPC handles in rank order (cyc_fused_connect's input)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_handles_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    blob = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert blob == b"".join(bytes([r]) * 64 for r in range(world))
