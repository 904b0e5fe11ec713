"""Row-sharded MAP over several GPUs, one process per GPU.

Partition: contiguous rows of the gather index, balanced by edge count — the
reference's own worker partition (map_engine.cpp:35-43), `shard_bounds`. The
reference's results are worker-count invariant (map_engine.hpp:46-49), so the
sharded run must reproduce the single-device verdict, witness, MapStats and
final vector bit for bit.

Per Jacobi step every rank computes the new values of its rows from the
replicated vector, then
  * all-gather of the row slices (equal-size padded slices), and
  * all-reduce(MAX) of {changed, -min self-witness},
so all ranks take the same stop / early-exit decision at the same step
(kernel_calls identical to one device). Demotion (map_engine.cpp:123-137) is
replicated on every rank from the gathered vector — no collective needed.

The protocol is backend-agnostic: the product runs `CudaShardBackend` (the
sm_100a step kernel through the C ABI, torch.distributed NCCL for the
collectives, the library ordered on torch's current stream); the CPU tests run
the same `run_map_sharded` over gloo with a host backend.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _abi
from .api import CsrSnapshot, MapStats, Verdict, shard_bounds

_NONE = 0xFFFFFFFF


@dataclass
class ShardedResult:
    verdict: Verdict
    stats: MapStats
    final_values: object  # torch tensor (int32 codes) on the backend's device


def plan(gather_offsets, world: int) -> np.ndarray:
    """Row bounds per rank (len world+1), edge-balanced."""
    return shard_bounds(gather_offsets, world)


class CudaShardBackend:
    """Dense step over this rank's rows with the engine's kernel (device only)."""

    def __init__(self, snap: CsrSnapshot, device):
        import torch

        self.torch = torch
        self.snap = snap
        self.n = snap.n
        self.device = device
        self.flags = torch.zeros(2, dtype=torch.int32, device=device)
        self.counts = torch.zeros(2, dtype=torch.int64, device=device)
        stream = torch.cuda.current_stream(device).cuda_stream
        _abi.check(_abi.lib().cyc_ctx_set_stream(snap.context.handle, C.c_void_p(stream), 1))

    def release(self):
        """Back to the context's own stream."""
        _abi.check(_abi.lib().cyc_ctx_set_stream(self.snap.context.handle, None, 0))

    def zeros(self, k: int):
        return self.torch.zeros(max(k, 1), dtype=self.torch.int32, device=self.device)

    def acc_tensor(self, words: np.ndarray):
        return self.torch.from_numpy(words.view(np.int64).copy()).to(self.device)

    def step(self, x, acc, lo: int, hi: int, out):
        _abi.check(_abi.lib().cyc_shard_step(self.snap.context.handle, self.snap.handle, lo, hi,
                                             _abi.ptr(x), _abi.ptr(acc), _abi.ptr(out),
                                             _abi.ptr(self.flags)))
        return self.flags

    def demote(self, x, acc):
        rem = self.torch.zeros_like(acc)
        _abi.check(_abi.lib().cyc_shard_demote(self.snap.context.handle, _abi.ptr(x), self.n,
                                               _abi.ptr(acc), _abi.ptr(rem), _abi.ptr(self.counts)))
        d, f = (int(v) for v in self.counts.cpu())
        return rem, d, f


def run_map_sharded(backend, dist, rank: int, world: int, bounds, acc_words: np.ndarray,
                    early_exit: bool = True, group=None) -> ShardedResult:
    """run_map (map_engine.cpp:139-162) with rows sharded over `world` ranks."""
    torch = backend.torch
    n = backend.n
    bounds = [int(b) for b in bounds]
    lo, hi = bounds[rank], bounds[rank + 1]
    maxrows = max(bounds[r + 1] - bounds[r] for r in range(world))
    x = backend.zeros(n)
    send = backend.zeros(maxrows)
    gathered = [backend.zeros(maxrows) for _ in range(world)]
    acc = backend.acc_tensor(np.ascontiguousarray(acc_words, dtype=np.uint64))
    red = torch.zeros(2, dtype=torch.int64, device=x.device)
    stats = MapStats()
    verdict = Verdict.no_cycle()
    fsize = int(np.unpackbits(np.ascontiguousarray(acc_words, dtype=np.uint64).view(np.uint8)).sum())
    while fsize > 0:  # front.any()
        x.zero_()
        steps = 0
        witness = _NONE
        while True:
            flags = backend.step(x, acc, lo, hi, send)
            dist.all_gather(gathered, send, group=group)
            for r in range(world):
                k = bounds[r + 1] - bounds[r]
                if k:
                    x[bounds[r]: bounds[r + 1]].copy_(gathered[r][:k])
            red[0] = flags[0].to(torch.int64)
            red[1] = -(flags[1].to(torch.int64) & 0xFFFFFFFF)
            dist.all_reduce(red, op=dist.ReduceOp.MAX, group=group)
            changed, wit = (int(v) for v in red.cpu())
            wit = -wit
            steps += 1
            if early_exit and wit != _NONE:
                witness = wit
                break
            if not changed:
                witness = wit
                break
        stats.iterations += 1
        stats.kernel_calls += steps
        if witness != _NONE:
            stats.cycle_witness = witness
            verdict = Verdict.cycle(witness)
            break
        acc, dcount, fsize = backend.demote(x, acc)
        stats.demoted_total += dcount
        if dcount == 0:
            break
    return ShardedResult(verdict, stats, x[:n] if n else x[:0])
