"""Host-side mirror of the reference's MAP interface, over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/cycheck/{types,bitset,graph,map_engine}.hpp so a
caller of the reference (cycheck_main.cpp:88-97, explore.cpp:71-124) can switch
to the B200 engine call for call:

    log = EdgeLog();  v = log.add_vertex(True); log.append_edge(v, v)
    snap = build_snapshot(log, Orientation.transposed)
    verdict, stats = run_map(snap, snap.accepting)

Map vectors are numpy uint32 arrays of codes (id+1, 0 = NIL; map_engine.hpp:16-29).
Accepting sets are `Bitset`s (bitset.hpp:12-72) or anything `as_bitset` accepts.
All compute runs in the CUDA library; snapshots live in device memory.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import ContractError, CudaError, CycheckError, ParseError, ResourceLimitError, check, ptr

NIL = 0
_NONE = 0xFFFFFFFF


class Orientation(enum.IntEnum):
    """types.hpp:12."""

    forward = _abi.CYC_FORWARD
    transposed = _abi.CYC_TRANSPOSED


class Outcome(enum.Enum):
    cycle_found = "cycle_found"
    no_accepting_cycle = "no_accepting_cycle"


@dataclass(frozen=True)
class Verdict:
    """types.hpp:18-27."""

    outcome: Outcome = Outcome.no_accepting_cycle
    witness: Optional[int] = None

    @staticmethod
    def cycle(w: int) -> "Verdict":
        return Verdict(Outcome.cycle_found, int(w))

    @staticmethod
    def no_cycle() -> "Verdict":
        return Verdict(Outcome.no_accepting_cycle, None)

    def cycle_found(self) -> bool:
        return self.outcome is Outcome.cycle_found


# --------------------------------------------------------------------- Bitset
class Bitset:
    """Fixed-size bit sequence in uint64 words with trimmed tail (bitset.hpp:12-72)."""

    __slots__ = ("_size", "_words")

    def __init__(self, size: int = 0, value: bool = False):
        self._size = int(size)
        nw = (self._size + 63) // 64
        self._words = np.full(nw, np.uint64(0xFFFFFFFFFFFFFFFF) if value else 0, dtype=np.uint64)
        self.trim()

    @classmethod
    def all_set(cls, size: int) -> "Bitset":
        return cls(size, True)

    @classmethod
    def from_words(cls, words, size: int) -> "Bitset":
        b = cls(size)
        w = np.asarray(words, dtype=np.uint64)
        b._words[: min(len(w), len(b._words))] = w[: len(b._words)]
        b.trim()
        return b

    @classmethod
    def from_indices(cls, size: int, idx: Iterable[int]) -> "Bitset":
        b = cls(size)
        for i in idx:
            b.set(int(i))
        return b

    @classmethod
    def from_bools(cls, flags) -> "Bitset":
        f = np.asarray(flags, dtype=bool)
        b = cls(len(f))
        if len(f):
            packed = np.packbits(f, bitorder="little")
            pad = (-len(packed)) % 8
            b._words = np.frombuffer(np.concatenate([packed, np.zeros(pad, np.uint8)]).tobytes(),
                                     dtype=np.uint64).copy()[: (len(f) + 63) // 64]
        return b

    def size(self) -> int:
        return self._size

    def __len__(self) -> int:
        return self._size

    def empty(self) -> bool:
        return self._size == 0

    def test(self, i: int) -> bool:
        return bool((int(self._words[i >> 6]) >> (i & 63)) & 1)

    def set(self, i: int) -> None:
        if not 0 <= i < self._size:
            raise ContractError(f"bit {i} out of range [0, {self._size})")
        self._words[i >> 6] |= np.uint64(1 << (i & 63))

    def reset(self, i: int) -> None:
        self._words[i >> 6] &= np.uint64(~(1 << (i & 63)) & 0xFFFFFFFFFFFFFFFF)

    def count(self) -> int:
        return int(np.unpackbits(self._words.view(np.uint8)).sum())

    def any(self) -> bool:
        return bool(self._words.any())

    def none(self) -> bool:
        return not self.any()

    def to_bools(self) -> np.ndarray:
        return np.unpackbits(self._words.view(np.uint8), bitorder="little")[: self._size].astype(bool)

    def indices(self) -> np.ndarray:
        return np.flatnonzero(self.to_bools()).astype(np.uint32)

    def words(self) -> np.ndarray:
        return self._words

    def trim(self) -> None:
        if self._size & 63:
            self._words[-1] &= np.uint64((1 << (self._size & 63)) - 1)

    def __eq__(self, other) -> bool:
        return isinstance(other, Bitset) and self._size == other._size and bool(
            np.array_equal(self._words, other._words))

    def __repr__(self) -> str:
        return f"Bitset(size={self._size}, count={self.count()})"


def as_bitset(acc, n: int) -> Bitset:
    """Accepts a Bitset, a bool array of length n, or an iterable of ids."""
    if isinstance(acc, Bitset):
        if acc.size() != n:
            raise ContractError(f"accepting set size {acc.size()} != vertex count {n}")
        return acc
    a = np.asarray(acc)
    if a.dtype == bool:
        if len(a) != n:
            raise ContractError(f"accepting set size {len(a)} != vertex count {n}")
        return Bitset.from_bools(a)
    return Bitset.from_indices(n, a.ravel().tolist())


# ------------------------------------------------------------------- context
class Context:
    """One GPU and one CUDA stream; every call of the context is ordered on it."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(_abi.lib().cyc_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def synchronize(self) -> None:
        check(_abi.lib().cyc_ctx_synchronize(self._h))

    def reserve(self, m_log: int, n: int, background: bool = True) -> None:
        """Allocate what a build of an m_log-edge log over n vertices uses
        ahead of the first call (cyc_ctx_reserve); (0, 0) waits for a
        background reserve."""
        check(_abi.lib().cyc_ctx_reserve(self._h, int(m_log), int(n), int(background)))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().cyc_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None
_ctx_lock = threading.Lock()


def default_context() -> Context:
    global _default_ctx
    with _ctx_lock:
        if _default_ctx is None:
            _default_ctx = Context(0)
        return _default_ctx


def launch_count() -> int:
    """Kernels launched by the engine library in this process."""
    return int(_abi.lib().cyc_launch_count())


# ------------------------------------------------------------------- EdgeLog
class EdgeLog:
    """Append-only vertex/edge store (graph.hpp:49-91), host memory."""

    @dataclass
    class Limits:
        max_vertices: int = 1 << 24
        max_edges: int = 1 << 28

    def __init__(self, limits: Optional["EdgeLog.Limits"] = None):
        self._limits = limits or EdgeLog.Limits()
        self._acc = np.zeros(1024, dtype=bool)
        self._n = 0
        self._edges = np.zeros((1024, 2), dtype=np.uint32)
        self._m = 0

    @classmethod
    def from_arrays(cls, n: int, edges, accepting=None,
                    limits: Optional["EdgeLog.Limits"] = None) -> "EdgeLog":
        """Bulk fill (equivalent to fill_log, graph.cpp:305-310)."""
        log = cls(limits or EdgeLog.Limits(max(int(n), 1), max(len(edges), 1)))
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        if int(n) > log._limits.max_vertices:
            raise ResourceLimitError(f"vertex capacity exceeded ({log._limits.max_vertices})")
        if len(e) > log._limits.max_edges:
            raise ResourceLimitError(f"edge capacity exceeded ({log._limits.max_edges})")
        if len(e) and int(e.max()) >= int(n):
            raise ContractError("append_edge: endpoint not interned")
        acc = np.zeros(int(n), dtype=bool)
        if accepting is not None:
            acc = as_bitset(accepting, int(n)).to_bools()
        log._acc, log._n = acc, int(n)
        log._edges, log._m = e, len(e)
        return log

    def limits(self) -> "EdgeLog.Limits":
        return self._limits

    def add_vertex(self, accepting: bool) -> int:
        if self._n >= self._limits.max_vertices:
            raise ResourceLimitError(f"vertex capacity exceeded ({self._limits.max_vertices})")
        if self._n == len(self._acc):
            self._acc = np.concatenate([self._acc, np.zeros(len(self._acc), bool)])
        self._acc[self._n] = bool(accepting)
        self._n += 1
        return self._n - 1

    def append_edge(self, src: int, dst: int) -> None:
        if src >= self._n or dst >= self._n or src < 0 or dst < 0:
            raise ContractError(
                f"append_edge: endpoint not interned ({src} -> {dst}, n={self._n})")
        if self._m >= self._limits.max_edges:
            raise ResourceLimitError(f"edge capacity exceeded ({self._limits.max_edges})")
        if self._m == len(self._edges):
            self._edges = np.concatenate([self._edges, np.zeros_like(self._edges)])
        self._edges[self._m] = (src, dst)
        self._m += 1

    def vertex_count(self) -> int:
        return self._n

    def edge_count(self) -> int:
        return self._m

    def is_accepting(self, v: int) -> bool:
        return bool(self._acc[v])

    def edge(self, i: int):
        return int(self._edges[i, 0]), int(self._edges[i, 1])

    def edges(self, m: Optional[int] = None) -> np.ndarray:
        m = self._m if m is None else m
        return np.ascontiguousarray(self._edges[:m])

    def accepting_prefix(self, n: int) -> Bitset:
        return Bitset.from_bools(self._acc[:n])


# ------------------------------------------------------------------ snapshot
class CsrSnapshot:
    """Device-resident snapshot (graph.hpp:27-42) plus its gather index.

    row_offsets / col_indices / accepting are copied out lazily on access.
    """

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self._h = handle
        self._ctx = ctx
        n, m, o, r = C.c_uint32(), C.c_uint64(), C.c_int(), C.c_int()
        check(_abi.lib().cyc_graph_info(handle, C.byref(n), C.byref(m), C.byref(o), C.byref(r)))
        self.n = int(n.value)
        self.m = int(m.value)
        self.orientation = Orientation(o.value)
        self.restricted = bool(r.value)
        self._csr = None
        self._acc = None
        self._kept = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @property
    def context(self) -> Context:
        return self._ctx

    def _export(self):
        if self._csr is None:
            off = np.zeros(self.n + 1, dtype=np.uint64)
            col = np.zeros(max(self.m, 1), dtype=np.uint32)
            acc = np.zeros(max((self.n + 63) // 64, 1), dtype=np.uint64)
            kept = np.zeros(max(self.n, 1), dtype=np.uint32) if self.restricted else None
            check(_abi.lib().cyc_graph_export(self._h, ptr(off), ptr(col), ptr(acc), ptr(kept)))
            self._csr = (off, col[: self.m])
            self._acc = Bitset.from_words(acc, self.n)
            self._kept = kept[: self.n] if kept is not None else None
        return self._csr

    @property
    def row_offsets(self) -> np.ndarray:
        return self._export()[0]

    @property
    def col_indices(self) -> np.ndarray:
        return self._export()[1]

    @property
    def accepting(self) -> Bitset:
        self._export()
        return self._acc

    @property
    def kept(self) -> Optional[np.ndarray]:
        self._export()
        return self._kept

    def row(self, v: int) -> np.ndarray:
        off, col = self._export()
        return col[int(off[v]): int(off[v + 1])]

    def edge_list(self):
        off, col = self._export()
        rows = np.repeat(np.arange(self.n, dtype=np.uint32), np.diff(off).astype(np.int64))
        return list(zip(rows.tolist(), col.tolist()))

    def gather_index(self):
        """The MaxPropagation gather index (map_engine.cpp:9-19)."""
        off = np.zeros(self.n + 1, dtype=np.uint64)
        col = np.zeros(max(self.m, 1), dtype=np.uint32)
        check(_abi.lib().cyc_graph_export_gather(self._h, ptr(off), ptr(col)))
        return off, col[: self.m]

    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().cyc_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_snapshot(log, orientation: Orientation = Orientation.transposed,
                   m: Optional[int] = None, n: Optional[int] = None,
                   ctx: Optional[Context] = None) -> CsrSnapshot:
    """build_snapshot (graph.hpp:97-101, graph.cpp:63-111) on the device.

    ``log`` is an EdgeLog, or a tuple (n, edges[m,2], accepting) for bulk use.
    """
    ctx = ctx or default_context()
    if isinstance(log, EdgeLog):
        mm = log.edge_count() if m is None else int(m)
        nn = log.vertex_count() if n is None else int(n)
        if mm > log.edge_count():
            raise ContractError("build_snapshot: prefix beyond log")
        edges = log.edges(mm)
        acc = log.accepting_prefix(nn).words()
    else:
        nn, edges, acc = log
        edges = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        mm = len(edges) if m is None else int(m)
        acc = as_bitset(acc, int(nn)).words() if acc is not None else None
    h = C.c_void_p()
    check(_abi.lib().cyc_graph_build(ctx.handle, ptr(edges), C.c_uint64(mm), C.c_uint32(int(nn)),
                                     ptr(acc), int(orientation), C.byref(h)))
    return CsrSnapshot(h, ctx)


def extend_snapshot(prev: CsrSnapshot, log, m: Optional[int] = None, n: Optional[int] = None) -> CsrSnapshot:
    """Incremental snapshot: the snapshot of the log prefix
    (m, n) from ``prev`` (the snapshot of a shorter prefix of the same log) and
    the new edges only. Equal to ``build_snapshot(log, prev.orientation, m, n)``
    — the explorer's per-round rebuild (explore.cpp:71-124).

    ``log`` is an EdgeLog, or a tuple (n, new_edges[k,2], accepting) holding
    only the edges after prev's prefix."""
    ctx = prev.context
    m_prev = C.c_uint64()
    check(_abi.lib().cyc_graph_log_prefix(prev.handle, C.byref(m_prev)))
    if isinstance(log, EdgeLog):
        mm = log.edge_count() if m is None else int(m)
        nn = log.vertex_count() if n is None else int(n)
        if mm > log.edge_count():
            raise ContractError("build_snapshot: prefix beyond log")
        if mm < m_prev.value:
            raise ContractError("extend_snapshot: edge prefix shrinks")
        new = log.edges(mm)[m_prev.value:]
        acc = log.accepting_prefix(nn).words()
    else:
        nn, new, acc = log
        new = np.asarray(new, dtype=np.uint32).reshape(-1, 2)
        acc = as_bitset(acc, int(nn)).words() if acc is not None else None
    new = np.ascontiguousarray(new)
    h = C.c_void_p()
    check(_abi.lib().cyc_graph_extend(ctx.handle, prev.handle, ptr(new), C.c_uint64(len(new)),
                                      C.c_uint32(int(nn)), ptr(acc), C.byref(h)))
    return CsrSnapshot(h, ctx)


# ------------------------------------------------------- explicit graphs
@dataclass
class ExplicitGraph:
    """ExplicitGraph (graph.hpp:140-144): accepting ids in file order."""
    n: int
    accepting: np.ndarray
    edges: np.ndarray  # [m, 2] (src, dst)


class DeviceExplicitGraph:
    """A parsed explicit graph held on the device (cyc_explicit)."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self._h, self._ctx = handle, ctx
        n, na, m = C.c_uint32(), C.c_uint64(), C.c_uint64()
        check(_abi.lib().cyc_explicit_info(handle, C.byref(n), C.byref(na), C.byref(m)))
        self.n, self.n_accepting, self.m = int(n.value), int(na.value), int(m.value)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().cyc_explicit_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export(self) -> ExplicitGraph:
        acc = np.zeros(max(self.n_accepting, 1), np.uint32)
        e = np.zeros((max(self.m, 1), 2), np.uint32)
        check(_abi.lib().cyc_explicit_export(self._h, ptr(acc), ptr(e)))
        return ExplicitGraph(self.n, acc[: self.n_accepting], e[: self.m])

    def snapshot(self, orientation: Orientation = Orientation.transposed) -> CsrSnapshot:
        """fill_log (graph.cpp:305-310) + build_snapshot, on the device."""
        h = C.c_void_p()
        check(_abi.lib().cyc_explicit_snapshot(self._ctx.handle, self._h, int(orientation), C.byref(h)))
        return CsrSnapshot(h, self._ctx)


def parse_explicit_device(text, ctx: Optional[Context] = None) -> DeviceExplicitGraph:
    """parse_explicit_graph (graph.cpp:259-297) on the device; the graph stays
    there. Raises ParseError with the reference's message on malformed text."""
    ctx = ctx or default_context()
    data = text.encode() if isinstance(text, str) else bytes(text)
    buf = np.frombuffer(data, dtype=np.uint8) if data else np.zeros(1, np.uint8)
    h = C.c_void_p()
    check(_abi.lib().cyc_explicit_parse(ctx.handle, ptr(buf), C.c_uint64(len(data)), C.byref(h)))
    return DeviceExplicitGraph(h, ctx)


def parse_explicit_graph(text, ctx: Optional[Context] = None) -> ExplicitGraph:
    """parse_explicit_graph (graph.hpp:146) with the parse on the device."""
    return parse_explicit_device(text, ctx).export()


def load_explicit_graph(path: str, ctx: Optional[Context] = None) -> ExplicitGraph:
    """load_explicit_graph (graph.cpp:299-303)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise ParseError(f"0:0: error[syntax]: cannot open '{path}'", 0, 0, 0) from None
    return parse_explicit_graph(data, ctx)


def write_binary_graph(n: int, edges, accepting, path: Optional[str] = None) -> bytes:
    """The binary edge list read by cyc_explicit_load_binary: "CYCGRAPH", u32
    version 1, u32 n, u64 m, u64 accepting words, u32 (src, dst) pairs."""
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
    words = as_bitset(accepting, int(n)).words() if accepting is not None else np.zeros((int(n) + 63) // 64,
                                                                                          np.uint64)
    words = np.ascontiguousarray(words[: (int(n) + 63) // 64], dtype=np.uint64)
    hdr = b"CYCGRAPH" + np.array([1, int(n)], np.uint32).tobytes() + np.array([len(e)], np.uint64).tobytes()
    data = hdr + words.tobytes() + e.tobytes()
    if path is not None:
        with open(path, "wb") as f:
            f.write(data)
    return data


def load_binary_graph(data_or_path, ctx: Optional[Context] = None) -> DeviceExplicitGraph:
    ctx = ctx or default_context()
    if isinstance(data_or_path, str):
        with open(data_or_path, "rb") as f:
            data = f.read()
    else:
        data = bytes(data_or_path)
    buf = np.frombuffer(data, dtype=np.uint8)
    h = C.c_void_p()
    check(_abi.lib().cyc_explicit_load_binary(ctx.handle, ptr(buf), C.c_uint64(len(data)), C.byref(h)))
    return DeviceExplicitGraph(h, ctx)


@dataclass
class SccRestriction:
    """graph.hpp:105-108."""

    snapshot: CsrSnapshot
    kept: np.ndarray


def restrict_to_accepting_sccs(snap: CsrSnapshot) -> SccRestriction:
    """graph.hpp:110-114, graph.cpp:190-221."""
    h = C.c_void_p()
    check(_abi.lib().cyc_graph_restrict(snap.context.handle, snap.handle, C.byref(h)))
    r = CsrSnapshot(h, snap.context)
    return SccRestriction(r, r.kept if r.kept is not None else np.zeros(0, np.uint32))


# ---------------------------------------------------------------- map engine
@dataclass
class MapOptions:
    """map_engine.hpp:33-36 (+ device step selection)."""

    workers: int = 1
    early_exit: bool = True
    mode: str = "auto"            # "auto" | "pull" | "push"
    push_alpha: int = 0
    trace_cap: int = 0            # > 0: keep a per-step device trace (map_trace)
    layout: str = "auto"          # "auto" | "identity" | "degree": storage order (same results)

    def to_c(self, max_iterations: int = 0, max_steps: int = 0) -> _abi.MapOptionsC:
        modes = {"auto": _abi.CYC_MODE_AUTO, "pull": _abi.CYC_MODE_PULL, "push": _abi.CYC_MODE_PUSH}
        layouts = {"auto": _abi.CYC_LAYOUT_AUTO, "identity": _abi.CYC_LAYOUT_IDENTITY,
                   "degree": _abi.CYC_LAYOUT_DEGREE}
        if self.mode not in modes:
            raise ContractError(f"unknown mode {self.mode!r}")
        if self.layout not in layouts:
            raise ContractError(f"unknown layout {self.layout!r}")
        return _abi.MapOptionsC(int(bool(self.early_exit)), modes[self.mode], max_iterations,
                                max_steps, int(self.push_alpha), int(self.trace_cap), layouts[self.layout], 0)


@dataclass
class StepResult:
    """map_engine.hpp:38-44."""

    changed: bool = False
    self_witness: Optional[int] = None


@dataclass
class FixpointResult:
    """map_engine.hpp:75-79."""

    values: np.ndarray
    steps: int = 0
    witness: Optional[int] = None


@dataclass
class DemoteResult:
    """map_engine.hpp:91-94."""

    remaining: Bitset
    demoted: np.ndarray


@dataclass
class MapStats:
    """map_engine.hpp:101-106 plus device evidence."""

    iterations: int = 0
    kernel_calls: int = 0
    demoted_total: int = 0
    cycle_witness: Optional[int] = None
    device: dict = field(default_factory=dict)


def _acc_words(accepting, n: int) -> np.ndarray:
    return as_bitset(accepting, n).words()


def _vector(x, n: int) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.uint32))
    if a.shape != (n,):
        raise ContractError(f"propagate_step: vector length {a.size} != vertex count {n}")
    return a


class MaxPropagation:
    """map_engine.hpp:46-65. The gather index already lives with the snapshot."""

    def __init__(self, snap: CsrSnapshot):
        self._snap = snap

    def vertex_count(self) -> int:
        return self._snap.n

    def step(self, x, accepting, out: Optional[np.ndarray] = None) -> StepResult:
        n = self._snap.n
        xv = _vector(x, n)
        acc = _acc_words(accepting, n)
        o = out if out is not None else np.zeros(n, dtype=np.uint32)
        if o.shape != (n,) or o.dtype != np.uint32:
            raise ContractError("propagate_step: output vector mismatch")
        ch, w = C.c_int32(), C.c_uint32()
        check(_abi.lib().cyc_map_step(self._snap.context.handle, self._snap.handle, ptr(acc),
                                      ptr(xv), ptr(o), C.byref(ch), C.byref(w)))
        self.last_out = o
        return StepResult(bool(ch.value), None if w.value == _NONE else int(w.value))


def init_vector(snap: CsrSnapshot) -> np.ndarray:
    """map_engine.cpp:81-83: all NIL."""
    return np.zeros(snap.n, dtype=np.uint32)


def propagate_step(snap: CsrSnapshot, x, accepting):
    """map_engine.cpp:85-92 -> (x', changed)."""
    k = MaxPropagation(snap)
    out = np.zeros(snap.n, dtype=np.uint32)
    r = k.step(x, accepting, out)
    return out, r.changed


def fixpoint(snap: CsrSnapshot, accepting, options: Optional[MapOptions] = None,
             max_steps: int = 0) -> FixpointResult:
    """map_engine.cpp:94-121 (max_steps > 0 stops after that many steps)."""
    options = options or MapOptions()
    n = snap.n
    acc = _acc_words(accepting, n)
    vals = np.zeros(max(n, 1), dtype=np.uint32)
    steps, w = C.c_uint64(), C.c_uint32()
    opt = options.to_c(1, max_steps)
    check(_abi.lib().cyc_fixpoint(snap.context.handle, snap.handle, ptr(acc), C.byref(opt),
                                  ptr(vals), C.byref(steps), C.byref(w)))
    return FixpointResult(vals[:n], int(steps.value), None if w.value == _NONE else int(w.value))


def demote(values, accepting, ctx: Optional[Context] = None) -> DemoteResult:
    """map_engine.cpp:123-137."""
    ctx = ctx or default_context()
    x = np.ascontiguousarray(np.asarray(values, dtype=np.uint32))
    n = len(x)
    acc = _acc_words(accepting, n)
    rem = np.zeros(max((n + 63) // 64, 1), dtype=np.uint64)
    dem = np.zeros(max(n, 1), dtype=np.uint32)
    nd = C.c_uint64()
    check(_abi.lib().cyc_demote(ctx.handle, ptr(x) if n else None, n, ptr(acc), ptr(rem), ptr(dem),
                                C.byref(nd)))
    return DemoteResult(Bitset.from_words(rem, n), dem[: nd.value].copy())


@dataclass
class MapRun:
    verdict: Verdict
    stats: MapStats
    final_values: Optional[np.ndarray]
    iter_hash: np.ndarray
    iter_steps: np.ndarray


def run_map_detailed(snap: CsrSnapshot, accepting=None, options: Optional[MapOptions] = None,
                     want_values: bool = True, hash_cap: int = 4096) -> MapRun:
    """run_map plus the per-iteration evidence used by parity tests."""
    options = options or MapOptions()
    n = snap.n
    acc = _acc_words(accepting, n) if accepting is not None else None
    st = _abi.MapStatsC()
    vals = np.zeros(max(n, 1), dtype=np.uint32) if want_values else None
    hh = np.zeros(max(hash_cap, 1), dtype=np.uint64)
    hs = np.zeros(max(hash_cap, 1), dtype=np.uint64)
    opt = options.to_c()
    check(_abi.lib().cyc_map_run(snap.context.handle, snap.handle, ptr(acc), C.byref(opt),
                                 C.byref(st), ptr(vals), ptr(hh), ptr(hs), C.c_uint64(hash_cap)))
    k = min(int(st.iterations), hash_cap)
    verdict = Verdict.cycle(st.witness) if st.cycle_found else Verdict.no_cycle()
    stats = MapStats(int(st.iterations), int(st.kernel_calls), int(st.demoted_total),
                     int(st.witness) if st.cycle_found else None, stats_dict(st))
    return MapRun(verdict, stats, vals[:n] if vals is not None else None, hh[:k], hs[:k])


def run_map(snap: CsrSnapshot, accepting=None, options: Optional[MapOptions] = None):
    """map_engine.cpp:139-162 -> (Verdict, MapStats)."""
    if accepting is not None and as_bitset(accepting, snap.n).size() != snap.n:
        raise ContractError("run_map: accepting set size mismatch")
    r = run_map_detailed(snap, accepting, options, want_values=False, hash_cap=0)
    return r.verdict, r.stats


def map_trace(snap: CsrSnapshot, cap: int = 1 << 16) -> np.ndarray:
    """Per-step device trace of the snapshot's last run with trace_cap > 0.
    Columns: mode (1 pull, 2 push), step in fixpoint, frontier edges, raised,
    t_start, t_phase0, t_phase1, t_flags, t_end (globaltimer ns), input chunks."""
    buf = np.zeros((cap, 64), dtype=np.uint64)
    n = C.c_uint32()
    check(_abi.lib().cyc_map_trace(snap.handle, ptr(buf), cap, C.byref(n)))
    t = buf[: n.value]
    t = t[(t[:, 0] >> np.uint64(60)) > 0]
    out = np.zeros((len(t), 10), dtype=np.int64)
    out[:, 0] = (t[:, 0] >> np.uint64(60)).astype(np.int64)
    out[:, 1] = (t[:, 0] & np.uint64(0xFFFFFF)).astype(np.int64)
    out[:, 2] = t[:, 1].astype(np.int64)
    out[:, 3] = t[:, 2].astype(np.int64)
    out[:, 4] = t[:, 3].astype(np.int64)
    for ph in range(3):
        out[:, 5 + ph] = t[:, 16 + 16 * ph: 32 + 16 * ph].max(axis=1).astype(np.int64)
    out[:, 8] = t[:, 7].astype(np.int64)
    out[:, 9] = ((t[:, 0] >> np.uint64(24)) & np.uint64((1 << 36) - 1)).astype(np.int64)
    return out


def stats_dict(st: _abi.MapStatsC) -> dict:
    return {name: getattr(st, name) for name, _ in st._fields_}


def check_graph(n: int, edges, accepting, orientation: Orientation = Orientation.transposed,
                scc_restriction: bool = False, options: Optional[MapOptions] = None,
                ctx: Optional[Context] = None):
    """One call from an edge log to a verdict: the `cycheck graph` / final
    explore round pipeline (cycheck_main.cpp:88-97, explore.cpp:71-124)."""
    ctx = ctx or default_context()
    options = options or MapOptions()
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
    acc = _acc_words(accepting, int(n))
    st = _abi.MapStatsC()
    ms = (C.c_double * 4)()
    opt = options.to_c()
    check(_abi.lib().cyc_check(ctx.handle, ptr(e), C.c_uint64(len(e)), C.c_uint32(int(n)), ptr(acc),
                               int(orientation), int(bool(scc_restriction)), C.byref(opt),
                               C.byref(st), ms))
    verdict = Verdict.cycle(st.witness) if st.cycle_found else Verdict.no_cycle()
    stats = MapStats(int(st.iterations), int(st.kernel_calls), int(st.demoted_total),
                     int(st.witness) if st.cycle_found else None, stats_dict(st))
    stats.device["phase_ms"] = list(ms)
    return verdict, stats


@dataclass
class OracleVerdict:
    """oracle.hpp:20-23."""

    verdict: Verdict
    cyclic_accepting: np.ndarray


def scc_verdict(snap: CsrSnapshot) -> OracleVerdict:
    """scc_verdict (oracle.cpp:32-98) on the device, over the snapshot relation
    (SCCs do not depend on orientation)."""
    cyc_, w, cnt = C.c_int32(), C.c_uint32(), C.c_uint64()
    out = np.zeros(max(snap.n, 1), dtype=np.uint32)
    check(_abi.lib().cyc_scc_verdict(snap.context.handle, snap.handle, C.byref(cyc_), C.byref(w),
                                     ptr(out), C.byref(cnt)))
    v = Verdict.cycle(w.value) if cyc_.value else Verdict.no_cycle()
    return OracleVerdict(v, out[: cnt.value].copy())


@dataclass
class OwctyStats:
    """OwctyStats (owcty.hpp:12-17)."""
    outer_iterations: int = 0
    reach_ms: float = 0.0
    elim_ms: float = 0.0
    final_size: int = 0


def run_owcty(snap: CsrSnapshot, accepting=None) -> "tuple[Verdict, OwctyStats]":
    """run_owcty (owcty.hpp:28-31, owcty.cpp:56-87) on the device over the
    snapshot relation; the reference runs it on a forward snapshot."""
    cyc_, w, st = C.c_int32(), C.c_uint32(), _abi.OwctyStatsC()
    aw = None if accepting is None else _acc_words(accepting, snap.n)
    check(_abi.lib().cyc_owcty(snap.context.handle, snap.handle, None if aw is None else ptr(aw),
                               C.byref(cyc_), C.byref(w), C.byref(st)))
    v = Verdict.cycle(w.value) if cyc_.value else Verdict.no_cycle()
    return v, OwctyStats(st.outer_iterations, st.reach_ms, st.elim_ms, st.final_size)


def shard_bounds(row_offsets: Sequence[int], parts: int) -> np.ndarray:
    """Edge-balanced contiguous row ranges (map_engine.cpp:35-43)."""
    off = np.ascontiguousarray(np.asarray(row_offsets, dtype=np.uint64))
    n = len(off) - 1
    b = np.zeros(parts + 1, dtype=np.uint32)
    check(_abi.lib().cyc_shard_bounds(ptr(off), n, int(parts), ptr(b)))
    return b


__all__ = [
    "Bitset", "CsrSnapshot", "Context", "ContractError", "CudaError", "CycheckError", "DemoteResult",
    "EdgeLog", "FixpointResult", "MapOptions", "MapRun", "MapStats", "MaxPropagation", "NIL",
    "Orientation", "Outcome", "ResourceLimitError", "SccRestriction", "StepResult", "Verdict",
    "as_bitset", "build_snapshot", "check_graph", "default_context", "demote", "fixpoint",
    "init_vector", "launch_count", "propagate_step", "restrict_to_accepting_sccs", "run_map",
    "run_map_detailed", "shard_bounds", "map_trace", "scc_verdict", "OracleVerdict", "OwctyStats",
    "run_owcty", "extend_snapshot", "ExplicitGraph", "DeviceExplicitGraph", "ParseError",
    "parse_explicit_graph", "parse_explicit_device", "load_explicit_graph", "write_binary_graph",
    "load_binary_graph",
]
