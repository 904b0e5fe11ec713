"""TEST INFRASTRUCTURE ONLY — the parity checker for the B200 engine.

Two CPU implementations of the reference MAP path, loaded with ctypes:

* ``Restatement`` — oracle/cyc_oracle.c, a plain-C restatement of
  /root/reference/proj/src/{graph,map_engine}.cpp (each function cites the
  lines it follows), built into oracle/_build/libcyo.so.
* ``Reference`` — the reference itself, compiled from its own sources by
  oracle/Makefile into oracle/_ref/libcycheck_ref.so and driven through its
  public API (oracle/ref_driver.cpp). Present wherever that .so was built
  (here, and on the GPU box as a shipped prebuilt file).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package. The engine (paper_0912_2555_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "_build", "libcyo.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libcycheck_ref.so")
NONE = 0xFFFFFFFF

_P = C.c_void_p


def build(quiet: bool = True) -> None:
    """Builds both oracle libraries (the reference only if its sources exist)."""
    subprocess.run(["make", "-C", HERE, "-j4"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _words(acc, n: int) -> np.ndarray:
    nw = max((n + 63) // 64, 1)
    if acc is None:
        return np.zeros(nw, np.uint64)
    if hasattr(acc, "words"):
        w = np.asarray(acc.words(), dtype=np.uint64)
    else:
        a = np.asarray(acc)
        if a.dtype == bool:
            w = np.zeros(nw, np.uint64)
            idx = np.flatnonzero(a)
            np.bitwise_or.at(w, idx >> 6, (np.uint64(1) << (idx & 63).astype(np.uint64)))
        else:
            w = np.asarray(a, dtype=np.uint64)
    out = np.zeros(nw, np.uint64)
    out[: min(len(w), nw)] = w[:nw]
    if n & 63 and n:
        out[(n - 1) >> 6] &= np.uint64((1 << (n & 63)) - 1)
    return out


def bools_from_words(words, n: int) -> np.ndarray:
    w = np.asarray(words, dtype=np.uint64)
    return np.unpackbits(w.view(np.uint8), bitorder="little")[:n].astype(bool)


class GenParams(C.Structure):
    """Mirror of cyc_gen_params (include/cyc_gen.h), kept here so the checker
    never imports the engine package (the reference arm must not map it)."""

    _fields_ = [("kind", C.c_int32), ("n", C.c_uint32), ("m", C.c_uint64), ("seed", C.c_uint64),
                ("deg", C.c_uint32), ("acc_thr", C.c_uint64), ("L", C.c_uint32), ("W", C.c_uint32),
                ("S", C.c_uint32), ("exit_all", C.c_uint32), ("acc_all", C.c_uint32),
                ("scale", C.c_uint32), ("edgefactor", C.c_uint32), ("thr_a", C.c_uint64),
                ("thr_ab", C.c_uint64), ("thr_abc", C.c_uint64), ("perm_mul1", C.c_uint64),
                ("perm_mul2", C.c_uint64), ("grid_bits", C.c_uint32), ("region", C.c_uint32),
                ("plant", C.c_uint32), ("reserved", C.c_uint32)]


class _Csr(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint64), ("off", C.POINTER(C.c_uint64)),
                ("col", C.POINTER(C.c_uint32))]


@dataclass
class Csr:
    n: int
    off: np.ndarray  # u64[n+1]
    col: np.ndarray  # u32[m]

    @property
    def m(self) -> int:
        return int(self.off[-1]) if len(self.off) else 0


@dataclass
class MapResult:
    cycle: bool
    witness: Optional[int]
    iterations: int
    kernel_calls: int
    demoted_total: int
    final_x: np.ndarray
    iter_hash: np.ndarray
    iter_steps: np.ndarray


class Restatement:
    """The C restatement (cyc_oracle.c)."""

    def __init__(self, path: str = RESTATEMENT_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.cyo_build_snapshot.argtypes = [_P, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(_Csr)]
        L.cyo_transpose.argtypes = [C.POINTER(_Csr), C.POINTER(_Csr)]
        L.cyo_csr_free.argtypes = [C.POINTER(_Csr)]
        L.cyo_scc_keep_mask.argtypes = [C.POINTER(_Csr), _P, _P]
        L.cyo_restrict.argtypes = [C.POINTER(_Csr), _P, C.POINTER(_Csr), _P, _P, C.POINTER(C.c_uint32)]
        L.cyo_step.argtypes = [C.POINTER(_Csr), _P, _P, _P, C.POINTER(C.c_int), C.POINTER(C.c_uint32)]
        L.cyo_fixpoint.argtypes = [C.POINTER(_Csr), _P, C.c_int, _P, _P, C.POINTER(C.c_uint32)]
        L.cyo_fixpoint.restype = C.c_uint64
        L.cyo_demote.argtypes = [_P, C.c_uint32, _P, _P, _P]
        L.cyo_demote.restype = C.c_uint64
        L.cyo_run_map.argtypes = [C.POINTER(_Csr), _P, C.c_int, _P, _P, _P, _P, C.c_uint64]
        L.cyo_run_owcty.argtypes = [C.POINTER(_Csr), _P, C.POINTER(C.c_int), C.POINTER(C.c_uint32),
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.cyo_vector_hash.argtypes = [_P, C.c_uint32]
        L.cyo_vector_hash.restype = C.c_uint64
        L.cyo_generate.argtypes = [_P, _P, _P]
        L.cyo_gen_preset.argtypes = [C.c_int, _P]
        L.cyo_gen_prepare.argtypes = [_P]

    # --- marshalling
    @staticmethod
    def _to_c(g: Csr) -> _Csr:
        c = _Csr()
        c.n = g.n
        c.m = g.m
        c.off = g.off.ctypes.data_as(C.POINTER(C.c_uint64))
        col = g.col if len(g.col) else np.zeros(1, np.uint32)
        c.col = col.ctypes.data_as(C.POINTER(C.c_uint32))
        c._keep = (g.off, col)  # keep arrays alive across the call
        return c

    def _from_c(self, c: _Csr) -> Csr:
        n, m = int(c.n), int(c.m)
        off = np.ctypeslib.as_array(c.off, shape=(n + 1,)).copy()
        col = np.ctypeslib.as_array(c.col, shape=(max(m, 1),))[:m].copy() if m else np.zeros(0, np.uint32)
        self.lib.cyo_csr_free(C.byref(c))
        return Csr(n, off, col)

    # --- graph_core
    def build_snapshot(self, n: int, edges, transposed: bool = True) -> Csr:
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        out = _Csr()
        rc = self.lib.cyo_build_snapshot(e.ctypes.data if len(e) else None, len(e), n, int(transposed),
                                         C.byref(out))
        if rc != 0:
            raise ValueError("build_snapshot: edge endpoint out of range")
        return self._from_c(out)

    def transpose(self, g: Csr) -> Csr:
        out = _Csr()
        self.lib.cyo_transpose(C.byref(self._to_c(g)), C.byref(out))
        return self._from_c(out)

    def keep_mask(self, g: Csr, acc) -> np.ndarray:
        keep = np.zeros(max(g.n, 1), np.uint8)
        aw = _words(acc, g.n)
        self.lib.cyo_scc_keep_mask(C.byref(self._to_c(g)), aw.ctypes.data,
                                   keep.ctypes.data)
        return keep[: g.n].astype(bool)

    def restrict(self, g: Csr, acc):
        out = _Csr()
        oacc = np.zeros(max((g.n + 63) // 64, 1), np.uint64)
        kept = np.zeros(max(g.n, 1), np.uint32)
        k = C.c_uint32()
        aw = _words(acc, g.n)
        self.lib.cyo_restrict(C.byref(self._to_c(g)), aw.ctypes.data, C.byref(out),
                              oacc.ctypes.data, kept.ctypes.data, C.byref(k))
        r = self._from_c(out)
        return r, oacc[: max((k.value + 63) // 64, 1)], kept[: k.value].copy()

    # --- map_engine (all take the GATHER index)
    def step(self, gather: Csr, x, acc):
        x = np.ascontiguousarray(np.asarray(x, np.uint32))
        out = np.zeros(max(gather.n, 1), np.uint32)
        ch, w = C.c_int(), C.c_uint32()
        aw = _words(acc, gather.n)
        self.lib.cyo_step(C.byref(self._to_c(gather)), x.ctypes.data, aw.ctypes.data,
                          out.ctypes.data, C.byref(ch), C.byref(w))
        return out[: gather.n], bool(ch.value), (None if w.value == NONE else int(w.value))

    def fixpoint(self, gather: Csr, acc, early_exit: bool = True):
        x = np.zeros(max(gather.n, 1), np.uint32)
        tmp = np.zeros_like(x)
        w = C.c_uint32()
        aw = _words(acc, gather.n)
        steps = self.lib.cyo_fixpoint(C.byref(self._to_c(gather)), aw.ctypes.data,
                                      int(early_exit), x.ctypes.data, tmp.ctypes.data, C.byref(w))
        return x[: gather.n], int(steps), (None if w.value == NONE else int(w.value))

    def demote(self, x, acc):
        x = np.ascontiguousarray(np.asarray(x, np.uint32))
        n = len(x)
        rem = np.zeros(max((n + 63) // 64, 1), np.uint64)
        dem = np.zeros(max(n, 1), np.uint32)
        aw = _words(acc, n)
        nd = self.lib.cyo_demote(x.ctypes.data if n else None, n, aw.ctypes.data,
                                 rem.ctypes.data, dem.ctypes.data)
        return rem, dem[:nd].copy()

    def run_map(self, gather: Csr, acc, early_exit: bool = True, cap: int = 1 << 16) -> MapResult:
        st = (C.c_uint64 * 5)()

        class _St(C.Structure):
            _fields_ = [("cycle_found", C.c_int), ("witness", C.c_uint32), ("iterations", C.c_uint64),
                        ("kernel_calls", C.c_uint64), ("demoted_total", C.c_uint64)]

        s = _St()
        fx = np.zeros(max(gather.n, 1), np.uint32)
        hh = np.zeros(cap, np.uint64)
        hs = np.zeros(cap, np.uint64)
        aw = _words(acc, gather.n)
        self.lib.cyo_run_map(C.byref(self._to_c(gather)), aw.ctypes.data,
                             int(early_exit), C.byref(s), fx.ctypes.data, hh.ctypes.data,
                             hs.ctypes.data, cap)
        del st
        k = min(int(s.iterations), cap)
        return MapResult(bool(s.cycle_found), int(s.witness) if s.cycle_found else None,
                         int(s.iterations), int(s.kernel_calls), int(s.demoted_total),
                         fx[: gather.n], hh[:k], hs[:k])

    def vector_hash(self, x) -> int:
        x = np.ascontiguousarray(np.asarray(x, np.uint32))
        return int(self.lib.cyo_vector_hash(x.ctypes.data if len(x) else None, len(x)))

    # --- generators (include/cyc_gen.h)
    def preset(self, index: int):
        p = GenParams()
        if self.lib.cyo_gen_preset(index, C.byref(p)) != 0:
            raise ValueError(f"unknown config {index}")
        return p

    def prepare(self, p):
        if self.lib.cyo_gen_prepare(C.byref(p)) != 0:
            raise ValueError("bad generator params")
        return p

    def run_owcty(self, snap: Csr, acc):
        """owcty.cpp:56-87 over the rows of `snap` -> (cycle, witness|None, outer_iterations, final_size)."""
        c, w, it, fs = C.c_int(), C.c_uint32(), C.c_uint64(), C.c_uint64()
        aw = _words(acc, snap.n)
        self.lib.cyo_run_owcty(C.byref(self._to_c(snap)), aw.ctypes.data, C.byref(c), C.byref(w),
                               C.byref(it), C.byref(fs))
        return bool(c.value), (w.value if c.value else None), int(it.value), int(fs.value)

    def generate(self, p):
        e = np.zeros((int(p.m), 2), np.uint32)
        acc = np.zeros(max((int(p.n) + 63) // 64, 1), np.uint64)
        self.lib.cyo_generate(C.byref(p), e.ctypes.data if p.m else None, acc.ctypes.data)
        return int(p.n), e, acc


class RefParseError(RuntimeError):
    """cycheck::ParseError raised by the reference; str() = what()."""


class Reference:
    """The reference implementation (compiled from /root/reference sources)."""

    def __init__(self, path: str = REFERENCE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference build missing: {path}")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_snapshot_new.argtypes = [_P, C.c_uint64, C.c_uint32, _P, C.c_int, C.POINTER(_P)]
        L.ref_snapshot_gen.argtypes = [_P, C.c_int, C.POINTER(_P)]
        L.ref_snapshot_free.argtypes = [_P]
        L.ref_snapshot_info.argtypes = [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)]
        L.ref_snapshot_export.argtypes = [_P, _P, _P, _P, _P]
        L.ref_restrict.argtypes = [_P, C.POINTER(_P)]
        L.ref_step.argtypes = [_P, _P, _P, C.c_int, _P, C.POINTER(C.c_int), C.POINTER(C.c_uint32)]
        L.ref_fixpoint.argtypes = [_P, _P, C.c_int, C.c_int, _P, C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_uint32)]
        L.ref_demote.argtypes = [_P, C.c_uint32, _P, _P, _P, C.POINTER(C.c_uint64)]
        L.ref_run_map.argtypes = [_P, _P, C.c_int, C.c_int, _P, _P, _P, _P, C.c_uint64, C.c_int]
        L.ref_scc_verdict.argtypes = [_P, C.POINTER(C.c_int)]
        L.ref_run_owcty.argtypes = [_P, _P, _P]
        L.ref_explicit_parse.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(_P)]
        L.ref_explicit_info.argtypes = [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.ref_explicit_info.restype = None
        L.ref_explicit_export.argtypes = [_P, _P, _P]
        L.ref_explicit_export.restype = None
        L.ref_explicit_free.argtypes = [_P]
        L.ref_explicit_free.restype = None
        L.ref_explicit_snapshot.argtypes = [_P, C.c_int, C.POINTER(_P)]
        L.ref_time_steps.argtypes = [_P, C.c_int, C.c_uint64, C.c_double, _P, C.POINTER(C.c_uint64)]
        L.ref_time_build.argtypes = [_P, C.c_int, C.POINTER(C.c_double)]
        L.ref_hw_threads.restype = C.c_int
        L.ref_ttv.argtypes = [_P, C.c_int, C.c_int, C.c_int, _P, C.c_int, _P, _P]
        L.ref_snapshot_gen_fast.argtypes = [_P, C.c_int, C.c_int, C.POINTER(_P)]

    def _ok(self, rc: int) -> None:
        if rc != 0:
            msg = self.lib.ref_last_error().decode(errors="replace")
            raise {1: ValueError, 2: MemoryError, 5: RefParseError}.get(rc, RuntimeError)(msg)

    def parse_explicit(self, text: bytes):
        """parse_explicit_graph (graph.cpp:259-297) -> (n, accepting ids, edges[m,2]);
        raises RefParseError(ParseError::what()) on malformed text."""
        h = _P()
        self._ok(self.lib.ref_explicit_parse(text, len(text), C.byref(h)))
        try:
            n, na, m = C.c_uint32(), C.c_uint64(), C.c_uint64()
            self.lib.ref_explicit_info(h, C.byref(n), C.byref(na), C.byref(m))
            acc = np.zeros(max(na.value, 1), np.uint32)
            e = np.zeros((max(m.value, 1), 2), np.uint32)
            self.lib.ref_explicit_export(h, acc.ctypes.data, e.ctypes.data)
            return int(n.value), acc[: na.value], e[: m.value]
        finally:
            self.lib.ref_explicit_free(h)

    def explicit_snapshot(self, text: bytes, transposed: bool = True) -> "RefSnapshot":
        """load + fill_log + build_snapshot, all by the reference."""
        h = _P()
        self._ok(self.lib.ref_explicit_parse(text, len(text), C.byref(h)))
        try:
            sh = _P()
            self._ok(self.lib.ref_explicit_snapshot(h, int(transposed), C.byref(sh)))
            return RefSnapshot(self, sh)
        finally:
            self.lib.ref_explicit_free(h)

    def snapshot(self, n: int, edges, acc, transposed: bool = True) -> "RefSnapshot":
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        h = _P()
        aw = _words(acc, n)
        self._ok(self.lib.ref_snapshot_new(e.ctypes.data if len(e) else None, len(e), n,
                                           aw.ctypes.data, int(transposed), C.byref(h)))
        return RefSnapshot(self, h)

    def snapshot_gen(self, params, transposed: bool = True) -> "RefSnapshot":
        h = _P()
        self._ok(self.lib.ref_snapshot_gen(C.byref(params), int(transposed), C.byref(h)))
        return RefSnapshot(self, h)

    def snapshot_gen_fast(self, params, transposed: bool = True, threads: int = 0) -> "RefSnapshot":
        """SETUP ONLY: build_snapshot's result for a generated config, built
        with `threads` host threads (ref_driver.cpp ref_snapshot_gen_fast)."""
        h = _P()
        self._ok(self.lib.ref_snapshot_gen_fast(C.byref(params), int(transposed), threads or (os.cpu_count() or 1),
                                                C.byref(h)))
        return RefSnapshot(self, h)

    def demote(self, x, acc):
        x = np.ascontiguousarray(np.asarray(x, np.uint32))
        n = len(x)
        rem = np.zeros(max((n + 63) // 64, 1), np.uint64)
        dem = np.zeros(max(n, 1), np.uint32)
        nd = C.c_uint64()
        aw = _words(acc, n)
        self._ok(self.lib.ref_demote(x.ctypes.data if n else None, n, aw.ctypes.data,
                                     rem.ctypes.data, dem.ctypes.data, C.byref(nd)))
        return rem, dem[: nd.value].copy()

    def time_build(self, params, transposed: bool = True) -> float:
        s = C.c_double()
        self._ok(self.lib.ref_time_build(C.byref(params), int(transposed), C.byref(s)))
        return float(s.value)

    def ttv(self, params, workers=(1,), transposed: bool = True, restrict: bool = False, early_exit: bool = True):
        """CPU time to verdict, phase by phase (ref_driver.cpp ref_ttv): returns
        {"log_fill_s", "build_snapshot_s", "restrict_s", "run_map_s": {w: s},
        "stats": {w: (cycle, witness, iterations, kernel_calls, demoted)}}."""
        w = np.asarray(list(workers), np.int32)
        t = np.zeros(3 + len(w), np.float64)
        st = np.zeros(5 * len(w), np.uint64)
        self._ok(self.lib.ref_ttv(C.byref(params), int(transposed), int(restrict), int(early_exit),
                                  w.ctypes.data, len(w), t.ctypes.data, st.ctypes.data))
        return {"log_fill_s": float(t[0]), "build_snapshot_s": float(t[1]), "restrict_s": float(t[2]),
                "run_map_s": {int(x): float(t[3 + i]) for i, x in enumerate(w)},
                "stats": {int(x): tuple(int(v) for v in st[5 * i:5 * i + 5]) for i, x in enumerate(w)}}

    def hw_threads(self) -> int:
        return int(self.lib.ref_hw_threads())


class RefSnapshot:
    def __init__(self, ref: Reference, h):
        self.ref, self.h = ref, h
        n, m = C.c_uint32(), C.c_uint64()
        ref.lib.ref_snapshot_info(h, C.byref(n), C.byref(m))
        self.n, self.m = int(n.value), int(m.value)

    def __del__(self):
        try:
            self.ref.lib.ref_snapshot_free(self.h)
        except Exception:
            pass

    def export(self):
        off = np.zeros(self.n + 1, np.uint64)
        col = np.zeros(max(self.m, 1), np.uint32)
        acc = np.zeros(max((self.n + 63) // 64, 1), np.uint64)
        kept = np.zeros(max(self.n, 1), np.uint32)
        self.ref.lib.ref_snapshot_export(self.h, off.ctypes.data, col.ctypes.data, acc.ctypes.data,
                                         kept.ctypes.data)
        return Csr(self.n, off, col[: self.m]), acc, kept[: self.n]

    def restrict(self) -> "RefSnapshot":
        h = _P()
        self.ref._ok(self.ref.lib.ref_restrict(self.h, C.byref(h)))
        return RefSnapshot(self.ref, h)

    def step(self, x, acc=None, workers: int = 1):
        x = np.ascontiguousarray(np.asarray(x, np.uint32))
        out = np.zeros(max(self.n, 1), np.uint32)
        ch, w = C.c_int(), C.c_uint32()
        aw = None if acc is None else _words(acc, self.n)
        self.ref._ok(self.ref.lib.ref_step(self.h, x.ctypes.data if self.n else None,
                                           None if aw is None else aw.ctypes.data,
                                           workers, out.ctypes.data, C.byref(ch), C.byref(w)))
        return out[: self.n], bool(ch.value), (None if w.value == NONE else int(w.value))

    def fixpoint(self, acc=None, early_exit: bool = True, workers: int = 1):
        vals = np.zeros(max(self.n, 1), np.uint32)
        steps, w = C.c_uint64(), C.c_uint32()
        aw = None if acc is None else _words(acc, self.n)
        self.ref._ok(self.ref.lib.ref_fixpoint(self.h, None if aw is None else aw.ctypes.data,
                                               int(early_exit), workers, vals.ctypes.data,
                                               C.byref(steps), C.byref(w)))
        return vals[: self.n], int(steps.value), (None if w.value == NONE else int(w.value))

    def run_map(self, acc=None, early_exit: bool = True, workers: int = 1, cap: int = 1 << 16,
                check_run_map: bool = True) -> MapResult:
        st = np.zeros(5, np.uint64)
        fx = np.zeros(max(self.n, 1), np.uint32)
        hh = np.zeros(cap, np.uint64)
        hs = np.zeros(cap, np.uint64)
        aw = None if acc is None else _words(acc, self.n)
        self.ref._ok(self.ref.lib.ref_run_map(self.h, None if aw is None else aw.ctypes.data,
                                              int(early_exit), workers, st.ctypes.data, fx.ctypes.data,
                                              hh.ctypes.data, hs.ctypes.data, cap, int(check_run_map)))
        k = min(int(st[2]), cap)
        return MapResult(bool(st[0]), int(st[1]) if st[0] else None, int(st[2]), int(st[3]), int(st[4]),
                         fx[: self.n], hh[:k], hs[:k])

    def scc_verdict(self) -> bool:
        c = C.c_int()
        self.ref._ok(self.ref.lib.ref_scc_verdict(self.h, C.byref(c)))
        return bool(c.value)

    def run_owcty(self, acc=None):
        """run_owcty (owcty.cpp:56-87) -> (cycle, witness|None, outer_iterations, final_size)."""
        out = np.zeros(4, np.uint64)
        aw = None if acc is None else _words(acc, self.n)
        self.ref._ok(self.ref.lib.ref_run_owcty(self.h, None if aw is None else aw.ctypes.data,
                                                out.ctypes.data))
        return bool(out[0]), (int(out[1]) if out[0] else None), int(out[2]), int(out[3])

    def time_steps(self, workers: int, max_steps: int, max_seconds: float):
        t = np.zeros(2, np.float64)
        k = C.c_uint64()
        self.ref._ok(self.ref.lib.ref_time_steps(self.h, workers, max_steps, max_seconds, t.ctypes.data,
                                                 C.byref(k)))
        return float(t[0]), float(t[1]), int(k.value)


def reference_available() -> bool:
    return os.path.exists(REFERENCE_SO)
