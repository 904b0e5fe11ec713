"""ctypes binding of the C ABI in include/cycheck_b200.h.

The shared library is built in-tree (paper_0912_2555_b200/_lib/) by
``__graft_entry__.build()``. There is no fallback: if the library is missing,
importing this module raises, so nothing can silently run on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CYC_LIB_PATH: an alternative build of the same library (tuning experiments)
LIB_PATH = os.environ.get("CYC_LIB_PATH") or os.path.join(_HERE, "_lib", "libcycheck_b200.so")


class CycheckError(RuntimeError):
    """Base of the errors raised across the C ABI."""


class ContractError(CycheckError, ValueError):
    """cycheck::ContractError (reference errors.hpp:10-14)."""


class ResourceLimitError(CycheckError):
    """cycheck::ResourceLimitError (reference errors.hpp:16-20), incl. device OOM."""


class CudaError(CycheckError):
    """CUDA runtime failure inside the engine."""


class ParseError(CycheckError):
    """cycheck::ParseError (reference errors.hpp:32-45): code (DiagCode), line, col;
    str() is ParseError::what()."""

    def __init__(self, msg: str, code: int = 0, line: int = 0, col: int = 0):
        super().__init__(msg)
        self.code, self.line, self.col = code, line, col


_ERRORS = {1: ContractError, 2: ResourceLimitError, 3: CudaError, 4: CycheckError, 5: ParseError}

CYC_FORWARD, CYC_TRANSPOSED = 0, 1
CYC_MODE_AUTO, CYC_MODE_PULL, CYC_MODE_PUSH = 0, 1, 2
CYC_LAYOUT_AUTO, CYC_LAYOUT_IDENTITY, CYC_LAYOUT_DEGREE = 0, 1, 2


class MapOptionsC(C.Structure):
    _fields_ = [
        ("early_exit", C.c_int32),
        ("mode", C.c_int32),
        ("max_iterations", C.c_uint64),
        ("max_steps", C.c_uint64),
        ("push_alpha", C.c_uint32),
        ("trace_cap", C.c_uint32),
        ("layout", C.c_int32),
        ("reserved", C.c_int32),
    ]


class OwctyStatsC(C.Structure):
    _fields_ = [
        ("outer_iterations", C.c_uint64),
        ("final_size", C.c_uint64),
        ("reach_ms", C.c_double),
        ("elim_ms", C.c_double),
    ]


class MapStatsC(C.Structure):
    _fields_ = [
        ("cycle_found", C.c_int32),
        ("witness", C.c_uint32),
        ("iterations", C.c_uint64),
        ("kernel_calls", C.c_uint64),
        ("demoted_total", C.c_uint64),
        ("steps_last", C.c_uint64),
        ("pull_steps", C.c_uint64),
        ("push_steps", C.c_uint64),
        ("edges_touched", C.c_uint64),
        ("rows_touched", C.c_uint64),
        ("algorithmic_bytes", C.c_uint64),
        ("loop_ms", C.c_double),
        ("grid_blocks", C.c_uint32),
        ("block_threads", C.c_uint32),
        ("plan_ms", C.c_double),
        ("layout", C.c_int32),
        ("world", C.c_int32),
        ("exchanged_rows", C.c_uint64),
    ]


class GenParams(C.Structure):
    """Mirror of cyc_gen_params (include/cyc_gen.h)."""

    _fields_ = [
        ("kind", C.c_int32),
        ("n", C.c_uint32),
        ("m", C.c_uint64),
        ("seed", C.c_uint64),
        ("deg", C.c_uint32),
        ("acc_thr", C.c_uint64),
        ("L", C.c_uint32),
        ("W", C.c_uint32),
        ("S", C.c_uint32),
        ("exit_all", C.c_uint32),
        ("acc_all", C.c_uint32),
        ("scale", C.c_uint32),
        ("edgefactor", C.c_uint32),
        ("thr_a", C.c_uint64),
        ("thr_ab", C.c_uint64),
        ("thr_abc", C.c_uint64),
        ("perm_mul1", C.c_uint64),
        ("perm_mul2", C.c_uint64),
        ("grid_bits", C.c_uint32),
        ("region", C.c_uint32),
        ("plant", C.c_uint32),
        ("reserved", C.c_uint32),
    ]


_P = C.c_void_p
_U32P = C.POINTER(C.c_uint32)
_U64P = C.POINTER(C.c_uint64)

_SIGS = {
    "cyc_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "cyc_ctx_destroy": (None, [_P]),
    "cyc_last_error": (C.c_char_p, []),
    "cyc_launch_count": (C.c_uint64, []),
    "cyc_ctx_synchronize": (C.c_int, [_P]),
    "cyc_ctx_stream": (_P, [_P]),
    "cyc_ctx_set_stream": (C.c_int, [_P, _P, C.c_int]),
    "cyc_ctx_reserve": (C.c_int, [_P, C.c_uint64, C.c_uint32, C.c_int]),
    "cyc_graph_build": (C.c_int, [_P, _P, C.c_uint64, C.c_uint32, _P, C.c_int, C.POINTER(_P)]),
    "cyc_graph_from_csr": (C.c_int, [_P, _P, _P, C.c_uint32, C.c_uint64, _P, C.c_int, C.POINTER(_P)]),
    "cyc_graph_extend": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_uint32, _P, C.POINTER(_P)]),
    "cyc_graph_log_prefix": (C.c_int, [_P, _U64P]),
    "cyc_graph_restrict": (C.c_int, [_P, _P, C.POINTER(_P)]),
    "cyc_graph_destroy": (None, [_P]),
    "cyc_graph_info": (C.c_int, [_P, _U32P, _U64P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "cyc_graph_export": (C.c_int, [_P, _P, _P, _P, _P]),
    "cyc_graph_export_gather": (C.c_int, [_P, _P, _P]),
    "cyc_map_step": (C.c_int, [_P, _P, _P, _P, _P, C.POINTER(C.c_int32), _U32P]),
    "cyc_fixpoint": (C.c_int, [_P, _P, _P, C.POINTER(MapOptionsC), _P, _U64P, _U32P]),
    "cyc_demote": (C.c_int, [_P, _P, C.c_uint32, _P, _P, _P, _U64P]),
    "cyc_map_run": (C.c_int, [_P, _P, _P, C.POINTER(MapOptionsC), C.POINTER(MapStatsC), _P, _P, _P,
                              C.c_uint64]),
    "cyc_explicit_parse": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(_P)]),
    "cyc_explicit_load_binary": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(_P)]),
    "cyc_last_parse_error": (C.c_int, [C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "cyc_explicit_info": (C.c_int, [_P, _U32P, _U64P, _U64P]),
    "cyc_explicit_export": (C.c_int, [_P, _P, _P]),
    "cyc_explicit_snapshot": (C.c_int, [_P, _P, C.c_int, C.POINTER(_P)]),
    "cyc_explicit_destroy": (None, [_P]),
    "cyc_check": (C.c_int, [_P, _P, C.c_uint64, C.c_uint32, _P, C.c_int, C.c_int,
                            C.POINTER(MapOptionsC), C.POINTER(MapStatsC), C.POINTER(C.c_double)]),
    "cyc_scc_verdict": (C.c_int, [_P, _P, C.POINTER(C.c_int32), _U32P, _P, _U64P]),
    "cyc_owcty": (C.c_int, [_P, _P, _P, C.POINTER(C.c_int32), _U32P, C.POINTER(OwctyStatsC)]),
    "cyc_gen_fill": (C.c_int, [_P, _P, _P, _P]),  # any cyc_gen_params mirror (oracle has its own)
    "cyc_gen_preset": (C.c_int, [C.c_int, C.POINTER(GenParams)]),
    "cyc_gen_prepare": (C.c_int, [C.POINTER(GenParams)]),
    "cyc_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_P)]),
    "cyc_host_free": (None, [_P]),
    "cyc_device_alloc": (C.c_int, [_P, C.c_size_t, C.POINTER(_P)]),
    "cyc_device_free": (None, [_P, _P]),
    "cyc_memcpy": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "cyc_memcpy_async": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "cyc_flush_l2": (C.c_int, [_P, C.c_size_t]),
    "cyc_shard_bounds": (C.c_int, [_P, C.c_uint32, C.c_int, _P]),
    "cyc_map_trace": (C.c_int, [_P, _P, C.c_uint32, C.POINTER(C.c_uint32)]),
    "cyc_shard_step": (C.c_int, [_P, _P, C.c_uint32, C.c_uint32, _P, _P, _P, _P, _P, C.c_int]),
    "cyc_shard_post": (C.c_int, [_P, _P, _P, _P, _P, C.c_int, C.c_uint32, _P]),
    "cyc_shard_collect": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P, _P, C.c_uint32, _P, _P, C.c_int, _P, _P,
                                    _P, _P, _P]),
    "cyc_shard_push": (C.c_int, [_P, _P, C.c_uint32, C.c_uint32, _P, C.c_int, C.c_uint32, _P, _P, _P, _P, _P,
                                 _P]),
    "cyc_shard_post_sparse": (C.c_int, [_P, _P, _P, _P, C.c_int, C.c_uint32, _P]),
    "cyc_shard_demote": (C.c_int, [_P, _P, C.c_uint32, _P, _P, _P]),
    "cyc_fused_open": (C.c_int, [_P, _P, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.POINTER(_P), _P]),
    "cyc_fused_connect": (C.c_int, [_P, _P]),
    "cyc_fused_run": (C.c_int, [_P, _P, C.c_int, C.POINTER(MapStatsC), _P]),
    "cyc_fused_close": (None, [_P]),
    "cyc_shard_build": (C.c_int, [_P, _P, C.c_uint64, C.c_uint32, _P, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(_P)]),
    "cyc_shard_info": (C.c_int, [_P, _U32P, _U32P, _U64P, _U64P]),
    "cyc_shard_handle": (C.c_int, [_P, _P]),
    "cyc_shard_connect": (C.c_int, [_P, _P]),
    "cyc_shard_connect_local": (C.c_int, [_P, C.c_int]),
    "cyc_shard_run_map": (C.c_int, [_P, C.c_int, _P, C.POINTER(MapOptionsC), C.POINTER(MapStatsC), _P, _P, _P,
                                    C.c_uint64]),
    "cyc_shard_destroy": (None, [_P]),
}
SHARD_HANDLE_BYTES = 512  # CYC_SHARD_HANDLE_BYTES

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def lib() -> C.CDLL:
    """Loads the in-tree engine library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"B200 engine library missing at {LIB_PATH}; run __graft_entry__.build() "
                "(there is no CPU fallback)"
            )
        lib_ = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib_, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib_
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().cyc_last_error().decode(errors="replace")
        if status == 5:
            c, ln, col = C.c_int(), C.c_int(), C.c_int()
            lib().cyc_last_parse_error(C.byref(c), C.byref(ln), C.byref(col))
            raise ParseError(msg, c.value, ln.value, col.value)
        raise _ERRORS.get(status, CycheckError)(msg)


def ptr(a) -> C.c_void_p | None:
    """Address of a numpy array, a torch tensor, or an int; None passes NULL."""
    if a is None:
        return None
    if isinstance(a, int):
        return C.c_void_p(a)
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ContractError("array must be C-contiguous")
        return C.c_void_p(a.ctypes.data)
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    raise TypeError(f"cannot pass {type(a)!r} across the C ABI")


def preset(index: int) -> GenParams:
    p = GenParams()
    check(lib().cyc_gen_preset(index, C.byref(p)))
    return p


def prepare(p: GenParams) -> GenParams:
    check(lib().cyc_gen_prepare(C.byref(p)))
    return p
