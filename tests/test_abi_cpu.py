"""CPU tests of the C-ABI library: it loads without a GPU, exports every symbol
include/cycheck_b200.h declares, its host-only helpers behave, and compute
entry points fail loudly (no silent CPU fallback) when no GPU is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cycheck_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:[A-Za-z_][\w\s\*]*?)\b(cyc_\w+)\s*\(", src, flags=re.M)))


def test_header_declarations_match_binding(eng):
    decl = declared_functions()
    assert len(decl) >= 25
    assert sorted(eng.EXPORTED_SYMBOLS) == decl


def test_library_exports_every_declared_symbol(eng):
    lib = C.CDLL(eng.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(ROOT, "paper_0912_2555_b200", "_lib", "libcycheck_b200.so")],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout and "sm_80" not in out.stdout


def test_generator_presets_match_oracle(eng, R):
    for idx in (1, 2, 3, 4, 5):
        a, b = eng.preset(idx), R.preset(idx)
        for f, _ in a._fields_:
            assert getattr(a, f) == getattr(b, f), (idx, f)


def test_shard_bounds_matches_reference_partition(eng):
    # map_engine.cpp:35-43 bounds[w] = lower_bound(offsets, total*w/W), capped at n
    rng = np.random.default_rng(5)
    for _ in range(50):
        n = int(rng.integers(1, 300))
        deg = rng.integers(0, 20, size=n)
        off = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
        for parts in (1, 2, 3, 4, 8):
            b = eng.shard_bounds(off, parts)
            total = int(off[-1])
            want = [0] + [min(int(np.searchsorted(off, total * w // parts, side="left")), n)
                          for w in range(1, parts)] + [n]
            assert b.tolist() == want


def test_bitset_semantics(eng):
    b = eng.Bitset(70)
    for i in (0, 63, 64, 69):
        b.set(i)
    assert b.count() == 4 and b.test(69) and not b.test(1)
    b.reset(63)
    assert b.count() == 3
    assert eng.Bitset.all_set(70).count() == 70  # tail trimmed (bitset.hpp:65-67)
    assert eng.Bitset.from_bools(b.to_bools()) == b
    with pytest.raises(eng.ContractError):
        b.set(70)


def test_edgelog_contract_and_limits(eng):
    log = eng.EdgeLog(eng.EdgeLog.Limits(max_vertices=2, max_edges=1))
    assert log.add_vertex(True) == 0 and log.add_vertex(False) == 1
    with pytest.raises(eng.ResourceLimitError):
        log.add_vertex(False)
    with pytest.raises(eng.ContractError):
        log.append_edge(0, 5)  # graph.cpp:43-46
    log.append_edge(0, 1)
    with pytest.raises(eng.ResourceLimitError):
        log.append_edge(1, 0)
    assert log.accepting_prefix(2).to_bools().tolist() == [True, False]


def test_no_silent_cpu_fallback_without_gpu(eng):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(eng.CycheckError):
        eng.Context(0)
