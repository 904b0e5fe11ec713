"""GPU parity: every engine entry point, called through the C ABI, against the
oracle restatement (pinned to the reference in test_oracle.py) and the golden
fixtures made by the reference itself. Integer work: bit-exact everywhere."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.json")
MODES = ("auto", "pull", "push")
G1 = [(0, 1), (1, 2), (2, 1)]


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def snap_of(eng, n, edges, acc, transposed=True):
    o = eng.Orientation.transposed if transposed else eng.Orientation.forward
    return eng.build_snapshot((n, np.asarray(edges, np.uint32).reshape(-1, 2), acc), o)


def oracle_run(R, n, edges, acc, transposed, early):
    gat = R.transpose(R.build_snapshot(n, edges, transposed))
    return R.run_map(gat, acc, early)


def assert_same_run(run, ref):
    got = (run.verdict.cycle_found(), run.verdict.witness, run.stats.iterations,
           run.stats.kernel_calls, run.stats.demoted_total)
    want = (ref.cycle, ref.witness, ref.iterations, ref.kernel_calls, ref.demoted_total)
    assert got == want
    assert np.array_equal(run.final_values, ref.final_x)
    assert np.array_equal(run.iter_hash, ref.iter_hash[: len(run.iter_hash)])
    assert np.array_equal(run.iter_steps, ref.iter_steps[: len(run.iter_steps)])


# ------------------------------------------------------------------ KATs
def test_kat_snapshot(eng):
    s = snap_of(eng, 3, G1, [False, True, False], True)
    assert s.row_offsets.tolist() == [0, 0, 2, 3] and s.col_indices.tolist() == [0, 2, 1]
    off, col = s.gather_index()
    assert off.tolist() == [0, 1, 2, 3] and col.tolist() == [1, 2, 1]
    f = snap_of(eng, 3, G1, [False, True, False], False)
    assert f.row_offsets.tolist() == [0, 1, 2, 3] and f.col_indices.tolist() == [1, 2, 1]
    e = snap_of(eng, 0, np.zeros((0, 2)), np.zeros(0, bool))
    assert e.row_offsets.tolist() == [0] and e.m == 0


def test_kat_steps_and_fixpoint(eng):
    s = snap_of(eng, 3, G1, [False, True, False])
    x1, ch = eng.propagate_step(s, eng.init_vector(s), s.accepting)
    assert x1.tolist() == [2, 0, 2] and ch
    r = eng.MaxPropagation(s).step(x1, s.accepting)
    assert r.changed and r.self_witness == 1
    for mode in MODES:
        fr = eng.fixpoint(s, s.accepting, eng.MapOptions(mode=mode))
        assert fr.witness == 1 and fr.steps == 2 and fr.values.tolist() == [2, 2, 2]
    chain = snap_of(eng, 3, [(0, 1), (1, 2)], [False, False, True])
    for mode in MODES:
        fr = eng.fixpoint(chain, chain.accepting, eng.MapOptions(mode=mode))
        assert fr.values.tolist() == [3, 3, 0] and fr.steps == 3 and fr.witness is None
    empty = snap_of(eng, 0, np.zeros((0, 2)), np.zeros(0, bool))
    fr = eng.fixpoint(empty, empty.accepting)
    assert fr.steps == 1 and fr.witness is None
    nof = snap_of(eng, 4, [(0, 1), (1, 2)], [False] * 4)
    fr = eng.fixpoint(nof, nof.accepting)
    assert fr.steps == 1 and fr.values.tolist() == [0, 0, 0, 0]


def test_kat_demote(eng):
    d = eng.demote([3, 3, 0], [False, False, True])
    assert d.demoted.tolist() == [2] and d.remaining.count() == 0
    d = eng.demote([0, 0, 0, 0], [True, False, True, True])
    assert d.demoted.tolist() == [] and d.remaining.indices().tolist() == [0, 2, 3]
    d = eng.demote([4, 0, 4, 0], [False, True, False, True])
    assert d.demoted.tolist() == [3] and d.remaining.indices().tolist() == [1]


def test_kat_run_map(eng):
    s = snap_of(eng, 1, [(0, 0)], [True])
    v, st = eng.run_map(s, s.accepting)
    assert v.cycle_found() and v.witness == 0 and st.iterations == 1
    dag = snap_of(eng, 3, [(0, 1), (1, 2)], [True, True, True])
    v, st = eng.run_map(dag, dag.accepting)
    assert not v.cycle_found()
    none = snap_of(eng, 2, [(0, 1)], [False, False])
    v, st = eng.run_map(none, none.accepting)
    assert not v.cycle_found() and st.iterations == 0 and st.kernel_calls == 0


def test_kat_restrict(eng):
    s = snap_of(eng, 3, G1, [False, True, False])
    r = eng.restrict_to_accepting_sccs(s)
    assert r.kept.tolist() == [1, 2] and r.snapshot.n == 2
    assert r.snapshot.row_offsets.tolist() == [0, 1, 2] and r.snapshot.col_indices.tolist() == [1, 0]
    assert r.snapshot.accepting.indices().tolist() == [0]
    c = snap_of(eng, 3, [(0, 1), (1, 2)], [False, False, True])
    assert eng.restrict_to_accepting_sccs(c).kept.tolist() == []


def test_contract_errors(eng):
    with pytest.raises(eng.ContractError):
        snap_of(eng, 2, [(0, 5)], [False, False])
    s = snap_of(eng, 3, G1, [False, True, False])
    with pytest.raises(eng.ContractError):
        eng.propagate_step(s, np.zeros(4, np.uint32), s.accepting)
    with pytest.raises(eng.ContractError):
        eng.run_map(s, np.zeros(5, bool))


# -------------------------------------------------------------- golden
def test_golden_random(eng, golden):
    for case in golden["random"]:
        n = case["n"]
        acc = np.zeros(n, bool)
        acc[case["accepting"]] = True
        s = snap_of(eng, n, case["edges"], acc)
        assert s.row_offsets.tolist() == case["row_offsets"]
        assert s.col_indices.tolist() == case["col_indices"]
        x1, ch = eng.propagate_step(s, eng.init_vector(s), acc)
        assert x1.tolist() == case["step1"] and ch == case["step1_changed"]
        for mode in MODES:
            for key, early in (("early", True), ("full", False)):
                run = eng.run_map_detailed(s, acc, eng.MapOptions(early_exit=early, mode=mode))
                want = case[key]
                assert (run.verdict.cycle_found(), run.verdict.witness, run.stats.iterations,
                        run.stats.kernel_calls, run.stats.demoted_total) == (
                    want["cycle"], want["witness"], want["iterations"], want["kernel_calls"],
                    want["demoted_total"]), (mode, key)
                assert run.final_values.tolist() == case["final_x_" + key]
                assert [int(h) for h in run.iter_hash] == want["iter_hash"]


@pytest.mark.parametrize("name", ["c1", "c2_L16", "c5_L16", "c3_s12", "c4_g6"])
def test_golden_configs(eng, R, golden, name):
    cfg = golden["configs"][name]
    p = R.preset(cfg["config"])
    for k, v in cfg["overrides"].items():
        setattr(p, k, v)
    R.prepare(p)
    n, e, accw = R.generate(p)
    # the device generator reproduces the same log
    de = np.zeros_like(e)
    da = np.zeros_like(accw)
    from paper_0912_2555_b200 import _abi
    ctx = eng.default_context()
    _abi.check(_abi.lib().cyc_gen_fill(ctx.handle, _abi.C.byref(p), _abi.ptr(de), _abi.ptr(da)))
    assert np.array_equal(de, e) and np.array_equal(da, accw)
    acc = eng.Bitset.from_words(accw, n)
    for orient, tr in (("transposed", True), ("forward", False)):
        s = snap_of(eng, n, e, acc, tr)
        want = cfg[orient]
        assert s.m == want["m"]
        assert digest(s.row_offsets) == want["off_digest"] and digest(s.col_indices) == want["col_digest"]
        for mode in MODES:
            for key, early in (("early", True), ("full", False)):
                run = eng.run_map_detailed(s, acc, eng.MapOptions(early_exit=early, mode=mode))
                w = want[key]
                assert (run.verdict.cycle_found(), run.verdict.witness, run.stats.iterations,
                        run.stats.kernel_calls, run.stats.demoted_total) == (
                    w["cycle"], w["witness"], w["iterations"], w["kernel_calls"], w["demoted_total"]), (
                    orient, mode, key)
                assert digest(run.final_values) == w["final_x_digest"]
                assert [int(h) for h in run.iter_hash[:256]] == w["iter_hash"]
        wo = want["owcty"]
        v, st = eng.run_owcty(s)
        assert (v.cycle_found(), v.witness, st.outer_iterations, st.final_size) == (
            wo["cycle"], wo["witness"], wo["outer_iterations"], wo["final_size"])
        r = eng.restrict_to_accepting_sccs(s)
        wr = want["restricted"]
        assert (r.snapshot.n, r.snapshot.m) == (wr["n"], wr["m"])
        assert digest(r.kept) == wr["kept_digest"]
        assert digest(r.snapshot.row_offsets) == wr["off_digest"]
        assert digest(r.snapshot.col_indices) == wr["col_digest"]
        if wr["n"]:
            v, st = eng.run_map(r.snapshot, r.snapshot.accepting)
            w = wr["early"]
            assert (v.cycle_found(), st.iterations, st.kernel_calls) == (w["cycle"], w["iterations"],
                                                                         w["kernel_calls"])
            if w["cycle"]:
                assert int(r.kept[v.witness]) == w["witness_original"]


# ------------------------------------------------------- differential
def random_graph(rng, n, m, hubs=0):
    e = rng.integers(0, n, size=(m, 2)).astype(np.uint32)
    if hubs:
        # a few hub rows/columns beyond the small/medium/heavy thresholds
        for h in range(hubs):
            d = int(rng.integers(300, 9000))
            hub = int(rng.integers(0, n))
            other = rng.integers(0, n, size=d).astype(np.uint32)
            pair = np.stack([np.full(d, hub, np.uint32), other], 1) if h % 2 else \
                np.stack([other, np.full(d, hub, np.uint32)], 1)
            e = np.concatenate([e, pair])
    return e


@pytest.mark.parametrize("seed", range(6))
def test_differential_random(eng, R, seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(200, 20000))
    m = int(n * rng.choice([1, 2, 4, 8]))
    e = random_graph(rng, n, m, hubs=seed % 3)
    acc = rng.random(n) < rng.choice([0.001, 0.01, 0.05, 0.3])
    for tr in (True, False):
        s = snap_of(eng, n, e, acc, tr)
        g = R.build_snapshot(n, e, tr)
        assert np.array_equal(s.row_offsets, g.off) and np.array_equal(s.col_indices, g.col)
        gat = R.transpose(g)
        off, col = s.gather_index()
        assert np.array_equal(off, gat.off) and np.array_equal(col, gat.col)
        for early in (True, False):
            ref = R.run_map(gat, acc, early)
            for mode in MODES:
                run = eng.run_map_detailed(s, acc, eng.MapOptions(early_exit=early, mode=mode))
                assert_same_run(run, ref)


def test_per_step_vectors(eng, R):
    # Jacobi step-for-step: x after k steps, all step kinds
    rng = np.random.default_rng(77)
    n, m = 3000, 6000
    e = random_graph(rng, n, m, hubs=2)
    acc = rng.random(n) < 0.02
    s = snap_of(eng, n, e, acc)
    gat = R.transpose(R.build_snapshot(n, e, True))
    x = np.zeros(n, np.uint32)
    for k in range(1, 12):
        x, ch, w = R.step(gat, x, acc)
        for mode in MODES:
            fr = eng.fixpoint(s, acc, eng.MapOptions(early_exit=False, mode=mode), max_steps=k)
            assert fr.steps <= k
            assert np.array_equal(fr.values, x), (k, mode)
        if not ch:
            break


def test_dense_step_matches_oracle_on_arbitrary_vectors(eng, R):
    rng = np.random.default_rng(9)
    n = 5000
    e = random_graph(rng, n, 20000, hubs=2)
    acc = rng.random(n) < 0.1
    s = snap_of(eng, n, e, acc)
    gat = R.transpose(R.build_snapshot(n, e, True))
    for _ in range(5):
        x = rng.integers(0, n + 1, size=n).astype(np.uint32)
        want = R.step(gat, x, acc)
        r = eng.MaxPropagation(s)
        res = r.step(x, acc)
        assert np.array_equal(r.last_out, want[0])
        assert res.changed == want[1] and res.self_witness == want[2]


def test_restrict_differential(eng, R):
    rng = np.random.default_rng(31)
    for t in range(8):
        n = int(rng.integers(50, 5000))
        e = random_graph(rng, n, int(n * rng.choice([1, 2, 3])), hubs=t % 2)
        acc = rng.random(n) < rng.choice([0.01, 0.1, 0.5])
        for tr in (True, False):
            s = snap_of(eng, n, e, acc, tr)
            g = R.build_snapshot(n, e, tr)
            rg, racc, kept = R.restrict(g, acc)
            r = eng.restrict_to_accepting_sccs(s)
            assert np.array_equal(r.kept, kept)
            assert np.array_equal(r.snapshot.row_offsets, rg.off)
            assert np.array_equal(r.snapshot.col_indices, rg.col)
            assert np.array_equal(r.snapshot.accepting.words()[: len(racc)], racc[: len(r.snapshot.accepting.words())])
            # verdict preserved under restriction (graph.hpp:110-113)
            v1, _ = eng.run_map(s, acc)
            v2, _ = eng.run_map(r.snapshot, r.snapshot.accepting)
            assert v1.cycle_found() == v2.cycle_found()


def test_check_pipeline(eng, R):
    rng = np.random.default_rng(4)
    n = 4000
    e = random_graph(rng, n, 12000)
    acc = rng.random(n) < 0.05
    for restrict in (False, True):
        v, st = eng.check_graph(n, e, acc, eng.Orientation.transposed, restrict)
        g = R.build_snapshot(n, e, True)
        if restrict:
            rg, racc, kept = R.restrict(g, acc)
            ref = R.run_map(R.transpose(rg), racc, True)
            wit = int(kept[ref.witness]) if ref.cycle else None
        else:
            ref = R.run_map(R.transpose(g), acc, True)
            wit = ref.witness
        assert (v.cycle_found(), v.witness, st.iterations, st.kernel_calls) == (
            ref.cycle, wit, ref.iterations, ref.kernel_calls)


# ------------------------------------------------------- full-size properties
def test_c2_full_size_closed_form(eng):
    """Config 2 at 2^22: iterations = L+1 = 65, kernel_calls = (L+1)^2 = 4225,
    no cycle, one connector demoted per round."""
    p = eng.preset(2)
    from paper_0912_2555_b200 import _abi
    ctx = eng.default_context()
    e = np.zeros((p.m, 2), np.uint32)
    a = np.zeros((p.n + 63) // 64, np.uint64)
    _abi.check(_abi.lib().cyc_gen_fill(ctx.handle, _abi.C.byref(p), _abi.ptr(e), _abi.ptr(a)))
    s = snap_of(eng, p.n, e, eng.Bitset.from_words(a, p.n))
    for mode in MODES:
        v, st = eng.run_map(s, s.accepting, eng.MapOptions(mode=mode))
        assert not v.cycle_found()
        assert (st.iterations, st.kernel_calls, st.demoted_total) == (65, 65 ** 2, 64), mode


def test_monotone_and_idempotent(eng, R):
    rng = np.random.default_rng(12)
    n = 20000
    e = random_graph(rng, n, 60000)
    acc = rng.random(n) < 0.01
    s = snap_of(eng, n, e, acc)
    fr = eng.fixpoint(s, acc, eng.MapOptions(early_exit=False))
    # idempotence at the fixpoint
    x2, ch = eng.propagate_step(s, fr.values, acc)
    assert not ch and np.array_equal(x2, fr.values)


# ------------------------------------------------------- larger instances
@pytest.mark.parametrize("scale", [14, 16])
def test_rmat_parity(eng, R, scale):
    """R-MAT (config 3 family) with real hubs: build (all row classes incl. the
    tiled hub sort), gather index, run_map in both modes and all step kinds,
    restriction."""
    p = R.preset(3)
    p.scale = scale
    R.prepare(p)
    n, e, accw = R.generate(p)
    acc = eng.Bitset.from_words(accw, n)
    s = snap_of(eng, n, e, acc)
    g = R.build_snapshot(n, e, True)
    assert np.array_equal(s.row_offsets, g.off) and np.array_equal(s.col_indices, g.col)
    gat = R.transpose(g)
    off, col = s.gather_index()
    assert np.array_equal(off, gat.off) and np.array_equal(col, gat.col)
    for early in (True, False):
        ref = R.run_map(gat, accw, early)
        for mode in MODES:
            assert_same_run(eng.run_map_detailed(s, acc, eng.MapOptions(early_exit=early, mode=mode)), ref)
    rg, racc, kept = R.restrict(g, accw)
    r = eng.restrict_to_accepting_sccs(s)
    assert np.array_equal(r.kept, kept)
    assert np.array_equal(r.snapshot.row_offsets, rg.off) and np.array_equal(r.snapshot.col_indices, rg.col)


def test_chain_family_closed_form(eng, R):
    """Config 5 family (only the sink connector accepting, ring exits from
    member S/2): one MAP iteration of L*(S/2+2)+7-ish dense-equivalent steps,
    equal to the oracle in every step kind."""
    p = R.preset(5)
    p.L, p.W, p.S = 12, 16, 32
    R.prepare(p)
    n, e, accw = R.generate(p)
    s = snap_of(eng, n, e, eng.Bitset.from_words(accw, n))
    ref = R.run_map(R.transpose(R.build_snapshot(n, e, True)), accw, True)
    assert ref.iterations == 1 and not ref.cycle
    for mode in MODES:
        assert_same_run(eng.run_map_detailed(s, eng.Bitset.from_words(accw, n), eng.MapOptions(mode=mode)), ref)


def test_forward_orientation_with_restriction(eng, R):
    """The explorer's map_orientation may be forward (explore.hpp:40): the
    whole pipeline (build, restrict, run_map, witness back-mapping) in the
    forward orientation."""
    p = R.preset(1)
    p.n = 1 << 14
    R.prepare(p)
    n, e, accw = R.generate(p)
    acc = eng.Bitset.from_words(accw, n)
    for restrict in (False, True):
        v, st = eng.check_graph(n, e, acc, eng.Orientation.forward, restrict)
        g = R.build_snapshot(n, e, False)
        if restrict:
            rg, racc, kept = R.restrict(g, accw)
            ref = R.run_map(R.transpose(rg), racc, True)
            wit = int(kept[ref.witness]) if ref.cycle else None
        else:
            ref = R.run_map(R.transpose(g), accw, True)
            wit = ref.witness
        assert (v.cycle_found(), v.witness, st.iterations, st.kernel_calls) == (
            ref.cycle, wit, ref.iterations, ref.kernel_calls)


def test_device_scc_verdict(eng, R, REF):
    """scc_verdict on the device equals the reference's (oracle.cpp:32-98):
    verdict, witness (smallest) and the sorted cyclic accepting vertices; and
    agrees with MAP's verdict."""
    rng = np.random.default_rng(404)
    for t in range(12):
        n = int(rng.integers(2, 3000))
        e = random_graph(rng, n, int(n * rng.choice([1, 2])), hubs=t % 2)
        acc = rng.random(n) < rng.choice([0.01, 0.1, 0.4])
        s = snap_of(eng, n, e, acc)
        ov = eng.scc_verdict(s)
        keep = R.keep_mask(R.build_snapshot(n, e, True), acc)
        want = np.flatnonzero(keep & acc).astype(np.uint32)
        assert np.array_equal(ov.cyclic_accepting, want)
        assert ov.verdict.cycle_found() == (len(want) > 0)
        if len(want):
            assert ov.verdict.witness == int(want[0])
        rs = REF.snapshot(n, e, acc, True)
        assert ov.verdict.cycle_found() == rs.scc_verdict()
        v, _ = eng.run_map(s, s.accepting)
        assert v.cycle_found() == ov.verdict.cycle_found()


def test_device_owcty(eng, R, REF):
    """run_owcty on the device (owcty.cpp:56-87) equals the reference's on
    forward snapshots — verdict, witness, outer_iterations, final_size — and
    the restatement's on transposed ones; the verdict equals MAP's."""
    rng = np.random.default_rng(606)
    for t in range(16):
        n = int(rng.integers(2, 4000))
        e = random_graph(rng, n, int(n * rng.choice([1, 2])), hubs=2 * (t % 2))
        acc = rng.random(n) < rng.choice([0.01, 0.1, 0.4])
        fwd = t % 4 != 3
        s = snap_of(eng, n, e, acc, transposed=not fwd)
        v, st = eng.run_owcty(s)
        got = (v.cycle_found(), v.witness, st.outer_iterations, st.final_size)
        want = R.run_owcty(R.build_snapshot(n, e, not fwd), acc)
        assert got == want
        if fwd:
            assert got == REF.snapshot(n, e, acc, False).run_owcty()
        mv, _ = eng.run_map(s, s.accepting)
        assert mv.cycle_found() == v.cycle_found()
    # explicit accepting override and the C2 family (L+1 layers, no cycle)
    n = 50
    e = np.array([[i, (i + 1) % n] for i in range(n)], np.uint32)
    s = snap_of(eng, n, e, np.zeros(n, bool), transposed=False)
    assert not eng.run_owcty(s)[0].cycle_found()
    acc = np.zeros(n, bool)
    acc[[7, 30]] = True
    v, st = eng.run_owcty(s, acc)
    assert (v.witness, st.final_size, st.outer_iterations) == (7, n, 1)
    p = eng.preset(2)
    p.L, p.W, p.S = 8, 64, 8
    eng.prepare(p)
    gn, ge, ga = R.generate(p)
    s = eng.build_snapshot((gn, ge, eng.Bitset.from_words(ga, gn)), eng.Orientation.forward)
    v, st = eng.run_owcty(s)
    gacc = np.unpackbits(ga.view(np.uint8), bitorder="little")[:gn].astype(bool)
    want = REF.snapshot(gn, ge, gacc, False).run_owcty()
    assert (v.cycle_found(), v.witness, st.outer_iterations, st.final_size) == want


def test_extend_snapshot_equals_rebuild(eng, R):
    """Incremental snapshots: growing a device snapshot round by
    round, as the explorer's detector does (explore.cpp:71-124), gives exactly
    the snapshot a full rebuild of the prefix gives (graph.cpp:63-105) — both
    CSRs, accepting bits — and the same run_map."""
    rng = np.random.default_rng(1717)
    for trial in range(6):
        n_final = int(rng.integers(50, 6000))
        m_final = int(n_final * rng.choice([2, 4]))
        e = random_graph(rng, n_final, m_final, hubs=trial % 2)
        # make the log grow like an explorer: vertex v appears before its edges
        order = np.argsort(np.maximum(e[:, 0], e[:, 1]), kind="stable")
        e = np.ascontiguousarray(e[order])
        acc = rng.random(n_final) < 0.1
        tr = bool(trial % 3)
        o = eng.Orientation.transposed if tr else eng.Orientation.forward
        cuts = sorted(set(int(c) for c in rng.integers(1, len(e), size=4))) + [len(e)]
        m0 = cuts[0]
        n0 = int(e[:m0].max()) + 1
        s = eng.build_snapshot((n0, e[:m0], acc[:n0]), o)
        prev_m = m0
        for c in cuts[1:]:
            n1 = max(int(e[:c].max()) + 1, s.n)
            s = eng.extend_snapshot(s, (n1, e[prev_m:c], acc[:n1]))
            full = eng.build_snapshot((n1, e[:c], acc[:n1]), o)
            assert s.n == full.n and s.m == full.m
            assert np.array_equal(s.row_offsets, full.row_offsets)
            assert np.array_equal(s.col_indices, full.col_indices)
            assert np.array_equal(s.accepting.words(), full.accepting.words())
            go, gc = s.gather_index()
            fo, fc = full.gather_index()
            assert np.array_equal(go, fo) and np.array_equal(gc, fc)
            prev_m = c
        v1, st1 = eng.run_map(s, s.accepting)
        v2, st2 = eng.run_map(full, full.accepting)
        assert (v1.cycle_found(), v1.witness, st1.kernel_calls) == (v2.cycle_found(), v2.witness, st2.kernel_calls)
    # EdgeLog form (prefix semantics of the reference API) and contract errors
    log = eng.EdgeLog()
    for v in range(5):
        log.add_vertex(v % 2 == 0)
    for a, b in [(0, 1), (1, 2), (2, 0), (3, 4)]:
        log.append_edge(a, b)
    s = eng.build_snapshot(log, eng.Orientation.transposed, 2, 3)
    s2 = eng.extend_snapshot(s, log)
    full = eng.build_snapshot(log, eng.Orientation.transposed)
    assert s2.row_offsets.tolist() == full.row_offsets.tolist()
    assert s2.col_indices.tolist() == full.col_indices.tolist()
    with pytest.raises(eng.ContractError):
        eng.extend_snapshot(s2, (3, np.zeros((0, 2), np.uint32), [True] * 3))  # vertex prefix shrinks


# --------------------------------------------------- explicit-graph ingestion
def _explicit_same(eng, text, want):
    """device parse == reference result (dict with n/accepting/edges or error)."""
    if "error" in want:
        with pytest.raises(eng.ParseError) as ei:
            eng.parse_explicit_graph(text)
        assert str(ei.value) == want["error"]
        line = int(want["error"].split(":")[0])
        assert ei.value.line == line and ei.value.col == (0 if line == 0 and "cannot" in want["error"] else 1)
    else:
        g = eng.parse_explicit_graph(text)
        assert (g.n, g.accepting.tolist(), g.edges.tolist()) == (want["n"], want["accepting"], want["edges"])


def test_explicit_parse_golden(eng, golden):
    """parse_explicit_graph on the device reproduces the reference on the
    committed fixtures: the graph, or the same ParseError text and line."""
    import base64

    for rec in golden["explicit"]:
        _explicit_same(eng, base64.b64decode(rec["text_b64"]), rec)


def test_explicit_parse_fuzz_and_snapshot(eng, R, REF):
    import explicit_cases as X
    import oracle as O

    for text in X.cases(seed=77, count=300):
        try:
            n, acc, e = REF.parse_explicit(text)
            want = {"n": n, "accepting": acc.tolist(), "edges": e.tolist()}
        except O.RefParseError as ex:
            want = {"error": str(ex)}
        _explicit_same(eng, text, want)
    # a larger file: snapshot through the device parse == reference snapshot
    rng = np.random.default_rng(5)
    text, n, acc, edges = X.valid_text(rng, 3000, 20000, 0.05)
    dg = eng.parse_explicit_device(text)
    for tr in (True, False):
        s = dg.snapshot(eng.Orientation.transposed if tr else eng.Orientation.forward)
        rs = REF.explicit_snapshot(text, tr)
        c, racc, _ = rs.export()
        assert np.array_equal(s.row_offsets, c.off) and np.array_equal(s.col_indices, c.col)
        assert np.array_equal(s.accepting.words()[: len(racc)], racc[: len(s.accepting.words())])
    # binary round trip feeds the same snapshot
    g = dg.export()
    blob = eng.write_binary_graph(g.n, g.edges, eng.Bitset.from_indices(g.n, g.accepting))
    bg = eng.load_binary_graph(blob)
    assert (bg.n, bg.m) == (g.n, len(g.edges))
    b = bg.export()
    assert np.array_equal(b.edges, g.edges) and b.accepting.tolist() == sorted(set(g.accepting.tolist()))
    s1, s2 = bg.snapshot(), dg.snapshot()
    assert np.array_equal(s1.col_indices, s2.col_indices) and np.array_equal(s1.row_offsets, s2.row_offsets)
    with pytest.raises(eng.ContractError):
        eng.load_binary_graph(blob[:-4])
    with pytest.raises(eng.ParseError):
        eng.load_explicit_graph("/nonexistent/graph.txt")


def test_explicit_parse_large(eng, R):
    """A 2^20-edge file: every id parsed, order kept (device generator log)."""
    p = eng.preset(1)
    p.n, p.deg = 1 << 17, 8
    eng.prepare(p)
    gn, ge, ga = R.generate(p)
    acc = np.flatnonzero(np.unpackbits(ga.view(np.uint8), bitorder="little")[:gn])
    body = "\n".join(f"edge {s} {d}" for s, d in ge.tolist())
    text = f"graph {gn}\naccepting {' '.join(map(str, acc.tolist()))}\n{body}\n".encode()
    g = eng.parse_explicit_graph(text)
    assert g.n == gn and np.array_equal(g.edges, ge) and np.array_equal(g.accepting, acc.astype(np.uint32))


# ------------------------------------------- full BASELINE sizes (properties)
def _device_log(eng, cfg):
    from paper_0912_2555_b200 import _abi

    p = eng.preset(cfg)
    ctx = eng.default_context()
    L, C = _abi.lib(), _abi.C
    de, da = C.c_void_p(), C.c_void_p()
    _abi.check(L.cyc_device_alloc(ctx.handle, p.m * 8, C.byref(de)))
    _abi.check(L.cyc_device_alloc(ctx.handle, ((p.n + 63) // 64) * 8, C.byref(da)))
    _abi.check(L.cyc_gen_fill(ctx.handle, C.byref(p), de, da))
    return p, ctx, de, da


def _device_snapshot(eng, p, ctx, de, da, orientation):
    from paper_0912_2555_b200 import _abi

    L, C = _abi.lib(), _abi.C
    h = C.c_void_p()
    _abi.check(L.cyc_graph_build(ctx.handle, C.cast(de, C.POINTER(C.c_uint32)), p.m, p.n,
                                 C.cast(da, C.POINTER(C.c_uint64)), int(orientation), C.byref(h)))
    return eng.CsrSnapshot(h, ctx)


def test_c5_full_size_closed_form(eng):
    """Config 5 at 2^24: no cycle, one iteration, L*(S/2+2) + S/2 - 1 = 16767
    steps (the family's closed form, pinned on the CPU by the oracle and the
    reference); OWCTY and the SCC verdict agree."""
    from paper_0912_2555_b200 import _abi

    p, ctx, de, da = _device_log(eng, 5)
    try:
        s = _device_snapshot(eng, p, ctx, de, da, eng.Orientation.transposed)
        for mode in MODES:
            v, st = eng.run_map(s, s.accepting, eng.MapOptions(mode=mode))
            assert not v.cycle_found()
            assert (st.iterations, st.kernel_calls) == (1, 64 * 258 + 255), mode
        assert not eng.run_owcty(s)[0].cycle_found() and not eng.scc_verdict(s).verdict.cycle_found()
    finally:
        _abi.lib().cyc_device_free(ctx.handle, de)
        _abi.lib().cyc_device_free(ctx.handle, da)


@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_verdicts_agree(eng, cfg):
    """Configs 3 (R-MAT 2^26, 2^30 logged edges) and 4 (2^28-state product
    graph) at full size, where no CPU oracle finishes: MAP (with and without
    the final-round restriction), OWCTY and the SCC verdict agree; MAP's
    witness is an accepting vertex of a cyclic SCC; the restricted run maps its
    witness back to the unrestricted one (the cycle detector's contract)."""
    from paper_0912_2555_b200 import _abi

    p, ctx, de, da = _device_log(eng, cfg)
    try:
        s = _device_snapshot(eng, p, ctx, de, da, eng.Orientation.transposed)
        ov = eng.scc_verdict(s)
        cyc_acc = ov.cyclic_accepting
        assert ov.verdict.cycle_found() and len(cyc_acc) > 0
        r = eng.restrict_to_accepting_sccs(s)
        assert np.array_equal(np.intersect1d(r.kept, np.flatnonzero(
            np.unpackbits(s.accepting.words().view(np.uint8), bitorder="little")[: s.n])), cyc_acc)
        vr, _ = eng.run_map(r.snapshot, r.snapshot.accepting)
        w = int(r.kept[vr.witness])
        assert vr.cycle_found() and w in set(cyc_acc.tolist())
        if cfg == 3:  # unrestricted MAP on config 4 is MAP's worst case (49 K dense steps)
            v, _ = eng.run_map(s, s.accepting)
            assert v.cycle_found() and v.witness in set(cyc_acc.tolist())
        fwd = _device_snapshot(eng, p, ctx, de, da, eng.Orientation.forward)
        vo, so = eng.run_owcty(fwd)
        accb = np.unpackbits(fwd.accepting.words().view(np.uint8), bitorder="little")
        assert vo.cycle_found() and accb[vo.witness] and so.final_size > 0
    finally:
        _abi.lib().cyc_device_free(ctx.handle, de)
        _abi.lib().cyc_device_free(ctx.handle, da)


def test_build_long_rows_edge_cases(eng, R):
    """K1's long-row split sort (rows > 512): heavy duplication (one value
    range collapsing into an overfull sub-bucket, CTA and global fallbacks),
    narrow consecutive column ranges, and wide random ranges, in both CSRs."""
    rng = np.random.default_rng(31)
    n = 50000
    parts = [rng.integers(0, n, size=(60000, 2))]
    parts.append(np.stack([np.full(9000, 7), rng.integers(0, 3, size=9000)], 1))        # 9000 dups of 3 values
    parts.append(np.stack([np.full(6000, 11), np.full(6000, 12)], 1))                    # one value x 6000
    parts.append(np.stack([np.full(5000, 13), 20000 + np.arange(5000) % 2500], 1))       # narrow range, 2 copies
    parts.append(np.stack([np.full(70000, 17), rng.integers(0, n, size=70000)], 1))      # wide hub
    parts.append(np.stack([rng.integers(0, n, size=20000), np.full(20000, 19)], 1))      # hub in the other CSR
    e = np.concatenate(parts).astype(np.uint32)
    e = e[rng.permutation(len(e))]
    acc = rng.random(n) < 0.05
    for tr in (True, False):
        s = snap_of(eng, n, e, acc, tr)
        g = R.build_snapshot(n, e, tr)
        assert np.array_equal(s.row_offsets, g.off) and np.array_equal(s.col_indices, g.col)
        off, col = s.gather_index()
        gt = R.transpose(g)
        assert np.array_equal(off, gt.off) and np.array_equal(col, gt.col)


def test_fuzz_all_entry_points(eng, R, REF):
    """Randomised sweep over graph shapes (self loops, duplicate edges,
    isolated vertices, hubs in either CSR, 0-60 % accepting, both
    orientations): run_map in every step kind and both early-exit modes,
    restriction, OWCTY and the SCC verdict against the oracle / reference."""
    rng = np.random.default_rng(0xF022)
    for t in range(40):
        n = int(rng.integers(1, 3000))
        m = int(rng.integers(0, 6 * n + 1))
        e = rng.integers(0, n, size=(m, 2)).astype(np.uint32)
        if t % 3 == 0 and n > 1:  # self loops and duplicates
            k = int(rng.integers(1, 20))
            v = rng.integers(0, n, size=k).astype(np.uint32)
            e = np.concatenate([e, np.stack([v, v], 1), e[: min(len(e), 50)]])
        if t % 4 == 1:
            e = random_graph(rng, n, len(e), hubs=2)
        acc = rng.random(n) < rng.choice([0.0, 0.01, 0.1, 0.6])
        tr = bool(t % 2)
        s = snap_of(eng, n, e, acc, tr)
        g = R.build_snapshot(n, e, tr)
        gat = R.transpose(g)
        for early in (True, False):
            ref = R.run_map(gat, acc, early)
            for mode in MODES:
                assert_same_run(eng.run_map_detailed(s, acc, eng.MapOptions(early_exit=early, mode=mode)), ref)
        r = eng.restrict_to_accepting_sccs(s)
        _, _, kept = R.restrict(g, acc)
        assert np.array_equal(r.kept, kept)
        v, st = eng.run_owcty(s)
        assert (v.cycle_found(), v.witness, st.outer_iterations, st.final_size) == R.run_owcty(g, acc)
        assert eng.scc_verdict(s).verdict.cycle_found() == REF.snapshot(n, e, acc, tr).scc_verdict()


def test_restrict_hub_rows(eng, R):
    """Restriction of rows far longer than the compaction's chunk (8192):
    a hub inside the big SCC whose rows also reference dropped vertices (sink
    tails without a path back), in both CSRs and both orientations."""
    rng = np.random.default_rng(77)
    core, tail = 30000, 6000
    n = core + tail
    ring = np.stack([np.arange(core), (np.arange(core) + 1) % core], 1)
    hub_out = np.stack([np.zeros(n - 1, dtype=np.int64), np.arange(1, n)], 1)  # also into the tails
    hub_in = np.stack([np.arange(1, core), np.zeros(core - 1, dtype=np.int64)], 1)
    rnd = rng.integers(0, core, size=(40000, 2))
    tails = np.stack([rng.integers(core, n, size=5000), rng.integers(core, n, size=5000)], 1)
    e = np.concatenate([ring, hub_out, hub_in, rnd, tails]).astype(np.uint32)
    rng.shuffle(e)
    acc = np.zeros(n, dtype=bool)
    acc[rng.integers(0, n, size=200)] = True
    acc[5] = True
    for tr in (True, False):
        s = snap_of(eng, n, e, acc, tr)
        g = R.build_snapshot(n, e, tr)
        rg, racc, kept = R.restrict(g, acc)
        assert len(kept) == core
        r = eng.restrict_to_accepting_sccs(s)
        assert np.array_equal(r.kept, kept)
        assert np.array_equal(r.snapshot.row_offsets, rg.off)
        assert np.array_equal(r.snapshot.col_indices, rg.col)
        off, col = r.snapshot.gather_index()
        gt = R.transpose(rg)
        assert np.array_equal(off, gt.off) and np.array_equal(col, gt.col)


def test_overlapped_build_equals_sequential(eng, monkeypatch):
    """Logs of >= 2^24 edges build the gather index on a second stream by a
    helper thread (abi.cu build_graph); the result must equal the sequential
    build bit for bit (both CSRs)."""
    from paper_0912_2555_b200 import _abi

    p = eng.preset(3)
    p.scale, p.edgefactor = 20, 16
    eng.prepare(p)
    assert p.m >= 1 << 24
    ctx = eng.default_context()
    L, C = _abi.lib(), _abi.C
    de, da = C.c_void_p(), C.c_void_p()
    _abi.check(L.cyc_device_alloc(ctx.handle, p.m * 8, C.byref(de)))
    _abi.check(L.cyc_device_alloc(ctx.handle, ((p.n + 63) // 64) * 8, C.byref(da)))
    try:
        _abi.check(L.cyc_gen_fill(ctx.handle, C.byref(p), de, da))
        out = []
        for seq in (False, True):
            if seq:
                monkeypatch.setenv("CYC_BUILD_SEQUENTIAL", "1")
            s = _device_snapshot(eng, p, ctx, de, da, eng.Orientation.transposed)
            off, col = s.gather_index()
            out.append((s.row_offsets.copy(), s.col_indices.copy(), off.copy(), col.copy()))
        for a, b in zip(*out):
            assert np.array_equal(a, b)
    finally:
        L.cyc_device_free(ctx.handle, de)
        L.cyc_device_free(ctx.handle, da)
