"""CPU tests: the oracle restatement is pinned against the SPEC.md [OP]
known-answer examples, the committed golden fixtures (generated from the
reference itself, tests/golden/make_golden.py), and — where the reference
build is present — the reference on fresh random inputs."""
import hashlib
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.json")
NIL = 0


def code(v):  # map value of vertex v (map_engine.hpp:23)
    return v + 1


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


G1 = [(0, 1), (1, 2), (2, 1)]


# ---------------------------------------------------------------- SPEC KATs
def test_spec_snapshot_transposed(R):
    g = R.build_snapshot(3, G1, True)
    assert g.off.tolist() == [0, 0, 2, 3] and g.col.tolist() == [0, 2, 1]


def test_spec_snapshot_forward(R):
    g = R.build_snapshot(3, G1, False)
    assert g.off.tolist() == [0, 1, 2, 3] and g.col.tolist() == [1, 2, 1]


def test_spec_empty_snapshot(R):
    g = R.build_snapshot(0, [], True)
    assert g.off.tolist() == [0] and g.m == 0


def test_spec_dedup(R):  # SPEC.md:74-75, graph.cpp:89-101
    g = R.build_snapshot(2, [(0, 1), (0, 1), (1, 0)], True)
    assert g.m == 2


def test_spec_restrict_kept(R):
    g = R.build_snapshot(3, G1, True)
    r, acc, kept = R.restrict(g, np.array([False, True, False]))
    assert kept.tolist() == [1, 2]


def test_spec_restrict_chain_empty(R):
    g = R.build_snapshot(3, [(0, 1), (1, 2)], True)
    _, _, kept = R.restrict(g, np.array([False, False, True]))
    assert kept.tolist() == []


def test_spec_steps_g1(R):
    gat = R.transpose(R.build_snapshot(3, G1, True))
    acc = np.array([False, True, False])
    x1, ch1, _ = R.step(gat, np.zeros(3, np.uint32), acc)
    assert x1.tolist() == [code(1), NIL, code(1)] and ch1
    x2, ch2, w2 = R.step(gat, x1, acc)
    assert x2.tolist() == [code(1)] * 3 and ch2 and w2 == 1


def test_spec_fixpoint_g1_witness(R):
    gat = R.transpose(R.build_snapshot(3, G1, True))
    x, steps, w = R.fixpoint(gat, np.array([False, True, False]), True)
    assert w == 1 and steps == 2


def test_spec_chain_fixpoint(R):
    gat = R.transpose(R.build_snapshot(3, [(0, 1), (1, 2)], True))
    x, steps, w = R.fixpoint(gat, np.array([False, False, True]), True)
    assert x.tolist() == [code(2), code(2), NIL] and steps == 3 and w is None


def test_spec_empty_fixpoint(R):
    gat = R.transpose(R.build_snapshot(0, [], True))
    _, steps, w = R.fixpoint(gat, np.zeros(0, bool), True)
    assert steps == 1 and w is None


def test_spec_demote_chain(R):
    rem, d = R.demote([code(2), code(2), NIL], np.array([False, False, True]))
    assert d.tolist() == [2] and int(rem[0]) == 0


def test_spec_demote_nil(R):
    acc = np.array([True, False, True, True])
    rem, d = R.demote([NIL] * 4, acc)
    assert d.tolist() == [] and int(rem[0]) == 0b1101


def test_spec_demote_partial(R):  # only 3 appears as a value
    acc = np.array([False, True, False, True])
    rem, d = R.demote([code(3), NIL, code(3), NIL], acc)
    assert d.tolist() == [3] and int(rem[0]) == 0b0010


def test_spec_self_loop_cycle(R):
    gat = R.transpose(R.build_snapshot(1, [(0, 0)], True))
    r = R.run_map(gat, np.array([True]), True)
    assert r.cycle and r.witness == 0 and r.iterations == 1


def test_spec_dag_no_cycle(R):
    rng = np.random.default_rng(3)
    n = 30
    e = [(a, b) for a, b in rng.integers(0, n, (80, 2)).tolist() if a < b]
    gat = R.transpose(R.build_snapshot(n, e, True))
    for early in (True, False):
        assert not R.run_map(gat, rng.random(n) < 0.4, early).cycle


# -------------------------------------------------------------- golden
def test_golden_random_graphs(R, golden):
    for case in golden["random"]:
        n = case["n"]
        e = np.array(case["edges"], np.uint32).reshape(-1, 2)
        acc = np.zeros(n, bool)
        acc[case["accepting"]] = True
        g = R.build_snapshot(n, e, True)
        assert g.off.tolist() == case["row_offsets"] and g.col.tolist() == case["col_indices"]
        gat = R.transpose(g)
        x1, ch1, _ = R.step(gat, np.zeros(n, np.uint32), acc)
        assert x1.tolist() == case["step1"] and ch1 == case["step1_changed"]
        for mode, early in (("early", True), ("full", False)):
            r = R.run_map(gat, acc, early)
            want = case[mode]
            assert (r.cycle, r.witness, r.iterations, r.kernel_calls, r.demoted_total) == (
                want["cycle"], want["witness"], want["iterations"], want["kernel_calls"],
                want["demoted_total"])
            assert r.final_x.tolist() == case["final_x_" + mode]
            assert [int(h) for h in r.iter_hash] == want["iter_hash"]
            assert [int(s) for s in r.iter_steps] == want["iter_steps"]
        assert r.cycle == case["scc_cycle"]


@pytest.mark.parametrize("name", ["c1", "c2_L16", "c5_L16", "c3_s12", "c4_g6"])
def test_golden_configs(R, golden, name):
    cfg = golden["configs"][name]
    p = R.preset(cfg["config"])
    for k, v in cfg["overrides"].items():
        setattr(p, k, v)
    R.prepare(p)
    n, e, accw = R.generate(p)
    assert digest(e) == cfg["edges_digest"] and digest(accw) == cfg["acc_digest"]
    vec = np.load(os.path.join(os.path.dirname(GOLDEN), "golden_vectors.npz"))
    for orient, tr in (("transposed", True), ("forward", False)):
        g = R.build_snapshot(n, e, tr)
        want = cfg[orient]
        assert g.m == want["m"] and digest(g.off) == want["off_digest"] and digest(g.col) == want["col_digest"]
        gat = R.transpose(g)
        for mode, early in (("early", True), ("full", False)):
            r = R.run_map(gat, accw, early)
            w = want[mode]
            assert (r.cycle, r.witness, r.iterations, r.kernel_calls, r.demoted_total) == (
                w["cycle"], w["witness"], w["iterations"], w["kernel_calls"], w["demoted_total"])
            assert digest(r.final_x) == w["final_x_digest"]
            assert [int(h) for h in r.iter_hash[:256]] == w["iter_hash"]
            key = f"{name}_{orient}_{mode}_final_x"
            if key in vec:
                assert np.array_equal(vec[key], r.final_x)
        wo = want["owcty"]
        assert R.run_owcty(g, accw) == (wo["cycle"], wo["witness"], wo["outer_iterations"], wo["final_size"])
        rg, racc, kept = R.restrict(g, accw)
        wr = want["restricted"]
        assert rg.n == wr["n"] and rg.m == wr["m"] and digest(kept) == wr["kept_digest"]
        assert digest(rg.off) == wr["off_digest"] and digest(rg.col) == wr["col_digest"]


def test_closed_form_layered(R, golden):
    # C2 family has iterations = L+1, kernel_calls = (L+1)^2
    w = golden["configs"]["c2_L16"]["transposed"]["early"]
    assert w["iterations"] == 17 and w["kernel_calls"] == 17 ** 2 and not w["cycle"]


# ------------------------------------------- differential vs the reference
def test_random_differential_reference(R, REF):
    rng = np.random.default_rng(2555)
    for t in range(300):
        n = int(rng.integers(1, 50))
        m = int(rng.integers(0, 4 * n))
        e = rng.integers(0, n, size=(m, 2)).astype(np.uint32)
        acc = rng.random(n) < [0.1, 0.3][t % 2]
        for tr in (True, False):
            rs = REF.snapshot(n, e, acc, tr)
            c, racc, _ = rs.export()
            g = R.build_snapshot(n, e, tr)
            assert np.array_equal(g.off, c.off) and np.array_equal(g.col, c.col)
            gat = R.transpose(g)
            for early in (True, False):
                a, b = R.run_map(gat, acc, early), rs.run_map(None, early)
                assert (a.cycle, a.witness, a.iterations, a.kernel_calls, a.demoted_total) == (
                    b.cycle, b.witness, b.iterations, b.kernel_calls, b.demoted_total)
                assert np.array_equal(a.final_x, b.final_x)
                assert np.array_equal(a.iter_hash, b.iter_hash)
            rg, _, kept = R.restrict(g, acc)
            rr = rs.restrict()
            c2, _, k2 = rr.export()
            assert np.array_equal(kept, k2) and np.array_equal(rg.off, c2.off) and np.array_equal(rg.col, c2.col)
            # verdict equals the SCC oracle
            assert R.run_map(gat, acc, True).cycle == rs.scc_verdict()


def test_owcty_restatement_vs_reference(R, REF):
    # owcty.cpp:56-87 on forward snapshots (cycheck_main.cpp:98-106): verdict,
    # witness, outer_iterations and final_size agree; verdict equals MAP's
    rng = np.random.default_rng(1999)
    for t in range(300):
        n = int(rng.integers(1, 60))
        m = int(rng.integers(0, 3 * n))
        e = rng.integers(0, n, size=(m, 2)).astype(np.uint32)
        acc = rng.random(n) < [0.05, 0.3][t % 2]
        rs = REF.snapshot(n, e, acc, False)
        g = R.build_snapshot(n, e, False)
        got = R.run_owcty(g, acc)
        assert got == rs.run_owcty()
        assert got[0] == R.run_map(R.build_snapshot(n, e, True), acc, True).cycle
    # SPEC.md:182-183 shapes: self loop, DAG
    assert R.run_owcty(R.build_snapshot(1, [[0, 0]], False), [True])[:2] == (True, 0)
    assert not R.run_owcty(R.build_snapshot(3, [[0, 1], [1, 2]], False), [True] * 3)[0]
    assert R.run_owcty(R.build_snapshot(0, np.zeros((0, 2), np.uint32), False), [])[2] == 0


def test_explicit_golden_pinned(REF, golden):
    # the committed parse_explicit_graph fixtures (graph.cpp:259-297) are what
    # the compiled reference returns here
    import base64

    import oracle as O

    for rec in golden["explicit"]:
        text = base64.b64decode(rec["text_b64"])
        if "error" in rec:
            with pytest.raises(O.RefParseError) as ei:
                REF.parse_explicit(text)
            assert str(ei.value) == rec["error"]
        else:
            n, acc, e = REF.parse_explicit(text)
            assert (n, acc.tolist(), e.tolist()) == (rec["n"], rec["accepting"], rec["edges"])


def test_chain_family_closed_form_oracle(R, REF):
    # config 5 family: one MAP iteration of exactly L*(S/2+2) + S/2 - 1 steps,
    # independent of W (derived here on small members, checked against the
    # reference; pins the full-size GPU test, 64*258 + 255 = 16767)
    for L, S, W in ((2, 4, 1), (3, 8, 2), (4, 16, 4), (8, 32, 1), (5, 12, 3)):
        p = R.preset(5)
        p.L, p.W, p.S = L, W, S
        R.prepare(p)
        n, e, a = R.generate(p)
        r = R.run_map(R.transpose(R.build_snapshot(n, e, True)), a, True)
        assert (r.iterations, r.kernel_calls, r.cycle) == (1, L * (S // 2 + 2) + S // 2 - 1, False)
        if L <= 4:
            rr = REF.snapshot(n, e, a, True).run_map(None, True)
            assert rr.kernel_calls == r.kernel_calls


def test_reference_step_worker_invariance(REF):
    # map_engine.hpp:46-49: bitwise identical for every worker count
    rng = np.random.default_rng(7)
    n = 500
    e = rng.integers(0, n, size=(2000, 2)).astype(np.uint32)
    acc = rng.random(n) < 0.2
    rs = REF.snapshot(n, e, acc, True)
    x = rng.integers(0, n + 1, size=n).astype(np.uint32)
    outs = [rs.step(x, None, w) for w in (1, 2, 4)]
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and o[1:] == outs[0][1:]


def test_product_generator_shape(R):
    # C4 (cyc_gen.h): every one of the 4 G^2 product states is reachable and
    # ids follow BFS discovery order; accepting = automaton state q2 (1/4);
    # accepting cycles exist only with the planted reset (verdict by SCC)
    for gb, k, plant in ((2, 1, 1), (3, 2, 1), (4, 3, 0), (5, 8, 1), (5, 8, 0)):
        p = R.preset(4)
        p.grid_bits, p.region, p.plant = gb, k, plant
        R.prepare(p)
        n, e, aw = R.generate(p)
        G = 1 << gb
        assert n == 4 * G * G and len(e) == 12 * G * G + 6 * plant
        acc = np.unpackbits(aw.view(np.uint8), bitorder="little")[:n].astype(bool)
        assert acc.sum() == G * G and e[0].tolist() == [0, 1]
        # BFS order: sources appear in id order, every id > 0 is first named
        # as a destination before it appears as a source
        assert np.all(np.diff(e[:, 0].astype(np.int64)) >= 0)
        first = {}
        for i, d in enumerate(e[:, 1].tolist()):
            first.setdefault(d, i)
        starts = np.searchsorted(e[:, 0], np.arange(1, n))
        assert all(first[v] < starts[v - 1] for v in range(1, n))
        keep = R.keep_mask(R.build_snapshot(n, e, True), acc)
        assert bool((keep & acc).any()) == bool(plant)


def test_generators_deterministic(R):
    for idx in (1, 2, 5):
        p = R.preset(idx)
        if idx == 2:
            p.L, p.W, p.S = 4, 8, 4
        if idx == 5:
            p.L, p.W, p.S = 4, 2, 8
        R.prepare(p)
        a = R.generate(p)
        b = R.generate(p)
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    p = R.preset(2)
    assert (p.n, p.m) == (64 * (4096 * 16 + 1) + 1, 64 * 4096 * (1 + 16 + 16))


def test_fast_snapshot_setup_equals_build_snapshot(REF, R):
    """bench.py's CPU arm builds config 3's snapshot with the parallel setup
    builder (ref_driver.cpp ref_snapshot_gen_fast) before timing the
    reference's MaxPropagation; it must equal build_snapshot (graph.cpp:63-105)."""
    for cfg, over in ((1, {}), (3, {"scale": 16}), (2, {"L": 8, "W": 64, "S": 8}), (5, {"L": 8, "W": 4, "S": 16})):
        p = R.preset(cfg)
        for k, v in over.items():
            setattr(p, k, v)
        R.prepare(p)
        for tr in (True, False):
            a = REF.snapshot_gen(p, tr).export()
            b = REF.snapshot_gen_fast(p, tr, 4).export()
            assert np.array_equal(a[0].off, b[0].off) and np.array_equal(a[0].col, b[0].col)
            assert np.array_equal(a[1], b[1])
