"""GPU parity of the degree-ordered storage layout (csrc/plan.cu): run_map,
fixpoint and the per-step vectors with the map vector and both CSRs stored in
descending gather-count order must equal the oracle restatement bit for bit
(values are vertex ids, so only storage moves). Every case also runs the
identity layout on the same snapshot, so a stale plan or workspace between
layouts would show up here."""
import numpy as np
import pytest

from test_gpu_parity import MODES, assert_same_run, random_graph, snap_of

pytestmark = pytest.mark.gpu

LAYOUTS = ("degree", "identity", "auto")


@pytest.mark.parametrize("seed", range(5))
def test_layout_random(eng, R, seed):
    rng = np.random.default_rng(4200 + seed)
    n = int(rng.integers(100, 30000))
    m = int(n * rng.choice([1, 2, 4, 8]))
    e = random_graph(rng, n, m, hubs=1 + seed % 3)
    acc = rng.random(n) < rng.choice([0.002, 0.02, 0.1, 0.4])
    s = snap_of(eng, n, e, acc)
    gat = R.transpose(R.build_snapshot(n, e, True))
    for early in (True, False):
        ref = R.run_map(gat, acc, early)
        for layout in LAYOUTS:
            for mode in MODES:
                run = eng.run_map_detailed(s, acc, eng.MapOptions(early_exit=early, mode=mode, layout=layout))
                assert_same_run(run, ref)


@pytest.mark.parametrize("scale", [12, 15, 17])
def test_layout_rmat(eng, R, scale):
    """The family the layout is for: R-MAT hubs, 1 % accepting."""
    p = R.preset(3)
    p.scale = scale
    R.prepare(p)
    n, e, accw = R.generate(p)
    acc = eng.Bitset.from_words(accw, n)
    s = snap_of(eng, n, e, acc)
    gat = R.transpose(R.build_snapshot(n, e, True))
    for early in (True, False):
        ref = R.run_map(gat, accw, early)
        for mode in MODES:
            assert_same_run(eng.run_map_detailed(s, acc, eng.MapOptions(early_exit=early, mode=mode,
                                                                        layout="degree")), ref)
    # a different accepting set on the same plan (F is permuted per call)
    rng = np.random.default_rng(scale)
    acc2 = rng.random(n) < 0.05
    for early in (True, False):
        ref = R.run_map(gat, acc2, early)
        assert_same_run(eng.run_map_detailed(s, acc2, eng.MapOptions(early_exit=early, layout="degree")), ref)


def test_layout_per_step_vectors(eng, R):
    rng = np.random.default_rng(78)
    n, m = 4000, 12000
    e = random_graph(rng, n, m, hubs=2)
    acc = rng.random(n) < 0.03
    s = snap_of(eng, n, e, acc)
    gat = R.transpose(R.build_snapshot(n, e, True))
    x = np.zeros(n, np.uint32)
    for k in range(1, 12):
        x, ch, w = R.step(gat, x, acc)
        for mode in MODES:
            fr = eng.fixpoint(s, acc, eng.MapOptions(early_exit=False, mode=mode, layout="degree"), max_steps=k)
            assert np.array_equal(fr.values, x), (k, mode)
        if not ch:
            break


def test_layout_golden_configs(eng, R):
    """Scaled members of configs 1-5 (include/cyc_gen.h) under the degree layout."""
    for idx, over in ((1, {}), (2, {"L": 16, "W": 64, "S": 8}), (4, {"grid_bits": 6, "region": 16}),
                      (5, {"L": 16, "W": 4, "S": 16})):
        p = R.preset(idx)
        for k, v in over.items():
            setattr(p, k, v)
        R.prepare(p)
        n, e, accw = R.generate(p)
        for tr in (True, False):
            s = snap_of(eng, n, e, eng.Bitset.from_words(accw, n), tr)
            gat = R.transpose(R.build_snapshot(n, e, tr))
            for early in (True, False):
                ref = R.run_map(gat, accw, early)
                run = eng.run_map_detailed(s, eng.Bitset.from_words(accw, n),
                                           eng.MapOptions(early_exit=early, layout="degree"))
                assert_same_run(run, ref)


def test_layout_contract(eng):
    with pytest.raises(eng.ContractError):
        eng.MapOptions(layout="bogus").to_c()


@pytest.mark.parametrize("hot", ["0", "64", "704", "1048576"])
def test_layout_hot_staging_split(eng, R, hot, monkeypatch):
    """Pull steps skip gathers from positions < hot whose frontier bit (staged
    in shared memory) is clear; any split point must give the reference's
    results (0 = no filter, 2^20 = the whole graph filtered)."""
    monkeypatch.setenv("CYC_HOT_POS", hot)
    p = R.preset(3)
    p.scale = 13
    R.prepare(p)
    n, e, accw = R.generate(p)
    acc = eng.Bitset.from_words(accw, n)
    s = snap_of(eng, n, e, acc)
    gat = R.transpose(R.build_snapshot(n, e, True))
    for early in (True, False):
        ref = R.run_map(gat, accw, early)
        for mode in ("auto", "pull"):
            assert_same_run(eng.run_map_detailed(s, acc, eng.MapOptions(early_exit=early, mode=mode,
                                                                        layout="degree")), ref)


def test_auto_layout_builds_the_plan_from_the_second_loop(eng):
    """Auto layout: a graph's first MAP loop runs in id order (the plan costs
    more than one loop saves), the second builds and uses the degree-ordered
    plan; both loops give the same run (R-MAT scale 24: a 64 MB map vector
    whose hottest eighth takes most gathers, so auto picks the plan)."""
    import os

    from paper_0912_2555_b200 import _abi
    from test_gpu_parity import _device_snapshot

    if os.environ.get("CYC_LAYOUT"):
        pytest.skip("CYC_LAYOUT forces one layout for every run")
    p = eng.preset(3)
    p.scale = 24
    eng.prepare(p)
    ctx = eng.default_context()
    L, C = _abi.lib(), _abi.C
    de, da = C.c_void_p(), C.c_void_p()
    _abi.check(L.cyc_device_alloc(ctx.handle, p.m * 8, C.byref(de)))
    _abi.check(L.cyc_device_alloc(ctx.handle, ((p.n + 63) // 64) * 8, C.byref(da)))
    try:
        _abi.check(L.cyc_gen_fill(ctx.handle, C.byref(p), de, da))
        s = _device_snapshot(eng, p, ctx, de, da, eng.Orientation.transposed)
        opt = eng.MapOptions(early_exit=False)
        runs = [eng.run_map_detailed(s, s.accepting, opt, hash_cap=64) for _ in range(3)]
        assert [int(r.stats.device["layout"]) for r in runs] == [_abi.CYC_LAYOUT_IDENTITY, _abi.CYC_LAYOUT_DEGREE,
                                                        _abi.CYC_LAYOUT_DEGREE]
        pm = [r.stats.device["plan_ms"] for r in runs]
        assert pm[0] < 1.0 and pm[1] > 1.0 and pm[2] == 0.0  # first: only the decision; second: the plan; third: cached
        for r in runs[1:]:
            assert (r.verdict.cycle_found(), r.verdict.witness, r.stats.kernel_calls, r.stats.iterations) == (
                runs[0].verdict.cycle_found(), runs[0].verdict.witness, runs[0].stats.kernel_calls,
                runs[0].stats.iterations)
            assert np.array_equal(r.final_values, runs[0].final_values)
            assert np.array_equal(r.iter_hash, runs[0].iter_hash)
    finally:
        L.cyc_device_free(ctx.handle, de)
        L.cyc_device_free(ctx.handle, da)
