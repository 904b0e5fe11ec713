"""GPU: cyc_ctx_reserve (build memory allocated ahead, on a library thread)
changes nothing but when memory is first touched — builds and runs after a
background reserve equal the oracle bit for bit, a reserve far beyond the
device's memory is not an error, and a context can be destroyed while its
reserve is still running."""
import numpy as np
import pytest

from test_gpu_parity import assert_same_run, oracle_run, random_graph, snap_of

pytestmark = pytest.mark.gpu


def test_reserve_then_build(eng, R):
    rng = np.random.default_rng(91)
    ctx = eng.Context(0)
    try:
        n = 50000
        e = random_graph(rng, n, 8 * n, hubs=3)
        acc = rng.random(n) < 0.01
        ctx.reserve(len(e), n, background=True)  # the build below waits for it
        s = eng.build_snapshot((n, e, acc), eng.Orientation.transposed, ctx=ctx)
        for early in (True, False):
            assert_same_run(eng.run_map_detailed(s, s.accepting, eng.MapOptions(early_exit=early)),
                            oracle_run(R, n, e, acc, True, early))
        # larger than the arenas the first build left: reserve grows them
        n2 = 120000
        e2 = random_graph(rng, n2, 16 * n2, hubs=2)
        acc2 = rng.random(n2) < 0.02
        ctx.reserve(len(e2), n2, background=False)
        s2 = eng.build_snapshot((n2, e2, acc2), eng.Orientation.transposed, ctx=ctx)
        assert_same_run(eng.run_map_detailed(s2, s2.accepting, eng.MapOptions(early_exit=False)),
                        oracle_run(R, n2, e2, acc2, True, False))
        del s, s2
    finally:
        ctx.close()


def test_reserve_beyond_memory_is_not_an_error(eng, R):
    ctx = eng.Context(0)
    try:
        ctx.reserve(1 << 40, 1 << 30, background=False)  # ~50 TB: nothing reserved
        rng = np.random.default_rng(5)
        n = 3000
        e = random_graph(rng, n, 4 * n)
        acc = rng.random(n) < 0.05
        s = eng.build_snapshot((n, e, acc), eng.Orientation.transposed, ctx=ctx)
        assert_same_run(eng.run_map_detailed(s, s.accepting, eng.MapOptions(early_exit=False)),
                        oracle_run(R, n, e, acc, True, False))
        del s
    finally:
        ctx.close()


def test_destroy_while_reserving(eng):
    ctx = eng.Context(0)
    ctx.reserve(1 << 26, 1 << 22, background=True)
    ctx.close()  # joins the reserve thread, then frees
