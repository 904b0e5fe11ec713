"""GPU: the library is re-entrant per context (SURVEY §8b "one call in flight
per cyc_ctx"; the explorer's detector thread and the final round use
separate contexts). Threads with their own contexts build, restrict and run
MAP / OWCTY concurrently (ctypes releases the GIL) and get exactly the
results of a sequential run."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _work(eng, seed, ctx):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20000, 60000))
    e = rng.integers(0, n, size=(n * 4, 2)).astype(np.uint32)
    acc = rng.random(n) < 0.02
    s = eng.build_snapshot((n, e, acc), ctx=ctx)
    run = eng.run_map_detailed(s, acc, eng.MapOptions(early_exit=bool(seed % 2)))
    r = eng.restrict_to_accepting_sccs(s)
    v, st = eng.run_owcty(s)
    return (run.verdict.cycle_found(), run.verdict.witness, run.stats.iterations, run.stats.kernel_calls,
            int(np.asarray(run.final_values, np.uint64).sum()), r.kept.tobytes(), v.witness, st.outer_iterations)


def test_threads_with_own_contexts(eng):
    seeds = [11, 12, 13, 14]
    ctxs = [eng.Context(0) for _ in seeds]
    want = [_work(eng, sd, c) for sd, c in zip(seeds, ctxs)]
    for _ in range(3):
        got = [None] * len(seeds)

        def run(i):
            got[i] = _work(eng, seeds[i], ctxs[i])

        th = [threading.Thread(target=run, args=(i,)) for i in range(len(seeds))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert got == want
    for c in ctxs:
        c.close()
