"""GPU: the row-sharded engine (csrc/shard.cu + the sharded mode of
k_map_run) against the oracle, bit for bit.

One GPU holds W ranks here: each rank is built from the whole log but keeps
only its own rows (~1/W of the edges), and the W ranks run as ONE cooperative
grid (rank r = its own slice of the blocks) whose grid barrier stands in for
the cross-GPU barrier — the same kernel body, the same peer stores into the
other ranks' replicated vectors and the same record reduction as on W GPUs
(B200_PROFILING.md: ranks that wait on each other must not be separate
launches on one GPU). World 1 is the single-GPU engine on a shard."""
import numpy as np
import pytest

from test_gpu_parity import MODES, assert_same_run, random_graph

pytestmark = pytest.mark.gpu


def shards_of(eng, n, e, accw, world, layout, orientation=None):
    from paper_0912_2555_b200 import _abi
    from paper_0912_2555_b200.sharded import MapShard

    ctx = eng.default_context()
    o = _abi.CYC_TRANSPOSED if orientation is None else orientation
    sh = [MapShard(ctx, e, len(e), n, accw, world, r, orientation=o, layout=layout) for r in range(world)]
    MapShard.connect_local(sh)
    return sh


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("layout", ["identity", "degree"])
def test_shard_random(eng, R, world, layout):
    from paper_0912_2555_b200.sharded import MapShard

    rng = np.random.default_rng(700 + world)
    for trial in range(3):
        n = int(rng.integers(300, 20000))
        e = random_graph(rng, n, int(n * rng.choice([1, 2, 4, 8])), hubs=trial)
        acc = rng.random(n) < rng.choice([0.005, 0.05, 0.3])
        accw = eng.as_bitset(acc, n).words()
        sh = shards_of(eng, n, e, accw, world, layout)
        info = [s.info() for s in sh]
        assert info[0]["row_lo"] == 0 and all(info[i]["row_hi"] == info[i + 1]["row_lo"] for i in range(world - 1))
        gat = R.transpose(R.build_snapshot(n, e, True))
        assert sum(i["local_edges"] for i in info) == gat.m  # every snapshot edge on exactly one rank
        for early in (True, False):
            ref = R.run_map(gat, acc, early)
            for mode in MODES:
                assert_same_run(MapShard.run_map(sh, early_exit=early, mode=mode), ref)
        for s in sh:
            s.close()


@pytest.mark.parametrize("world", [2, 4])
def test_shard_rmat(eng, R, world):
    """R-MAT hubs: heavy rows on one rank, push steps over the replicated frontier."""
    from paper_0912_2555_b200.sharded import MapShard

    p = R.preset(3)
    p.scale = 15
    R.prepare(p)
    n, e, accw = R.generate(p)
    gat = R.transpose(R.build_snapshot(n, e, True))
    for layout in ("identity", "degree"):
        sh = shards_of(eng, n, e, accw, world, layout)
        for early in (True, False):
            ref = R.run_map(gat, accw, early)
            for mode in MODES:
                assert_same_run(MapShard.run_map(sh, early_exit=early, mode=mode), ref)
        # another accepting set on the same shards
        acc2 = np.random.default_rng(3).random(n) < 0.02
        ref = R.run_map(gat, acc2, False)
        assert_same_run(MapShard.run_map(sh, acc_words=eng.as_bitset(acc2, n).words(), early_exit=False), ref)
        for s in sh:
            s.close()


def test_shard_many_iterations_and_forward(eng, R):
    """Config-2 and config-5 families (many fixpoints / long chains), both orientations."""
    from paper_0912_2555_b200 import _abi
    from paper_0912_2555_b200.sharded import MapShard

    for idx, over in ((2, {"L": 16, "W": 64, "S": 8}), (5, {"L": 16, "W": 4, "S": 16}), (1, {})):
        p = R.preset(idx)
        for k, v in over.items():
            setattr(p, k, v)
        R.prepare(p)
        n, e, accw = R.generate(p)
        for tr in (True, False):
            gat = R.transpose(R.build_snapshot(n, e, tr))
            o = _abi.CYC_TRANSPOSED if tr else _abi.CYC_FORWARD
            for world in (2, 3):
                sh = shards_of(eng, n, e, accw, world, "degree", orientation=o)
                for early in (True, False):
                    assert_same_run(MapShard.run_map(sh, early_exit=early), R.run_map(gat, accw, early))
                for s in sh:
                    s.close()


def test_shard_memory_splits(eng, R):
    """Per-rank edge structures shrink with the world size (vectors are replicated)."""
    p = R.preset(3)
    p.scale = 16
    R.prepare(p)
    n, e, accw = R.generate(p)
    one = shards_of(eng, n, e, accw, 1, "degree")[0].info()["local_edges"]
    four = [s.info()["local_edges"] for s in shards_of(eng, n, e, accw, 4, "degree")]
    assert sum(four) == one
    assert max(four) < 0.4 * one  # edge-balanced (row-granular) split
