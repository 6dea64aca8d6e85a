"""GPU selection parity: given the identical RRR-set collection, the coverage
counts, seeds and marginals are bit-exact with the reference's select_seeds.

Re-expresses proj/tests/test_selection.cpp and acceptance.cpp criteria 01-03.
"""
import numpy as np
import pytest

import paper_2411_09473_b200 as P
from helpers import random_store

pytestmark = pytest.mark.gpu


def store_from_lists(n, lists):
    g = P.Graph(np.zeros(n + 1, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32))
    st = P.RRRStore(g)
    off = np.zeros(len(lists) + 1, np.uint64)
    for i, l in enumerate(lists):
        off[i + 1] = off[i] + len(l)
    mem = np.array([v for l in lists for v in l], np.uint32)
    if len(lists):
        st.import_sets(off, mem)
    return g, st


def test_hand_greedy(cuda):
    """test_selection.cpp:139-153."""
    g, st = store_from_lists(3, [[0, 1], [0], [2]])
    s = P.select_seeds(st, 3, 2)
    assert s.seeds == [0, 2] and s.marginal_counts == [2, 1]
    g, st = store_from_lists(4, [[1, 2], [1], [3]])
    s = P.select_seeds(st, 4, 1)
    assert s.seeds == [1] and s.marginal_counts == [2]


def test_k_bounds_and_empty_store_fill(cuda):
    """test_selection.cpp:155-164."""
    g, st = store_from_lists(3, [[0]])
    with pytest.raises(ValueError):
        P.select_seeds(st, 3, 4)
    with pytest.raises(ValueError):
        P.select_seeds(st, 3, 0)
    g, st = store_from_lists(5, [])
    s = P.select_seeds(st, 5, 3)
    assert s.seeds == [0, 1, 2] and s.marginal_counts == [0, 0, 0]


def test_ties_go_to_lowest_id(cuda):
    """test_selection.cpp:43-55 via one-round selection."""
    g, st = store_from_lists(3, [[0], [0], [0], [1], [2]])
    assert P.select_seeds(st, 3, 1).seeds == [0]
    g, st = store_from_lists(3, [[0], [0], [1], [1], [2]])
    assert P.select_seeds(st, 3, 1).seeds == [0]
    g, st = store_from_lists(5, [[4], [3], [3], [4]])
    assert P.select_seeds(st, 5, 1).seeds == [3]


def test_exhaustion_fill_skips_selected(cuda):
    g, st = store_from_lists(6, [[3], [3, 4], [5]])
    s = P.select_seeds(st, 6, 5)
    assert s.seeds == [3, 5, 0, 1, 2] and s.marginal_counts == [2, 1, 0, 0, 0]


@pytest.fixture(params=["scan", "index"])
def select_mode(request, monkeypatch):
    """Both ways of finding the sets that hold the round's seed: scanning the
    flat members (default up to 2^25 members) and the inverted index."""
    if request.param == "index":
        monkeypatch.setenv("RRGPU_SELECT_INDEX", "1")
    else:
        monkeypatch.delenv("RRGPU_SELECT_INDEX", raising=False)
    return request.param


@pytest.mark.parametrize("trial", range(12))
def test_random_stores_match_reference_with_round_counters(cuda, oracle, trial, select_mode):
    """acceptance.cpp:128-155 (criterion 02) + :111-126 (criterion 01)."""
    rng = np.random.default_rng(202 + trial)
    n = int(2 + rng.integers(0, 400))
    nsets = int(1 + rng.integers(0, 800))
    off, mem = random_store(n, nsets, rng, 0.15)
    k = int(1 + rng.integers(0, min(n, 10)))
    g, st = store_from_lists(n, [mem[off[i]:off[i + 1]].tolist() for i in range(nsets)])
    ref_counts = np.bincount(mem, minlength=n).astype(np.uint64)
    assert (st.counter() == ref_counts).all()
    seeds, marg, rc = oracle.select(n, off, np.concatenate(
        [np.sort(mem[off[i]:off[i + 1]]) for i in range(nsets)]).astype(np.uint32), k,
        capture=True)
    for prebuilt in (True, False):
        for thr in (0.0, 0.25, 1.0):
            s = P.select_seeds(st, n, k, thr, prebuilt=prebuilt, capture_round_counters=True)
            assert s.seeds == seeds
            assert s.marginal_counts == marg
            assert s.round_counters.shape == rc.shape
            assert (s.round_counters == rc).all()


@pytest.mark.parametrize("n,nsets,k", [(20000, 5000, 40), (70000, 3000, 60)])
def test_many_tiles_match_reference(cuda, oracle, select_mode, n, nsets, k):
    """Vertex counts spanning many argmax tiles (2048 vertices each): maxima kept
    per tile and re-reduced only where a count changed."""
    rng = np.random.default_rng(n + nsets)
    # skewed membership: a few hot vertices (ties across tiles) plus a long tail
    sizes = rng.integers(1, 40, nsets)
    hot = rng.choice(n, 64, replace=False)
    lists = []
    for sz in sizes:
        pool = np.concatenate([rng.choice(hot, min(sz // 3 + 1, 64), replace=False),
                               rng.integers(0, n, sz)])
        lists.append(np.unique(pool)[:sz].tolist())
    g, st = store_from_lists(n, lists)
    off = np.zeros(nsets + 1, np.uint64)
    off[1:] = np.cumsum([len(l) for l in lists])
    mem = np.concatenate([np.sort(np.array(l, np.uint32)) for l in lists]).astype(np.uint32)
    seeds, marg = oracle.select(n, off, mem, k)
    s = P.select_seeds(st, n, k)
    assert s.seeds == seeds and s.marginal_counts == marg


def test_sampled_store_selection_matches_reference(cuda, oracle, select_mode):
    """Selection over the GPU's own sampled store vs the reference's select_seeds
    over the reference's store (identical collections by the sampling parity)."""
    from paper_2411_09473_b200 import graphs
    cfg = graphs.scaled(graphs.CONFIGS["cfg1"], 1 << 12, 1 << 16)
    arrays = graphs.generate(cfg)
    g = P.Graph(*arrays)
    st = P.RRRStore(g)
    P.generate_batch(g, 0, 1, 20000, st)
    orc = oracle.graph(*arrays).sample(0, 1, 0, 20000, workers=4)
    seeds, marg = oracle.select(g.num_vertices, orc.offsets, orc.members, 50)
    s = P.select_seeds(st, g.num_vertices, 50)
    assert s.seeds == seeds and s.marginal_counts == marg
    # the store is left tombstoned; a second call revives everything (selection.hpp:215)
    s2 = P.select_seeds(st, g.num_vertices, 50)
    assert s2.seeds == seeds
    assert P.fraction_covered(st, s) == pytest.approx(sum(marg) / 20000, abs=0)


def test_fraction_covered(cuda):
    """test_selection.cpp:219-238."""
    g, st = store_from_lists(4, [[0], [1], [2]])
    assert P.fraction_covered(st, [0, 1, 2]) == 1.0
    assert P.fraction_covered(st, []) == 0.0
    rng = np.random.default_rng(53)
    off, mem = random_store(60, 80, rng)
    g, st = store_from_lists(60, [mem[off[i]:off[i + 1]].tolist() for i in range(80)])
    seeds = [1, 5, 17, 33]
    hit = sum(any(v in seeds for v in mem[off[i]:off[i + 1]]) for i in range(80))
    assert P.fraction_covered(st, seeds) == hit / 80


def test_coverage_of_prefixes_nondecreasing(cuda):
    """test_selection.cpp:240-253."""
    rng = np.random.default_rng(59)
    off, mem = random_store(80, 100, rng)
    g, st = store_from_lists(80, [mem[off[i]:off[i + 1]].tolist() for i in range(100)])
    s = P.select_seeds(st, 80, 10)
    prev = 0.0
    for L in range(1, 11):
        f = P.fraction_covered(st, s.seeds[:L])
        assert f >= prev
        prev = f


@pytest.mark.parametrize("cluster", ["0", "1"])
@pytest.mark.parametrize("threshold", [0.0, 0.25, 2.0])
@pytest.mark.parametrize("name", ["cfg1", "cfg4"])
def test_cluster_and_grid_selection_equal_reference(cuda, oracle, monkeypatch, cluster,
                                                    threshold, name):
    """The cluster-resident selection (one 16-block cluster, tile maxima replicated
    in shared memory, DSMEM tile flags) and the cooperative-grid one give the
    reference's seeds, marginals and covered count, with and without rebuilds."""
    from paper_2411_09473_b200 import graphs
    monkeypatch.setenv("RRGPU_SELECT_CLUSTER", cluster)
    cfg = graphs.scaled(graphs.CONFIGS[name], 1 << 13 if name == "cfg1" else 40000,
                        1 << 17 if name == "cfg1" else 600000)
    arrays = graphs.generate(cfg)
    n = arrays[0].size - 1
    g = P.Graph(*arrays)
    st = P.RRRStore(g)
    P.generate_batch(g, cfg.model, 3, 6000, st, density_divisor=0)  # list sets only
    off, mem = st.export()
    seeds, marg = oracle.select(n, off, mem, 40, threshold=threshold)
    for _ in range(2):  # the store is revived by every selection
        s = P.select_seeds(st, n, 40, adaptive_threshold=threshold)
        assert s.seeds == seeds and s.marginal_counts == marg
        assert st.live_count() == 6000 - sum(marg)
