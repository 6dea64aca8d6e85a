"""The rest of the reference's store / selection surface through the C ABI:
RRRStore::live_count / is_live after a selection (rrr_store.hpp:62, :84; the
store stays tombstoned, imm.hpp:194-195), a caller-held prebuilt Counter
(selection.hpp:209-218), SelectionStats round counters (:45-49, :237-239) and
BatchOutOfMemory{sets_generated} (sampling.hpp:148-154)."""
import numpy as np
import pytest

import paper_2411_09473_b200 as P
from paper_2411_09473_b200 import graphs

pytestmark = pytest.mark.gpu

IC = 0


def small(name="cfg1", n=1 << 11, m=1 << 15):
    return graphs.generate(graphs.scaled(graphs.CONFIGS[name], n, m))


@pytest.mark.parametrize("index", [False, True])
def test_live_count_and_flags_after_selection(cuda, oracle, monkeypatch, index):
    if index:
        monkeypatch.setenv("RRGPU_SELECT_INDEX", "1")
    arrays = small()
    n = arrays[0].size - 1
    g = P.Graph(*arrays)
    st = P.RRRStore(g)
    P.generate_batch(g, IC, 3, 3000, st)
    assert st.live_count() == 3000 and st.live_flags().all()
    sel = P.select_seeds(st, n, 15)
    off, mem = st.export()
    covered = np.array([bool(np.isin(sel.seeds, mem[off[i]:off[i + 1]]).any()) for i in range(3000)])
    assert st.live_count() == 3000 - sum(sel.marginal_counts) == int((~covered).sum())
    assert (st.live_flags() == ~covered).all()
    assert (st.live_flags(100, 50) == ~covered[100:150]).all()
    P.generate_batch(g, IC, 3, 10, st)  # an append revives every set (finalize)
    assert st.live_count() == 3010 and st.live_flags().all()


def test_prebuilt_counter_and_stats(cuda, oracle):
    arrays = small("cfg2")
    n = arrays[0].size - 1
    g = P.Graph(*arrays)
    st = P.RRRStore(g)
    P.generate_batch(g, 1, 5, 2500, st, fused=False)
    off, mem = st.export()
    tally = np.bincount(mem, minlength=n).astype(np.uint64)
    stats = P.SelectionStats(capture_round_counters=True)
    s = P.select_seeds(st, n, 12, prebuilt=tally, stats=stats)
    seeds, marg, rc = oracle.select(n, off, mem, 12, capture=True)
    assert s.seeds == seeds and s.marginal_counts == marg
    assert (stats.round_counters == rc).all()
    # a different starting tally changes the greedy exactly like the reference's
    skew = tally.copy()
    skew[7] += 100000
    s2 = P.select_seeds(st, n, 3, prebuilt=skew)
    assert s2.seeds[0] == 7


def test_batch_out_of_memory_keeps_a_consistent_store(cuda, oracle):
    arrays = small()
    n = arrays[0].size - 1
    g = P.Graph(*arrays)
    st = P.RRRStore(g)
    P.generate_batch(g, IC, 1, 500, st)
    mean = st.total_member_count() / 500
    limit = st.total_member_count() + int(5.5 * 1024 * mean)  # ~5 chunks of 1024 sets fit
    st.set_member_limit(limit)
    with pytest.raises(P.RRGOutOfMemory) as e:
        P.generate_batch(g, IC, 1, 200000, st)
    made = e.value.sets_generated
    assert 0 < made < 200000 and st.size() == 500 + made
    assert st.total_member_count() <= limit
    ref = oracle.graph(*arrays).sample(IC, 1, 0, 500 + made, workers=4)
    assert (st.counter() == ref.counter).all()
    off, mem = st.export()
    assert (np.diff(off.astype(np.int64)) == np.diff(ref.offsets.astype(np.int64))).all()
    st.set_member_limit(0)
    P.generate_batch(g, IC, 1, 100, st)  # the store keeps working past the failure
    assert st.size() == 600 + made


def test_graph_destroyed_before_its_store(cuda):
    """A caller's garbage collector may finalize a graph before its stores (e.g.
    both in a reference cycle): the graph stays alive until its last store goes."""
    arrays = small()
    g = P.Graph(*arrays)
    st = P.RRRStore(g)
    P.generate_batch(g, IC, 1, 100, st)
    g.close()
    assert st.size() == 100 and st.total_member_count() > 0
    st.close()


def _sets(g, model, seed, count):
    st = P.RRRStore(g)
    P.generate_batch(g, model, seed, count, st)
    off, mem = st.export()
    return off, mem, st.counter()


@pytest.mark.parametrize("name,model", [("cfg2", 1), ("cfg1", 0)])
def test_graph_created_with_a_model_hint_samples_the_same_sets(cuda, oracle, name, model):
    """rrg_graph_create_for: the LT layouts are built while the sources upload;
    the sets are the plain graph's (and the reference's)."""
    arrays = small(name, 1 << 12, 1 << 16)
    plain = _sets(P.Graph(*arrays), model, 7, 3000)
    hinted = _sets(P.Graph(*arrays, model=model), model, 7, 3000)
    for a, b in zip(plain, hinted):
        assert np.array_equal(a, b)
    ref = oracle.graph(*arrays).sample(model, 7, 0, 3000)
    assert np.array_equal(plain[2], ref.counter)
    # the other model on a hinted graph still works (the hint is only a hint)
    other = 1 - model
    a = _sets(P.Graph(*arrays), other, 3, 500)
    b = _sets(P.Graph(*arrays, model=model), other, 3, 500)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_model_hint_keeps_the_upload_checks(cuda):
    off, src, w = small("cfg2", 1 << 10, 1 << 13)
    bad_off = off.copy()
    bad_off[5] = bad_off[-1] + 7  # beyond m: the CDF kernels must never see it
    with pytest.raises(ValueError):
        P.Graph(bad_off, src, w, model=1)
    bad_src = src.copy()
    bad_src[11] = off.size + 3
    with pytest.raises(ValueError):
        P.Graph(off, bad_src, w, model=1)
    with pytest.raises(ValueError):
        P.Graph(off, src, w, model=7)


@pytest.mark.parametrize("hint", [None, 1])
def test_lite_guide_table_then_full_table(cuda, oracle, hint):
    """Small LT batches on an unprepared graph walk the lite guide table (8-byte
    entries built from the CDF alone -- with a model hint, while the sources
    upload); a large batch replaces it with the full table. Every batch is the
    reference's."""
    arrays = small("cfg2", 1 << 12, 1 << 16)
    og = oracle.graph(*arrays)
    g = P.Graph(*arrays, model=hint)
    st = P.RRRStore(g)
    done = 0
    for count in (2000, 3000, 1 << 17, 1000):  # lite, lite, full (large batch), full
        P.generate_batch(g, 1, 9, count, st)
        done += count
    off, mem = st.export()
    ref = og.sample(1, 9, 0, done)
    assert np.array_equal(np.diff(off.astype(np.int64)), np.diff(ref.offsets.astype(np.int64)))
    assert np.array_equal(st.counter(), ref.counter)
    for i in list(range(0, 5000, 97)) + list(range(done - 1000, done, 53)):
        assert np.array_equal(np.sort(mem[off[i]:off[i + 1]]),
                              ref.members[ref.offsets[i]:ref.offsets[i + 1]]), i


def test_model_hint_edge_cases(cuda, oracle):
    """rrg_graph_create_for on degenerate inputs: no vertices, no edges, and an
    LT graph whose CDF is not monotone (a negative weight: no lite table, the
    linear scan samples it) -- same behaviour as the plain constructor."""
    g0 = P.Graph(np.zeros(1, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32), model=1)
    assert g0.num_vertices == 0
    with pytest.raises(ValueError):
        P.generate_batch(g0, 1, 1, 4, P.RRRStore(g0))  # empty graph (sampling.hpp:165)
    g1 = P.Graph(np.zeros(6, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32), model=1)
    st = P.RRRStore(g1)
    P.generate_batch(g1, 1, 3, 50, st)
    off, mem = st.export()
    assert (np.diff(off.astype(np.int64)) == 1).all()  # isolated roots (test_sampling.cpp:44-50)
    rng = np.random.default_rng(5)
    n, m = 1500, 20000
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    keep = src != dst
    pairs = np.unique(np.stack([src[keep], dst[keep]]), axis=1)
    w = rng.uniform(0.0, 0.1, pairs.shape[1]).astype(np.float32)
    w[::53] = -0.02
    arrays = P.build_graph(n, pairs[0], pairs[1], w)
    a = _sets(P.Graph(*arrays), 1, 11, 2000)
    b = _sets(P.Graph(*arrays, model=1), 1, 11, 2000)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    ref = oracle.graph(*arrays).sample(1, 11, 0, 2000, workers=2)
    assert np.array_equal(a[2], ref.counter)
