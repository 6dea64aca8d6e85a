"""Parity at the full BASELINE sizes through size-independent properties:
the fused counter equals a recount of the exported store; every set has unique
members and the reference's root first; randomly chosen slots equal the
reference's sets (replayed by the checker at their slot ids); the LT search
modes agree set for set."""
import numpy as np
import pytest

import paper_2411_09473_b200 as P
from paper_2411_09473_b200 import graphs
from helpers import assert_sets_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg4_graph():
    cfg = graphs.CONFIGS["cfg4"]
    return cfg, graphs.generate(cfg)


def check_store(st, n):
    off, mem = st.export()
    sizes = np.diff(off.astype(np.int64))
    assert (sizes >= 1).all()
    counts = np.bincount(mem, minlength=n).astype(np.uint64)
    assert (counts == st.counter()).all(), "fused counter != recount"
    sid = np.repeat(np.arange(sizes.size), sizes)
    key = sid.astype(np.int64) * n + mem.astype(np.int64)
    assert np.unique(key).size == key.size, "duplicate member inside a set"
    return off, mem


def test_cfg4_full_size_lt(cuda, oracle, cfg4_graph):
    cfg, arrays = cfg4_graph
    n = arrays[0].size - 1
    g = P.Graph(*arrays)
    st_a = P.RRRStore(g)
    g.set_option("lt_scan", 1)
    P.generate_batch(g, 1, 1, 1 << 16, st_a)
    off, mem = check_store(st_a, n)
    og = oracle.graph(*arrays)
    rng = np.random.default_rng(4)
    for s in sorted(rng.choice(1 << 16, 64, replace=False).tolist()):
        ref = og.sample(1, 1, int(s), 1)
        assert_sets_equal(off[s:s + 2] - off[s], mem[off[s]:off[s + 1]], ref, first_slot=s)
    g.set_option("lt_scan", 0)
    st_b = P.RRRStore(g)
    P.generate_batch(g, 1, 1, 1 << 14, st_b)
    off_b, mem_b = st_b.export()
    assert (off_b == off[: off_b.size]).all() and (mem_b == mem[: mem_b.size]).all()
    g.set_option("lt_scan", 2)
    st_c = P.RRRStore(g)
    P.generate_batch(g, 1, 1, 1 << 16, st_c)
    off_c, mem_c = st_c.export()
    assert (off_c == off).all() and (mem_c == mem).all(), "guide mode != search mode"
    assert (st_c.counter() == st_a.counter()).all()


@pytest.mark.parametrize("name,count", [("cfg1", 1 << 20), ("cfg3", 1 << 20)])
def test_ic_full_size(cuda, oracle, name, count):
    cfg = graphs.CONFIGS[name]
    arrays = graphs.generate(cfg)
    n = arrays[0].size - 1
    g = P.Graph(*arrays)
    st = P.RRRStore(g)
    P.generate_batch(g, 0, 1, count, st)
    off, mem = check_store(st, n)
    og = oracle.graph(*arrays)
    rng = np.random.default_rng(5)
    picks = rng.choice(count, 64, replace=False).tolist()
    sizes = np.diff(off.astype(np.int64))
    picks += np.argsort(sizes)[-8:].tolist()  # the biggest sets (cooperative / big-set paths)
    for s in sorted(set(int(x) for x in picks)):
        ref = og.sample(0, 1, s, 1)
        assert_sets_equal(off[s:s + 2] - off[s], mem[off[s]:off[s + 1]], ref, first_slot=s)
