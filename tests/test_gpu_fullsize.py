"""Parity at the full BASELINE sizes.

* run_imm on every BASELINE config (cfg1-cfg5 at their full sizes, k = 50 / 100,
  epsilon = 0.5) against the reference's own run_imm (oracle/_ref): seeds,
  marginals, theta, theta', LB, sets generated, mean and max set size, all
  bit-exact (imm.hpp:214-251).
* per-slot sets: random slots plus the 16 largest sets of a batch on every
  config equal the reference's sets (replayed by the checker at their slot ids,
  sampling.hpp:159-199); size-independent properties over the whole batch (the
  fused counter equals a recount of the exported store, members are unique per
  set); the LT search modes agree set for set."""
import functools
import os

import numpy as np
import pytest

import paper_2411_09473_b200 as P
from paper_2411_09473_b200 import graphs
from helpers import assert_sets_equal

pytestmark = pytest.mark.gpu


@functools.lru_cache(maxsize=2)
def full_graph(name):
    cfg = graphs.CONFIGS[name]
    return cfg, graphs.generate(cfg)


@pytest.fixture(scope="module")
def cfg4_graph():
    return full_graph("cfg4")


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def check_slots(off, mem, og, model, picks):
    for s in sorted(set(int(x) for x in picks)):
        ref = og.sample(model, 1, s, 1)
        assert_sets_equal(off[s:s + 2] - off[s], mem[off[s]:off[s + 1]], ref, first_slot=s)


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


@pytest.mark.parametrize("name,count", [("cfg1", 1 << 20), ("cfg2", 1 << 20), ("cfg3", 1 << 20),
                                        ("cfg5", 1 << 13)])
def test_full_size_slots(cuda, oracle, name, count):
    """64 random slots + the 16 largest sets of a full-size batch (cfg5: the
    24M-inspected-edge sets that run the whole-list expansion and the in-window
    conflict repairs) equal the reference's; counter == recount over the batch."""
    cfg, arrays = full_graph(name)
    n = arrays[0].size - 1
    g = P.Graph(*arrays)
    st = P.RRRStore(g)
    P.generate_batch(g, cfg.model, 1, count, st)
    off, mem = check_store(st, n)
    og = oracle.graph(*arrays)
    rng = np.random.default_rng(5)
    picks = rng.choice(count, 64, replace=False).tolist()
    sizes = np.diff(off.astype(np.int64))
    picks += np.argsort(sizes, kind="stable")[-16:].tolist()  # the largest sets
    check_slots(off, mem, og, cfg.model, picks)
    st.close()
    g.close()


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_full_size_imm_matches_reference(cuda, oracle, name):
    """run_imm at the BASELINE sizes, GPU vs the reference's run_imm on all host
    cores: every field of ImmResult the reference computes deterministically."""
    cfg, arrays = full_graph(name)
    g = P.Graph(*arrays)
    res = P.run_imm(g, P.ImmConfig(k=cfg.k, epsilon=cfg.epsilon, model=cfg.model, rng_seed=1))
    g.close()
    ref = oracle.graph(*arrays).imm(k=cfg.k, epsilon=cfg.epsilon, model=cfg.model,
                                    workers=cores(), rng_seed=1)
    assert res.seeds.seeds == ref["seeds"]
    assert res.seeds.marginal_counts == ref["marginals"]
    assert (res.theta, res.theta_prime, res.lower_bound) == \
        (ref["theta"], ref["theta_prime"], ref["lower_bound"])
    assert res.sets_generated == ref["sets_generated"]
    assert res.max_set_size == ref["max_set_size"]
    assert res.mean_set_size == ref["mean_set_size"]
    assert res.mean_coverage_fraction == ref["mean_coverage_fraction"]
