"""Opt-in FAST IC sampling (RRG_OPT_IC_RNG = 1): counter-based
per-edge draws with geometric skipping. Sets are NOT the reference's slot by slot,
so parity is statistical, with the SURVEY 8(d) fallback criteria: two-sample KS on
set sizes (alpha 0.01), per-vertex coverage within binomial bounds, influence
estimate within 3 sigma -- all against the exact path, which the rest of the suite
pins to the reference. Draws are deterministic, so each check has one fixed outcome."""
import numpy as np
import pytest
from scipy import stats

import paper_2411_09473_b200 as P
from paper_2411_09473_b200 import graphs

pytestmark = pytest.mark.gpu

IC = 0
CASES = [("cfg1", 1 << 12, 1 << 16), ("cfg3", 30000, 500000), ("cfg5", 20000, 300000)]


def sample(arrays, rng_mode, count, seed=1):
    g = P.Graph(*arrays)
    g.set_option("ic_rng", rng_mode)
    st = P.RRRStore(g)
    P.generate_batch(g, IC, seed, count, st)
    off, mem = st.export()
    return g, st, off, mem


@pytest.mark.parametrize("name,n,m", CASES)
def test_fast_sets_are_distributed_like_the_reference(cuda, name, n, m):
    cfg = graphs.scaled(graphs.CONFIGS[name], n, m)
    arrays = graphs.generate(cfg)
    N = 20000
    _, st_f, off_f, mem_f = sample(arrays, 1, N, seed=3)
    _, st_e, off_e, mem_e = sample(arrays, 0, N, seed=3)
    # roots are the reference's (slot stream), the rest is resampled
    assert (mem_f[off_f[:-1].astype(np.int64)] == mem_e[off_e[:-1].astype(np.int64)]).all()
    sz_f = np.diff(off_f.astype(np.int64))
    sz_e = np.diff(off_e.astype(np.int64))
    assert stats.ks_2samp(sz_f, sz_e).pvalue > 0.01, (sz_f.mean(), sz_e.mean())
    # per-vertex coverage: |p_f - p_e| within 4 sigma of the pooled binomial
    cf = st_f.counter().astype(np.float64) / N
    ce = st_e.counter().astype(np.float64) / N
    pool = (cf + ce) / 2
    sig = np.sqrt(np.maximum(pool * (1 - pool), 1.0 / N) * 2.0 / N)
    bad = np.abs(cf - ce) > 4 * sig
    assert bad.mean() <= 1e-3, (bad.sum(), np.abs(cf - ce).max())
    # no set holds a vertex twice; every member is a vertex
    for i in range(0, N, 97):
        s = mem_f[off_f[i]:off_f[i + 1]]
        assert np.unique(s).size == s.size and (s < arrays[0].size - 1).all()


@pytest.mark.parametrize("name,n,m", CASES)
def test_fast_influence_estimate_within_three_sigma(cuda, name, n, m):
    """n F(S) for one seed set S over fast sets vs exact sets (selection.hpp:340-358).
    S is chosen on one exact collection (run_seed 11) and scored on two further,
    independent collections (fast run_seed 12, exact run_seed 13), so neither
    estimate is the in-sample coverage S was optimised for."""
    cfg = graphs.scaled(graphs.CONFIGS[name], n, m)
    arrays = graphs.generate(cfg)
    N = 30000
    _, st_e, _, _ = sample(arrays, 0, N, seed=11)
    seeds = P.select_seeds(st_e, arrays[0].size - 1, 10).seeds
    _, st_f, _, _ = sample(arrays, 1, N, seed=12)
    _, st_e2, _, _ = sample(arrays, 0, N, seed=13)
    f_f = P.fraction_covered(st_f, seeds)
    f_e = P.fraction_covered(st_e2, seeds)
    sig = np.sqrt(max(f_e * (1 - f_e), 1.0 / N) * 2.0 / N)
    assert abs(f_f - f_e) <= 3 * sig, (f_f, f_e, sig)


def test_fast_mode_deterministic_and_top_ups_continue(cuda):
    cfg = graphs.scaled(graphs.CONFIGS["cfg5"], 20000, 300000)
    arrays = graphs.generate(cfg)
    _, _, o1, m1 = sample(arrays, 1, 3000, seed=5)
    g = P.Graph(*arrays)
    g.set_option("ic_rng", 1)
    st = P.RRRStore(g)
    for c in (1000, 1500, 500):
        P.generate_batch(g, IC, 5, c, st)
    o2, m2 = st.export()
    assert (o1 == o2).all() and (m1 == m2).all()


def test_fast_giant_sets_use_the_bitmap_path(cuda):
    """Supercritical graph: sets beyond the 32K-member warp region go to the n-bit
    map variant; sizes stay distributed like the exact path's."""
    rng = np.random.default_rng(11)
    n, m = 60000, 600000
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    keep = src != dst
    w = np.full(keep.sum(), 0.3, np.float32)  # uniform weights: geometric skipping
    arrays = P.build_graph(n, src[keep], dst[keep], w)
    g, st, off, mem = sample(arrays, 1, 400, seed=17)
    sz = np.diff(off.astype(np.int64))
    assert sz.max() > 32 * 1024 and g.last_batch_stats().deferred > 0
    _, _, off_e, _ = sample(arrays, 0, 400, seed=17)
    assert stats.ks_2samp(sz, np.diff(off_e.astype(np.int64))).pvalue > 0.01


def test_fast_imm_runs_and_selects_good_seeds(cuda):
    """IMM with fast sampling: its seeds cover as much of an exact sample as the
    exact IMM's seeds do (within 3 sigma)."""
    cfg = graphs.scaled(graphs.CONFIGS["cfg5"], 20000, 300000)
    arrays = graphs.generate(cfg)
    gf = P.Graph(*arrays)
    gf.set_option("ic_rng", 1)
    rf = P.run_imm(gf, P.ImmConfig(k=10, model=IC))
    re = P.run_imm(P.Graph(*arrays), P.ImmConfig(k=10, model=IC))
    _, st, _, _ = sample(arrays, 0, 40000, seed=99)
    a = P.fraction_covered(st, rf.seeds.seeds)
    b = P.fraction_covered(st, re.seeds.seeds)
    assert a >= b - 3 * np.sqrt(b * (1 - b) / 40000), (a, b)


def test_ic_rng_option_validated(cuda):
    g = P.Graph.from_edges(3, [(0, 1, 0.5)])
    with pytest.raises(ValueError):
        g.set_option("ic_rng", 2)


@pytest.mark.parametrize("name,n,m", CASES)
def test_fast_variants_draw_the_same_sets(cuda, name, n, m):
    """Lane, warp and n-bit-map variants share the per-(slot, vertex, segment/edge)
    draws, so a slot deferred from one to the next is re-run to the same set (no
    selection bias from deferral)."""
    cfg = graphs.scaled(graphs.CONFIGS[name], n, m)
    arrays = graphs.generate(cfg)
    sets = []
    for mode in (1, 2):
        g = P.Graph(*arrays)
        g.set_option("ic_rng", 1)
        g.set_option("ic_mode", mode)
        st = P.RRRStore(g)
        P.generate_batch(g, IC, 21, 3000, st)
        sets.append(st.sets())
    assert all(np.array_equal(a, b) for a, b in zip(*sets))
