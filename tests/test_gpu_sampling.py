"""GPU sampling parity: every RRR set bit-identical to the reference's, slot by slot.

Re-expresses proj/tests/test_sampling.cpp and the per-slot parity contract of
SURVEY.md section 8(c) against the CUDA path (librrgpu.so through the C ABI).
"""
import numpy as np
import pytest

import paper_2411_09473_b200 as P
from paper_2411_09473_b200 import graphs
from helpers import assert_sets_equal

pytestmark = pytest.mark.gpu

IC, LT = 0, 1


def gpu_sample(arrays, model, run_seed, count, fused=True, chunks=1, **opts):
    g = P.Graph(*arrays)
    for k, v in opts.items():
        g.set_option(k, v)
    st = P.RRRStore(g)
    per = [count // chunks] * chunks
    per[-1] += count - sum(per)
    for c in per:
        P.generate_batch(g, model, run_seed, c, st, fused=fused)
    off, mem = st.export()
    return g, st, off, mem


SMALL = [
    ("cfg1", IC, 1 << 11, 1 << 15),
    ("cfg2", LT, 1 << 11, 1 << 15),
    ("cfg3", IC, 30000, 500000),
    ("cfg4", LT, 40000, 600000),
    ("cfg5", IC, 20000, 300000),
]


@pytest.mark.parametrize("name,model,n,m", SMALL)
def test_sets_match_reference_per_slot(cuda, oracle, name, model, n, m):
    cfg = graphs.scaled(graphs.CONFIGS[name], n, m)
    arrays = graphs.generate(cfg)
    count = 3000
    g, st, off, mem = gpu_sample(arrays, model, 1, count)
    ref = oracle.graph(*arrays).sample(model, 1, 0, count, workers=4)
    assert_sets_equal(off, mem, ref, msg=name)
    assert (st.counter() == ref.counter).all(), "fused counter differs"
    stats = g.last_batch_stats()
    assert stats.sets == count
    assert stats.members == ref.members.size


@pytest.mark.parametrize("model", [IC, LT])
def test_top_ups_continue_the_slot_stream(cuda, oracle, model):
    """Slots continue across generate_batch calls (rrr_store.hpp:34-39)."""
    cfg = graphs.scaled(graphs.CONFIGS["cfg1" if model == IC else "cfg2"], 1 << 10, 1 << 14)
    arrays = graphs.generate(cfg)
    _, st, off, mem = gpu_sample(arrays, model, 7, 2500, chunks=3)
    ref = oracle.graph(*arrays).sample(model, 7, 0, 2500, workers=4)
    assert_sets_equal(off, mem, ref)
    assert (st.counter() == ref.counter).all()


@pytest.mark.parametrize("kary", [2, 8, 16])
def test_lt_vertex_records_at_boundary_degrees(cuda, oracle, kary):
    """In-degrees around the vertex-record cases (whole list up to 8, 16-ary
    pivots above, step 1 below 16), the search arities and the warp-wide tail
    search (> 256), with zero weights (flat CDF runs) and sums below 1."""
    rng = np.random.default_rng(41)
    degs = list(range(0, 20)) + [31, 32, 33, 127, 128, 129, 255, 256, 257, 258, 1023, 1024,
                                 1025, 4095, 4096, 4097]
    n = len(degs)
    dst = np.repeat(np.arange(n, dtype=np.uint32), degs)
    src = rng.integers(0, n, dst.size).astype(np.uint32)
    w = rng.uniform(0.0, 1.0, dst.size).astype(np.float32)
    w[rng.random(dst.size) < 0.2] = 0.0
    roff, rsrc, rw = P.build_graph(n, src, dst, w)
    P.normalize_lt_weights(roff, rw)
    rw *= np.float32(0.97)  # leave "no in-neighbour chosen" reachable
    arrays = (roff, rsrc, rw)
    _, _, off_a, mem_a = gpu_sample(arrays, LT, 13, 6000, lt_scan=0)
    _, _, off_b, mem_b = gpu_sample(arrays, LT, 13, 6000, lt_scan=1, lt_kary=kary)
    assert (off_a == off_b).all() and (mem_a == mem_b).all()
    ref = oracle.graph(*arrays).sample(LT, 13, 0, 6000, workers=4)
    assert_sets_equal(off_b, mem_b, ref)


@pytest.mark.parametrize("kary", [2, 4, 8, 16])
def test_lt_search_mode_is_identical(cuda, oracle, kary):
    cfg = graphs.scaled(graphs.CONFIGS["cfg4"], 40000, 600000)
    arrays = graphs.generate(cfg)
    _, st_a, off_a, mem_a = gpu_sample(arrays, LT, 3, 4000, lt_scan=0)
    _, st_b, off_b, mem_b = gpu_sample(arrays, LT, 3, 4000, lt_scan=1, lt_kary=kary)
    assert (off_a == off_b).all() and (mem_a == mem_b).all()
    ref = oracle.graph(*arrays).sample(LT, 3, 0, 4000, workers=4)
    assert_sets_equal(off_b, mem_b, ref)


def _boundary_lt_graph(seed, skew=False):
    rng = np.random.default_rng(seed)
    degs = list(range(0, 20)) + [31, 32, 33, 127, 128, 129, 255, 256, 257, 258, 1023, 1024,
                                 1025, 4095, 4096, 4097]
    n = len(degs)
    dst = np.repeat(np.arange(n, dtype=np.uint32), degs)
    src = rng.integers(0, n, dst.size).astype(np.uint32)
    w = rng.uniform(0.0, 1.0, dst.size).astype(np.float32)
    w[rng.random(dst.size) < 0.2] = 0.0
    if skew:  # heavy-tailed weights: many CDF entries per guide bucket (search spans)
        w = (w ** 8).astype(np.float32)
    roff, rsrc, rw = P.build_graph(n, src, dst, w)
    P.normalize_lt_weights(roff, rw)
    rw *= np.float32(0.97)  # leave "no in-neighbour chosen" reachable
    return roff, rsrc, rw


@pytest.mark.parametrize("mult", [1, 2, 3, 16])
@pytest.mark.parametrize("skew", [False, True])
def test_lt_guide_mode_is_identical(cuda, oracle, mult, skew):
    """Guide-table steps (lt_scan 2, common.cuh) pick the reference's index:
    boundary degrees, zero weights (flat CDF runs = empty buckets), sums below 1,
    heavy-tailed weights (buckets spanning several entries), every multiplier."""
    arrays = _boundary_lt_graph(43, skew)
    _, _, off_a, mem_a = gpu_sample(arrays, LT, 13, 6000, lt_scan=0)
    g, _, off_b, mem_b = gpu_sample(arrays, LT, 13, 6000, lt_scan=2, lt_guide_mult=mult)
    assert (off_a == off_b).all() and (mem_a == mem_b).all()
    ref = oracle.graph(*arrays).sample(LT, 13, 0, 6000, workers=4)
    assert_sets_equal(off_b, mem_b, ref)


def test_lt_guide_mode_full_weight_and_exact_ties(cuda, oracle):
    """In-lists whose CDF reaches exactly 1.0, single in-edges of weight 1 and
    weights that are exact dyadic fractions (CDF entries on bucket edges)."""
    rng = np.random.default_rng(5)
    n = 3000
    degs = rng.integers(0, 9, n)
    dst = np.repeat(np.arange(n, dtype=np.uint32), degs)
    src = rng.integers(0, n, dst.size).astype(np.uint32)
    w = np.empty(dst.size, np.float32)
    pos = 0
    for v, d in enumerate(degs):
        if d:
            w[pos:pos + d] = np.float32(1.0 / d) if v % 3 else np.float32(2.0 ** -int(np.log2(d) + 1))
        pos += d
    arrays = P.build_graph(n, src, dst, w)
    for mult in (1, 2, 4):
        _, _, off_a, mem_a = gpu_sample(arrays, LT, 5, 5000, lt_scan=0)
        _, _, off_b, mem_b = gpu_sample(arrays, LT, 5, 5000, lt_scan=2, lt_guide_mult=mult)
        assert (off_a == off_b).all() and (mem_a == mem_b).all()
    ref = oracle.graph(*arrays).sample(LT, 5, 0, 5000, workers=4)
    assert_sets_equal(off_b, mem_b, ref)


def test_lt_guide_mode_long_walks(cuda, oracle):
    """Walks past the shared-memory filter (128 members: per-lane table from
    there, with growth) and past the lane budget (1024: big-set path), plus
    revisits at every distance: a weight-1 chain with random back edges."""
    rng = np.random.default_rng(8)
    n = 3000
    dst = np.arange(n - 1, dtype=np.uint32)
    src = dst + 1
    w = np.ones(n - 1, np.float32)
    # a quarter of the chain vertices also draw from a random earlier vertex
    extra = rng.choice(n - 1, (n - 1) // 4, replace=False).astype(np.uint32)
    src = np.concatenate([src, rng.integers(0, n, extra.size).astype(np.uint32)])
    dst = np.concatenate([dst, extra])
    w = np.concatenate([w, np.full(extra.size, 0.02, np.float32)])
    roff, rsrc, rw = P.build_graph(n, src, dst, w)
    P.normalize_lt_weights(roff, rw)
    arrays = (roff, rsrc, rw)
    _, _, off_a, mem_a = gpu_sample(arrays, LT, 21, 3000, lt_scan=0)
    g, _, off_b, mem_b = gpu_sample(arrays, LT, 21, 3000, lt_scan=2)
    sizes = np.diff(off_b.astype(np.int64))
    assert sizes.max() > 1024 and ((sizes > 128) & (sizes < 1024)).sum() > 100
    assert (off_a == off_b).all() and (mem_a == mem_b).all()
    ref = oracle.graph(*arrays).sample(LT, 21, 0, 3000, workers=4)
    assert_sets_equal(off_b, mem_b, ref)


def test_lt_guide_mode_cfg4_shape(cuda, oracle):
    cfg = graphs.scaled(graphs.CONFIGS["cfg4"], 40000, 600000)
    arrays = graphs.generate(cfg)
    _, st_a, off_a, mem_a = gpu_sample(arrays, LT, 3, 4000, lt_scan=0)
    _, st_b, off_b, mem_b = gpu_sample(arrays, LT, 3, 4000, lt_scan=2)
    assert (off_a == off_b).all() and (mem_a == mem_b).all()
    assert (st_a.counter() == st_b.counter()).all()
    ref = oracle.graph(*arrays).sample(LT, 3, 0, 4000, workers=4)
    assert_sets_equal(off_b, mem_b, ref)


def test_append_from_side_store_equals_direct_top_up(cuda):
    """Sets sampled ahead into a side store (generate_slots) and appended later are
    exactly the sets a direct top-up draws (slot j <- stream j)."""
    cfg = graphs.scaled(graphs.CONFIGS["cfg1"], 1 << 11, 1 << 15)
    arrays = graphs.generate(cfg)
    g = P.Graph(*arrays)
    direct = P.RRRStore(g)
    P.generate_batch(g, IC, 3, 3000, direct)
    main = P.RRRStore(g)
    P.generate_batch(g, IC, 3, 1000, main)
    side = P.RRRStore(g)
    P.generate_slots(g, IC, 3, 1000, 2500, side, fused=False)
    main.append_from(side, 0, 1200)
    main.append_from(side, 1200, 800)
    a, b = direct.export(), main.export()
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
    assert (direct.counter() == main.counter()).all()
    assert direct.max_set_size() == main.max_set_size()


def test_export_all_async_equals_sync_export(cuda):
    """The pipelined export (copy stream) returns exactly export() + counter()."""
    import torch
    cfg = graphs.scaled(graphs.CONFIGS["cfg2"], 1 << 11, 1 << 15)
    g = P.Graph(*graphs.generate(cfg))
    st = P.RRRStore(g)
    P.generate_batch(g, LT, 5, 3000, st)
    off, mem = st.export()
    o = torch.empty(st.size() + 1, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    m = torch.empty(st.total_member_count(), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
    c = torch.empty(g.num_vertices, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    s = torch.cuda.Stream()
    assert st.export_all_async(o, m, c, s.cuda_stream) == mem.size
    s.synchronize()
    assert (o == off).all() and (m == mem).all() and (c == st.counter()).all()
    # the compact 32-bit variant (u32 offsets and counts)
    o32 = torch.empty(st.size() + 1, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
    c32 = torch.empty(g.num_vertices, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
    m.fill(0)
    assert st.export_all_async(o32, m, c32, s.cuda_stream) == mem.size
    s.synchronize()
    assert (o32 == off).all() and (m == mem).all() and (c32 == st.counter()).all()


@pytest.mark.parametrize("coop_min", [2, 7, 64, 1 << 30])
def test_lt_cooperative_scan_threshold_changes_nothing(cuda, oracle, coop_min):
    cfg = graphs.scaled(graphs.CONFIGS["cfg2"], 1 << 10, 1 << 14)
    arrays = graphs.generate(cfg)
    _, _, off, mem = gpu_sample(arrays, LT, 11, 1500, lt_coop_min=coop_min)
    ref = oracle.graph(*arrays).sample(LT, 11, 0, 1500)
    assert_sets_equal(off, mem, ref)


@pytest.mark.parametrize("mode", [1, 2, 3])
@pytest.mark.parametrize("coop_min", [1, 33, 256, 1 << 30])
@pytest.mark.parametrize("name,n,m", [("cfg1", 1 << 11, 1 << 15), ("cfg5", 20000, 300000),
                                      ("cfg3", 30000, 500000)])
def test_ic_cooperative_expansion_is_exact(cuda, oracle, coop_min, name, n, m, mode):
    """Warp-cooperative in-list expansion with GF(2) jump-ahead segments draws the
    same stream positions as the serial loop, whatever the threshold, in both
    the lane-per-sample (1) and warp-per-sample (2) schedules."""
    cfg = graphs.scaled(graphs.CONFIGS[name], n, m)
    arrays = graphs.generate(cfg)
    _, st, off, mem = gpu_sample(arrays, IC, 21, 2000, ic_coop_min=coop_min, ic_mode=mode)
    ref = oracle.graph(*arrays).sample(IC, 21, 0, 2000, workers=4)
    assert_sets_equal(off, mem, ref, msg=f"{name} coop_min={coop_min}")
    assert (st.counter() == ref.counter).all()


@pytest.mark.parametrize("wc", [False, True])
@pytest.mark.parametrize("mode", [2, 3])
def test_ic_hub_lists_single_list_windows(cuda, oracle, mode, wc):
    """Duplicate-free hub in-lists around the block schedule's single-list fast
    window (>= 1024 remaining edges, 4096 per window) and whole-list expansion
    (>= 8192: 512-edge sub-windows, several per warp): lengths at the boundaries,
    sources that are already visited (hubs feed each other), certain accepts
    (weight 1) and a mix of small and near-zero weights."""
    rng = np.random.default_rng(2024)
    n = 100000
    hub_deg = [1023, 1024, 1025, 4095, 4096, 4097, 8191, 8192, 8193, 20000, 70001, 3000, 1500]
    src, dst, w = [], [], []
    for h, d in enumerate(hub_deg):
        s_ = rng.choice(np.arange(len(hub_deg), n), d - 4, replace=False)
        s_ = np.concatenate([s_, [(h + 1) % len(hub_deg), (h + 3) % len(hub_deg),
                                  (h + 5) % len(hub_deg), (h + 7) % len(hub_deg)]])
        ww = rng.uniform(0.0, 0.004, d)
        ww[rng.random(d) < 0.002] = 1.0
        ww[rng.random(d) < 0.05] = 0.0
        src.append(s_)
        dst.append(np.full(d, h))
        w.append(ww)
    m2 = 150000  # background edges: every vertex reaches the hubs
    src.append(rng.integers(0, n, m2))
    dst.append(rng.integers(0, n, m2))
    w.append(rng.uniform(0.0, 0.3, m2))
    src = np.concatenate(src).astype(np.uint32)
    dst = np.concatenate(dst).astype(np.uint32)
    w = np.concatenate(w).astype(np.float32)
    keep = src != dst
    pairs = np.unique(np.stack([src[keep], dst[keep]]), axis=1, return_index=True)[1]
    arrays = P.build_graph(n, src[keep][pairs], dst[keep][pairs], w[keep][pairs])
    if wc:  # weighted cascade: equal in-weights 1/indeg (the whole-list expansion path)
        roff = arrays[0].astype(np.int64)
        deg = np.diff(roff)
        arrays = (arrays[0], arrays[1],
                  np.repeat((1.0 / np.maximum(deg, 1)).astype(np.float32), deg))
    _, st, off, mem = gpu_sample(arrays, IC, 31, 1500, ic_mode=mode)
    ref = oracle.graph(*arrays).sample(IC, 31, 0, 1500, workers=4)
    assert_sets_equal(off, mem, ref)
    assert (st.counter() == ref.counter).all()


def test_ic_cooperative_expansion_with_duplicate_sources(cuda, oracle):
    """Parallel edges disable the cooperative path for that in-list only."""
    rng = np.random.default_rng(77)
    n, m = 3000, 60000
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, 40, m).astype(np.uint32)  # long in-lists with repeats
    keep = src != dst
    w = rng.uniform(0.0, 0.05, keep.sum()).astype(np.float32)
    arrays = P.build_graph(n, src[keep], dst[keep], w)
    ref = oracle.graph(*arrays).sample(IC, 4, 0, 1500)
    for mode in (1, 2, 3):
        _, st, off, mem = gpu_sample(arrays, IC, 4, 1500, ic_coop_min=1, ic_mode=mode)
        assert_sets_equal(off, mem, ref)


@pytest.mark.parametrize("inner", [1, 3, 32])
def test_ic_inner_steps_change_nothing(cuda, oracle, inner):
    cfg = graphs.scaled(graphs.CONFIGS["cfg1"], 1 << 10, 1 << 14)
    arrays = graphs.generate(cfg)
    _, _, off, mem = gpu_sample(arrays, IC, 5, 1500, ic_inner=inner)
    ref = oracle.graph(*arrays).sample(IC, 5, 0, 1500)
    assert_sets_equal(off, mem, ref)


def test_reference_synth_graphs(cuda, ref):
    """The reference's own fixtures (test_sampling.cpp:132-164) through the GPU."""
    for (kind, n, frac, gseed, wseed, model, rseed, count) in [
        (1, 300, 0.25, 13, 5, IC, 99, 500),
        (1, 120, 0.3, 3, 21, LT, 7, 400),
        (1, 200, 0.2, 17, 11, IC, 31, 200),
        (1, 200, 0.2, 17, 11, LT, 31, 200),
        (0, 64, 0.03, 77, 1, IC, 5, 300),
    ]:
        arrays = ref.synth_graph(kind, n, frac, gseed, wseed)
        _, st, off, mem = gpu_sample(arrays, model, rseed, count)
        orc = ref.graph(*arrays).sample(model, rseed, 0, count, workers=3)
        assert_sets_equal(off, mem, orc, msg=f"synth {kind} {n}")
        assert (st.counter() == orc.counter).all()


def test_big_set_path(cuda, oracle):
    """Dense IC (weights near 1) makes sets exceed the per-lane budget (1024),
    exercising the deferred warp-per-set path."""
    rng = np.random.default_rng(5)
    n, m = 6000, 60000
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    w = rng.uniform(0.2, 0.6, src.size).astype(np.float32)
    arrays = P.build_graph(n, src, dst, w)
    g, st, off, mem = gpu_sample(arrays, IC, 9, 600, ic_mode=1)
    assert g.last_batch_stats().deferred > 0
    ref = oracle.graph(*arrays).sample(IC, 9, 0, 600, workers=4)
    assert_sets_equal(off, mem, ref)
    assert (st.counter() == ref.counter).all()


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_giant_sets_all_schedules(cuda, oracle, mode):
    """Supercritical IC: sets of tens of thousands of members (> the 32K warp
    budget for some) go through the warp, block and big-set paths."""
    rng = np.random.default_rng(11)
    n, m = 40000, 400000
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    keep = src != dst
    w = rng.uniform(0.1, 0.45, keep.sum()).astype(np.float32)
    arrays = P.build_graph(n, src[keep], dst[keep], w)
    g, st, off, mem = gpu_sample(arrays, IC, 17, 300, ic_mode=mode)
    ref = oracle.graph(*arrays).sample(IC, 17, 0, 300, workers=8)
    assert np.diff(ref.offsets.astype(np.int64)).max() > 1024
    assert_sets_equal(off, mem, ref)
    assert (st.counter() == ref.counter).all()


@pytest.mark.parametrize("name,model,mode", [("cfg1", IC, 1), ("cfg1", IC, 2), ("cfg1", IC, 3),
                                             ("cfg2", LT, 0),
                                             ("cfg4", LT, 0)])
def test_inspected_edges_equal_reference_trip_count(cuda, port, name, model, mode):
    """edges_inspected (the roofline numerator) counts exactly the reference's
    loop trips (sampling.hpp:100-106, :130-136), including re-run slots."""
    cfg = graphs.scaled(graphs.CONFIGS[name], 1 << 12, 1 << 16) if name != "cfg4" else \
        graphs.scaled(graphs.CONFIGS[name], 40000, 600000)
    arrays = graphs.generate(cfg)
    for scan in ((0, 1, 2) if model == LT else (0,)):
        g = P.Graph(*arrays)
        g.set_option("lt_scan", scan)
        if model == IC:
            g.set_option("ic_mode", mode)
        st = P.RRRStore(g)
        P.generate_batch(g, model, 2, 5000, st)
        ref = port.graph(*arrays).sample(model, 2, 0, 5000, workers=4)
        assert g.last_batch_stats().edges_inspected == ref.inspected


def test_duplicate_edges_and_weights_edge_cases(cuda, oracle):
    """Parallel edges (kept by load_edge_list, graph.hpp:163-165), zero, one,
    subnormal and >1 weights, isolated vertices."""
    edges = [(0, 1, 0.5), (0, 1, 0.5), (2, 1, 1.0), (3, 1, 0.0), (4, 1, 1e-40),
             (1, 2, 2.0), (5, 2, 0.25), (5, 2, 0.25), (6, 0, 0.999999)]
    n = 8
    src = np.array([e[0] for e in edges], np.uint32)
    dst = np.array([e[1] for e in edges], np.uint32)
    w = np.array([e[2] for e in edges], np.float32)
    arrays = P.build_graph(n, src, dst, w)
    for model in (IC, LT):
        if model == LT:
            arrays = (arrays[0], arrays[1], P.normalize_lt_weights(arrays[0], arrays[2].copy()))
        _, st, off, mem = gpu_sample(arrays, model, 3, 2000)
        ref = oracle.graph(*arrays).sample(model, 3, 0, 2000)
        assert_sets_equal(off, mem, ref)


def test_single_vertex_and_count_zero(cuda):
    """test_sampling.cpp:111-130."""
    g = P.Graph.from_edges(1, [])
    st = P.RRRStore(g)
    assert P.generate_batch(g, IC, 1, 0, st) == 0
    assert st.size() == 0
    P.generate_batch_fused(g, IC, 1, 7, st)
    assert st.size() == 7
    assert st.counter().tolist() == [7]
    assert all(len(s) == 1 for s in st.sets())


def test_deterministic_sketches(cuda):
    """Isolated root; forced reverse edge (test_sampling.cpp:44-59, :80-87)."""
    g = P.Graph.from_edges(2, [(0, 1, 1.0)])
    for model in (IC, LT):
        st = P.RRRStore(g)
        P.generate_batch(g, model, 123, 200, st)
        for s in st.sets(sort=False):
            assert (s.tolist() == [0]) or (s.tolist() == [1, 0])


def test_bernoulli_and_categorical_rates(cuda):
    """test_sampling.cpp:61-72 (0.5 +- 0.01) and :89-109 (0.3/0.3/0.4 +- 0.01)."""
    g = P.Graph.from_edges(2, [(0, 1, 0.5)])
    st = P.RRRStore(g)
    P.generate_batch(g, IC, 4242, 100000, st)
    sets = st.sets()
    with_root1 = [s for s in sets if 1 in s]
    rate = np.mean([0 in s for s in with_root1])
    assert abs(rate - 0.5) < 0.01
    g = P.Graph.from_edges(3, [(0, 2, 0.3), (1, 2, 0.3)])
    st = P.RRRStore(g)
    P.generate_batch(g, LT, 777, 300000, st)
    rooted = [s for s in st.sets(sort=False) if s[0] == 2]
    a1 = np.mean([0 in s for s in rooted])
    a2 = np.mean([1 in s for s in rooted])
    assert abs(a1 - 0.3) < 0.01 and abs(a2 - 0.3) < 0.01 and abs(1 - a1 - a2 - 0.4) < 0.01


def test_empty_graph_is_rejected(cuda):
    g = P.Graph(np.zeros(1, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32))
    st = P.RRRStore(g)
    with pytest.raises(ValueError):
        P.generate_batch(g, IC, 1, 5, st)


@pytest.mark.timeout(300)
def test_lane_tags_after_failed_cooperative_expansion(cuda, oracle):
    """Regression: a lane whose cooperative hub expansion grows its table and
    then overflows the lane budget (the set is deferred) must start its next
    sample under a tag past the abandoned one. Every sample here does exactly
    that (root -> hub with a 3,000-edge duplicate-free in-list, ~1,350 accepted),
    several times per lane; before the fix, later samples on a lane found the
    abandoned entries live (endless probe chains: cfg3 1M lane batches hung in
    about half the runs)."""
    n, hubs, deg = 40000, 10, 3000
    rng = np.random.default_rng(17)
    src, dst, w = [], [], []
    for h in range(hubs):
        s_ = rng.choice(np.arange(hubs, n), deg, replace=False)
        src.append(s_)
        dst.append(np.full(deg, h))
        w.append(np.full(deg, 0.45))
    v = np.arange(hubs, n)
    src.append(v % hubs)
    dst.append(v)
    w.append(np.ones(v.size))
    arrays = P.build_graph(n, np.concatenate(src).astype(np.uint32),
                           np.concatenate(dst).astype(np.uint32),
                           np.concatenate(w).astype(np.float32))
    count = 200000
    g, st, off, mem = gpu_sample(arrays, IC, 3, count, ic_mode=1)
    assert g.last_batch_stats().deferred > count // 2
    ref = oracle.graph(*arrays).sample(IC, 3, 0, 4000, workers=8)
    assert_sets_equal(off[:4001], mem[:int(off[4000])], ref)


def test_lt_nonmonotone_cdf_falls_back_to_the_linear_scan(cuda, oracle):
    """A negative in-weight makes some in-list's CDF non-monotone: the
    guide table and search trees would be wrong there, so the graph samples LT
    with the reference's linear scan -- same sets as the reference."""
    rng = np.random.default_rng(23)
    n, m = 2000, 30000
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    keep = src != dst
    pairs = np.unique(np.stack([src[keep], dst[keep]]), axis=1)
    w = rng.uniform(0.0, 0.1, pairs.shape[1]).astype(np.float32)
    w[::97] = -0.05  # (NaN would do the same; the checker cannot round-trip NaN weights)
    arrays = P.build_graph(n, pairs[0], pairs[1], w)
    for scan in (2, 1, 0):
        _, st, off, mem = gpu_sample(arrays, LT, 9, 3000, lt_scan=scan)
        ref = oracle.graph(*arrays).sample(LT, 9, 0, 3000, workers=4)
        assert_sets_equal(off, mem, ref, msg=f"lt_scan {scan}")


@pytest.mark.parametrize("mode", [0, 3])
def test_ic_window_conflict_repairs(cuda, oracle, mode):
    """Near-critical IC on short in-lists: giant sets whose 4,096-edge windows of
    the block schedule hold many repeated sources: conflicts with >= 1,024 edges
    after them are repaired inside the window (stored draw words, epoch map;
    ~250 here), the rest cut (~5,900); every set must still be the reference's."""
    rng = np.random.default_rng(2411)
    n, deg = 30000, 24
    dst = np.repeat(np.arange(n, dtype=np.uint32), deg)
    z = (rng.zipf(1.6, dst.size) % n).astype(np.uint32)  # popular sources repeat
    u = rng.integers(0, n, dst.size).astype(np.uint32)
    src = np.where(rng.random(dst.size) < 0.5, z, u).astype(np.uint32)
    w = rng.uniform(0.0, 0.16, dst.size).astype(np.float32)  # ~87 of 400 sets > 2,000 members
    keep = src != dst
    pairs = np.unique(np.stack([src[keep], dst[keep]]), axis=1, return_index=True)[1]
    arrays = P.build_graph(n, src[keep][pairs], dst[keep][pairs], w[keep][pairs])
    _, st, off, mem = gpu_sample(arrays, IC, 5, 400, ic_mode=mode)
    sizes = np.diff(off.astype(np.int64))
    assert sizes.max() > 2000  # giant sets: multi-window, repair territory
    ref = oracle.graph(*arrays).sample(IC, 5, 0, 400, workers=4)
    assert_sets_equal(off, mem, ref)
    assert (st.counter() == ref.counter).all()
