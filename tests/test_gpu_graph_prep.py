"""On-device graph preparation: the transpose of an edge
list in detail::build_graph's in-list order (graph.hpp:69-115) and
normalize_lt_weights (graph.hpp:207-235), built on the GPU, must be
byte-identical to the host restatements (pinned to the reference by
tests/test_oracle_pin.py), and sampling on it must give the same sets."""
import numpy as np
import pytest

import paper_2411_09473_b200 as P
from helpers import assert_sets_equal

pytestmark = pytest.mark.gpu


def edge_list(seed, n, m, hub=0, dup=0.05, wlo=0.0, whi=1.0):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    if hub:  # one vertex with a long in-list, sources in random order
        src = np.concatenate([src, rng.integers(0, n, hub).astype(np.uint32)])
        dst = np.concatenate([dst, np.full(hub, n // 3, np.uint32)])
    k = int(dup * src.size)  # parallel edges, in shuffled positions
    pick = rng.integers(0, src.size, k)
    src = np.concatenate([src, src[pick]])
    dst = np.concatenate([dst, dst[pick]])
    perm = rng.permutation(src.size)
    src, dst = src[perm], dst[perm]
    w = rng.uniform(wlo, whi, src.size).astype(np.float32)
    w[rng.random(src.size) < 0.05] = 0.0
    return src, dst, w


def same_bits(a, b):
    return a.shape == b.shape and (a.view(np.uint32) == b.view(np.uint32)).all()


@pytest.mark.parametrize("n,m,hub", [(1, 0, 0), (7, 30, 0), (5000, 60000, 0),
                                     (40000, 300000, 120000), (70000, 50000, 0)])
def test_device_transpose_matches_build_graph(cuda, oracle, n, m, hub):
    src, dst, w = edge_list(n + m, n, m, hub)
    roff, rsrc, rw = oracle.build_graph(n, src, dst, w)  # detail::build_graph itself
    g = P.Graph.from_edge_arrays(n, src, dst, w)
    assert (g.reverse_offsets == roff).all()
    assert (g.reverse_sources == rsrc).all()
    assert same_bits(g.reverse_weights, rw)


@pytest.mark.parametrize("whi", [0.01, 0.3, 1.0, 3.0])
def test_device_normalize_matches_normalize_lt_weights(cuda, oracle, whi):
    """Sums below one (untouched), above one (deflation loop), exact ones."""
    n = 20000
    src, dst, w = edge_list(int(whi * 100), n, 200000, hub=60000, whi=whi)
    roff, rsrc, rw = oracle.build_graph(n, src, dst, w)
    rw_n = oracle.normalize_lt(roff, rw.copy())
    g = P.Graph.from_edge_arrays(n, src, dst, w, normalize_lt=True)
    assert (g.reverse_sources == rsrc).all()
    assert same_bits(g.reverse_weights, rw_n)


@pytest.mark.parametrize("whi", [0.01, 1.0, 3.0])
def test_device_normalize_hub_lists(cuda, oracle, whi):
    """Average in-degree ~260: many lists on either side of the warp-per-list
    threshold (256 in-edges, k_normalize_lt_hubs), chunk tails of every length."""
    n = 2000
    src, dst, w = edge_list(int(whi * 1000) + 7, n, 500000, hub=5000, whi=whi)
    roff, rsrc, rw = oracle.build_graph(n, src, dst, w)
    deg = np.diff(roff.astype(np.int64))
    assert (deg >= 256).sum() > 100 and (deg < 256).sum() > 10
    rw_n = oracle.normalize_lt(roff, rw.copy())
    g = P.Graph.from_edge_arrays(n, src, dst, w, normalize_lt=True)
    assert same_bits(g.reverse_weights, rw_n)


def test_device_normalize_hub_lists_with_rounding_adds(cuda, oracle):
    """Hub in-lists whose running sums ROUND (weights spanning 40 binades, tiny
    weights among ordinary ones, sums far above 1 so the deflation loop runs):
    the checked parallel scan of k_normalize_lt_hubs must fall back to the serial
    chain exactly where the reference's adds are inexact."""
    rng = np.random.default_rng(99)
    n = 64
    dsts, ws = [], []
    for v in range(n):
        deg = int(rng.integers(300, 6000))
        kind = v % 4
        if kind == 0:
            w = rng.random(deg) * 2.0 ** rng.integers(-45, -5, deg)
        elif kind == 1:
            w = rng.random(deg) / deg * 3.0           # sums ~1.5: deflated
            w[rng.integers(0, deg, 8)] = 1e-30
        elif kind == 2:
            w = rng.random(deg) * 5.0                 # sums in the thousands
        else:
            w = np.full(deg, 1.0 / deg) * (1 + 1e-3)  # equal weights just above 1
        dsts.append(np.full(deg, v, np.uint32))
        ws.append(w.astype(np.float32))
    dst = np.concatenate(dsts)
    w = np.concatenate(ws)
    src = rng.integers(0, 1 << 20, dst.size).astype(np.uint32) % 100000 + n  # no self-loops
    nn = 100000 + n
    roff, rsrc, rw = oracle.build_graph(nn, src, dst, w)
    rw_n = oracle.normalize_lt(roff, rw.copy())
    g = P.Graph.from_edge_arrays(nn, src, dst, w, normalize_lt=True)
    assert same_bits(g.reverse_weights, rw_n)


def test_device_normalize_negative_on_hub(cuda):
    src, dst, w = edge_list(5, 100, 50000, hub=3000)
    w[np.flatnonzero(dst == 33)[-1]] = -0.25  # inside the hub list of vertex 33
    with pytest.raises(ValueError, match="vertex 33"):
        P.Graph.from_edge_arrays(100, src, dst, w, normalize_lt=True)


def test_device_graph_errors(cuda):
    with pytest.raises(ValueError):
        P.Graph.from_edge_arrays(4, [0, 5], [1, 2], [0.5, 0.5])
    with pytest.raises(ValueError):
        P.Graph.from_edge_arrays(4, [0, 1], [1, 2], [0.5, -0.5], normalize_lt=True)
    g = P.Graph.from_edge_arrays(4, [0, 1], [1, 2], [0.5, -0.5])  # no normalization: kept
    assert g.reverse_weights.tolist() == [0.5, -0.5]
    # out-of-range targets are rejected before the sort and the offsets fill
    for bad_dst in (4, 5, 0xFFFFFFFF):
        with pytest.raises(ValueError, match="out of range"):
            P.Graph.from_edge_arrays(4, [0, 1, 2], [1, bad_dst, 3], [0.5, 0.5, 0.5])
    # the context is still usable afterwards
    g = P.Graph.from_edge_arrays(4, [0, 1, 2], [1, 3, 3], [0.5, 0.5, 0.5])
    assert g.reverse_offsets.tolist() == [0, 0, 1, 1, 3]
    with pytest.raises(ValueError, match="differ in length"):
        P.Graph.from_edge_arrays(4, [0, 1], [1], [0.5, 0.5])


def test_device_graph_long_empty_runs(cuda):
    """Targets only in the upper half of the id range (and a lone target at 0):
    the offsets of long zero-in-degree runs are filled in parallel."""
    n = 1 << 20
    src = np.array([5, 6, 7, 8], np.uint32)
    dst = np.array([0, n - 1, n - 1, n // 2], np.uint32)
    g = P.Graph.from_edge_arrays(n, src, dst, np.full(4, 0.25, np.float32))
    ref = P.build_graph(n, src, dst, np.full(4, 0.25, np.float32))
    assert (g.reverse_offsets == ref[0]).all()
    assert (g.reverse_sources == ref[1]).all()


@pytest.mark.parametrize("model", [0, 1])
def test_sampling_on_device_built_graph(cuda, oracle, model):
    n = 3000
    src, dst, w = edge_list(9, n, 40000, hub=5000, whi=0.2 if model == 0 else 1.0)
    g = P.Graph.from_edge_arrays(n, src, dst, w, normalize_lt=model == 1)
    st = P.RRRStore(g)
    P.generate_batch(g, model, 5, 3000, st)
    off, mem = st.export()
    arrays = (g.reverse_offsets, g.reverse_sources, g.reverse_weights)
    ref = oracle.graph(*arrays).sample(model, 5, 0, 3000, workers=4)
    assert_sets_equal(off, mem, ref)
