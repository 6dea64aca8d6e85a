"""The LT running sums (sampling.hpp:130-136: acc = 0.0, acc += (double)w[j] in
CSR order) as the device builds them (K0: k_build_cdf for short in-lists, the
exactness-checked parallel scan k_build_cdf_long for hubs) must be the host's
sequential fp64 sums bit for bit -- also where adds ROUND (tiny weights below
the sum's last place, sums past 1, binade crossings), which is where a parallel
scan would differ if its TwoSum check missed anything."""
import ctypes as C

import numpy as np
import pytest

import paper_2411_09473_b200 as P
from paper_2411_09473_b200 import _lib

pytestmark = pytest.mark.gpu


def host_cdf(off, w):
    """np.cumsum over float64 adds sequentially left to right (no pairwise
    blocking for cumsum), i.e. the reference's chain, per in-list."""
    out = np.empty(w.size, np.float64)
    wd = w.astype(np.float64)
    for v in range(off.size - 1):
        a, b = int(off[v]), int(off[v + 1])
        if b > a:
            out[a:b] = np.cumsum(wd[a:b])
    return out


def device_cdf(off, src, w, hint=None):
    g = P.Graph(off, src, w, model=hint)
    cdf = np.empty(w.size, np.float64)
    _lib.check(_lib.lib.rrg_debug_export_lt_cdf(g.handle, cdf.ctypes.data_as(C.POINTER(C.c_double))))
    g.close()
    return cdf


def lists_to_graph(lists, n):
    off = np.zeros(n + 1, np.uint64)
    for v, ws in enumerate(lists):
        off[v + 1] = off[v] + len(ws)
    w = np.concatenate([np.asarray(x, np.float32) for x in lists]) if lists else np.zeros(0, np.float32)
    rng = np.random.default_rng(1)
    src = rng.integers(0, n, w.size).astype(np.uint32)
    return off, src, w


def test_cumsum_is_the_sequential_chain():
    rng = np.random.default_rng(0)
    w = (rng.random(5000) * rng.choice([1e-12, 1e-6, 1e-2], 5000)).astype(np.float32).astype(np.float64)
    acc, ref = 0.0, np.empty(5000)
    for i, x in enumerate(w):
        acc = acc + x
        ref[i] = acc
    assert np.array_equal(np.cumsum(w), ref)


@pytest.mark.parametrize("hint", [None, 1])
def test_hub_cdf_is_the_serial_chain_bit_for_bit(cuda, hint):
    rng = np.random.default_rng(2411)
    lists = []
    # hubs (>= 4096 entries: k_build_cdf_long) of assorted lengths around the
    # 256-entry chunk and 512-entry stage boundaries, odd starts included
    for deg in (4096, 4097, 4351, 4352, 4353, 4607, 5000, 8191, 12289, 70001, 300007):
        u = rng.random(deg)
        lists.append((u / u.sum()).astype(np.float32))          # normalized: exact adds mostly
    # rounding adds everywhere: weights spanning 40 binades
    deg = 20000
    lists.append((rng.random(deg) * 2.0 ** rng.integers(-60, -10, deg) / 4).astype(np.float32))
    # a few tiny weights among ordinary ones (the cfg4 pattern), sums past 1 and 2
    w = (rng.random(50000) / 20000).astype(np.float32)
    w[rng.integers(0, 50000, 40)] = np.float32(1e-30)
    w[rng.integers(0, 50000, 40)] = np.float32(3e-41)  # denormal floats
    lists.append(w)
    # zeros, and a list of equal weights
    z = np.zeros(6000, np.float32)
    z[::7] = 1e-3
    lists.append(z)
    lists.append(np.full(9000, 1.0 / 9000, np.float32))
    # short lists in between (k_build_cdf) so hub starts land on odd offsets
    mixed = []
    for i, l in enumerate(lists):
        mixed.append(rng.random(1 + i % 5).astype(np.float32) / 8)
        mixed.append(l)
    n = len(mixed) + 3
    mixed += [np.zeros(0, np.float32)] * 3
    off, src, w = lists_to_graph(mixed, n)
    got = device_cdf(off, src, w, hint)
    want = host_cdf(off, w)
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, (bad[:5], got[bad[:5]], want[bad[:5]])
