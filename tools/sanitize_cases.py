#!/usr/bin/env python
"""Small parity fixtures for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py ic

Every IC schedule (lane, warp, block incl. the single-list windows, the whole-
list expansion and in-window conflict repairs, the big-set path, both fast-mode
variants), every LT mode (linear, search tree, guide table; walks past the
shared-memory filter and the lane budget) and both selection modes (member scan,
inverted index) run on graphs small enough for the sanitizer, and each result is
checked against the CPU port (test infrastructure, oracle/) so a run is also a
parity run. Used by tests/test_gpu_sanitizer.py. No torch import: the only CUDA
client in the process is librrgpu.so.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402
from oracle import Oracle  # noqa: E402

IC, LT = 0, 1
ORC = Oracle("port")


def check(arrays, model, seed, count, **opts):
    g = P.Graph(*arrays)
    for k, v in opts.items():
        g.set_option(k, v)
    st = P.RRRStore(g)
    P.generate_batch(g, model, seed, count, st)
    off, mem = st.export()
    if opts.get("ic_rng", 0) == 0:
        ref = ORC.graph(*arrays).sample(model, seed, 0, count, workers=4)
        assert (np.diff(off.astype(np.int64)) == np.diff(ref.offsets.astype(np.int64))).all(), opts
        for i in range(count):
            a = np.sort(mem[off[i]:off[i + 1]])
            assert np.array_equal(a, ref.members[ref.offsets[i]:ref.offsets[i + 1]]), (opts, i)
        assert (st.counter() == ref.counter).all(), opts
    else:
        sizes = np.diff(off.astype(np.int64))
        assert (sizes >= 1).all()
        assert (np.bincount(mem, minlength=arrays[0].size - 1) == st.counter()).all()
    stats = g.last_batch_stats()
    st.close()
    g.close()
    return off, stats


def hub_graph(n=30000, hub_deg=(1023, 1025, 4097, 8193, 12000), wc=True):
    rng = np.random.default_rng(2024)
    src, dst, w = [], [], []
    for h, d in enumerate(hub_deg):
        s_ = rng.choice(np.arange(len(hub_deg), n), d - 2, replace=False)
        s_ = np.concatenate([s_, [(h + 1) % len(hub_deg), (h + 3) % len(hub_deg)]])
        src.append(s_)
        dst.append(np.full(d, h))
        w.append(rng.uniform(0.0, 0.004, d))
    src.append(rng.integers(0, n, 60000))
    dst.append(rng.integers(0, n, 60000))
    w.append(rng.uniform(0.0, 0.3, 60000))
    src = np.concatenate(src).astype(np.uint32)
    dst = np.concatenate(dst).astype(np.uint32)
    w = np.concatenate(w).astype(np.float32)
    keep = src != dst
    pairs = np.unique(np.stack([src[keep], dst[keep]]), axis=1, return_index=True)[1]
    arrays = P.build_graph(n, src[keep][pairs], dst[keep][pairs], w[keep][pairs])
    if wc:
        deg = np.diff(arrays[0].astype(np.int64))
        arrays = (arrays[0], arrays[1], np.repeat((1.0 / np.maximum(deg, 1)).astype(np.float32), deg))
    return arrays


def conflict_graph(n=6000, deg=24):
    rng = np.random.default_rng(2411)
    dst = np.repeat(np.arange(n, dtype=np.uint32), deg)
    z = (rng.zipf(1.6, dst.size) % n).astype(np.uint32)
    u = rng.integers(0, n, dst.size).astype(np.uint32)
    src = np.where(rng.random(dst.size) < 0.5, z, u).astype(np.uint32)
    w = rng.uniform(0.0, 0.16, dst.size).astype(np.float32)
    keep = src != dst
    pairs = np.unique(np.stack([src[keep], dst[keep]]), axis=1, return_index=True)[1]
    return P.build_graph(n, src[keep][pairs], dst[keep][pairs], w[keep][pairs])


def dense_graph(n=3000, m=30000, lo=0.2, hi=0.6, seed=5):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    keep = src != dst
    w = rng.uniform(lo, hi, keep.sum()).astype(np.float32)
    return P.build_graph(n, src[keep], dst[keep], w)


def case_ic():
    small = graphs.generate(graphs.scaled(graphs.CONFIGS["cfg1"], 1 << 10, 1 << 14))
    for mode in (1, 2, 3):
        check(small, IC, 3, 256, ic_mode=mode)
    check(small, IC, 3, 256)                        # auto (pilot + schedule choice)
    hubs = hub_graph()
    for mode in (2, 3):                              # coop_expand / single-list / whole-list
        check(hubs, IC, 31, 96, ic_mode=mode)
    check(conflict_graph(), IC, 5, 64, ic_mode=3)   # in-window repairs and cuts
    _, stats = check(dense_graph(), IC, 9, 64, ic_mode=1)   # lane -> warp -> block -> big
    assert stats.deferred > 0
    for mode in (1, 2):                              # fast mode: lane / warp (+ big)
        check(hubs, IC, 7, 128, ic_rng=1, ic_mode=mode)
    print("ic ok")


def case_lt():
    small = graphs.generate(graphs.scaled(graphs.CONFIGS["cfg4"], 4000, 60000))
    for scan in (0, 1, 2):
        check(small, LT, 21, 512, lt_scan=scan)
    # walks past the 128-member filter and the 1024-member lane budget
    rng = np.random.default_rng(8)
    n = 1500
    dst = np.arange(n - 1, dtype=np.uint32)
    src = dst + 1
    w = np.ones(n - 1, np.float32)
    extra = rng.choice(n - 1, (n - 1) // 4, replace=False).astype(np.uint32)
    src = np.concatenate([src, rng.integers(0, n, extra.size).astype(np.uint32)])
    dst = np.concatenate([dst, extra])
    w = np.concatenate([w, np.full(extra.size, 0.02, np.float32)])
    roff, rsrc, rw = P.build_graph(n, src, dst, w)
    P.normalize_lt_weights(roff, rw)
    for scan in (0, 2):
        check((roff, rsrc, rw), LT, 21, 256, lt_scan=scan)
    print("lt ok")


def case_select():
    arrays = graphs.generate(graphs.scaled(graphs.CONFIGS["cfg1"], 1 << 10, 1 << 14))
    n = arrays[0].size - 1
    g = P.Graph(*arrays)
    st = P.RRRStore(g)
    P.generate_batch(g, IC, 1, 2000, st)
    off, mem = st.export()
    seeds, marg = ORC.select(n, off, mem, 20)
    for index in (False, True):
        if index:
            os.environ["RRGPU_SELECT_INDEX"] = "1"
        s = P.select_seeds(st, n, 20)
        assert s.seeds == seeds and s.marginal_counts == marg, (index, s.seeds, seeds)
        os.environ.pop("RRGPU_SELECT_INDEX", None)
    r = P.run_imm(g, P.ImmConfig(k=10, epsilon=0.5, model=IC, rng_seed=1))
    ref = ORC.graph(*arrays).imm(k=10, epsilon=0.5, model=IC, workers=2, rng_seed=1)
    assert r.seeds.seeds == ref["seeds"]
    print("select ok")


CASES = {"ic": case_ic, "lt": case_lt, "select": case_select}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
