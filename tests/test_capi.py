"""The C-ABI library (CPU only): loads, exports every symbol include/rrgpu.h
declares, and its host-side pieces behave (no device compute calls here)."""
import ctypes
import os
import re
import struct

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "rrgpu.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(rrg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_2411_09473_b200._lib as L
    lib = ctypes.CDLL(L.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    bound = {name for name, _, _ in L.SIGNATURES}
    assert set(syms) == bound, set(syms) ^ bound


def test_library_is_sm100a():
    import paper_2411_09473_b200._lib as L
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {L.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_version_and_errors():
    import paper_2411_09473_b200 as P
    assert "sm_100a" in P.version()
    with pytest.raises(ValueError):
        P.build_graph(3, [0, 5], [1, 1], [0.5, 0.5])  # id out of range
    # mismatched array lengths are rejected before any copy (no read past a buffer)
    with pytest.raises(ValueError, match="differ in length"):
        P.build_graph(3, [0, 1], [1], [0.5, 0.5])
    with pytest.raises(ValueError, match="differ in length"):
        P.build_graph(3, [0, 1], [1, 2], [0.5])
    with pytest.raises(ValueError, match="differ in length"):
        P.Graph(np.array([0, 1, 2], np.uint64), np.array([0, 1], np.uint32),
                np.array([0.5], np.float32))
    with pytest.raises(ValueError, match="differ in length"):
        P.Graph.from_edge_arrays(3, [0, 1], [1, 2], [0.5])


def f32_bits(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


def test_bernoulli_threshold_equals_double_compare():
    """uniform01() < (double)w  <=>  (x >> 11) < threshold(w)   (prng.hpp:46, :62)."""
    from paper_2411_09473_b200._lib import lib
    rng = np.random.default_rng(1)
    weights = list(rng.random(300).astype(np.float32)) + [
        0.0, -0.0, 1.0, 1.5, 1e-45, 1e-40, 1e-30, 2.0 ** -24, 2.0 ** -53, 2.0 ** -54,
        np.float32(0.1), np.float32(1 / 3), float("inf"), -1.0, float("nan"),
        np.nextafter(np.float32(1.0), np.float32(0.0))]
    for w in weights:
        w32 = np.float32(w)
        t = lib.rrg_debug_bernoulli_threshold(f32_bits(float(w32)))
        ks = [0, 1, 2, 2**52, 2**53 - 1, int(rng.integers(0, 2**53))]
        if 0 < t < 2**53:
            ks += [t - 1, t, t + 1]
        for k in ks:
            if k < 0 or k >= 2**53:
                continue
            expect = (k * 2.0 ** -53) < float(w32)
            assert (k < t) == expect, (w, k, t)


def test_record_threshold_high_word_decides_like_the_double_compare():
    """IC records keep T >> 21: x >> 32 < T_hi accepts, > rejects, a tie falls back to
    the full threshold -- identical to uniform01() < (double)w for every x."""
    from paper_2411_09473_b200._lib import lib
    rng = np.random.default_rng(2)
    weights = list(rng.random(200).astype(np.float32)) + [
        0.0, 1.0, 1.5, 1e-45, 2.0 ** -24, 2.0 ** -53, float("inf"), -1.0, float("nan"),
        np.float32(1 / 3), np.nextafter(np.float32(1.0), np.float32(0.0))]
    for w in weights:
        bits = f32_bits(float(np.float32(w)))
        t = lib.rrg_debug_bernoulli_threshold(bits)
        th = lib.rrg_debug_bernoulli_thr_hi(bits)
        xs = [int(x) for x in rng.integers(0, 2**63, 8, dtype=np.uint64)] + [0, 2**64 - 1]
        xs += [(th << 32) | int(lo) for lo in rng.integers(0, 2**32, 8)]  # ties
        xs += [(th << 32), (th << 32) | 0xFFFFFFFF]
        for x in xs:
            x &= 2**64 - 1
            kh, k = x >> 32, x >> 11
            got = kh < th or (kh == th and k < t)
            assert got == ((k * 2.0 ** -53) < float(np.float32(w))), (w, hex(x))


def test_jump_ahead_matches_sequential_draws(port):
    """T^k s == k calls of next_u64 (prng.hpp:33-43) for the GF(2) jump matrices."""
    import ctypes as C
    from paper_2411_09473_b200._lib import lib

    def splitmix_state(seed):
        s = []
        x = seed
        for _ in range(4):
            x = (x + 0x9e3779b97f4a7c15) & (2**64 - 1)
            z = x
            z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & (2**64 - 1)
            z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & (2**64 - 1)
            s.append(z ^ (z >> 31))
        return s

    def out_of(s):  # xoshiro256** output of state s
        r = (s[1] * 5) & (2**64 - 1)
        r = ((r << 7) | (r >> 57)) & (2**64 - 1)
        return (r * 9) & (2**64 - 1)

    seed = port.derive_stream_seed(1, 12345)
    draws = port.draws(seed, 5000)
    s0 = (C.c_uint64 * 4)(*splitmix_state(seed))
    for k in [0, 1, 2, 31, 32, 33, 1000, 4095, 4999]:
        out = (C.c_uint64 * 4)()
        lib.rrg_debug_jump(s0, k, out)
        assert out_of(list(out)) == int(draws[k]), k


def test_generators_are_deterministic_and_simple():
    from paper_2411_09473_b200 import graphs
    for name, n, m in [("cfg1", 1 << 10, 1 << 13), ("cfg3", 5000, 40000), ("cfg4", 5000, 40000),
                       ("cfg5", 3000, 20000)]:
        cfg = graphs.scaled(graphs.CONFIGS[name], n, m)
        a = graphs.generate(cfg, threads=1)
        b = graphs.generate(cfg, threads=5)
        for x, y in zip(a, b):
            assert (x == y).all()
        roff, rsrc, rw = a
        deg = np.diff(roff.astype(np.int64))
        dst = np.repeat(np.arange(deg.size), deg)
        key = dst * (1 << 32) + rsrc.astype(np.int64)
        assert (np.diff(key) > 0).all()  # in-lists by source ascending, no duplicates
        assert not (rsrc == dst).any()  # no self-loops
        expect_arcs = 2 * cfg.m if cfg.kind == graphs.CHUNG_LU_UNDIR else cfg.m
        assert rsrc.size == expect_arcs
        if cfg.weights == graphs.W_LT:
            sums = np.add.reduceat(rw.astype(np.float64), roff[:-1].astype(np.int64))[deg > 0]
            assert (sums <= 1.0).all() and (rw >= 0).all()
        if cfg.weights == graphs.W_WC:
            assert np.allclose(rw, np.repeat(1.0 / np.maximum(deg, 1), deg).astype(np.float32))


def test_undirected_generator_is_symmetric():
    from paper_2411_09473_b200 import graphs
    cfg = graphs.scaled(graphs.CONFIGS["cfg5"], 3000, 20000)
    roff, rsrc, _ = graphs.generate(cfg)
    deg = np.diff(roff.astype(np.int64))
    dst = np.repeat(np.arange(deg.size), deg)
    fwd = set(zip(rsrc.tolist(), dst.tolist()))
    assert all((d, s) in fwd for s, d in fwd)
