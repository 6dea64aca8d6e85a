"""Shared helpers for the parity tests."""
import numpy as np


def sorted_sets(offsets, members):
    return [np.sort(members[offsets[i]:offsets[i + 1]]) for i in range(offsets.size - 1)]


def assert_sets_equal(gpu_off, gpu_mem, orc, first_slot=0, msg=""):
    """GPU store slice (visit order) vs oracle Sketches (sorted)."""
    n_sets = gpu_off.size - 1
    assert n_sets == orc.offsets.size - 1, msg
    sizes_g = np.diff(gpu_off.astype(np.int64))
    sizes_o = np.diff(orc.offsets.astype(np.int64))
    bad = np.nonzero(sizes_g != sizes_o)[0]
    assert bad.size == 0, f"{msg}: set sizes differ at slots {first_slot + bad[:10]}"
    # roots: first member in visit order == reference RRRSet::root
    if n_sets:
        roots = gpu_mem[gpu_off[:-1].astype(np.int64)] if gpu_mem.size else np.zeros(0)
        nz = sizes_g > 0
        assert (roots[nz] == orc.roots[nz]).all(), f"{msg}: roots differ"
    gs = sorted_sets(gpu_off, gpu_mem)
    for i, (a, b) in enumerate(zip(gs, orc.sets())):
        if not np.array_equal(a, b):
            raise AssertionError(f"{msg}: set {first_slot + i} differs: gpu={a[:20]} ref={b[:20]}")


def random_store(n, nsets, rng, max_frac=0.2):
    """proj/tests/test_util.hpp:77-99 analogue: distinct members, root first."""
    max_size = max(1, int(max_frac * n))
    off = [0]
    mem = []
    for _ in range(nsets):
        size = int(rng.integers(1, max_size + 1))
        mem.extend(rng.choice(n, size=size, replace=False).tolist())
        off.append(len(mem))
    return np.array(off, np.uint64), np.array(mem, np.uint32)
