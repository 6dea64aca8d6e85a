"""Randomized parity sweep against the CPU checker (oracle/_ref when built, else
the port): random graphs (sizes, degree skew, weight scales incl. hub in-lists
past the warp-per-list thresholds), both models, random seeds / k / batch sizes,
plain and model-hinted graph creation, device-built graphs (LT normalization),
generate_batch + select_seeds + run_imm. Prints one line per case; exits non-zero
at the first mismatch. tests/test_gpu_fuzz.py runs a bounded number of cases;
longer sweeps: python tests/fuzz_parity.py [seconds=240] [seed=1]"""
import sys
import time

import os  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2411_09473_b200 as P  # noqa: E402
from oracle import Oracle, available  # noqa: E402


def run(budget=240.0, seed=1, max_cases=None, verbose=True):
    rng = np.random.default_rng(seed)
    orc = Oracle("reference" if available("reference") else "port")
    t_end = time.time() + budget
    case = 0
    while time.time() < t_end and (max_cases is None or case < max_cases):
        case += 1
        one_case(rng, orc, case, verbose)
    return case, orc.kind


def one_case(rng, orc, case, verbose):
    n = int(rng.choice([50, 400, 3000, 20000]))
    m = int(n * rng.choice([2, 8, 30]))
    hubs = int(rng.integers(0, 4))
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    for h in range(hubs):  # hub in-lists of 300 .. 20000 edges
        deg = int(rng.integers(300, 20000))
        src = np.concatenate([src, rng.integers(0, n, deg).astype(np.uint32)])
        dst = np.concatenate([dst, np.full(deg, int(rng.integers(0, n)), np.uint32)])
    keep = src != dst
    pairs = np.unique(np.stack([src[keep], dst[keep]]), axis=1)
    src, dst = pairs[0], pairs[1]
    model = int(rng.integers(0, 2))
    scale = float(rng.choice([0.02, 0.3, 1.0, 4.0]))
    if rng.random() < 0.3:  # weighted cascade / equal weights per in-list
        indeg = np.bincount(dst, minlength=n).astype(np.float64)
        w = (1.0 / indeg[dst]).astype(np.float32)
    else:
        w = (rng.random(src.size) * scale * 2.0 ** rng.integers(-20, 1, src.size)
             if rng.random() < 0.3 else rng.random(src.size) * scale).astype(np.float32)
    if model == 0:
        w = np.minimum(w, np.float32(1.0))
    device_built = model == 1 and rng.random() < 0.5
    if device_built:
        g = P.Graph.from_edge_arrays(n, src, dst, w, normalize_lt=True)
        arrays = (g.reverse_offsets, g.reverse_sources, g.reverse_weights)
        roff, rsrc, rw = orc.build_graph(n, src, dst, w)
        rw = orc.normalize_lt(roff, rw.copy())
        assert np.array_equal(arrays[0], roff) and np.array_equal(arrays[1], rsrc)
        assert np.array_equal(arrays[2].view(np.uint32), rw.view(np.uint32)), "normalize_lt"
    else:
        roff, rsrc, rw = orc.build_graph(n, src, dst, w)
        if model == 1:
            rw = orc.normalize_lt(roff, rw.copy())
        arrays = (roff, rsrc, rw)
        g = P.Graph(*arrays, model=(model if rng.random() < 0.5 else None))
    og = orc.graph(*arrays)
    seed = int(rng.integers(1, 1 << 40))
    count = int(rng.choice([1, 37, 1000, 9000]))
    st = P.RRRStore(g)
    P.generate_batch(g, model, seed, count, st)
    off, mem = st.export()
    ref = og.sample(model, seed, 0, count, workers=4)
    assert np.array_equal(np.diff(off.astype(np.int64)), np.diff(ref.offsets.astype(np.int64))), "sizes"
    assert np.array_equal(st.counter(), ref.counter), "counter"
    for i in rng.integers(0, count, min(count, 40)):
        assert np.array_equal(np.sort(mem[off[i]:off[i + 1]]),
                              ref.members[ref.offsets[i]:ref.offsets[i + 1]]), f"set {i}"
    k = int(rng.integers(1, min(n, 30) + 1))
    s = P.select_seeds(st, n, k)
    seeds, marg = orc.select(n, ref.offsets, ref.members, k)
    assert s.seeds == seeds and s.marginal_counts == marg, "select"
    eps = float(rng.choice([0.3, 0.5, 0.8]))
    r = P.run_imm(g, P.ImmConfig(k=k, epsilon=eps, model=model, rng_seed=seed))
    rr = og.imm(k=k, epsilon=eps, model=model, workers=4, rng_seed=seed)
    assert r.seeds.seeds == rr["seeds"] and r.seeds.marginal_counts == rr["marginals"], "imm seeds"
    assert (r.theta, r.theta_prime, r.lower_bound, r.sets_generated) == \
        (rr["theta"], rr["theta_prime"], rr["lower_bound"], rr["sets_generated"]), "imm theta"
    if verbose:
        print(f"case {case}: n {n} m {src.size} hubs {hubs} model {model} scale {scale} "
              f"{'device-built ' if device_built else ''}count {count} k {k} eps {eps} "
              f"theta {r.theta} ok", flush=True)
    st.close()
    g.close()

if __name__ == "__main__":
    n_cases, kind = run(float(sys.argv[1]) if len(sys.argv) > 1 else 240.0,
                        int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    print(f"{n_cases} cases ok ({kind} checker)")
