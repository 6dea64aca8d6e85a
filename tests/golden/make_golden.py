"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists and oracle/_ref is
built):   python tests/golden/make_golden.py

Every vector below is computed by the unmodified reference headers through
oracle/_ref/librrflow_ref.so; the port oracle and the GPU path are checked
against these files, so parity stays pinned on the GPU box where the
reference sources are absent.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Oracle  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402


def kat(ref):
    out = {"streams": [], "theta": {}}
    for run_seed, slot in [(1, 0), (1, 1), (1, 12345), (7, 2**40 + 3), (2**63 + 5, 99)]:
        s = ref.derive_stream_seed(run_seed, slot)
        d = ref.draws(s, 4)
        below, nxt = ref.uniform_below(s, 65536)
        below_n, _ = ref.uniform_below(s, 4_847_571)
        out["streams"].append({
            "run_seed": run_seed, "slot": slot, "stream_seed": int(s),
            "draws": [int(x) for x in d], "below_65536": int(below), "next_u01": nxt,
            "below_4847571": int(below_n)})
    out["theta"] = {
        "lambda_prime_1e4_50": ref.lambda_prime(10000, 50, 0.5, 1.0),
        "theta_round1_1e4_50": int(ref.theta_for_round(10000, 50, 0.5, 1.0, 1)),
        "lambda_star_100_2": ref.lambda_star(100, 2, 0.5, 1.0),
        "set_theta_100_2_lb10": int(ref.set_theta(100, 2, 0.5, 1.0, 10.0)),
        "effective_ell_65536": ref.effective_ell(1.0, 65536),
        "sampling_rounds": {str(n): int(ref.sampling_rounds(n))
                            for n in [1, 4, 5, 65536, 1632803, 3072441, 4847571]},
        "theta_rounds_cfg4": [int(ref.theta_for_round(4847571, 50, 0.5,
                                                       ref.effective_ell(1.0, 4847571), i))
                              for i in range(1, 6)],
        "set_theta_cfg5": int(ref.set_theta(3072441, 100, 0.5,
                                            ref.effective_ell(1.0, 3072441), 12345.678)),
    }
    return out


def sketch_fixtures(ref):
    cases = {}
    # the reference's own synthetic fixtures (proj/tests/test_sampling.cpp:132-178)
    for name, (kind, n, frac, gseed, wseed, model, rseed, count) in {
        "scc300_ic": (1, 300, 0.25, 13, 5, 0, 99, 500),
        "scc120_lt": (1, 120, 0.3, 3, 21, 1, 7, 400),
        "er64_ic": (0, 64, 0.03, 77, 1, 0, 5, 300),
    }.items():
        arrays = ref.synth_graph(kind, n, frac, gseed, wseed)
        cases[name] = (arrays, model, rseed, count)
    # scaled-down BASELINE generators
    for name, (cfg, n, m) in {
        "rmat_ic": ("cfg1", 1 << 10, 1 << 13),
        "rmat_lt": ("cfg2", 1 << 10, 1 << 13),
        "cl_corr_lt": ("cfg4", 3000, 30000),
        "cl_undir_ic": ("cfg5", 2000, 12000),
    }.items():
        c = graphs.scaled(graphs.CONFIGS[cfg], n, m)
        cases[name] = (graphs.generate(c), c.model, 1, 600)
    out = {}
    for name, ((roff, rsrc, rw), model, rseed, count) in cases.items():
        sk = ref.graph(roff, rsrc, rw).sample(model, rseed, 0, count, workers=4)
        out[f"{name}/roff"] = roff
        out[f"{name}/rsrc"] = rsrc
        out[f"{name}/rw"] = rw
        out[f"{name}/meta"] = np.array([model, rseed, count], np.uint64)
        out[f"{name}/offsets"] = sk.offsets
        out[f"{name}/members"] = sk.members
        out[f"{name}/roots"] = sk.roots
        out[f"{name}/counter"] = sk.counter
    return out


def selection_fixtures(ref):
    rng = np.random.default_rng(2411)
    out = {}
    for t in range(8):
        n = int(2 + rng.integers(0, 300))
        nsets = int(rng.integers(0, 500))
        off = [0]
        mem = []
        for _ in range(nsets):
            size = int(rng.integers(1, max(1, int(0.15 * n)) + 1))
            mem.extend(sorted(rng.choice(n, size=size, replace=False).tolist()))
            off.append(len(mem))
        off = np.array(off, np.uint64)
        mem = np.array(mem, np.uint32)
        k = int(1 + rng.integers(0, min(n, 10)))
        seeds, marg, rc = ref.select(n, off, mem, k, capture=True)
        out[f"s{t}/meta"] = np.array([n, k], np.uint64)
        out[f"s{t}/offsets"] = off
        out[f"s{t}/members"] = mem
        out[f"s{t}/seeds"] = np.array(seeds, np.uint32)
        out[f"s{t}/marginals"] = np.array(marg, np.uint64)
        out[f"s{t}/round_counters"] = rc
    return out


def imm_fixtures(ref):
    out = []
    for cfg, n, m, k in [("cfg1", 1 << 10, 1 << 13, 10), ("cfg2", 1 << 10, 1 << 13, 10),
                         ("cfg4", 3000, 30000, 5), ("cfg3", 3000, 40000, 5)]:
        c = graphs.scaled(graphs.CONFIGS[cfg], n, m)
        arrays = graphs.generate(c)
        r = ref.graph(*arrays).imm(k=k, model=c.model, workers=4)
        r.pop("t_generate"), r.pop("t_select"), r.pop("t_total")
        out.append({"cfg": cfg, "n": n, "m": m, "k": k, "model": c.model, "result": r})
    return out


def main():
    ref = Oracle("reference")
    assert ref.kind == "reference"
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat(ref), f, indent=1)
    np.savez_compressed(os.path.join(HERE, "sketches.npz"), **sketch_fixtures(ref))
    np.savez_compressed(os.path.join(HERE, "selection.npz"), **selection_fixtures(ref))
    with open(os.path.join(HERE, "imm.json"), "w") as f:
        json.dump(imm_fixtures(ref), f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
