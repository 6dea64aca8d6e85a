"""Pins the CPU checkers (CPU only, no GPU).

* the port restatement (oracle/port.cpp) against the golden vectors the
  reference produced (tests/golden/, tests/golden/make_golden.py);
* the port against the reference library itself where oracle/_ref is built;
* the reference's frozen known-answer values (proj/tests/test_imm.cpp:36-42,
  :52-57) and SURVEY.md Appendix A.
"""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load_kat():
    with open(os.path.join(GOLD, "kat.json")) as f:
        return json.load(f)


def test_appendix_a_kats(port):
    """SURVEY.md Appendix A, computed from prng.hpp."""
    rows = [(1, 0, 0xe99ff867dbf682c9, 0x2f5b5f3017c3f107, 0x64296db5b7c65d61, 12123,
             0.39125714956733171),
            (1, 1, 0xf893a2eefb32555e, 0x89faeafca43b9699, 0x06a6b64f63462214, 35322,
             0.025981325513634079),
            (1, 12345, 0x1a7807bc728ce4ed, 0xca114aef00f41d9a, 0x4171d1ce0514f259, 51729,
             0.25564299850255501)]
    for run_seed, slot, ss, d0, d1, below, u in rows:
        s = port.derive_stream_seed(run_seed, slot)
        assert s == ss
        d = port.draws(s, 2)
        assert int(d[0]) == d0 and int(d[1]) == d1
        b, nxt = port.uniform_below(s, 65536)
        assert b == below and nxt == u


def test_golden_streams(port):
    for row in load_kat()["streams"]:
        s = port.derive_stream_seed(row["run_seed"], row["slot"])
        assert s == row["stream_seed"]
        assert [int(x) for x in port.draws(s, 4)] == row["draws"]
        b, nxt = port.uniform_below(s, 65536)
        assert b == row["below_65536"] and nxt == row["next_u01"]
        assert port.uniform_below(s, 4_847_571)[0] == row["below_4847571"]


def test_frozen_theta_values(port):
    """proj/tests/test_imm.cpp:36-42 and :52-57 (1e-12 relative, as Catch::Approx there)."""
    assert port.lambda_prime(10000, 50, 0.5, 1.0) == pytest.approx(16000551.4717494, rel=1e-12)
    assert port.theta_for_round(10000, 50, 0.5, 1.0, 1) == 3201
    assert port.lambda_star(100, 2, 0.5, 1.0) == pytest.approx(15552.279899859497, rel=1e-12)
    assert port.set_theta(100, 2, 0.5, 1.0, 10.0) == 1556
    t = load_kat()["theta"]
    assert port.lambda_prime(10000, 50, 0.5, 1.0) == t["lambda_prime_1e4_50"]
    assert port.lambda_star(100, 2, 0.5, 1.0) == t["lambda_star_100_2"]
    assert port.effective_ell(1.0, 65536) == t["effective_ell_65536"]
    for n, r in t["sampling_rounds"].items():
        assert port.sampling_rounds(int(n)) == r
    ell = port.effective_ell(1.0, 4847571)
    assert [port.theta_for_round(4847571, 50, 0.5, ell, i) for i in range(1, 6)] == \
        t["theta_rounds_cfg4"]
    assert port.set_theta(3072441, 100, 0.5, port.effective_ell(1.0, 3072441), 12345.678) == \
        t["set_theta_cfg5"]


def test_theta_doubling(port):
    """test_imm.cpp:17-29."""
    n = 1 << 12
    for i in range(1, port.sampling_rounds(n)):
        a = port.theta_for_round(n, 10, 0.5, 1.0, i)
        b = port.theta_for_round(n, 10, 0.5, 1.0, i + 1)
        assert 2 * a - 1 <= b <= 2 * a


def sketch_cases():
    z = np.load(os.path.join(GOLD, "sketches.npz"))
    names = sorted({k.split("/")[0] for k in z.files})
    return z, names


@pytest.mark.parametrize("case", sketch_cases()[1])
def test_port_reproduces_reference_sketches(port, case):
    z, _ = sketch_cases()
    g = port.graph(z[f"{case}/roff"], z[f"{case}/rsrc"], z[f"{case}/rw"])
    model, rseed, count = (int(x) for x in z[f"{case}/meta"])
    sk = g.sample(model, rseed, 0, count, workers=3)
    assert (sk.offsets == z[f"{case}/offsets"]).all()
    assert (sk.members == z[f"{case}/members"]).all()
    assert (sk.roots == z[f"{case}/roots"]).all()
    assert (sk.counter == z[f"{case}/counter"]).all()
    # replay from a non-zero first slot (slot j <- stream j)
    part = g.sample(model, rseed, 37, 50)
    o = z[f"{case}/offsets"]
    assert (part.members == z[f"{case}/members"][o[37]:o[87]]).all()


@pytest.mark.parametrize("i", range(8))
def test_port_selection_matches_reference_golden(port, i):
    z = np.load(os.path.join(GOLD, "selection.npz"))
    n, k = (int(x) for x in z[f"s{i}/meta"])
    seeds, marg, rc = port.select(n, z[f"s{i}/offsets"], z[f"s{i}/members"], k, capture=True)
    assert seeds == z[f"s{i}/seeds"].tolist()
    assert marg == z[f"s{i}/marginals"].tolist()
    assert rc.shape == z[f"s{i}/round_counters"].shape
    assert (rc == z[f"s{i}/round_counters"]).all()


def test_port_imm_matches_reference_golden(port):
    with open(os.path.join(GOLD, "imm.json")) as f:
        cases = json.load(f)
    from paper_2411_09473_b200 import graphs
    for c in cases:
        cfg = graphs.scaled(graphs.CONFIGS[c["cfg"]], c["n"], c["m"])
        r = port.graph(*graphs.generate(cfg)).imm(k=c["k"], model=c["model"])
        for key, val in c["result"].items():
            assert r[key] == val, (c["cfg"], key)


def test_port_vs_reference_live(port, ref):
    """Direct cross-check on a fresh graph when the reference library is built."""
    from paper_2411_09473_b200 import graphs
    for name, n, m in [("cfg1", 1 << 11, 1 << 15), ("cfg4", 8000, 90000)]:
        cfg = graphs.scaled(graphs.CONFIGS[name], n, m)
        arrays = graphs.generate(cfg)
        a = ref.graph(*arrays).sample(cfg.model, 3, 0, 1500, workers=4)
        b = port.graph(*arrays).sample(cfg.model, 3, 0, 1500, workers=2)
        assert (a.members == b.members).all() and (a.offsets == b.offsets).all()
        assert (a.counter == b.counter).all()
        ra = ref.graph(*arrays).imm(k=8, model=cfg.model, workers=4)
        rb = port.graph(*arrays).imm(k=8, model=cfg.model)
        for key in ("seeds", "marginals", "theta", "theta_prime", "lower_bound",
                    "sets_generated", "max_set_size", "mean_set_size"):
            assert ra[key] == rb[key], key


def test_reference_build_graph_and_normalize_match_host_code(ref):
    """The product's host transpose + LT normalization equal the reference's."""
    import paper_2411_09473_b200 as P
    rng = np.random.default_rng(7)
    n, m = 300, 5000
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    w = (rng.random(m) * 0.9).astype(np.float32)
    a = P.build_graph(n, src, dst, w)
    b = ref.build_graph(n, src, dst, w)
    for x, y in zip(a, b):
        assert (x == y).all()
    rw = a[2].copy()
    P.normalize_lt_weights(a[0], rw)
    assert (rw == ref.normalize_lt(a[0], a[2])).all()
    assert not (rw == a[2]).all()  # some in-lists were infeasible and got rescaled


def test_port_sampling_phase_and_baseline_match_reference(port, ref):
    """The C++ restatement's sampling_phase and baseline run_imm against the reference
    headers (imm.hpp:169-209; Strategy::baseline, imm.hpp:147-153)."""
    for (kind, n, frac, gseed, wseed, k, seed, model) in [
        (1, 200, 0.25, 19, 23, 3, 7, 0), (1, 150, 0.2, 5, 9, 4, 31, 1)]:
        arrays = ref.synth_graph(kind, n, frac, gseed, wseed)
        a = port.graph(*arrays).sampling_phase(k=k, model=model, rng_seed=seed, workers=2)
        b = ref.graph(*arrays).sampling_phase(k=k, model=model, rng_seed=seed, workers=2)
        assert a["lower_bound"] == b["lower_bound"] and a["theta_prime"] == b["theta_prime"]
        assert (a["counter"] == b["counter"]).all()
        ra = port.graph(*arrays).imm(k=k, model=model, rng_seed=seed, workers=2, strategy=1)
        rb = ref.graph(*arrays).imm(k=k, model=model, rng_seed=seed, workers=2, strategy=1)
        assert ra["seeds"] == rb["seeds"] and ra["marginals"] == rb["marginals"]
        assert ra["theta"] == rb["theta"]
