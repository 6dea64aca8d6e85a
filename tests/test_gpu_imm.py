"""IMM end to end on the GPU vs the reference's run_imm: seeds, marginals,
theta, theta', LB bit-exact (proj/tests/test_imm.cpp)."""
import math

import numpy as np
import pytest

import paper_2411_09473_b200 as P
from paper_2411_09473_b200 import graphs

pytestmark = pytest.mark.gpu


def compare(res, ref):
    assert res.seeds.seeds == ref["seeds"]
    assert res.seeds.marginal_counts == ref["marginals"]
    assert res.theta == ref["theta"]
    assert res.theta_prime == ref["theta_prime"]
    assert res.lower_bound == ref["lower_bound"]
    assert res.sets_generated == ref["sets_generated"]
    assert res.max_set_size == ref["max_set_size"]
    assert res.mean_set_size == ref["mean_set_size"]


@pytest.mark.parametrize("name,n,m,k", [
    ("cfg1", 1 << 12, 1 << 16, 20),
    ("cfg2", 1 << 12, 1 << 16, 20),
    ("cfg3", 30000, 500000, 10),
    ("cfg4", 40000, 600000, 10),
    ("cfg5", 20000, 300000, 10),
])
def test_imm_matches_reference(cuda, oracle, name, n, m, k):
    cfg = graphs.scaled(graphs.CONFIGS[name], n, m)
    arrays = graphs.generate(cfg)
    g = P.Graph(*arrays)
    res = P.run_imm(g, P.ImmConfig(k=k, epsilon=0.5, model=cfg.model, rng_seed=1))
    ref = oracle.graph(*arrays).imm(k=k, epsilon=0.5, model=cfg.model, workers=4, rng_seed=1)
    compare(res, ref)


def test_reference_fixture_graphs(cuda, ref):
    for (kind, n, frac, gseed, wseed, k, seed, model) in [
        (1, 200, 0.25, 19, 23, 3, 7, 0),
        (1, 120, 0.3, 2, 6, 5, 44, 0),
        (1, 150, 0.2, 5, 9, 4, 31, 1),
        (0, 12, 0.2, 3, 4, 12, 1, 0),
    ]:
        arrays = ref.synth_graph(kind, n, frac, gseed, wseed)
        g = P.Graph(*arrays)
        res = P.run_imm(g, P.ImmConfig(k=k, model=model, rng_seed=seed))
        compare(res, ref.graph(*arrays).imm(k=k, model=model, rng_seed=seed, workers=2))


def test_star_center_and_k_equals_n(cuda):
    """test_imm.cpp:129-153."""
    g = P.Graph.from_edges(9, [(3, v, 1.0) for v in range(9) if v != 3])
    assert P.run_imm(g, P.ImmConfig(k=1, workers=2)).seeds.seeds == [3]
    rng = np.random.default_rng(3)
    edges = [(u, v, float(rng.random())) for u in range(12) for v in range(12)
             if u != v and rng.random() < 0.2]
    g = P.Graph.from_edges(12, edges)
    r = P.run_imm(g, P.ImmConfig(k=12))
    assert sorted(r.seeds.seeds) == list(range(12))


def test_complete_graph_stops_in_round_one(cuda, oracle):
    """test_imm.cpp:59-79."""
    n = 6
    g = P.Graph.from_edges(n, [(u, v, 1.0) for u in range(n) for v in range(n) if u != v])
    r = P.run_imm(g, P.ImmConfig(k=2, epsilon=0.5, workers=2))
    ell = oracle.effective_ell(1.0, n)
    assert r.theta_prime == oracle.theta_for_round(n, 2, 0.5, ell, 1)
    assert r.lower_bound == pytest.approx(n / (1 + math.sqrt(2) * 0.5), rel=1e-12)


def test_single_vertex_lb_one(cuda):
    """test_imm.cpp:81-88 (through run_imm: LB = max(., k) = 1)."""
    g = P.Graph.from_edges(1, [])
    r = P.run_imm(g, P.ImmConfig(k=1))
    assert r.lower_bound == 1.0 and r.seeds.seeds == [0]


def test_validation(cuda):
    """test_imm.cpp:166-177."""
    g = P.Graph.from_edges(3, [(0, 1, 0.5)])
    for cfg in (P.ImmConfig(k=4), P.ImmConfig(k=1, epsilon=1.0), P.ImmConfig(k=1, workers=0),
                P.ImmConfig(k=0)):
        with pytest.raises(ValueError):
            P.run_imm(g, cfg)


@pytest.mark.parametrize("name,n,m,k", [("cfg1", 1 << 12, 1 << 16, 20), ("cfg4", 40000, 600000, 10)])
def test_sampling_phase_matches_reference(cuda, oracle, name, n, m, k):
    """sampling_phase (imm.hpp:169-209): LB, theta' and the phase's fused counter."""
    cfg = graphs.scaled(graphs.CONFIGS[name], n, m)
    arrays = graphs.generate(cfg)
    g = P.Graph(*arrays)
    got = P.sampling_phase(g, P.ImmConfig(k=k, model=cfg.model, rng_seed=3))
    ref = oracle.graph(*arrays).sampling_phase(k=k, model=cfg.model, rng_seed=3, workers=4)
    assert got.lower_bound == ref["lower_bound"]
    assert got.theta_prime == ref["theta_prime"] == got.store.size()
    assert (got.store.counter() == ref["counter"]).all()


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_baseline_strategy_same_seeds(cuda, oracle, name):
    """Strategy::baseline (unfused sampling + baseline_select) returns the fused
    strategy's seeds (test_selection.cpp:188-200); both match the reference's."""
    cfg = graphs.scaled(graphs.CONFIGS[name], *((1 << 12, 1 << 16) if name == "cfg2"
                                               else (30000, 500000)))
    arrays = graphs.generate(cfg)
    g = P.Graph(*arrays)
    k = 10
    base = P.run_imm(g, P.ImmConfig(k=k, model=cfg.model, strategy=P.parse_strategy("baseline")))
    ref = oracle.graph(*arrays).imm(k=k, model=cfg.model, workers=4, strategy=1)
    compare(base, ref)
    fused = P.run_imm(g, P.ImmConfig(k=k, model=cfg.model))
    assert fused.seeds == base.seeds and fused.theta == base.theta


def test_unknown_strategy_rejected(cuda):
    g = P.Graph.from_edges(3, [(0, 1, 0.5), (1, 2, 0.5)])
    with pytest.raises(ValueError):
        P.run_imm(g, P.ImmConfig(k=1, strategy=7))
    with pytest.raises(ValueError):
        P.parse_strategy("nope")


_SPEC_CHILD = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import paper_2411_09473_b200 as P
from paper_2411_09473_b200 import graphs
out = {}
for name, n, m, k in (("cfg1", 1 << 12, 1 << 16, 20), ("cfg3", 30000, 500000, 10)):
    cfg = graphs.scaled(graphs.CONFIGS[name], n, m)
    g = P.Graph(*graphs.generate(cfg))
    icfg = P.ImmConfig(k=k, epsilon=0.5, model=cfg.model, rng_seed=1)
    P.run_imm(g, icfg)       # the first run measures the graph's mean inspected edges,
    r = P.run_imm(g, icfg)   # the second one speculates with it
    out[name] = [r.seeds.seeds, r.seeds.marginal_counts, r.theta, r.theta_prime,
                 r.lower_bound, r.sets_generated, r.max_set_size, r.mean_set_size]
print(json.dumps(out))
"""


def test_speculation_settings_never_change_the_result(cuda):
    """The driver samples later rounds' (and the final top-up's) slots ahead when
    they look cheap; the main store only ever receives the reference's slots, so
    every setting of the tuning variables must give the same ImmResult -- also
    with the trial selections cut short once they provably cannot trigger
    (RRGPU_IMM_EARLY_EXIT)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    results = []
    for free, final, early in (("0", "0", "0"), ("1e15", "1", "1"), ("67108864", "1", "1"),
                               ("1e15", "0", "0"), ("0", "0", "1")):
        env = dict(os.environ, RRGPU_IMM_FREE_EDGES=free, RRGPU_IMM_SPEC_FINAL=final,
                   RRGPU_IMM_EARLY_EXIT=early)
        p = subprocess.run([sys.executable, "-c", _SPEC_CHILD, root], env=env, check=True,
                           capture_output=True, text=True, timeout=300)
        results.append(json.loads(p.stdout.strip().splitlines()[-1]))
    for r in results[1:]:
        assert r == results[0]
