"""Multi-GPU IMM through the drop-in (rrg_run_imm_sharded).

Only one GPU is available to the test suite, so the sharding is proven two
ways: (1) the shard split + ordered assembly run in one process for N = 2, 3, 8
simulated ranks (each rank's slot range sampled separately, appended in rank
order) -- seeds, marginals, theta, theta', LB and set statistics equal
rrg_run_imm's, which equal the reference's; (2) the NCCL transport itself on a
one-rank communicator (the broadcast of every shard array from device memory,
the header AllGather, the ordered append)."""
import numpy as np
import pytest

import paper_2411_09473_b200 as P
from paper_2411_09473_b200 import graphs

pytestmark = pytest.mark.gpu


def same(a, b):
    assert a.seeds.seeds == b.seeds.seeds
    assert a.seeds.marginal_counts == b.seeds.marginal_counts
    assert (a.theta, a.theta_prime, a.lower_bound) == (b.theta, b.theta_prime, b.lower_bound)
    assert (a.sets_generated, a.mean_set_size, a.max_set_size) == \
        (b.sets_generated, b.mean_set_size, b.max_set_size)


@pytest.mark.parametrize("name,n,m,k", [("cfg1", 1 << 12, 1 << 16, 20), ("cfg2", 1 << 12, 1 << 16, 20),
                                        ("cfg3c", 30000, 560000, 10), ("cfg5", 20000, 300000, 10)])
@pytest.mark.parametrize("ranks", [2, 3, 8])
def test_sharded_imm_equals_single_gpu(cuda, oracle, name, n, m, k, ranks):
    cfg = graphs.scaled(graphs.CONFIGS[name], n, m)
    arrays = graphs.generate(cfg)
    g = P.Graph(*arrays)
    icfg = P.ImmConfig(k=k, epsilon=0.5, model=cfg.model, rng_seed=1)
    one = P.run_imm(g, icfg)
    shard = P.run_imm_sharded(g, icfg, sim_ranks=ranks)
    same(shard, one)
    if ranks == 2:
        ref = oracle.graph(*arrays).imm(k=k, epsilon=0.5, model=cfg.model, workers=4, rng_seed=1)
        assert shard.seeds.seeds == ref["seeds"] and shard.theta == ref["theta"]


def test_sharded_imm_over_nccl_one_rank(cuda):
    cfg = graphs.scaled(graphs.CONFIGS["cfg3c"], 30000, 560000)
    arrays = graphs.generate(cfg)
    g = P.Graph(*arrays)
    icfg = P.ImmConfig(k=10, epsilon=0.5, model=cfg.model, rng_seed=1)
    comm = P.NcclComm(P.nccl_unique_id(), 1, 0)
    try:
        got = P.run_imm_sharded(g, icfg, comm)
    finally:
        comm.close()
    same(got, P.run_imm(g, icfg))


def test_sharded_needs_a_transport(cuda):
    arrays = graphs.generate(graphs.scaled(graphs.CONFIGS["cfg1"], 1 << 10, 1 << 13))
    g = P.Graph(*arrays)
    with pytest.raises(ValueError):
        P.run_imm_sharded(g, P.ImmConfig(k=5), None, 0)
