"""parallel.sharded_imm driven by the CUDA sampler and selector (one rank,
no process group): equals the reference's run_imm."""
import numpy as np
import pytest

import paper_2411_09473_b200 as P
from paper_2411_09473_b200 import graphs, parallel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_sharded_imm_on_gpu(cuda, oracle, name):
    cfg = graphs.scaled(graphs.CONFIGS[name], 1 << 11, 1 << 15)
    arrays = graphs.generate(cfg)
    g = P.Graph(*arrays)
    n = g.num_vertices
    k = 12

    def sample_fn(first, count):
        st = P.RRRStore(g)
        P.generate_slots(g, cfg.model, 1, first, count, st)
        off, mem = st.export()
        return off, mem, st.counter()

    def select_fn(off, mem, counter):
        gs = P.Graph(np.zeros(n + 1, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32))
        st = P.RRRStore(gs)
        st.import_sets(off, mem)
        assert (st.counter() == counter).all()
        s = P.select_seeds(st, n, k)
        return s.seeds, s.marginal_counts

    res = parallel.sharded_imm(n, k, 0.5, 1.0, sample_fn, select_fn)
    ref = oracle.graph(*arrays).imm(k=k, model=cfg.model, workers=4)
    assert res.seeds == ref["seeds"] and res.marginals == ref["marginals"]
    assert (res.theta, res.theta_prime, res.lower_bound) == \
        (ref["theta"], ref["theta_prime"], ref["lower_bound"])
