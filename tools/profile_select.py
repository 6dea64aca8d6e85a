"""select_seeds on a sampled store of a BASELINE config (the command profiled by
ncu: `ncu -k regex:k_select -s 1 -c 1 ...`); prints the per-call wall time."""
import argparse
import sys
import time

sys.path.insert(0, ".")
import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--sets", type=int, default=8192)
ap.add_argument("--k", type=int, default=0)
ap.add_argument("--repeat", type=int, default=5)
a = ap.parse_args()
cfg = graphs.CONFIGS[a.workload]
arrays = graphs.generate(cfg)
g = P.Graph(*arrays)
st = P.RRRStore(g)
P.generate_batch(g, cfg.model, 1, a.sets, st)
k = a.k or cfg.k
for i in range(a.repeat):
    t = time.perf_counter()
    s = P.select_seeds(st, g.num_vertices, k)
    dt = time.perf_counter() - t
    print(f"{cfg.name} sets {a.sets} members {st.total_member_count()} k {k} select {1e3 * dt:.3f} ms "
          f"covered {sum(s.marginal_counts)}", flush=True)
