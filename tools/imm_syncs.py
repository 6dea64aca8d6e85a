"""run_imm per config: wall time (median of 5 after a warm-up) and the host
syncs / kernel launches of one run (rrg_host_sync_count, rrg_launch_count)."""
import statistics
import sys
import time

sys.path.insert(0, ".")
import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402

for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4"]:
    cfg = graphs.CONFIGS[name]
    g = P.Graph(*graphs.generate(cfg))
    icfg = P.ImmConfig(k=cfg.k, epsilon=cfg.epsilon, model=cfg.model)
    P.run_imm(g, icfg)
    ts = []
    for _ in range(5):
        s0, l0 = P.host_sync_count(), P.launch_count()
        t0 = time.perf_counter()
        r = P.run_imm(g, icfg)
        ts.append(time.perf_counter() - t0)
        syncs, launches = P.host_sync_count() - s0, P.launch_count() - l0
    print(f"{name} imm {1e3 * statistics.median(ts):.2f} ms syncs {syncs} launches {launches} "
          f"seeds {r.seeds.seeds[:3]}", flush=True)
    g.close()
