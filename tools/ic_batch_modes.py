"""IMM-sized IC batches under each IC schedule (tools, not product): the device
time of generate_batch for N sets at slot 0 per ic_mode (0 auto, 1 lane, 2 warp,
3 block), median of --repeat runs after a warm-up on a fresh graph."""
import argparse
import statistics
import sys

sys.path.insert(0, ".")
import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("sets", type=int, nargs="+")
ap.add_argument("--modes", default="0,1,2,3")
ap.add_argument("--repeat", type=int, default=3)
ap.add_argument("--budgets", default="0", help="warp-schedule window budgets to try (mode 2)")
a = ap.parse_args()
cfg = graphs.CONFIGS[a.workload]
arrays = graphs.generate(cfg)
runs = [(int(m), 0) for m in a.modes.split(",")]
runs += [(2, int(b)) for b in a.budgets.split(",") if int(b)]
for mode, budget in runs:
    g = P.Graph(*arrays)
    g.set_option("ic_mode", mode)
    g.set_option("ic_warp_budget", budget)
    st = P.RRRStore(g)
    P.generate_batch(g, 0, 1, 2048, st)  # warm-up (auto: the pilot)
    for N in a.sets:
        ts = []
        for _ in range(a.repeat):
            st.clear()
            P.generate_batch(g, 0, 1, N, st)
            ts.append(g.last_batch_stats().total_ms)
        b = g.last_batch_stats()
        print(f"{a.workload} mode {mode} budget {budget} sets {N} total {statistics.median(ts):.3f} ms "
              f"sample {b.sample_ms:.3f} ms deferred {b.deferred} insp/set {b.edges_inspected / N:.0f}",
              flush=True)
    st.close()
    g.close()
