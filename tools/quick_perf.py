"""Quick throughput probe of the samplers and selection at BASELINE sizes (dev tool)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402


def run(name, count, **opts):
    cfg = graphs.CONFIGS[name]
    t = time.time()
    arrays = graphs.generate(cfg)
    tg = time.time() - t
    t = time.time()
    g = P.Graph(*arrays)
    g.prepare(cfg.model)
    tu = time.time() - t
    for k, v in opts.items():
        g.set_option(k, v)
    st = P.RRRStore(g)
    P.generate_batch(g, cfg.model, 99, min(count, 4096), st)  # warm
    st.clear()
    P.generate_batch(g, cfg.model, 1, count, st)
    s = g.last_batch_stats()
    print(f"{name} {opts} gen {tg:.1f}s upload+prep {tu:.2f}s | sets {s.sets} members {s.members} "
          f"insp/set {s.edges_inspected / s.sets:.0f} deferred {s.deferred} | sample {s.sample_ms:.2f} ms "
          f"total {s.total_ms:.2f} ms | {s.sets / s.sample_ms * 1e3:.3e} sets/s "
          f"{s.edges_inspected / s.sample_ms * 1e3:.3e} edges/s "
          f"{8 * s.edges_inspected / s.sample_ms / 1e6:.1f} GB/s", flush=True)
    t = time.time()
    sel = P.select_seeds(st, g.num_vertices, cfg.k)
    print(f"   select k={cfg.k}: {1e3 * (time.time() - t):.2f} ms, covered {sel.covered}", flush=True)
    t = time.time()
    r = P.run_imm(g, P.ImmConfig(k=cfg.k, model=cfg.model))
    print(f"   imm: {1e3 * (time.time() - t):.1f} ms theta {r.theta} theta' {r.theta_prime} "
          f"timings {r.timings}", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg1", "cfg2", "cfg4", "cfg3", "cfg5"]
    counts = {"cfg1": 1 << 20, "cfg2": 1 << 20, "cfg3": 1 << 22, "cfg4": 1 << 16, "cfg5": 1 << 15}
    for w in which:
        run(w, counts[w])
        if graphs.CONFIGS[w].model == 1:
            run(w, counts[w], lt_scan=1)
