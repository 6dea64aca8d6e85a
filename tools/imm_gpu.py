"""GPU-only IMM wall time (median of 5 after a warm-up) on BASELINE configs, for
A/B runs of library builds (RRGPU_LIB=...); no CPU reference."""
import statistics
import sys
import time

sys.path.insert(0, ".")
import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402

for name in sys.argv[1:] or ["cfg1", "cfg3", "cfg5"]:
    cfg = graphs.CONFIGS[name]
    g = P.Graph(*graphs.generate(cfg))
    g.prepare(cfg.model)
    icfg = P.ImmConfig(k=cfg.k, epsilon=cfg.epsilon, model=cfg.model)
    P.run_imm(g, icfg)
    walls = []
    for _ in range(5):
        t = time.time()
        r = P.run_imm(g, icfg)
        walls.append(time.time() - t)
    print(f"{name} imm {1e3 * statistics.median(walls):.2f} ms seeds {r.seeds.seeds[:3]}", flush=True)
