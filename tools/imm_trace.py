"""Per-launch trace (RRGPU_DEBUG=1) of one warmed-up IMM run on BASELINE configs:
which sampler launches a run makes, their device times, deferrals and windows."""
import os
import sys
import time

os.environ["RRGPU_DEBUG"] = "1"
sys.path.insert(0, ".")
import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402

for name in sys.argv[1:] or ["cfg1", "cfg3"]:
    cfg = graphs.CONFIGS[name]
    g = P.Graph(*graphs.generate(cfg))
    g.prepare(cfg.model)
    icfg = P.ImmConfig(k=cfg.k, epsilon=cfg.epsilon, model=cfg.model)
    P.run_imm(g, icfg)
    P.run_imm(g, icfg)
    sys.stderr.flush()
    print(f"==== {name} measured run", file=sys.stderr, flush=True)
    t = time.time()
    r = P.run_imm(g, icfg)
    w = time.time() - t
    print(f"==== {name} imm {1e3 * w:.2f} ms generate {1e3 * r.timings["generate_rrrsets"]:.2f} "
          f"select {1e3 * r.timings["find_most_influential"]:.2f} theta {r.theta} sets {r.sets_generated} "
          f"max {r.max_set_size}", file=sys.stderr, flush=True)
