"""run_imm on a BASELINE config (the command for an ncu launch list of the
whole IMM driver: sampling top-ups + selections)."""
import argparse
import sys
import time

sys.path.insert(0, ".")
import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--repeat", type=int, default=3)
ap.add_argument("--ic-mode", type=int, default=0)
ap.add_argument("--ic-rng", type=int, default=0, help="1 = fast statistical IC sampling")
a = ap.parse_args()
cfg = graphs.CONFIGS[a.workload]
arrays = graphs.generate(cfg)
g = P.Graph(*arrays)
g.prepare(cfg.model)
g.set_option("ic_mode", a.ic_mode)
g.set_option("ic_rng", a.ic_rng)
for i in range(a.repeat):
    t = time.time()
    r = P.run_imm(g, P.ImmConfig(k=cfg.k, epsilon=cfg.epsilon, model=cfg.model))
    print(f"{cfg.name} mode {a.ic_mode} rng {a.ic_rng} imm {1e3 * (time.time() - t):.1f} ms theta {r.theta} theta' {r.theta_prime} "
          f"lb {r.lower_bound:.1f} timings {r.timings}", flush=True)
