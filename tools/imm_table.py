"""IMM end to end on every BASELINE config: the GPU driver (graph resident;
median of 3 after a warm-up) next to the reference's run_imm on all host cores,
with the seeds / marginals / theta parity flags. Prints one JSON line per config."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, ".")
import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402
from oracle import Oracle, available  # noqa: E402

names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
orc = Oracle("reference" if available("reference") else "port")
cores = len(os.sched_getaffinity(0))
# CUDA context + module load happen once per process: keep them out of the
# first config's upload time.
_w = P.Graph(*graphs.generate(graphs.scaled(graphs.CONFIGS["cfg1"], 1024, 8192)))
_w.prepare(0)
_w.prepare(1)
del _w
for name in names:
    cfg = graphs.CONFIGS[name]
    t = time.time()
    arrays = graphs.generate(cfg)
    gen_s = time.time() - t
    t = time.time()
    g = P.Graph(*arrays)
    g.prepare(cfg.model)
    up_s = time.time() - t
    icfg = P.ImmConfig(k=cfg.k, epsilon=cfg.epsilon, model=cfg.model)
    P.run_imm(g, icfg)
    walls, r = [], None
    for _ in range(3):
        t = time.time()
        r = P.run_imm(g, icfg)
        walls.append(time.time() - t)
    og = orc.graph(*arrays)  # rrflow::Graph construction is not part of run_imm
    cpu_walls = []
    for _ in range(3):  # median of 3, like the GPU side
        t = time.time()
        rr = og.imm(k=cfg.k, epsilon=cfg.epsilon, model=cfg.model, workers=cores)
        cpu_walls.append(time.time() - t)
    cpu_s = statistics.median(cpu_walls)
    print(json.dumps({
        "cfg": name, "k": cfg.k, "n": int(arrays[0].size - 1), "arcs": int(arrays[1].size),
        "gpu_imm_s": statistics.median(walls), "gpu_upload_k0_s": up_s,
        "gpu_timings": r.timings, "cpu_ref_imm_s": cpu_s, "cpu_cores": cores,
        "cpu_kind": orc.kind, "speedup": cpu_s / statistics.median(walls),
        "theta": r.theta, "theta_prime": r.theta_prime, "sets": r.sets_generated,
        "mean_set_size": r.mean_set_size,
        "seeds_match": r.seeds.seeds == rr["seeds"],
        "marginals_match": r.seeds.marginal_counts == rr["marginals"],
        "theta_match": (r.theta, r.theta_prime, r.lower_bound) ==
                       (rr["theta"], rr["theta_prime"], rr["lower_bound"]),
        "cpu_timings": {"generate": rr["t_generate"], "select": rr["t_select"]},
        "graph_gen_s": gen_s}), flush=True)
