"""Golden run_imm results at FULL BASELINE sizes, computed by the REFERENCE
(oracle/_ref, the unmodified rrflow headers) in the build container:

    python tests/golden/make_imm_full.py cfg3c [cfg1 ...]

Writes tests/golden/imm_full_<cfg>.json. Used where the reference's own
run_imm is too slow to repeat on every GPU test / bench run (cfg3c: the
correlated-degree cfg3 with giant sets, ~8 min on 8 cores); the inputs are the
pinned generators (rrgen), so the GPU box rebuilds the identical graph.
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Oracle  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402


def main(names):
    ref = Oracle("reference")
    for name in names:
        cfg = graphs.CONFIGS[name]
        arrays = graphs.generate(cfg)
        og = ref.graph(*arrays)
        t0 = time.perf_counter()
        res = og.imm(k=cfg.k, epsilon=cfg.epsilon, model=cfg.model, workers=os.cpu_count(),
                     rng_seed=1)
        dt = time.perf_counter() - t0
        out = {"cfg": name, "n": int(arrays[0].size - 1), "arcs": int(arrays[1].size),
               "k": cfg.k, "epsilon": cfg.epsilon, "model": cfg.model, "rng_seed": 1,
               "result": {k: v for k, v in res.items() if not k.startswith("t_")},
               "reference_wall_s": dt, "reference_workers": os.cpu_count()}
        with open(os.path.join(HERE, f"imm_full_{name}.json"), "w") as f:
            json.dump(out, f, indent=1)
        print(name, dt, out["result"]["theta"], out["result"]["seeds"][:5], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg3c"])
