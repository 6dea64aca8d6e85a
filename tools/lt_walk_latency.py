"""Latency of single LT walks (the batch tail): time one-slot batches of the
longest and a median walk among the first N slots of a config."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
cfg = graphs.CONFIGS[name]
arrays = graphs.generate(cfg)
g = P.Graph(*arrays)
g.prepare(cfg.model)
g.set_option("lt_scan", int(sys.argv[3]) if len(sys.argv) > 3 else 2)
st = P.RRRStore(g)
P.generate_slots(g, cfg.model, 1, 0, N, st)
off, _ = st.export()
L = np.diff(off.astype(np.int64))
order = np.argsort(L)
for slot in [int(order[-1]), int(order[-2]), int(order[len(L) // 2])]:
    ts = []
    for _ in range(5):
        s1 = P.RRRStore(g)
        P.generate_slots(g, cfg.model, 1, slot, 1, s1)
        ts.append(g.last_batch_stats().sample_ms)
        s1.close()
    t = min(ts)
    print(f"slot {slot} len {L[slot]} sample_ms {t:.3f} us/step {1e3 * t / L[slot]:.2f}")
