"""Sample one given slot (twice: warm-up + measured) in a given IC schedule; the
command profiled by ncu for a single giant set's latency."""
import sys

sys.path.insert(0, ".")
import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402

name, slot, mode = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = graphs.CONFIGS[name]
g = P.Graph(*graphs.generate(cfg))
g.set_option("ic_mode", mode)
st = P.RRRStore(g)
for _ in range(2):
    st.clear()
    P.generate_slots(g, cfg.model, 1, slot, 1, st)
b = g.last_batch_stats()
print(f"{name} slot {slot} mode {mode} insp {b.edges_inspected} sample {b.sample_ms:.2f} ms")
