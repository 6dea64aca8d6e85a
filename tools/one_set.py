"""Latency of the single largest IC set of a batch (the batch's tail): finds it,
then re-samples that slot alone in each schedule."""
import argparse
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--sets", type=int, default=4096)
ap.add_argument("--top", type=int, default=1)
a = ap.parse_args()
cfg = graphs.CONFIGS[a.workload]
arrays = graphs.generate(cfg)
g = P.Graph(*arrays)
st = P.RRRStore(g)
P.generate_batch(g, 0, 1, a.sets, st)
off, mem = st.export()
indeg = np.diff(arrays[0].astype(np.int64))
insp = np.add.reduceat(indeg[mem], off[:-1].astype(np.int64))
for slot in np.argsort(insp)[::-1][:a.top]:
    for mode in (2, 3):
        g.set_option("ic_mode", mode)
        s1 = P.RRRStore(g)
        P.generate_slots(g, 0, 1, int(slot), 1, s1)
        s1.clear()
        P.generate_slots(g, 0, 1, int(slot), 1, s1)
        b = g.last_batch_stats()
        print(f"{cfg.name} slot {slot} insp {insp[slot]} members {off[slot+1]-off[slot]} mode {mode} "
              f"sample {b.sample_ms:.2f} ms -> {insp[slot] / b.sample_ms / 1e3:.1f} M edges/s", flush=True)
        s1.close()
