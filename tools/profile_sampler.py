"""One warm-up batch + one measured batch of the sampler on a BASELINE config
(the command profiled by ncu: `ncu -k regex:k_sample -s 1 -c 1 ...`)."""
import argparse
import sys
import time

sys.path.insert(0, ".")
import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--sets", type=int, default=1 << 16)
ap.add_argument("--lt-scan", type=int, default=0)
ap.add_argument("--n", type=int, default=0, help="scaled-down vertex count (0 = full size)")
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--ic-coop-min", type=int, default=0)
ap.add_argument("--lt-kary", type=int, default=0)
ap.add_argument("--ic-mode", type=int, default=0)
ap.add_argument("--lt-guide-mult", type=int, default=0)
ap.add_argument("--ic-rng", type=int, default=0, help="1 = fast statistical IC sampling")
ap.add_argument("--l2-fetch", type=int, default=0,
                help="cudaLimitMaxL2FetchGranularity hint in bytes (32 / 64 / 128); 0 = leave")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
if a.l2_fetch:
    import ctypes
    import torch
    torch.cuda.init()
    rt = ctypes.CDLL("libcudart.so.12")
    got = ctypes.c_size_t(0)
    rc = rt.cudaDeviceSetLimit(5, ctypes.c_size_t(a.l2_fetch))  # cudaLimitMaxL2FetchGranularity
    rt.cudaDeviceGetLimit(ctypes.byref(got), 5)
    print(f"l2 fetch granularity: set rc {rc}, now {got.value}")
cfg = graphs.CONFIGS[a.workload]
if a.n:
    cfg = graphs.scaled(cfg, a.n, a.m)
arrays = graphs.generate(cfg)
g = P.Graph(*arrays)
g.set_option("lt_scan", a.lt_scan)
if a.lt_guide_mult:
    g.set_option("lt_guide_mult", a.lt_guide_mult)
t = time.time()
g.prepare(cfg.model)
print(f"prepare {1e3 * (time.time() - t):.1f} ms (lt_scan {a.lt_scan})")
if a.ic_coop_min:
    g.set_option("ic_coop_min", a.ic_coop_min)
if a.lt_kary:
    g.set_option("lt_kary", a.lt_kary)
g.set_option("ic_mode", a.ic_mode)
g.set_option("ic_rng", a.ic_rng)
st = P.RRRStore(g)
P.generate_batch(g, cfg.model, 99, a.sets, st)
for _ in range(a.reps - 1):
    st.clear()
    P.generate_batch(g, cfg.model, 1, a.sets, st)
    print(f"rep sample {g.last_batch_stats().sample_ms:.3f} ms")
st.clear()
t = time.time()
P.generate_batch(g, cfg.model, 1, a.sets, st)
s = g.last_batch_stats()
print(f"{cfg.name} scan {a.lt_scan} mult {a.lt_guide_mult} rng {a.ic_rng} coop_min {a.ic_coop_min} kary {a.lt_kary} mode {a.ic_mode} sets {s.sets} insp/set {s.edges_inspected / s.sets:.0f} members/set "
      f"{s.members / s.sets:.1f} deferred {s.deferred} sample {s.sample_ms:.2f} ms "
      f"{s.sets / s.sample_ms * 1e3:.3e} sets/s {s.edges_inspected / s.sample_ms * 1e3:.3e} edges/s "
      f"wall {1e3 * (time.time() - t):.1f} ms")
