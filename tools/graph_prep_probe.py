"""Breakdown of rrg_graph_create_from_edges on a BASELINE config: the whole call
(best of 3) beside a bare pinned H2D of the same three edge arrays, so the
device-side share (sort, scatter, normalize, allocations) is the difference.
Run it under `ncu --metrics gpu__time_duration.sum` for the kernel times."""
import argparse
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_09473_b200 as P  # noqa: E402
from paper_2411_09473_b200 import graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="cfg4")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = graphs.CONFIGS[a.workload]
roff, rsrc, rw = graphs.generate(cfg)
n, m = roff.size - 1, rsrc.size
perm = np.random.default_rng(2411).permutation(m)
dst = np.repeat(np.arange(n, dtype=np.uint32), np.diff(roff.astype(np.int64)))
pin = [torch.from_numpy(x[perm]).pin_memory() for x in (rsrc, dst, rw)]
lib = P.lib
for r in range(a.reps):
    h = C.c_void_p()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.check(lib.rrg_graph_create_from_edges(
        n, m, C.cast(pin[0].data_ptr(), C.POINTER(C.c_uint32)),
        C.cast(pin[1].data_ptr(), C.POINTER(C.c_uint32)),
        C.cast(pin[2].data_ptr(), C.POINTER(C.c_float)), 1 if cfg.model == 1 else 0, C.byref(h)))
    t1 = time.perf_counter()
    lib.rrg_graph_destroy(h)
    print(f"{cfg.name} create_from_edges m={m} {1e3 * (t1 - t0):.1f} ms")
dev = [torch.empty(x.shape, dtype=x.dtype, device="cuda") for x in pin]
for r in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for d, x in zip(dev, pin):
        d.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"pinned H2D {3 * m * 4 / 1e6:.0f} MB {1e3 * (t1 - t0):.1f} ms "
          f"({3 * m * 4 / (t1 - t0) / 1e9:.1f} GB/s)")
