"""CPU checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package. It loads one of

  oracle/_ref/librrflow_ref.so  the unmodified reference headers (kind "reference")
  oracle/liboracle_port.so      the C++17 restatement in port.cpp (kind "port")

through the common C API of oracle/oracle.h. The product package
(paper_2411_09473_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PATH = os.path.join(HERE, "_ref", "librrflow_ref.so")
PORT_PATH = os.path.join(HERE, "liboracle_port.so")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
vp = C.c_void_p


class ImmConfigC(C.Structure):
    _fields_ = [("k", C.c_uint32), ("epsilon", C.c_double), ("model", C.c_int),
                ("workers", C.c_uint32), ("rng_seed", C.c_uint64), ("ell", C.c_double),
                ("adaptive_threshold", C.c_double), ("strategy", C.c_int)]


class ImmResultC(C.Structure):
    _fields_ = [("theta", C.c_uint64), ("theta_prime", C.c_uint64), ("lower_bound", C.c_double),
                ("sets_generated", C.c_uint64), ("mean_set_size", C.c_double),
                ("max_set_size", C.c_uint32), ("mean_coverage_fraction", C.c_double),
                ("t_generate", C.c_double), ("t_select", C.c_double), ("t_total", C.c_double)]


_SIG = [
    ("orc_kind", C.c_char_p, []),
    ("orc_last_error", C.c_char_p, []),
    ("orc_graph_new", vp, [C.c_uint32, C.c_uint64, u64p, u32p, f32p]),
    ("orc_graph_free", None, [vp]),
    ("orc_derive_stream_seed", C.c_uint64, [C.c_uint64, C.c_uint64]),
    ("orc_prng_draws", None, [C.c_uint64, C.c_uint64, u64p]),
    ("orc_uniform_below", C.c_uint64, [C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]),
    ("orc_sample", vp, [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32]),
    ("orc_store_sets", C.c_uint64, [vp]),
    ("orc_store_members", C.c_uint64, [vp]),
    ("orc_store_export", None, [vp, u64p, u32p]),
    ("orc_store_counter", None, [vp, u64p]),
    ("orc_store_roots", None, [vp, u32p]),
    ("orc_store_inspected", C.c_uint64, [vp]),
    ("orc_store_free", None, [vp]),
    ("orc_select", C.c_int, [C.c_uint32, C.c_uint64, u64p, u32p, C.c_uint32, C.c_double,
                             C.c_uint32, u32p, u64p, u64p, u32p]),
    ("orc_imm", C.c_int, [vp, C.POINTER(ImmConfigC), u32p, u64p, C.POINTER(ImmResultC)]),
    ("orc_sampling_phase", C.c_int, [vp, C.POINTER(ImmConfigC), C.POINTER(C.c_double), u64p, u64p]),
    ("orc_log_binomial", C.c_double, [C.c_uint64, C.c_uint64]),
    ("orc_effective_ell", C.c_double, [C.c_double, C.c_uint64]),
    ("orc_lambda_prime", C.c_double, [C.c_uint64, C.c_uint64, C.c_double, C.c_double]),
    ("orc_sampling_rounds", C.c_uint32, [C.c_uint64]),
    ("orc_theta_for_round", C.c_uint64, [C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                         C.c_uint32]),
    ("orc_lambda_star", C.c_double, [C.c_uint64, C.c_uint64, C.c_double, C.c_double]),
    ("orc_set_theta", C.c_uint64, [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double]),
    ("orc_build_graph", C.c_int, [C.c_uint32, C.c_uint64, u32p, u32p, f32p, u64p, u32p, f32p]),
    ("orc_normalize_lt", C.c_int, [C.c_uint32, u64p, f32p]),
    ("orc_activation_probability", C.c_double, [vp, u32p, C.c_uint32, C.c_uint32, C.c_int,
                                                C.c_uint64, C.c_uint64]),
    ("orc_exact_spread", C.c_double, [vp, u32p, C.c_uint32, C.c_int]),
    ("orc_synth_graph", C.c_uint64, [C.c_int, C.c_uint32, C.c_double, C.c_uint64, C.c_int,
                                     C.c_uint64, u64p, u32p, f32p]),
]


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


def available(kind: str) -> bool:
    return os.path.exists(REF_PATH if kind == "reference" else PORT_PATH)


@dataclass
class Sketches:
    offsets: np.ndarray   # u64[count+1]
    members: np.ndarray   # u32, ascending within each set
    roots: np.ndarray     # u32[count]
    counter: np.ndarray   # u64[n]
    inspected: int

    def sets(self):
        return [self.members[self.offsets[i]:self.offsets[i + 1]]
                for i in range(self.offsets.size - 1)]


class Oracle:
    def __init__(self, kind: str = "reference"):
        path = REF_PATH if kind == "reference" else PORT_PATH
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -f oracle/Makefile)")
        self.lib = C.CDLL(path)
        for name, res, args in _SIG:
            f = getattr(self.lib, name)
            f.restype = res
            f.argtypes = args
        self.kind = self.lib.orc_kind().decode()

    def err(self) -> str:
        return self.lib.orc_last_error().decode()

    # -- graph handles --------------------------------------------------------
    def graph(self, roff, rsrc, rw):
        roff = np.ascontiguousarray(roff, np.uint64)
        rsrc = np.ascontiguousarray(rsrc, np.uint32)
        rw = np.ascontiguousarray(rw, np.float32)
        h = self.lib.orc_graph_new(roff.size - 1, rsrc.size, _p(roff, C.c_uint64),
                                   _p(rsrc, C.c_uint32), _p(rw, C.c_float))
        if not h:
            raise ValueError(self.err())
        return OracleGraph(self, h, roff.size - 1)

    # -- prng -------------------------------------------------------------------
    def derive_stream_seed(self, run_seed, stream):
        return self.lib.orc_derive_stream_seed(run_seed, stream)

    def draws(self, seed, count):
        out = np.zeros(count, np.uint64)
        self.lib.orc_prng_draws(seed, count, _p(out, C.c_uint64))
        return out

    def uniform_below(self, seed, bound):
        nxt = C.c_double()
        v = self.lib.orc_uniform_below(seed, bound, C.byref(nxt))
        return v, nxt.value

    # -- selection ------------------------------------------------------------
    def select(self, n, offsets, members, k, threshold=0.25, workers=1, capture=False):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        members = np.ascontiguousarray(members, np.uint32)
        seeds = np.zeros(k, np.uint32)
        marg = np.zeros(k, np.uint64)
        rc = np.zeros(k * n, np.uint64) if capture else None
        rounds = C.c_uint32()
        st = self.lib.orc_select(n, offsets.size - 1, _p(offsets, C.c_uint64),
                                 _p(members, C.c_uint32), k, threshold, workers,
                                 _p(seeds, C.c_uint32), _p(marg, C.c_uint64),
                                 _p(rc, C.c_uint64), C.byref(rounds))
        if st != 0:
            raise ValueError(self.err())
        out = ([int(x) for x in seeds], [int(x) for x in marg])
        if capture:
            return out + (rc.reshape(k, n)[: rounds.value],)
        return out

    # -- theta math -------------------------------------------------------------
    def log_binomial(self, n, k):
        return self.lib.orc_log_binomial(n, k)

    def effective_ell(self, ell, n):
        return self.lib.orc_effective_ell(ell, n)

    def lambda_prime(self, n, k, e, l):
        return self.lib.orc_lambda_prime(n, k, e, l)

    def sampling_rounds(self, n):
        return self.lib.orc_sampling_rounds(n)

    def theta_for_round(self, n, k, e, l, i):
        return self.lib.orc_theta_for_round(n, k, e, l, i)

    def lambda_star(self, n, k, e, l):
        return self.lib.orc_lambda_star(n, k, e, l)

    def set_theta(self, n, k, e, l, lb):
        return self.lib.orc_set_theta(n, k, e, l, lb)

    # -- graph prep -------------------------------------------------------------
    def build_graph(self, n, src, dst, w):
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        w = np.ascontiguousarray(w, np.float32)
        roff = np.zeros(n + 1, np.uint64)
        rsrc = np.zeros(src.size, np.uint32)
        rw = np.zeros(src.size, np.float32)
        st = self.lib.orc_build_graph(n, src.size, _p(src, C.c_uint32), _p(dst, C.c_uint32),
                                      _p(w, C.c_float), _p(roff, C.c_uint64),
                                      _p(rsrc, C.c_uint32), _p(rw, C.c_float))
        if st != 0:
            raise ValueError(self.err())
        return roff, rsrc, rw

    def normalize_lt(self, roff, rw):
        roff = np.ascontiguousarray(roff, np.uint64)
        rw = np.array(rw, np.float32, copy=True)
        if self.lib.orc_normalize_lt(roff.size - 1, _p(roff, C.c_uint64), _p(rw, C.c_float)):
            raise ValueError(self.err())
        return rw

    def synth_graph(self, kind, n, param, seed, ic_weights_seed=None):
        m = self.lib.orc_synth_graph(kind, n, param, seed, ic_weights_seed is not None,
                                     ic_weights_seed or 0, None, None, None)
        if m == 2**64 - 1:
            raise ValueError(self.err())
        roff = np.zeros(n + 1, np.uint64)
        rsrc = np.zeros(m, np.uint32)
        rw = np.zeros(m, np.float32)
        self.lib.orc_synth_graph(kind, n, param, seed, ic_weights_seed is not None,
                                 ic_weights_seed or 0, _p(roff, C.c_uint64),
                                 _p(rsrc, C.c_uint32), _p(rw, C.c_float))
        return roff, rsrc, rw


class OracleGraph:
    def __init__(self, orc: Oracle, h, n):
        self.orc, self.h, self.n = orc, h, n

    def __del__(self):
        try:
            self.orc.lib.orc_graph_free(self.h)
        except Exception:
            pass

    def sample(self, model, run_seed, first_slot, count, workers=1) -> Sketches:
        lib = self.orc.lib
        st = lib.orc_sample(self.h, int(model), run_seed, first_slot, count, workers)
        if not st:
            raise ValueError(self.orc.err())
        try:
            nsets = lib.orc_store_sets(st)
            nmem = lib.orc_store_members(st)
            off = np.zeros(nsets + 1, np.uint64)
            mem = np.zeros(nmem, np.uint32)
            roots = np.zeros(nsets, np.uint32)
            cnt = np.zeros(self.n, np.uint64)
            lib.orc_store_export(st, _p(off, C.c_uint64), _p(mem, C.c_uint32))
            lib.orc_store_roots(st, _p(roots, C.c_uint32))
            lib.orc_store_counter(st, _p(cnt, C.c_uint64))
            insp = lib.orc_store_inspected(st)
        finally:
            lib.orc_store_free(st)
        return Sketches(off, mem, roots, cnt, insp)

    def sampling_phase(self, k=50, epsilon=0.5, model=0, workers=1, rng_seed=1, ell=1.0,
                       adaptive_threshold=0.25, strategy=0):
        cfg = ImmConfigC(k, epsilon, model, workers, rng_seed, ell, adaptive_threshold, strategy)
        lb = C.c_double()
        tp = np.zeros(1, np.uint64)
        cnt = np.zeros(self.n, np.uint64)
        if self.orc.lib.orc_sampling_phase(self.h, C.byref(cfg), C.byref(lb), _p(tp, C.c_uint64),
                                           _p(cnt, C.c_uint64)):
            raise ValueError(self.orc.err())
        return {"lower_bound": lb.value, "theta_prime": int(tp[0]), "counter": cnt}

    def imm(self, k=50, epsilon=0.5, model=0, workers=1, rng_seed=1, ell=1.0,
            adaptive_threshold=0.25, strategy=0):
        cfg = ImmConfigC(k, epsilon, model, workers, rng_seed, ell, adaptive_threshold, strategy)
        seeds = np.zeros(max(k, 1), np.uint32)
        marg = np.zeros(max(k, 1), np.uint64)
        res = ImmResultC()
        if self.orc.lib.orc_imm(self.h, C.byref(cfg), _p(seeds, C.c_uint32),
                                _p(marg, C.c_uint64), C.byref(res)):
            raise ValueError(self.orc.err())
        return {
            "seeds": [int(x) for x in seeds], "marginals": [int(x) for x in marg],
            "theta": res.theta, "theta_prime": res.theta_prime, "lower_bound": res.lower_bound,
            "sets_generated": res.sets_generated, "mean_set_size": res.mean_set_size,
            "max_set_size": res.max_set_size,
            "mean_coverage_fraction": res.mean_coverage_fraction,
            "t_generate": res.t_generate, "t_select": res.t_select, "t_total": res.t_total,
        }

    def activation_probability(self, sources, target, model, trials, seed):
        s = np.ascontiguousarray(sources, np.uint32)
        return self.orc.lib.orc_activation_probability(self.h, _p(s, C.c_uint32), s.size, target,
                                                       model, trials, seed)

    def exact_spread(self, seeds, model):
        s = np.ascontiguousarray(seeds, np.uint32)
        return self.orc.lib.orc_exact_spread(self.h, _p(s, C.c_uint32), s.size, model)
