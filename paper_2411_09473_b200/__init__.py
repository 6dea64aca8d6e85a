"""paper_2411_09473_b200 -- B200-native IMM hot path (RRR sampling + greedy seed selection).

Python mirror of the reference's operator API (rrflow 0.1.0, proj/include/rrflow),
same names, argument meaning and error classes, over the C ABI of librrgpu.so:

  Graph            rrflow::Graph transpose view (graph.hpp:34-59), device-resident
  RRRStore         RRRStore + fused Counter (rrr_store.hpp:20-120, counter.hpp:15-62)
  generate_batch   sampling.hpp:159-199
  select_seeds     selection.hpp:209-243
  fraction_covered selection.hpp:340-358
  run_imm          imm.hpp:214-251 (driver in C++17, csrc/imm.cpp)
  build_graph      detail::build_graph (graph.hpp:69-115), host
  normalize_lt_weights graph.hpp:207-235, host

Every compute call runs the sm_100a kernels in csrc/; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import RRGError, RRGOutOfMemory, check, lib, ptr

__all__ = [
    "DiffusionModel", "Graph", "RRRStore", "SeedSet", "ImmConfig", "ImmResult",
    "generate_batch", "generate_batch_fused", "select_seeds", "fraction_covered",
    "run_imm", "build_graph", "normalize_lt_weights", "RRGError", "RRGOutOfMemory",
    "version", "BatchStats", "SelectionStats", "run_imm_sharded", "NcclComm",
    "nccl_unique_id",
]

kDefaultDensityDivisor = 64  # rrr_set.hpp:13


class DiffusionModel(enum.IntEnum):
    IC = 0
    LT = 1


def version() -> str:
    return lib.rrg_version().decode()


def _model(m) -> int:
    if isinstance(m, str):
        s = m.lower()
        if s not in ("ic", "lt"):
            raise ValueError(f"unknown diffusion model: {m}")  # graph.hpp:24-28
        return 0 if s == "ic" else 1
    return int(DiffusionModel(m))


def build_graph(n: int, src, dst, w):
    """Transpose arrays of detail::build_graph (graph.hpp:69-115) for an edge list."""
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    if not (src.size == dst.size == w.size):
        raise ValueError(f"build_graph: src, dst and w differ in length "
                         f"({src.size}, {dst.size}, {w.size})")
    m = src.size
    roff = np.zeros(n + 1, dtype=np.uint64)
    rsrc = np.zeros(m, dtype=np.uint32)
    rw = np.zeros(m, dtype=np.float32)
    check(lib.rrg_build_transpose(n, m, ptr(src, C.c_uint32), ptr(dst, C.c_uint32),
                                  ptr(w, C.c_float), ptr(roff, C.c_uint64),
                                  ptr(rsrc, C.c_uint32), ptr(rw, C.c_float)))
    return roff, rsrc, rw


def normalize_lt_weights(roff, rw):
    """normalize_lt_weights (graph.hpp:207-235), in place on transpose weights."""
    n = roff.size - 1
    check(lib.rrg_normalize_lt_weights(n, ptr(roff, C.c_uint64), ptr(rw, C.c_float)))
    return rw


class Graph:
    """Device-resident transpose CSR (the reverse arrays of rrflow::Graph)."""

    def __init__(self, rev_offsets, rev_sources, rev_weights, model=None):
        """model (optional: IC / LT, as generate_batch takes it): the diffusion
        model the graph will be sampled under -- the upload then overlaps that
        model's device layouts (rrg_graph_create_for); results are the same."""
        self.reverse_offsets = np.ascontiguousarray(rev_offsets, dtype=np.uint64)
        self.reverse_sources = np.ascontiguousarray(rev_sources, dtype=np.uint32)
        self.reverse_weights = np.ascontiguousarray(rev_weights, dtype=np.float32)
        if self.reverse_offsets.size < 1:
            raise ValueError("Graph: reverse_offsets needs n + 1 >= 1 entries")
        if self.reverse_weights.size != self.reverse_sources.size:
            raise ValueError("Graph: reverse_sources and reverse_weights differ in length "
                             f"({self.reverse_sources.size} vs {self.reverse_weights.size})")
        self.num_vertices = int(self.reverse_offsets.size - 1)
        self.num_edges = int(self.reverse_sources.size)
        h = C.c_void_p()
        check(lib.rrg_graph_create_for(
            self.num_vertices, self.num_edges, ptr(self.reverse_offsets, C.c_uint64),
            ptr(self.reverse_sources, C.c_uint32), ptr(self.reverse_weights, C.c_float),
            -1 if model is None else _model(model), C.byref(h)))
        self._h = h

    @classmethod
    def from_edges(cls, n: int, edges):
        """Like proj/tests/test_util.hpp:46-52 graph_from_edges: [(src, dst, w), ...]."""
        if len(edges):
            arr = np.array(edges, dtype=np.float64)
            src, dst, w = arr[:, 0].astype(np.uint32), arr[:, 1].astype(np.uint32), arr[:, 2]
        else:
            src = dst = np.zeros(0, np.uint32)
            w = np.zeros(0, np.float32)
        return cls(*build_graph(n, src, dst, w))

    @classmethod
    def from_edge_arrays(cls, n: int, src, dst, w, normalize_lt: bool = False) -> "Graph":
        """Device-built transpose of an edge list (rrg_graph_create_from_edges):
        detail::build_graph's in-list order and, with normalize_lt,
        normalize_lt_weights -- both on the GPU. The host copies of the reverse
        arrays are fetched back (export_transpose) so the object reads like one
        built from host arrays."""
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        w = np.ascontiguousarray(w, dtype=np.float32)
        if not (src.size == dst.size == w.size):
            raise ValueError("from_edge_arrays: src, dst and w differ in length "
                             f"({src.size}, {dst.size}, {w.size})")
        h = C.c_void_p()
        check(lib.rrg_graph_create_from_edges(n, src.size, ptr(src, C.c_uint32),
                                              ptr(dst, C.c_uint32), ptr(w, C.c_float),
                                              1 if normalize_lt else 0, C.byref(h)))
        g = cls.__new__(cls)
        g._h = h
        g.num_vertices = int(n)
        g.num_edges = int(src.size)
        g.reverse_offsets, g.reverse_sources, g.reverse_weights = g.export_transpose()
        return g

    def export_transpose(self):
        """(reverse_offsets u64[n+1], reverse_sources u32[m], reverse_weights f32[m])
        as held on the device."""
        roff = np.zeros(self.num_vertices + 1, np.uint64)
        rsrc = np.zeros(self.num_edges, np.uint32)
        rw = np.zeros(self.num_edges, np.float32)
        check(lib.rrg_graph_export_transpose(self._h, ptr(roff, C.c_uint64),
                                             ptr(rsrc, C.c_uint32), ptr(rw, C.c_float)))
        return roff, rsrc, rw

    @property
    def handle(self):
        return self._h

    def in_degree(self, v: int) -> int:
        return int(self.reverse_offsets[v + 1] - self.reverse_offsets[v])

    def prepare(self, model) -> None:
        check(lib.rrg_graph_prepare(self._h, _model(model)))

    def set_stream(self, cuda_stream_handle: int) -> None:
        check(lib.rrg_graph_set_stream(self._h, C.c_void_p(cuda_stream_handle or None)))

    def set_option(self, opt: str, value: int) -> None:
        code = {"lt_scan": 0, "lt_coop_min": 1, "ic_inner": 2, "ic_coop_min": 3,
                "lt_kary": 4, "ic_mode": 5, "ic_warp_min_insp": 6, "ic_rng": 7,
                "lt_guide_mult": 8, "ic_warp_budget": 9}[opt]
        check(lib.rrg_graph_set_option(self._h, code, int(value)))

    def last_batch_stats(self) -> "BatchStats":
        st = _lib.BatchStats()
        check(lib.rrg_last_batch_stats(self._h, C.byref(st)))
        return BatchStats(st.sets, st.members, st.edges_inspected, st.entries_read,
                          st.deferred, st.sample_ms, st.total_ms)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.rrg_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class BatchStats:
    sets: int
    members: int
    edges_inspected: int
    entries_read: int
    deferred: int
    sample_ms: float
    total_ms: float


class RRRStore:
    """Slot-ordered device store of RRR sets plus the fused occurrence counter."""

    def __init__(self, graph: Graph):
        self.graph = graph
        h = C.c_void_p()
        check(lib.rrg_store_create(graph.handle, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def size(self) -> int:
        s = C.c_uint64()
        check(lib.rrg_store_info(self._h, C.byref(s), None, None))
        return s.value

    def total_member_count(self) -> int:
        m = C.c_uint64()
        check(lib.rrg_store_info(self._h, None, C.byref(m), None))
        return m.value

    def max_set_size(self) -> int:
        x = C.c_uint32()
        check(lib.rrg_store_info(self._h, None, None, C.byref(x)))
        return x.value

    def live_count(self) -> int:
        """RRRStore::live_count (rrr_store.hpp:84): sets the last select_seeds left
        uncovered; every append revives all sets (finalize)."""
        x = C.c_uint64()
        check(lib.rrg_store_live_count(self._h, C.byref(x)))
        return x.value

    def live_flags(self, first: int = 0, count: Optional[int] = None) -> np.ndarray:
        """RRRStore::is_live (rrr_store.hpp:62) for sets [first, first+count)."""
        if count is None:
            count = self.size() - first
        out = np.zeros(max(count, 1), dtype=np.uint8)
        check(lib.rrg_store_live_flags(self._h, first, count, ptr(out, C.c_uint8)))
        return out[:count].astype(bool)

    def set_counter(self, counts) -> None:
        """A caller-held tally becomes the prebuilt Counter of select_seeds."""
        c = np.ascontiguousarray(counts, dtype=np.uint64)
        if c.size != self.graph.num_vertices:
            raise ValueError("set_counter: need one count per vertex")
        check(lib.rrg_store_set_counter(self._h, ptr(c, C.c_uint64)))

    def set_member_limit(self, max_members: int) -> None:
        """RRG_ENOMEM (RRGOutOfMemory) for a batch chunk past max_members (0: none)."""
        check(lib.rrg_store_set_member_limit(self._h, int(max_members)))

    def dense_info(self) -> dict:
        """The dense arm (rrr_set.hpp:73-90): n-bit map rows, their members and
        bytes, and the rebuild rounds of the last select_seeds on this store."""
        v = [C.c_uint64() for _ in range(4)]
        check(lib.rrg_store_dense_info(self._h, *[C.byref(x) for x in v]))
        return {"dense_sets": v[0].value, "dense_members": v[1].value,
                "dense_bytes": v[2].value, "rebuild_rounds": v[3].value}

    def clear(self) -> None:
        check(lib.rrg_store_clear(self._h))

    def export(self, first: int = 0, count: Optional[int] = None):
        """(offsets u64[count+1], members u32[...]) in slot order, visit order per set."""
        if count is None:
            count = self.size() - first
        off = np.zeros(count + 1, dtype=np.uint64)
        check(lib.rrg_store_export(self._h, first, count, ptr(off, C.c_uint64), None))
        mem = np.zeros(int(off[-1]), dtype=np.uint32)
        check(lib.rrg_store_export(self._h, first, count, ptr(off, C.c_uint64),
                                   ptr(mem, C.c_uint32)))
        return off, mem

    def export_into(self, offsets: np.ndarray, members: np.ndarray, first: int = 0,
                    count: Optional[int] = None) -> int:
        """Like export() but into caller-owned (e.g. pinned) host arrays; returns
        the member count written. offsets needs count+1 entries."""
        if count is None:
            count = self.size() - first
        check(lib.rrg_store_export(self._h, first, count, ptr(offsets, C.c_uint64), None))
        total = int(offsets[count])
        if total > members.size:
            raise ValueError("members buffer too small")
        check(lib.rrg_store_export(self._h, first, count, ptr(offsets, C.c_uint64),
                                   ptr(members, C.c_uint32)))
        return total

    def export_all_async(self, offsets: np.ndarray, members: np.ndarray,
                         counts: Optional[np.ndarray], stream: int) -> int:
        """Enqueues the D2H copies of the whole store (offsets, members, counter) on
        the CUDA stream handle `stream` and returns the member count without
        waiting; synchronize the stream before reading the buffers or touching
        the store again. u32 `offsets` / `counts` arrays select the compact
        32-bit export (fewer bytes over PCIe)."""
        total = self.total_member_count()
        if offsets.size < self.size() + 1 or members.size < total:
            raise ValueError("export buffers too small")
        if offsets.dtype == np.uint32:  # compact: u32 offsets and counts
            if counts is not None and counts.dtype != np.uint32:
                raise ValueError("export_all_async: u32 offsets need u32 counts")
            check(lib.rrg_store_export_all_async32(
                self._h, ptr(offsets, C.c_uint32), ptr(members, C.c_uint32),
                ptr(counts, C.c_uint32) if counts is not None else None, C.c_void_p(stream)))
            return total
        check(lib.rrg_store_export_all_async(
            self._h, ptr(offsets, C.c_uint64), ptr(members, C.c_uint32),
            ptr(counts, C.c_uint64) if counts is not None else None, C.c_void_p(stream)))
        return total

    def counter_into(self, out: np.ndarray) -> np.ndarray:
        check(lib.rrg_store_counter(self._h, ptr(out, C.c_uint64)))
        return out

    def sets(self, first: int = 0, count: Optional[int] = None, sort: bool = True):
        off, mem = self.export(first, count)
        out = [mem[off[i]:off[i + 1]] for i in range(off.size - 1)]
        return [np.sort(s) for s in out] if sort else out

    def import_sets(self, offsets, members) -> None:
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        members = np.ascontiguousarray(members, dtype=np.uint32)
        check(lib.rrg_store_import(self._h, offsets.size - 1, ptr(offsets, C.c_uint64),
                                   ptr(members, C.c_uint32)))

    def append_from(self, src: "RRRStore", first: int, count: int) -> None:
        """Appends src's sets [first, first+count) (device to device)."""
        check(lib.rrg_store_append_from(self._h, src.handle, int(first), int(count)))

    def counter(self) -> np.ndarray:
        out = np.zeros(self.graph.num_vertices, dtype=np.uint64)
        check(lib.rrg_store_counter(self._h, ptr(out, C.c_uint64)))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.rrg_store_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def generate_batch(g: Graph, model, run_seed: int, count: int, store: RRRStore,
                   fused: bool = True, density_divisor: int = kDefaultDensityDivisor) -> int:
    """sampling.hpp:159-199: appends `count` sets at slots [size, size+count)."""
    made = C.c_uint64()
    st = lib.rrg_generate_batch(g.handle, _model(model), int(run_seed) & (2**64 - 1), int(count),
                                store.handle, 1 if fused else 0, int(density_divisor),
                                C.byref(made))
    check(st, made.value)
    return made.value


def generate_slots(g: Graph, model, run_seed: int, first_slot: int, count: int,
                   store: RRRStore, fused: bool = True,
                   density_divisor: int = kDefaultDensityDivisor) -> int:
    """Appends the sets of slots [first_slot, first_slot+count) (one shard of a
    slot range split across GPUs; slot j depends only on (run_seed, j))."""
    made = C.c_uint64()
    st = lib.rrg_generate_slots(g.handle, _model(model), int(run_seed) & (2**64 - 1),
                                int(first_slot), int(count), store.handle, 1 if fused else 0,
                                int(density_divisor), C.byref(made))
    check(st, made.value)
    return made.value


def host_sync_count() -> int:
    """Host waits on the device (stream synchronizations) by librrgpu.so so far."""
    return int(lib.rrg_host_sync_count())


def launch_count() -> int:
    """Kernels librrgpu.so has launched in this process."""
    return int(lib.rrg_launch_count())


def generate_batch_fused(g: Graph, model, run_seed: int, count: int, store: RRRStore,
                         density_divisor: int = kDefaultDensityDivisor) -> int:
    """sampling.hpp:201-206."""
    return generate_batch(g, model, run_seed, count, store, True, density_divisor)


@dataclass
class SeedSet:
    """selection.hpp:19-22."""
    seeds: List[int] = field(default_factory=list)
    marginal_counts: List[int] = field(default_factory=list)
    round_counters: Optional[np.ndarray] = None
    covered: int = 0


@dataclass
class SelectionStats:
    """selection.hpp:45-49. touches (the reference's CPU touch tally) has no
    device counterpart and stays 0; rebuild_rounds counts the rounds that took
    rebuild_update (selection.hpp:161-203)."""
    touches: int = 0
    capture_round_counters: bool = False
    round_counters: Optional[np.ndarray] = None
    rebuild_rounds: int = 0


def select_seeds(store: RRRStore, n: int, k: int, adaptive_threshold: float = 0.25,
                 prebuilt=True, capture_round_counters: bool = False,
                 stats: Optional[SelectionStats] = None) -> SeedSet:
    """selection.hpp:209-243 (k rounds resident on the GPU). prebuilt: True = the
    store's fused counter, False = recount (build_counter), or a per-vertex
    array = the caller's Counter as the starting tally."""
    if not isinstance(prebuilt, bool):
        store.set_counter(prebuilt)
        prebuilt = True
    if stats is not None and stats.capture_round_counters:
        capture_round_counters = True
    if n != store.graph.num_vertices:
        raise ValueError("select_seeds: n does not match the store's graph")
    if k < 1:
        raise ValueError("select_seeds: k must be >= 1")
    if k > n:
        raise ValueError("select_seeds: k exceeds vertex count")
    seeds = np.zeros(k, dtype=np.uint32)
    marg = np.zeros(k, dtype=np.uint64)
    snap = np.zeros(k * n, dtype=np.uint64) if capture_round_counters else None
    rounds = C.c_uint32()
    covered = C.c_uint64()
    check(lib.rrg_select_seeds(store.handle, k, float(adaptive_threshold), 1 if prebuilt else 0,
                               ptr(seeds, C.c_uint32), ptr(marg, C.c_uint64),
                               ptr(snap, C.c_uint64), C.byref(rounds), C.byref(covered)))
    rc = snap.reshape(k, n)[: rounds.value] if snap is not None else None
    if stats is not None:
        stats.round_counters = rc
        stats.rebuild_rounds = store.dense_info()["rebuild_rounds"]
    return SeedSet([int(x) for x in seeds], [int(x) for x in marg], rc, covered.value)


def fraction_covered(store: RRRStore, seeds) -> float:
    """selection.hpp:340-358."""
    s = np.ascontiguousarray(list(seeds.seeds if isinstance(seeds, SeedSet) else seeds),
                             dtype=np.uint32)
    out = C.c_double()
    check(lib.rrg_fraction_covered(store.handle, ptr(s, C.c_uint32), s.size, C.byref(out)))
    return out.value


@dataclass
class ImmConfig:
    """imm.hpp:27-36 defaults."""
    k: int = 50
    epsilon: float = 0.5
    model: int = DiffusionModel.IC
    workers: int = 1
    rng_seed: int = 1
    ell: float = 1.0
    adaptive_threshold: float = 0.25
    strategy: int = 0  # Strategy::fused (imm.hpp:33); 1 = baseline (same seeds, unfused)


class Strategy:
    FUSED, BASELINE = 0, 1


def parse_strategy(s: str) -> int:
    """parse_strategy (imm.hpp:20-24)."""
    if s == "fused":
        return Strategy.FUSED
    if s == "baseline":
        return Strategy.BASELINE
    raise ValueError("unknown strategy: " + s)


@dataclass
class ImmResult:
    """imm.hpp:44-54."""
    seeds: SeedSet
    theta: int
    theta_prime: int
    lower_bound: float
    timings: dict
    sets_generated: int
    mean_set_size: float
    max_set_size: int
    mean_coverage_fraction: float


def _imm_config(cfg: ImmConfig):
    return _lib.ImmConfigC(int(cfg.k), float(cfg.epsilon), _model(cfg.model), int(cfg.workers),
                           int(cfg.rng_seed) & (2**64 - 1), float(cfg.ell),
                           float(cfg.adaptive_threshold), int(cfg.strategy))


@dataclass
class SamplingPhaseResult:
    """imm.hpp:157-162: the store (its fused counter is the phase's Counter)."""
    store: RRRStore
    lower_bound: float
    theta_prime: int
    timings: dict


def sampling_phase(g: Graph, cfg: ImmConfig) -> SamplingPhaseResult:
    """sampling_phase (imm.hpp:169-209) into a fresh device store."""
    c = _imm_config(cfg)
    st = RRRStore(g)
    lb = C.c_double()
    tp = C.c_uint64()
    r = _lib.ImmResultC()
    check(lib.rrg_sampling_phase(g.handle, C.byref(c), st.handle, C.byref(lb), C.byref(tp),
                                 C.byref(r)))
    return SamplingPhaseResult(st, lb.value, int(tp.value),
                               {"generate_rrrsets": r.t_generate,
                                "find_most_influential": r.t_select})


def run_imm(g: Graph, cfg: ImmConfig) -> ImmResult:
    """imm.hpp:214-251, driven by the C++17 driver in csrc/imm.cpp."""
    return _run_imm(g, cfg, None, 0)


def run_imm_sharded(g: Graph, cfg: ImmConfig, comm: Optional["NcclComm"] = None,
                    sim_ranks: int = 0) -> ImmResult:
    """Multi-GPU run_imm: every rank of `comm` samples its shard
    of each top-up, the shards are exchanged over NCCL from device memory, and
    every rank returns run_imm's result. comm=None with sim_ranks >= 1 runs the
    same shard split in one process."""
    return _run_imm(g, cfg, comm, sim_ranks, sharded=True)


class NcclComm:
    """An NCCL communicator for rrg_run_imm_sharded: one per rank, created with
    this process's GPU current (torch.cuda.set_device) from the 128-byte id of
    nccl_unique_id() on rank 0, passed to all ranks."""

    def __init__(self, uid: bytes, nranks: int, rank: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        check(lib.rrg_nccl_comm_create(buf, int(nranks), int(rank), C.byref(h)))
        self._h = h
        self.nranks, self.rank = nranks, rank

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.rrg_nccl_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib.rrg_nccl_unique_id(buf))
    return bytes(buf)


def _run_imm(g: Graph, cfg: ImmConfig, comm, sim_ranks: int, sharded: bool = False) -> ImmResult:
    c = _imm_config(cfg)
    k = max(int(cfg.k), 1)
    seeds = np.zeros(k, dtype=np.uint32)
    marg = np.zeros(k, dtype=np.uint64)
    r = _lib.ImmResultC()
    if not sharded:
        check(lib.rrg_run_imm(g.handle, C.byref(c), ptr(seeds, C.c_uint32),
                              ptr(marg, C.c_uint64), C.byref(r)))
    else:
        check(lib.rrg_run_imm_sharded(g.handle, C.byref(c), comm.handle if comm else None,
                                      int(sim_ranks), ptr(seeds, C.c_uint32),
                                      ptr(marg, C.c_uint64), C.byref(r)))
    return ImmResult(
        seeds=SeedSet([int(x) for x in seeds], [int(x) for x in marg]),
        theta=r.theta, theta_prime=r.theta_prime, lower_bound=r.lower_bound,
        timings={"generate_rrrsets": r.t_generate, "find_most_influential": r.t_select,
                 "total": r.t_total},
        sets_generated=r.sets_generated, mean_set_size=r.mean_set_size,
        max_set_size=r.max_set_size, mean_coverage_fraction=r.mean_coverage_fraction)
