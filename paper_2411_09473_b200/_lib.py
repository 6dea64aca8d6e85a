"""ctypes binding of librrgpu.so (include/rrgpu.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2411_09473_b200/csrc``). There is no fallback: importing this
module without the library raises, so no caller can silently run on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RRGPU_LIB") or os.path.join(_HERE, "librrgpu.so")

RRG_OK, RRG_EINVAL, RRG_ENOMEM, RRG_ECUDA = 0, 1, 2, 3

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
vp = C.c_void_p


class BatchStats(C.Structure):
    _fields_ = [
        ("sets", C.c_uint64),
        ("members", C.c_uint64),
        ("edges_inspected", C.c_uint64),
        ("entries_read", C.c_uint64),
        ("deferred", C.c_uint64),
        ("sample_ms", C.c_float),
        ("total_ms", C.c_float),
    ]


class ImmConfigC(C.Structure):
    _fields_ = [
        ("k", C.c_uint32),
        ("epsilon", C.c_double),
        ("model", C.c_int),
        ("workers", C.c_uint32),
        ("rng_seed", C.c_uint64),
        ("ell", C.c_double),
        ("adaptive_threshold", C.c_double),
        ("strategy", C.c_int),
    ]


class ImmResultC(C.Structure):
    _fields_ = [
        ("theta", C.c_uint64),
        ("theta_prime", C.c_uint64),
        ("lower_bound", C.c_double),
        ("sets_generated", C.c_uint64),
        ("mean_set_size", C.c_double),
        ("max_set_size", C.c_uint32),
        ("mean_coverage_fraction", C.c_double),
        ("t_generate", C.c_double),
        ("t_select", C.c_double),
        ("t_total", C.c_double),
    ]


# (name, restype, argtypes) for every symbol of include/rrgpu.h
SIGNATURES = [
    ("rrg_graph_create", C.c_int, [C.c_uint32, C.c_uint64, u64p, u32p, f32p, C.POINTER(vp)]),
    ("rrg_graph_create_for", C.c_int,
     [C.c_uint32, C.c_uint64, u64p, u32p, f32p, C.c_int, C.POINTER(vp)]),
    ("rrg_graph_create_from_edges", C.c_int,
     [C.c_uint32, C.c_uint64, u32p, u32p, f32p, C.c_int, C.POINTER(vp)]),
    ("rrg_graph_export_transpose", C.c_int, [vp, u64p, u32p, f32p]),
    ("rrg_graph_destroy", None, [vp]),
    ("rrg_graph_prepare", C.c_int, [vp, C.c_int]),
    ("rrg_graph_set_stream", C.c_int, [vp, vp]),
    ("rrg_graph_num_vertices", C.c_uint32, [vp]),
    ("rrg_graph_num_edges", C.c_uint64, [vp]),
    ("rrg_graph_set_option", C.c_int, [vp, C.c_int, C.c_int64]),
    ("rrg_store_create", C.c_int, [vp, C.POINTER(vp)]),
    ("rrg_store_destroy", None, [vp]),
    ("rrg_store_clear", C.c_int, [vp]),
    ("rrg_store_dense_info", C.c_int, [vp, u64p, u64p, u64p, u64p]),
    ("rrg_host_sync_count", C.c_uint64, []),
    ("rrg_nccl_unique_id", C.c_int, [u8p]),
    ("rrg_nccl_comm_create", C.c_int, [u8p, C.c_int, C.c_int, C.POINTER(vp)]),
    ("rrg_nccl_comm_destroy", None, [vp]),
    ("rrg_run_imm_sharded", C.c_int, [vp, C.POINTER(ImmConfigC), vp, C.c_int, u32p, u64p,
                                      C.POINTER(ImmResultC)]),
    ("rrg_store_live_count", C.c_int, [vp, u64p]),
    ("rrg_store_live_flags", C.c_int, [vp, C.c_uint64, C.c_uint64, u8p]),
    ("rrg_store_set_counter", C.c_int, [vp, u64p]),
    ("rrg_store_set_member_limit", C.c_int, [vp, C.c_uint64]),
    ("rrg_store_info", C.c_int, [vp, u64p, u64p, u32p]),
    ("rrg_generate_batch", C.c_int,
     [vp, C.c_int, C.c_uint64, C.c_uint64, vp, C.c_int, C.c_uint32, u64p]),
    ("rrg_generate_slots", C.c_int,
     [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, vp, C.c_int, C.c_uint32, u64p]),
    ("rrg_last_batch_stats", C.c_int, [vp, C.POINTER(BatchStats)]),
    ("rrg_launch_count", C.c_uint64, []),
    ("rrg_select_seeds", C.c_int,
     [vp, C.c_uint32, C.c_double, C.c_int, u32p, u64p, u64p, u32p, u64p]),
    ("rrg_fraction_covered", C.c_int, [vp, u32p, C.c_uint32, C.POINTER(C.c_double)]),
    ("rrg_imm_config_default", None, [C.POINTER(ImmConfigC)]),
    ("rrg_run_imm", C.c_int, [vp, C.POINTER(ImmConfigC), u32p, u64p, C.POINTER(ImmResultC)]),
    ("rrg_sampling_phase", C.c_int,
     [vp, C.POINTER(ImmConfigC), vp, C.POINTER(C.c_double), u64p, C.POINTER(ImmResultC)]),
    ("rrg_store_export", C.c_int, [vp, C.c_uint64, C.c_uint64, u64p, u32p]),
    ("rrg_store_import", C.c_int, [vp, C.c_uint64, u64p, u32p]),
    ("rrg_store_append_from", C.c_int, [vp, vp, C.c_uint64, C.c_uint64]),
    ("rrg_store_counter", C.c_int, [vp, u64p]),
    ("rrg_store_export_all_async", C.c_int, [vp, u64p, u32p, u64p, vp]),
    ("rrg_store_export_all_async32", C.c_int, [vp, u32p, u32p, u32p, vp]),
    ("rrg_build_transpose", C.c_int,
     [C.c_uint32, C.c_uint64, u32p, u32p, f32p, u64p, u32p, f32p]),
    ("rrg_normalize_lt_weights", C.c_int, [C.c_uint32, u64p, f32p]),
    ("rrg_last_error", C.c_char_p, []),
    ("rrg_version", C.c_char_p, []),
    ("rrg_debug_bernoulli_threshold", C.c_uint64, [C.c_uint32]),
    ("rrg_debug_bernoulli_thr_hi", C.c_uint32, [C.c_uint32]),
    ("rrg_debug_export_lt_cdf", C.c_int, [vp, C.POINTER(C.c_double)]),
    ("rrg_debug_jump", None, [u64p, C.c_uint64, u64p]),
]


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with __graft_entry__.build() or "
            "`make -C paper_2411_09473_b200/csrc` (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()


class RRGError(RuntimeError):
    """RRG_ECUDA: std::runtime_error in the reference."""


class RRGOutOfMemory(MemoryError):
    """RRG_ENOMEM: BatchOutOfMemory / std::bad_alloc (sampling.hpp:148-154)."""

    def __init__(self, msg: str, sets_generated: int = 0):
        super().__init__(msg)
        self.sets_generated = sets_generated


def check(status: int, sets_generated: int = 0) -> None:
    if status == RRG_OK:
        return
    msg = (lib.rrg_last_error() or b"").decode()
    if status == RRG_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if status == RRG_ENOMEM:
        raise RRGOutOfMemory(msg, sets_generated)
    raise RRGError(msg)


def ptr(arr, ctype):
    """ctypes pointer into a contiguous numpy array (or None)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(C.POINTER(ctype))
