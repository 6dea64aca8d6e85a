"""Multi-GPU split of the IMM hot path.

Slot j of a run depends only on (run_seed, j) (sampling.hpp:179), so each rank
samples a contiguous slice of every top-up's slot range with no communication.
The one real exchange is before selection: the ranks' flat buffers are
all-gathered in slot order (sigma|R| is a few MB at the BASELINE
configs) and every rank runs the deterministic selection on the full
collection, so all ranks hold the same seeds without a broadcast. The fused
occurrence counters merge with one all-reduce (sum) for the prebuilt tally.

The host logic is written against two callables so it can be exercised with
any sampler/selector (the CUDA path on GPUs; the CPU checkers in the gloo
tests of tests/test_parallel.py):

  sample_fn(first_slot, count) -> (offsets u64[count+1], members u32[...], counter u64[n])
  select_fn(offsets, members, counter) -> (seeds list, marginals list)
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, List, Optional, Tuple

import numpy as np


def shard(lo: int, hi: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous slice [first, first+count) of slots [lo, hi) owned by `rank`."""
    total = hi - lo
    q, r = divmod(total, world)
    first = lo + rank * q + min(rank, r)
    count = q + (1 if rank < r else 0)
    return first, count


def _all_gather_varlen(arr: np.ndarray, group=None) -> List[np.ndarray]:
    """All-gather 1-D numpy arrays of different lengths (rank order)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = _comm_device(group)
    n = torch.tensor([arr.size], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    width = max(max(sizes), 1)
    buf = torch.zeros(width, dtype=torch.int64, device=dev)
    buf[: arr.size] = torch.from_numpy(arr.astype(np.int64))
    outs = [torch.zeros(width, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return [o[:s].cpu().numpy() for o, s in zip(outs, sizes)]


def _comm_device(group=None):
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_sets(offsets: np.ndarray, members: np.ndarray, group=None):
    """Concatenate every rank's (offsets, members) shard in rank = slot order."""
    sizes = np.diff(offsets.astype(np.int64))
    all_sizes = _all_gather_varlen(sizes, group)
    all_members = _all_gather_varlen(members.astype(np.int64), group)
    sizes = np.concatenate(all_sizes) if all_sizes else np.zeros(0, np.int64)
    off = np.zeros(sizes.size + 1, np.uint64)
    np.cumsum(sizes, out=off[1:])
    mem = np.concatenate(all_members).astype(np.uint32) if all_members else np.zeros(0, np.uint32)
    return off, mem


def merge_counters(counter: np.ndarray, group=None) -> np.ndarray:
    """Sum of the ranks' fused occurrence counters (one all-reduce)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(counter.astype(np.int64)).to(_comm_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy().astype(np.uint64)


# ---- theta math (imm.hpp:57-120), same expression order ---------------------
def log_binomial(n: int, k: int) -> float:
    s = 0.0
    for j in range(n - k + 1, n + 1):
        s += math.log(float(j))
    for j in range(1, k + 1):
        s -= math.log(float(j))
    return s


def effective_ell(ell: float, n: int) -> float:
    if n < 2:
        return ell
    return ell * (1.0 + math.log(2.0) / math.log(float(n)))


def lambda_prime(n: int, k: int, eps: float, ell: float) -> float:
    nd = float(n)
    ep = math.sqrt(2.0) * eps
    l2 = max(1.0, math.log2(nd))
    terms = log_binomial(n, k) + ell * math.log(nd) + math.log(l2)
    return (2.0 + (2.0 / 3.0) * ep) * terms * nd / (ep * ep)


def sampling_rounds(n: int) -> int:
    if n <= 4:
        return 1
    r = int(math.floor(math.log2(float(n)))) - 1
    return 1 if r < 1 else r


def round_target(n: int, i: int) -> float:
    if n <= 4:
        return max(1.0, float(n) / 2.0)
    return float(n) / math.pow(2.0, float(i))


def theta_for_round(n: int, k: int, eps: float, ell: float, i: int) -> int:
    t = math.ceil(lambda_prime(n, k, eps, ell) / round_target(n, i))
    return 1 if not (t >= 1.0) else int(t)


def lambda_star(n: int, k: int, eps: float, ell: float) -> float:
    nd = float(n)
    c = 1.0 - 1.0 / math.exp(1.0)
    a = math.sqrt(ell * math.log(nd) + math.log(2.0))
    b = math.sqrt(c * (log_binomial(n, k) + ell * math.log(nd) + math.log(2.0)))
    s = c * a + b
    return 2.0 * nd * s * s / (eps * eps)


def set_theta(n: int, k: int, eps: float, ell: float, lb: float) -> int:
    t = math.ceil(lambda_star(n, k, eps, ell) / lb)
    return 1 if not (t >= 1.0) else int(t)


@dataclass
class ShardedImmResult:
    seeds: List[int]
    marginals: List[int]
    theta: int
    theta_prime: int
    lower_bound: float
    sets_generated: int


def sharded_imm(n: int, k: int, epsilon: float, ell: float,
                sample_fn: Callable, select_fn: Callable, group=None) -> ShardedImmResult:
    """run_imm (imm.hpp:214-251) with each top-up split across the ranks."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    ell_eff = effective_ell(ell, n)
    eps_prime = math.sqrt(2.0) * epsilon
    local_off = [np.zeros(1, np.uint64)]
    local_mem: List[np.ndarray] = []
    counter = np.zeros(n, np.uint64)
    size = 0
    full: Optional[Tuple[np.ndarray, np.ndarray]] = None
    shards: List[Tuple[np.ndarray, np.ndarray]] = []

    def top_up(target: int):
        nonlocal size, counter, full
        if target <= size:
            return
        first, count = shard(size, target, world, rank)
        off, mem, cnt = sample_fn(first, count)
        counter = counter + cnt
        if world > 1:
            g_off, g_mem = gather_sets(off, mem, group)
        else:
            g_off, g_mem = off, mem
        shards.append((g_off, g_mem))
        size = target
        full = None

    def collection():
        nonlocal full
        if full is None:
            sizes = np.concatenate([np.diff(o.astype(np.int64)) for o, _ in shards])
            off = np.zeros(sizes.size + 1, np.uint64)
            np.cumsum(sizes, out=off[1:])
            mem = np.concatenate([m for _, m in shards]).astype(np.uint32)
            full = (off, mem)
        return full

    rounds = sampling_rounds(n)
    spread, triggered = 0.0, False
    for i in range(1, rounds + 1):
        top_up(theta_for_round(n, k, epsilon, ell_eff, i))
        off, mem = collection()
        merged = merge_counters(counter, group) if world > 1 else counter
        _, marg = select_fn(off, mem, merged)
        spread = float(n) * (float(sum(marg)) / float(size))
        if spread >= (1.0 + eps_prime) * round_target(n, i):
            triggered = True
            break
    lb = spread / (1.0 + eps_prime) if triggered else max(spread / (1.0 + eps_prime), float(k))
    theta_prime = size
    theta = set_theta(n, k, epsilon, ell_eff, lb)
    top_up(theta)
    off, mem = collection()
    merged = merge_counters(counter, group) if world > 1 else counter
    seeds, marg = select_fn(off, mem, merged)
    del local_off, local_mem
    return ShardedImmResult(list(seeds), list(marg), theta, theta_prime, lb, size)


def share_unique_id(make_id: Callable[[], bytes], group=None) -> bytes:
    """Rank 0's NCCL unique id (128 bytes), handed to every rank over the
    torch.distributed group (gloo or nccl)."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def run_imm_distributed(g, cfg, group=None):
    """run_imm over every rank of `group`, one GPU each (the current device):
    rrg_run_imm_sharded with an NCCL communicator of the group's ranks -- each
    top-up's shards sampled locally and exchanged as device buffers over NCCL;
    every rank returns the same ImmResult as single-GPU run_imm."""
    import torch.distributed as dist
    from . import NcclComm, nccl_unique_id, run_imm_sharded
    uid = share_unique_id(nccl_unique_id, group)
    comm = NcclComm(uid, dist.get_world_size(group), dist.get_rank(group))
    try:
        return run_imm_sharded(g, cfg, comm)
    finally:
        comm.close()
