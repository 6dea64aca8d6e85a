"""Multi-rank host logic of paper_2411_09473_b200/parallel.py on CPU (gloo,
world size 2): slot sharding, ordered set gather, counter all-reduce and the
sharded IMM driver reproduce the single-process reference result exactly.
The per-rank sampler here is the CPU checker (test-only injection); on GPUs
the same functions drive the CUDA sampler (tests/test_gpu_parallel.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2411_09473_b200 import parallel


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_partitions_every_range():
    for lo, hi, world in [(0, 10, 3), (5, 5, 2), (7, 100, 8), (0, 3, 4)]:
        got = []
        for r in range(world):
            f, c = parallel.shard(lo, hi, world, r)
            got.extend(range(f, f + c))
        assert got == list(range(lo, hi))


def test_theta_math_matches_oracle(port):
    for n, k in [(10000, 50), (65536, 50), (4847571, 50), (3072441, 100), (100, 2)]:
        ell = parallel.effective_ell(1.0, n)
        assert ell == port.effective_ell(1.0, n)
        assert parallel.lambda_prime(n, k, 0.5, ell) == port.lambda_prime(n, k, 0.5, ell)
        assert parallel.sampling_rounds(n) == port.sampling_rounds(n)
        for i in range(1, 6):
            assert parallel.theta_for_round(n, k, 0.5, ell, i) == \
                port.theta_for_round(n, k, 0.5, ell, i)
        assert parallel.set_theta(n, k, 0.5, ell, 1234.5) == port.set_theta(n, k, 0.5, ell, 1234.5)


def _worker(rank, world, port_no, arrays, model, k, q):
    import torch.distributed as dist
    from oracle import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle("port")
    g = orc.graph(*arrays)
    n = arrays[0].size - 1

    def sample_fn(first, count):
        sk = g.sample(model, 1, first, count)
        return sk.offsets, sk.members, sk.counter

    def select_fn(off, mem, counter):
        # the merged counter must be the histogram of the gathered collection
        assert (np.bincount(mem, minlength=n).astype(np.uint64) == counter).all()
        return orc.select(n, off, mem, k)

    res = parallel.sharded_imm(n, k, 0.5, 1.0, sample_fn, select_fn)
    q.put((rank, res.seeds, res.marginals, res.theta, res.theta_prime, res.lower_bound,
           res.sets_generated))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("model,name", [(0, "cfg1"), (1, "cfg2")])
def test_sharded_imm_world2_equals_single_process(port, model, name):
    from paper_2411_09473_b200 import graphs
    cfg = graphs.scaled(graphs.CONFIGS[name], 1 << 10, 1 << 13)
    arrays = graphs.generate(cfg)
    k = 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, arrays, model, k, q))
             for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = port.graph(*arrays).imm(k=k, model=model)
    for _, seeds, marg, theta, theta_p, lb, sets in results:
        assert seeds == ref["seeds"]
        assert marg == ref["marginals"]
        assert theta == ref["theta"] and theta_p == ref["theta_prime"]
        assert lb == ref["lower_bound"]
        assert sets == ref["sets_generated"]


def _uid_worker(rank, world, port_no, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []

    def make_id():
        calls.append(rank)
        return bytes(range(128))[::-1]

    uid = parallel.share_unique_id(make_id)
    q.put((rank, uid, calls))
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_unique_id_reaches_every_rank():
    """rrg_run_imm_sharded's communicator setup: only rank 0 makes the 128-byte
    NCCL id, every rank receives the same bytes (world size 3, gloo)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = free_port()
    procs = [ctx.Process(target=_uid_worker, args=(r, 3, port_no, q)) for r in range(3)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = bytes(range(128))[::-1]
    assert all(uid == want for _, uid, _ in results)
    assert [calls for _, _, calls in results] == [[0], [], []]
