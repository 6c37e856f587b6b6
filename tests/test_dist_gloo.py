"""World-size-2 gloo tests of the multi-GPU control plane (no GPU): the NCCL
unique-id broadcast, per-rank batch streams, max-over-ranks timing, the
merge cadence of DataParallelWorker, and the model-averaging semantics."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2004_08771_b200 import parallel as P

    P.init_process_group(dist)  # CPU box: plain gloo (on a GPU box "cpu:gloo,cuda:nccl")

    out = {}
    uid = bytes(range(128)) if rank == 0 else None
    out["uid"] = P.broadcast_bytes(dist, uid, 0)
    out["max"] = P.max_over_ranks(dist, 1.5 + rank)
    out["seed"] = P.shard_seed(42, rank)
    out["starts"] = P.batch_starts(64700, 8192, 10)

    class FakeReplica:
        def __init__(self):
            self.merges = 0
            self.steps = []

        def comm_init(self, uid, nranks, r):
            self.comm = (len(uid), nranks, r)

        def step(self, start, rows, eta, merge=False, **kw):
            self.steps.append(start)
            self.merges += int(merge)

        def merge_allreduce(self):
            self.merges += 1

    import paper_2004_08771_b200.parallel as par

    orig = par.GpuReplica.nccl_unique_id
    par.GpuReplica.nccl_unique_id = staticmethod(lambda: bytes([7]) * 128)
    try:
        rep = FakeReplica()
        w = P.DataParallelWorker(rep, dist, merge_every=3)
        for s in range(7):
            w.step(s, 10, 0.1)
        out["merges"] = rep.merges
        out["comm"] = rep.comm
    finally:
        par.GpuReplica.nccl_unique_id = orig
    P.barrier(dist)  # the bench's host-side barrier (a CPU all-reduce)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_control_plane_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0]["uid"] == res[1]["uid"] == bytes(range(128))
    assert res[0]["max"] == res[1]["max"] == 2.5
    assert res[0]["seed"] != res[1]["seed"]
    assert res[0]["starts"] == res[1]["starts"] and max(res[0]["starts"]) <= 64700 - 8192
    assert res[0]["merges"] == res[1]["merges"] == 2  # every 3rd of 7 steps
    assert res[0]["comm"] == (128, 2, 0) and res[1]["comm"] == (128, 2, 1)


def test_average_models_host():
    from paper_2004_08771_b200.parallel import average_models_host

    a = [np.ones((2, 2)), np.zeros(3)]
    b = [3 * np.ones((2, 2)), np.ones(3)]
    avg = average_models_host([a, b])
    assert np.array_equal(avg[0], 2 * np.ones((2, 2))) and np.array_equal(avg[1], 0.5 * np.ones(3))


def test_merge_every_validation():
    from paper_2004_08771_b200.parallel import DataParallelWorker

    with pytest.raises(ValueError):
        DataParallelWorker(object(), None, merge_every=0)
