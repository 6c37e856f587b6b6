"""Multi-GPU data parallelism for the GPU replica workers.

One process per B200 (torchrun), each running its own GPU replica worker on
its own stream of batches (the paper's "separate GPU worker" per device,
PAPER.md:321).  The only exchange is the GPU-replica merge: every
`merge_every` steps the device models are averaged, either with an NCCL
allreduce issued by the C library on its own stream (hb_merge_allreduce) or
over peer memory (transport="peer": the library's one-shot reduce kernel reads
and writes every rank's exchange buffer directly, NVLink P2P / CUDA IPC).  The NCCL
unique id travels over `torch.distributed` (any backend, gloo included) as a
128-byte tensor, so the control plane here is testable on CPU.
"""

from __future__ import annotations

import os

import numpy as np

from .replica import GpuReplica


def dist_env() -> tuple:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def broadcast_bytes(dist, payload: bytes | None, src: int = 0, length: int = 128) -> bytes:
    """Broadcast a fixed-length byte string from `src` to every rank."""
    import torch

    if payload is not None and len(payload) != length:
        raise ValueError(f"payload must be {length} bytes")
    t = torch.tensor(list(payload) if payload is not None else [0] * length, dtype=torch.uint8)
    dist.broadcast(t, src)
    return bytes(t.tolist())


def broadcast_float(dist, value: float, src: int = 0) -> float:
    """Rank `src`'s float on every rank (CPU tensor: the gloo half of the group)."""
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64)
    dist.broadcast(t, src)
    return float(t.item())


def barrier(dist) -> None:
    """Host-side barrier as a one-element CPU all-reduce: it runs on the CPU
    (gloo) half of a "cpu:gloo,cuda:nccl" process group, so it needs no GPU
    tensor and no device-side NCCL communicator of torch's."""
    import torch

    dist.all_reduce(torch.zeros(1))


def init_process_group(dist) -> None:
    """torch.distributed for the control plane: CPU tensors over gloo, CUDA
    tensors over NCCL; the replica merge itself is the library's own NCCL
    communicator (hb_comm_init / hb_merge_allreduce)."""
    import torch

    dist.init_process_group("cpu:gloo,cuda:nccl" if torch.cuda.is_available() else "gloo")


def max_over_ranks(dist, value: float) -> float:
    """The slowest rank's time: the multi-GPU timing rule (max over ranks)."""
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard_seed(seed: int, rank: int) -> int:
    """Per-rank data seed: every GPU worker draws its own batch stream."""
    return int(seed) * 1_000_003 + int(rank)


def batch_starts(n_rows: int, batch: int, steps: int, offset: int = 0) -> list:
    """Contiguous batch ranges cycling through an epoch of n_rows (full batches only)."""
    n_batches = max(1, (n_rows - batch) // batch + 1)
    return [((offset + i) % n_batches) * batch for i in range(steps)]


def init_replica_comm(replica: GpuReplica, dist, rank: int, world: int) -> None:
    """Create the NCCL communicator of a replica (unique id from rank 0)."""
    uid = GpuReplica.nccl_unique_id() if rank == 0 else None
    replica.comm_init(broadcast_bytes(dist, uid, 0), world, rank)


def all_gather_bytes(dist, payload: bytes, world: int) -> list:
    """Every rank's fixed-length byte string, in rank order (CPU tensors)."""
    import torch

    t = torch.tensor(list(payload), dtype=torch.uint8)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [bytes(o.tolist()) for o in out]


def init_replica_peers(replica: GpuReplica, dist, rank: int, world: int) -> None:
    """Peer-memory merge group across processes: the exchange-buffer handles
    (CUDA IPC) travel over torch.distributed, then every rank maps the others."""
    replica.peer_attach(all_gather_bytes(dist, replica.peer_handle(), world), rank)


def local_peer_group(replicas) -> None:
    """Peer-memory merge group of replicas in this process (one per GPU worker
    thread, as the reference engine runs its roster, engine.py:131-134), or
    several replicas on one device.  Every replica must then merge the same
    number of times, each from its own thread."""
    handles = [r.peer_handle() for r in replicas]
    for rank, r in enumerate(replicas):
        r.peer_attach(handles, rank)


class DataParallelWorker:
    """A GPU replica worker that averages its model with its peers every
    `merge_every` steps (model averaging over NVLink)."""

    def __init__(self, replica: GpuReplica, dist=None, merge_every: int = 1, transport: str = "nccl"):
        if merge_every < 1:
            raise ValueError("merge_every must be >= 1")
        if transport not in ("nccl", "peer"):
            raise ValueError(f"transport must be 'nccl' or 'peer', got {transport!r}")
        self.replica = replica
        self.dist = dist
        self.rank, self.world, _ = dist_env()
        self.merge_every = merge_every
        self.transport = transport
        self.steps = 0
        if self.world > 1:
            if transport == "peer":
                init_replica_peers(replica, dist, self.rank, self.world)
            else:
                init_replica_comm(replica, dist, self.rank, self.world)

    def step(self, start: int, rows: int, eta: float, **kw):
        # the merge rides on the step's stream (HB_STEP_MERGE): no extra sync
        self.steps += 1
        due = self.world > 1 and self.steps % self.merge_every == 0
        return self.replica.step(start, rows, eta, merge=due, **kw)


def average_models_host(models: list) -> list:
    """Reference semantics of the merge on host arrays (used by tests)."""
    return [np.mean(np.stack(ws), axis=0) for ws in zip(*models)]
