"""The GPU replica worker behind the reference's own worker interface.

Drop-in seam: the reference's `WorkerThread._execute` calls
the module-global `execute_batch_replica(model, batch, eta, speed_factor)`
(pkg/src/hogtrain/workers.py:204-206) and `_evaluate` calls
`loss_sum(eval_model, x, y)` (workers.py:214).  `execute_gpu_replica` and
`gpu_loss_sum` here have exactly those signatures and semantics and run the
whole step on a B200; `install()` rebinds them into a live `hogtrain` module
(the reference's own injection mechanism, test_engine_modes.py:59).

`WorkerMode.GPU_REPLICA` / `WorkerConfig(device=...)` extend the reference's
config surface (workers.py:38-77; harness.py:153-177 reads `worker.N.mode`)
for rosters that name the GPU worker explicitly.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass
from enum import Enum

import numpy as np

from .data import CsrBatchRef, CsrDataset
from .nn import layer_sizes_of
from ._native import HB_DENSIFY_MAX_DIN as N_DENSIFY_MAX_DIN
from .replica import GpuReplica


class WorkerMode(Enum):  # workers.py:38-40 plus the B200 worker
    HOGWILD_SHARDED = "hogwild_sharded"
    BATCH_REPLICA = "batch_replica"
    GPU_REPLICA = "gpu_replica"


class ReplicaMode(Enum):  # workers.py:43-45
    REFERENCE = "reference"
    DEEP_COPY = "deep_copy"


_REQUIRED_REPLICA = {  # workers.py:48-51
    WorkerMode.HOGWILD_SHARDED: ReplicaMode.REFERENCE,
    WorkerMode.BATCH_REPLICA: ReplicaMode.DEEP_COPY,
    WorkerMode.GPU_REPLICA: ReplicaMode.DEEP_COPY,
}


@dataclass(frozen=True)
class WorkerConfig:  # workers.py:54-77, plus device / precision / sync_every for GPU workers
    worker_id: str
    mode: WorkerMode
    threads: int = 1
    replica_mode: ReplicaMode | None = None
    speed_factor: float = 0.0
    min_batch: int = 1
    max_batch: int = 1
    device: int = 0
    precision: str = "3xtf32"

    def __post_init__(self):
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.speed_factor < 0:
            raise ValueError("speed_factor must be >= 0")
        if not (1 <= self.min_batch <= self.max_batch):
            raise ValueError(f"need 1 <= min_batch <= max_batch, got [{self.min_batch}, {self.max_batch}]")
        if self.device < 0:
            raise ValueError("device must be >= 0")
        required = _REQUIRED_REPLICA[self.mode]
        if self.replica_mode is None:
            object.__setattr__(self, "replica_mode", required)
        elif self.replica_mode is not required:
            raise ValueError(f"{self.mode.value} workers require replica_mode={required.value}")


# ------------------------------------------------------------------------
# Per-thread device contexts: a context is affine to the worker thread that
# created it (include/hogbatch_b200.h "Conventions").
_tls = threading.local()
_DEFAULT_MAX_BATCH = 8192
# worker id -> device, for the reference's worker threads (named
# "worker-<worker_id>", workers.py:154), which the caller does not control
_worker_devices: dict = {}
_sole_writer = False
_speed_feed = None  # DeviceSpeedFeed fed by every replica step (install(feed=...))


def set_worker_device(device: int, max_batch: int | None = None, precision: str = "3xtf32") -> None:
    """Select the GPU (and batch capacity / precision) for replica calls made
    on the *calling* thread.  For the reference engine's worker threads use
    set_worker_devices (they are created by the engine, engine.py:131-134)."""
    _tls.device = int(device)
    _tls.precision = precision
    if max_batch is not None:
        _tls.max_batch = int(max_batch)


def set_worker_devices(mapping: dict, max_batch: int | None = None) -> None:
    """Map reference worker ids to GPUs, e.g. {"gpu0": 0, "gpu1": 1}: a replica
    call on the engine's thread "worker-gpu1" (workers.py:154) runs on cuda:1.
    Unmapped threads without set_worker_device use cuda:0."""
    global _DEFAULT_MAX_BATCH
    _worker_devices.clear()
    _worker_devices.update({str(k): int(v) for k, v in mapping.items()})
    if max_batch is not None:
        _DEFAULT_MAX_BATCH = int(max_batch)


def set_sole_writer(on: bool) -> None:
    """Declare that this GPU replica is the only writer of the shared host
    model (no CPU Hogwild pool, a single replica; HB_STEP_SOLE_WRITER): the
    float64 merge then runs on a device-resident copy of the model, merged
    layers are DMA'd back and later calls skip the snapshot.  Off by default,
    since the device's layer-wide read-merge-write would drop concurrent host
    updates that the reference's per-element np.add (linalg.py:79) keeps."""
    global _sole_writer
    _sole_writer = bool(on)


def _worker_id() -> str | None:
    name = threading.current_thread().name
    return name[len("worker-"):] if name.startswith("worker-") else None


def _thread_device() -> int | None:
    """Device of this thread, or None if it is not a GPU worker thread."""
    d = getattr(_tls, "device", None)
    if d is not None:
        return d
    wid = _worker_id()
    return _worker_devices.get(wid) if wid is not None else None


def _replica(sizes, rows: int, sparse: bool, purpose: str) -> GpuReplica:
    cache = getattr(_tls, "contexts", None)
    if cache is None:
        cache = _tls.contexts = {}
    device = _thread_device()
    device = 0 if device is None else device
    precision = getattr(_tls, "precision", "3xtf32")
    key = (purpose, device, sizes, sparse, precision)
    ctx = cache.get(key)
    want = max(rows, getattr(_tls, "max_batch", _DEFAULT_MAX_BATCH))
    if ctx is None or ctx.max_batch < rows:
        if ctx is not None:
            ctx.close()
        ctx = cache[key] = GpuReplica(sizes, want, device=device, sparse=sparse, precision=precision)
    return ctx


def release_thread_contexts() -> None:
    for ctx in getattr(_tls, "contexts", {}).values():
        ctx.close()
    _tls.contexts = {}


def _stage_for(ctx: GpuReplica, batch) -> None:
    """Stage the array a BatchRef views (the epoch copy) once; later batches of
    the same epoch only pass (start, length)."""
    if isinstance(batch, CsrBatchRef):
        if not ctx.is_staged(GpuReplica.key_of(batch.data)):
            ctx.stage(batch.data)
        return
    if not ctx.is_staged(GpuReplica.key_of(batch.features)):
        ctx.stage(batch.features, batch.labels)


# A dense epoch array wider than this whose sampled rows are at most this dense
# is sparse data densified by the reference loader (data.py:128-140): its
# replica stages it as CSR and runs layer 0 on the CSR kernels.
_SPARSE_DENSITY = 0.05


def _is_wide_sparse(features) -> bool:
    if features.ndim != 2 or features.shape[1] <= N_DENSIFY_MAX_DIN:
        return False
    key = GpuReplica.key_of(features)
    memo = getattr(_tls, "sparse_memo", None)
    if memo is None:
        memo = _tls.sparse_memo = {}
    if key not in memo:
        n = features.shape[0]
        rows = features[np.linspace(0, n - 1, num=min(n, 256)).astype(np.int64)]
        memo.clear()  # one epoch array at a time
        memo[key] = np.count_nonzero(rows) <= _SPARSE_DENSITY * rows.size
    return memo[key]


def execute_gpu_replica(model, batch, eta: float, speed_factor: float = 0.0) -> float:
    """GPU version of execute_batch_replica (workers.py:126-138).

    Gradient on a snapshot of the *current* shared model, then a stale merge
    of that gradient into whatever the shared model holds at merge time:
      snapshot  host float64 model -> device fp32 mirror     (deep_copy, :132)
      step      forward/backward on the device              (:133-134)
      merge     W_host -= eta * g, float64, in place         (apply_update, :135)
    Returns the update-count delta 1.0.  `speed_factor` keeps the reference's
    emulation contract (sleep speed_factor x elapsed); real devices pass 0."""
    start_t = time.perf_counter()
    sizes = layer_sizes_of(model)
    sparse = isinstance(batch, CsrBatchRef) or _is_wide_sparse(batch.features)
    ctx = _replica(sizes, batch.length, sparse, "train")
    _tls.gpu_worker = True
    _stage_for(ctx, batch)
    # snapshot, step and stale merge in one call; the shared model is
    # page-locked once and its DMAs overlap the compute layer by layer
    ctx.replica_step(model.weights, batch.start, batch.length, eta, timed=True, sole_writer=_sole_writer)
    book_device_step(batch.length, ctx.last_step_ms)
    if speed_factor > 0:
        time.sleep(speed_factor * (time.perf_counter() - start_t))
    return 1.0


# replica steps begun (execute_gpu_replica_begin) whose stale merge has not
# landed yet; the pipelined coordinator wrapper waits for zero before it
# snapshots the shared model for an evaluation (feed.pipelined)
_inflight = threading.Condition()
_inflight_n = 0


def execute_gpu_replica_begin(model, batch, eta: float) -> None:
    """First half of execute_gpu_replica: stage (once per epoch array) and
    enqueue snapshot, step and gradient copies, then return while the step
    runs.  execute_gpu_replica_end on the same thread applies the stale merge;
    nothing else may run on this thread's replica in between."""
    global _inflight_n
    sizes = layer_sizes_of(model)
    sparse = isinstance(batch, CsrBatchRef) or _is_wide_sparse(batch.features)
    ctx = _replica(sizes, batch.length, sparse, "train")
    _tls.gpu_worker = True
    _stage_for(ctx, batch)
    ctx.replica_begin(model.weights, batch.start, batch.length, eta, timed=True, sole_writer=_sole_writer)
    _tls.pending = (ctx, batch.length)
    with _inflight:
        _inflight_n += 1


def execute_gpu_replica_end() -> float:
    """Second half: the stale merge lands in the shared model; returns the
    step's device time in seconds (booked like execute_gpu_replica)."""
    global _inflight_n
    ctx, rows = _tls.pending
    _tls.pending = None
    try:
        ctx.replica_end()
    finally:
        with _inflight:
            _inflight_n -= 1
            _inflight.notify_all()
    ms = ctx.last_step_ms
    book_device_step(rows, ms)
    return ms / 1000.0


def wait_merges_landed(timeout: float | None = None) -> bool:
    """Block until every begun replica step has merged into the shared model."""
    with _inflight:
        return _inflight.wait_for(lambda: _inflight_n == 0, timeout)


def book_device_step(rows: int, ms: float) -> None:
    """Account one device-timed replica step on this thread: last / total
    device time, and the installed DeviceSpeedFeed under this thread's
    reference worker id."""
    _tls.last_device_ms = ms
    _tls.device_busy_s = getattr(_tls, "device_busy_s", 0.0) + ms / 1000.0
    feed, wid = _speed_feed, _worker_id()
    if feed is not None and wid is not None:
        feed.record(wid, rows, ms)


def last_device_ms() -> float:
    """CUDA-event time of the last replica step on this thread (controller feed)."""
    return float(getattr(_tls, "last_device_ms", 0.0))


def device_busy_seconds() -> float:
    """Sum of the device-timed replica steps run on this thread -- the GPU
    worker's busy time without queue / host latency (workers.py:207 books wall
    time; the device-timed install replaces it with this)."""
    return float(getattr(_tls, "device_busy_s", 0.0))


def gpu_loss_sum(model, features, labels, chunk: int = 4096) -> float:
    """GPU version of loss_sum (nn.py:139-146): sum over rows of
    -log max(p_y, 1e-12) of `model` on (features, labels)."""
    sizes = layer_sizes_of(model)
    if not isinstance(features, CsrDataset) and _is_wide_sparse(features):
        ctx = _replica(sizes, chunk, True, "eval")
        if not ctx.is_staged(GpuReplica.key_of(features)):
            ctx.stage(features, np.asarray(labels, dtype=np.int64))
        ctx.set_weights(model.weights)
        return ctx.eval_loss_sum(0, features.shape[0])
    if isinstance(features, CsrDataset):
        ctx = _replica(sizes, chunk, True, "eval")
        if not ctx.is_staged(GpuReplica.key_of(features)):
            ctx.stage(features)
        n = features.n_examples
    else:
        if features.ndim != 2 or features.shape[1] != sizes[0]:
            raise ValueError(f"batch shape {features.shape} incompatible with input dim {sizes[0]}")
        ctx = _replica(sizes, chunk, False, "eval")
        if not ctx.is_staged(GpuReplica.key_of(features)):
            ctx.stage(features, np.asarray(labels, dtype=np.int64))
        n = features.shape[0]
    ctx.set_weights(model.weights)
    return ctx.eval_loss_sum(0, n)


def is_gpu_thread() -> bool:
    """True on a thread that runs (or is mapped to run) GPU replica steps."""
    return getattr(_tls, "gpu_worker", False) or _thread_device() is not None


def routed_loss_sum(reference_loss_sum):
    """loss_sum for WorkerThread._evaluate (workers.py:212-222): on the GPU for
    GPU worker threads, the reference's own loss_sum everywhere else (CPU
    Hogwild workers keep their evaluation slices on the host)."""

    def loss_sum(model, features, labels):
        if is_gpu_thread():
            return gpu_loss_sum(model, features, labels)
        return reference_loss_sum(model, features, labels)

    loss_sum.reference = reference_loss_sum
    return loss_sum


def set_host_merge_threads(threads: int, spin: int = 20000) -> None:
    """Size the library's host merge pool (caller included) and its post-layer
    spin (hb_host_merge_threads): leave the cores to a CPU Hogwild pool
    sharing the process, e.g. set_host_merge_threads(2, spin=0)."""
    from . import _native as N

    N.check(N.load().hb_host_merge_threads(int(threads), int(spin)))


def install(hogtrain_module=None, devices: dict | None = None, sole_writer: bool = False, feed=None,
            cpu_pool_threads: int = 0) -> None:
    """Route the reference's BATCH_REPLICA workers to the B200 path by
    rebinding `hogtrain.workers.execute_batch_replica`, and the GPU workers'
    evaluation slices by wrapping `loss_sum`.  devices: worker id -> GPU
    (set_worker_devices); feed: a DeviceSpeedFeed that every replica step
    records its device-timed examples/s into (the coordinator's eval split,
    engine.py:335-351, can read it; see feed.device_timed); cpu_pool_threads:
    threads of a CPU Hogwild worker in the same roster, whose cores the merge
    pool then leaves alone."""
    global _speed_feed
    if cpu_pool_threads > 0:
        # the roster's CPU Hogwild pool keeps its cores: the merge pool takes
        # what is left (at least 2 threads) and never spins between layers
        import os

        set_host_merge_threads(max(2, min(12, (os.cpu_count() or 4) - int(cpu_pool_threads))), spin=0)
    if hogtrain_module is None:
        import hogtrain.workers as hogtrain_module  # noqa: F811  (reference package, if present)
    if devices is not None:
        set_worker_devices(devices)
    set_sole_writer(sole_writer)
    _speed_feed = feed
    hogtrain_module.execute_batch_replica = execute_gpu_replica
    ref = getattr(hogtrain_module.loss_sum, "reference", hogtrain_module.loss_sum)
    hogtrain_module.loss_sum = routed_loss_sum(ref)
