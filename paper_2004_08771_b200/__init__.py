"""B200-native GPU replica worker for heterogeneous CPU+GPU (Adaptive) Hogbatch SGD.

The hot path of arXiv:2004.08771's GPU worker -- the large-batch synchronous
MLP step `execute_batch_replica` of the reference package `hogtrain`
(pkg/src/hogtrain/workers.py:126-138) and its loss evaluation
(nn.py:139-146) -- rebuilt as hand-written sm_100a CUDA (TMA + tcgen05/TMEM
GEMMs with fused epilogues, CSR-gather SpMM first layer) behind a C ABI
(include/hogbatch_b200.h), bound here with ctypes.

Drop-in: `execute_gpu_replica` / `gpu_loss_sum` have the reference's
signatures; `install()` rebinds them into a live `hogtrain`.
"""

from ._native import device_count, load as load_library
from .data import (
    BatchRef,
    CsrBatchRef,
    CsrDataset,
    Dataset,
    LabelMapping,
    LibsvmParseError,
    epoch_shuffle_seed,
    load_libsvm,
    load_libsvm_csr,
    reorder,
    shuffle_epoch,
    synthetic_blobs,
    synthetic_csr,
)
from .nn import Architecture, InitScheme, Model, deep_copy, init_model
from .feed import DeviceSpeedFeed, device_timed, pipelined, share_host
from .replica import GpuReplica
from .trainer import TrainResult, train_gpu
from .workers import (
    WorkerConfig,
    WorkerMode,
    execute_gpu_replica,
    execute_gpu_replica_begin,
    execute_gpu_replica_end,
    gpu_loss_sum,
    device_busy_seconds,
    install,
    last_device_ms,
    set_sole_writer,
    set_worker_device,
    set_worker_devices,
)

__all__ = [
    "Architecture", "BatchRef", "CsrBatchRef", "CsrDataset", "Dataset", "DeviceSpeedFeed", "GpuReplica",
    "InitScheme", "LabelMapping", "LibsvmParseError", "Model", "TrainResult", "WorkerConfig", "WorkerMode",
    "deep_copy", "device_busy_seconds", "device_count", "device_timed", "pipelined", "share_host", "epoch_shuffle_seed", "execute_gpu_replica", "execute_gpu_replica_begin", "execute_gpu_replica_end",
    "gpu_loss_sum", "init_model", "install", "last_device_ms", "load_libsvm", "load_libsvm_csr", "load_library",
    "reorder", "set_sole_writer", "set_worker_device", "set_worker_devices", "shuffle_epoch", "synthetic_blobs",
    "synthetic_csr", "train_gpu",
]

__version__ = "0.1.0"
