"""Deterministic single-GPU-worker training driver (the engine's caller edge).

`train_gpu` reproduces the schedule of the reference coordinator with one
replica worker and a uniform batch size (engine.py:175-316 with
UniformHogbatch; identical to tests/helpers.py:54-74, which the reference
asserts bitwise-equal to the engine): per-epoch reshuffle seeded
(run_seed, epoch), contiguous batches over the shuffled copy with a short
tail batch (drain_tail), and a loss sample over the unshuffled dataset
before training and after every epoch, with evaluation excluded from the
training clock (engine.py:158-171, 229-236).

Because the GPU is the only writer of the model in this mode, the device
mirror stays authoritative between steps (no per-step snapshot/merge) and
the host model is written back at the end -- the per-step stale merge of
execute_gpu_replica is only needed when other workers write the host model.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

from .data import CsrDataset, epoch_shuffle_seed, shuffle_epoch
from .nn import layer_sizes_of
from .replica import GpuReplica


@dataclass
class LossSample:  # engine.py:31-35
    wall_ms: float
    epoch_fraction: float
    loss: float


@dataclass
class TrainResult:
    samples: list = field(default_factory=list)
    steps: int = 0
    examples: int = 0
    training_wall_ms: float = 0.0
    device_ms: float = 0.0
    time_to_target_ms: float | None = None

    @property
    def curve(self) -> list:
        return [s.loss for s in self.samples]

    @property
    def samples_per_s(self) -> float:
        return self.examples / (self.training_wall_ms / 1000.0) if self.training_wall_ms > 0 else 0.0


def train_gpu(dataset, model, batch_size: int, eta: float, epochs: int, seed: int, device: int = 0,
              precision: str = "3xtf32", shuffle_each_epoch: bool = True, drain_tail: bool = True,
              target_loss: float | None = None, timed_steps: bool = False) -> TrainResult:
    """Train `model` (host float64, updated in place at the end) on `dataset`
    (Dataset or CsrDataset) with one GPU replica worker."""
    sizes = layer_sizes_of(model)
    sparse = isinstance(dataset, CsrDataset)
    n = dataset.n_examples
    if dataset.class_count > sizes[-1]:
        raise ValueError(f"dataset has {dataset.class_count} classes but the model only emits {sizes[-1]}")
    b = int(batch_size)
    train_ctx = GpuReplica(sizes, min(b, n), device=device, sparse=sparse, precision=precision)
    eval_ctx = GpuReplica(sizes, min(4096, n), device=device, sparse=sparse, precision=precision)
    try:
        train_ctx.set_weights(model.weights)
        if sparse:
            eval_ctx.stage(dataset)
        else:
            eval_ctx.stage(dataset.features, dataset.labels)
        res = TrainResult()
        train_s = 0.0

        def evaluate(fraction):
            eval_ctx.set_weights(train_ctx.get_weights())
            loss = eval_ctx.eval_loss_sum(0, n) / n
            res.samples.append(LossSample(train_s * 1000.0, fraction, loss))
            if target_loss is not None and res.time_to_target_ms is None and loss <= target_loss:
                res.time_to_target_ms = train_s * 1000.0
            return loss

        evaluate(0.0)
        # the dataset is staged once; every epoch's shuffled copy is gathered
        # on the device (same rows/CSC as staging reorder(dataset, perm))
        if sparse:
            train_ctx.stage(dataset)
        else:
            train_ctx.stage(dataset.features, dataset.labels)
        shuffled = False
        for epoch in range(epochs):
            if not shuffled or shuffle_each_epoch:
                train_ctx.permute_epoch(shuffle_epoch(n, epoch_shuffle_seed(seed, epoch if shuffle_each_epoch else 0)))
                shuffled = True
            t0 = time.perf_counter()
            cursor = 0
            while cursor < n:
                length = min(b, n - cursor)
                if length < b and not drain_tail:
                    break
                train_ctx.step(cursor, length, eta, timed=timed_steps, blocking=timed_steps)
                if timed_steps:
                    res.device_ms += train_ctx.last_step_ms
                cursor += length
                res.steps += 1
                res.examples += length
            train_ctx.synchronize()
            train_s += time.perf_counter() - t0
            evaluate(float(epoch + 1))
        res.training_wall_ms = train_s * 1000.0
        train_ctx.write_weights_into(model.weights)
        return res
    finally:
        train_ctx.close()
        eval_ctx.close()
