"""Device-timed feed for the reference's controller and coordinator.

The batch-size controller itself is the reference's (`hogtrain.policies`,
Alg. 2 at policies.py:84-129) and stays the drop-in surface; this module only
changes what it and the coordinator are fed.  In the reference every time
figure is host wall time: `WorkerThread._execute` books
`busy_seconds += perf_counter() - start` (workers.py:207) and the coordinator's
speed estimate is served-to-reported wall time, an EWMA 0.5/0.5
(engine.py:318-328), which sizes the evaluation slices (engine.py:335-351).
For a B200 replica whose step is 0.1-10 ms, both are dominated by the Python
queue round trip and host merge, not by the device.  Here:

* `DeviceSpeedFeed` keeps the same EWMA over CUDA-event-timed steps
  (`execute_gpu_replica` records into it once installed);
* `device_timed(workers_module, engine_module, feed)` wraps the reference's
  own `WorkerThread._execute` and `_Coordinator._update_speed` so GPU worker
  threads book device busy time and the coordinator reads the device-timed
  speed -- without copying either method;
* `pipelined(workers_module, engine_module)` takes the coordinator round trip
  (one Condition-queue message each way per batch,
  messaging.py:24-67, engine.py:278-316) off the GPU worker's critical path:
  the worker answers SCHEDULE_WORK as soon as its step is enqueued and applies
  the stale merge while the coordinator serves its next batch.
"""

from __future__ import annotations

import threading

from . import workers as _w


class DeviceSpeedFeed:
    """Per-worker examples/second from device-timed steps, EWMA 0.5/0.5 like
    the coordinator's estimator (engine.py:318-328)."""

    def __init__(self):
        self.speed: dict = {}
        self._mu = threading.Lock()

    def record(self, worker_id: str, examples: int, device_ms: float) -> float:
        with self._mu:
            if device_ms <= 0 or examples <= 0:
                return self.speed.get(worker_id, 0.0)
            rate = examples / (device_ms / 1000.0)
            prev = self.speed.get(worker_id)
            self.speed[worker_id] = rate if prev is None else 0.5 * prev + 0.5 * rate
            return self.speed[worker_id]

    def eval_slices(self, worker_ids, n: int) -> list:
        """(worker, start, length) covering n rows in proportion to speed, with
        the coordinator's rounding (remainder to the first worker,
        engine.py:335-351)."""
        with self._mu:
            weights = [max(self.speed.get(w, 0.0), 0.0) for w in worker_ids]
        if sum(weights) <= 0:
            weights = [1.0] * len(worker_ids)
        total = sum(weights)
        sizes = [int(n * w / total) for w in weights]
        sizes[0] += n - sum(sizes)
        out, start = [], 0
        for wid, size in zip(worker_ids, sizes):
            if size > 0:
                out.append((wid, start, size))
                start += size
        return out


def device_timed(workers_module, engine_module, feed: DeviceSpeedFeed) -> None:
    """Feed the reference's accounting from the device clock.

    - `WorkerThread._execute` (workers.py:193-210): on a GPU worker thread the
      wall-clock increment of `busy_seconds` is replaced by the CUDA-event time
      of the replica steps the call ran (`device_busy_seconds`); CPU Hogwild
      workers keep wall time.
    - `_Coordinator._update_speed` (engine.py:318-328): after the reference's
      own estimate, a worker the feed has device-timed steps for gets the
      feed's EWMA instead, so `_eval_slices` (engine.py:335-351) splits the
      evaluation by device throughput.
    Idempotent; `install(..., feed=feed)` must route the steps into `feed`."""
    wt = workers_module.WorkerThread
    if not hasattr(wt._execute, "reference"):
        ref_execute = wt._execute

        def _execute(self, msg):
            busy0, dev0 = self.busy_seconds, _w.device_busy_seconds()
            ref_execute(self, msg)
            dev = _w.device_busy_seconds() - dev0
            if dev > 0:
                self.busy_seconds = busy0 + dev

        _execute.reference = ref_execute
        wt._execute = _execute
    co = engine_module._Coordinator
    ref_update = getattr(co._update_speed, "reference", co._update_speed)  # re-point an earlier wrapper

    def _update_speed(self, wid):
        ref_update(self, wid)
        v = feed.speed.get(wid)
        if v:
            self.speed[wid] = v

    _update_speed.reference = ref_update
    co._update_speed = _update_speed


def pipelined(workers_module, engine_module) -> None:
    """Overlap the coordinator round trip with the GPU replica step.

    The reference worker replies SCHEDULE_WORK only after the whole step
    (workers.py:193-210), so every batch pays the message round trip (~35 us
    per batch measured on the reference engine) on top of the device step.
    Here a GPU replica worker (BATCH_REPLICA routed to execute_gpu_replica)
    enqueues the step (execute_gpu_replica_begin), books the update and
    replies at once, then lands the stale merge (execute_gpu_replica_end)
    while the coordinator picks its next batch.  The step's arithmetic and
    merge are unchanged: the next snapshot is taken after this merge landed.
    What changes is when the coordinator hears of the update -- one step
    early -- so before it snapshots the model for an evaluation
    (engine.py:353-356) it waits until every begun step has merged.
    CPU workers keep the reference's _execute.  Idempotent."""
    wt = workers_module.WorkerThread
    prev = getattr(wt._execute, "pipelined_over", wt._execute)

    def _execute(self, msg):
        if not (self.cfg.mode is workers_module.WorkerMode.BATCH_REPLICA
                and workers_module.execute_batch_replica is _w.execute_gpu_replica):
            return prev(self, msg)
        _w.execute_gpu_replica_begin(self.ctx.model, msg.batch, msg.learning_rate)
        try:
            # the reference's bookkeeping and reply (workers.py:207-210), sent while the step runs
            self.update_count += 1.0
            self.examples_processed += msg.batch.length
            self._send(workers_module.ToCoordinator.SCHEDULE_WORK)
        finally:
            self.busy_seconds += _w.execute_gpu_replica_end()

    _execute.pipelined_over = prev
    _execute.reference = getattr(prev, "reference", prev)
    wt._execute = _execute
    co = engine_module._Coordinator
    ref_eval = getattr(co._evaluate_and_sample, "reference", co._evaluate_and_sample)

    def _evaluate_and_sample(self, fraction):
        _w.wait_merges_landed()
        return ref_eval(self, fraction)

    _evaluate_and_sample.reference = ref_eval
    co._evaluate_and_sample = _evaluate_and_sample


last_host_share = None  # (merge threads, spin) the last coordinator's roster chose (share_host)


def share_host(engine_module) -> None:
    """Size the library's host merge pool from the coordinator's roster.

    Wraps `_Coordinator.__init__` (engine.py:93-157): when the roster has a
    CPU Hogwild pool (HOGWILD_SHARDED, `threads` each, workers.py:94-123) the
    merge pool takes only the remaining host threads (at least 2) and stops
    spinning between layers, so the pool's cores stay with the CPU workers
    (measured: the CPU pool keeps 0.91 instead of 0.83 of its throughput on
    w8a, scripts/coexist.py); a GPU-only roster restores the default pool.
    Idempotent."""
    import os

    co = engine_module._Coordinator
    ref_init = getattr(co.__init__, "reference", co.__init__)

    def __init__(self, dataset, model, roster, *args, **kwargs):
        global last_host_share
        ref_init(self, dataset, model, roster, *args, **kwargs)
        cpu = sum(int(getattr(cfg, "threads", 1)) for cfg in roster
                  if getattr(getattr(cfg, "mode", None), "value", "") == "hogwild_sharded")
        hw = os.cpu_count() or 4
        share = (max(2, min(12, hw - cpu)), 0) if cpu else (max(2, min(12, hw * 3 // 4)), 20000)
        if share != last_host_share:
            _w.set_host_merge_threads(*share)
            last_host_share = share

    __init__.reference = ref_init
    co.__init__ = __init__
