"""Host-CPU Hogbatch: the reference's sharded Hogwild/Hogbatch CPU worker,
restated for timing (test / baseline infrastructure only).

`execute_hogwild_sharded` (pkg/src/hogtrain/workers.py:94-123) splits the
coordinator's batch into `threads` contiguous shards (`split_batch`,
workers.py:80-91); every shard runs forward / backward / apply_update on the
*shared* model by reference, with no lock, in a ThreadPoolExecutor.  This is
the "host-CPU Hogbatch" that BASELINE.json's metric compares against.
BASELINE.md §2 / SURVEY.md §8d fix how it is run: threads = host cores,
64 examples per thread, and one BLAS thread per worker thread
(OPENBLAS_NUM_THREADS=1; the default oversubscribes the cores ~10x).
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor, wait

import numpy as np

from . import ref_nn


def split_batch(n, parts):
    """(start, length) sub-ranges, remainder one-extra on the leading ones (workers.py:80-91)."""
    k = min(parts, n)
    base, extra = divmod(n, k)
    bounds, start = [], 0
    for i in range(k):
        length = base + (1 if i < extra else 0)
        bounds.append((start, length))
        start += length
    return bounds


def execute_hogwild_sharded(weights, x, y, threads, eta, beta=1.0, pool=None):
    """One sharded Hogbatch step on the shared `weights` (workers.py:94-123).
    Returns the update-count delta t' * beta."""
    bounds = split_batch(x.shape[0], threads)

    def shard_step(start, length):
        sx, sy = x[start:start + length], y[start:start + length]
        tape = ref_nn.forward(weights, sx)
        ref_nn.apply_update(weights, ref_nn.backward(weights, tape, sy), eta)

    if pool is None or len(bounds) == 1:
        for s, n in bounds:
            shard_step(s, n)
    else:
        futures = [pool.submit(shard_step, s, n) for s, n in bounds]
        wait(futures)
        for f in futures:
            f.result()
    return len(bounds) * beta


def _blas_single_thread():
    """threadpoolctl limit to one BLAS thread (OPENBLAS_NUM_THREADS=1 at run time)."""
    try:
        from threadpoolctl import threadpool_limits

        return threadpool_limits(limits=1, user_api="blas")
    except Exception:  # pragma: no cover - threadpoolctl is in the image
        import contextlib

        return contextlib.nullcontext()


def run_hogbatch(weights, batches, eta, budget_s, threads=None, per_thread=64, min_batches=1, on_batch=None):
    """Run Hogbatch over `batches` (an iterator of (x, y) float64/int64 arrays of
    threads*per_thread rows) until `budget_s` of training time has elapsed.
    Returns dict(samples, seconds, batches, threads).  `on_batch(i, seconds)`
    (optional) runs outside the clock after every batch (loss sampling)."""
    threads = threads or os.cpu_count() or 1
    done = samples = 0
    seconds = 0.0
    with _blas_single_thread(), ThreadPoolExecutor(max_workers=threads, thread_name_prefix="hogbatch") as pool:
        for x, y in batches:
            t0 = time.perf_counter()
            execute_hogwild_sharded(weights, x, y, threads, eta, 1.0, pool)
            seconds += time.perf_counter() - t0
            done += 1
            samples += x.shape[0]
            if on_batch is not None:
                on_batch(done, seconds)
            if seconds >= budget_s and done >= min_batches:
                break
    return {"samples": samples, "seconds": seconds, "batches": done, "threads": threads,
            "per_thread": per_thread}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def blas_info() -> list:
    try:
        from threadpoolctl import threadpool_info

        return [{k: i.get(k) for k in ("internal_api", "version", "num_threads", "architecture")}
                for i in threadpool_info() if i.get("user_api") == "blas"]
    except Exception:
        return []


__all__ = ["blas_info", "cpu_model", "execute_hogwild_sharded", "run_hogbatch", "split_batch"]
