#!/usr/bin/env python
"""Benchmark of the B200 GPU replica step (Hogbatch / Adaptive Hogbatch MLP worker).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config scaled] [--impl ours|reference]

One "step" = one replica SGD step (forward, fused softmax-CE, backward, fused
SGD update) over one batch of the named BASELINE.json configuration.  The
default workload is configs[4], the headline "1/2/4/8 B200" configuration: the
scaled synthetic dense 10M x 1024 set (every row staged in HBM, generated on
the device), MLP 1024-4096-4096-4096-1000, GPU batch 8192.  N>1 (torchrun)
runs one GPU worker per rank on its own batch stream over its own 10M/N-row
shard (weak scaling per step) and averages the replicas with NCCL allreduce
every `--merge-every` steps (the GPU-replica merge).

Prints ONE JSON line (rank 0).  `value` is device-timed throughput with the
data resident in HBM; `e2e` is the same metric through the drop-in replica
call (host float64 model snapshot H2D, batch H2D from pinned host memory, the
gradient D2H and float64 stale merge on the host, loss D2H) -- the exact
semantics of the reference's execute_batch_replica.  `cpu_baseline` is the
reference's host-CPU Hogbatch (execute_hogwild_sharded, all host cores, 64
examples per thread, one BLAS thread each) timed on this box, next to the
single-worker replica step; `time_to_target` compares training-clock time to
the loss the reference reaches.  `--impl reference` prints the host-CPU
Hogbatch line alone (the reference arm).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2004_08771_b200.parallel import (  # noqa: E402
    barrier,
    batch_starts,
    broadcast_float,
    init_process_group,
    init_replica_comm,
    init_replica_peers,
    max_over_ranks,
    shard_seed,
)

METRIC = "MLP train samples/sec"
UNIT = "samples/s"

# BASELINE.json configs
CONFIGS = {
    "covtype": dict(sizes=(54, 512, 512, 512, 2), n=581012, kind="dense", classes=2, batch=512, eta=0.5,
                    desc="covtype-shaped synthetic dense 581012x54, MLP 54-512-512-512-2, b=512"),
    "w8a": dict(sizes=(300, 512, 512, 512, 2), n=64700, kind="csr", nnz=12, binary=True, normalize=False,
                classes=2, batch=8192, eta=0.5,
                desc="w8a-shaped synthetic sparse 64700x300 (12 nnz/row, ~4%), MLP 300-512-512-512-2, GPU batch 8192"),
    "delicious": dict(sizes=(500, 1024, 1024, 983), n=16105, kind="dense", classes=983, batch=8192, eta=0.5,
                      desc="delicious-shaped synthetic dense 16105x500, 983 labels, MLP 500-1024-1024-983, GPU batch 8192"),
    "realsim": dict(sizes=(20958, 1024, 1024, 2), n=72309, kind="csr", nnz=52, binary=False, normalize=True,
                    classes=2, batch=8192, eta=0.5,
                    desc="real-sim-shaped synthetic sparse 72309x20958 (52 nnz/row), MLP 20958-1024-1024-2, GPU batch 8192"),
    "scaled": dict(sizes=(1024, 4096, 4096, 4096, 1000), n=10_000_000, kind="blobs", classes=1000, batch=8192,
                   eta=0.1, separation=2.5,
                   desc="scaled synthetic dense 10Mx1024, 1000 classes (all 10M rows staged in HBM, generated on the "
                        "device), MLP 1024-4096-4096-4096-1000, GPU batch 8192"),
}
DEFAULT_CONFIG = "scaled"


def dense_flops_per_sample(sizes, sparse_first):
    """6*sum(d_l d_{l+1}) - 2 d_0 d_1 (no dX for layer 0); the sparse first layer
    is counted as bytes instead."""
    pairs = list(zip(sizes[:-1], sizes[1:]))
    tot = sum(6 * a * b for a, b in pairs) - 2 * sizes[0] * sizes[1]
    if sparse_first:
        tot -= 4 * sizes[0] * sizes[1]  # the dense-equivalent fwd+dW of layer 0
    return tot


def hb_sparse_kernels(cfg):
    """The CSR first layer runs on the gather kernels (else it is densified on
    the device and runs as a tensor-core GEMM): paper_2004_08771_b200.replica."""
    from paper_2004_08771_b200 import _native as N

    return cfg["kind"] == "csr" and cfg["sizes"][0] > N.HB_DENSIFY_MAX_DIN


def make_data(cfg, seed, rank=0, n=None):
    """Host dataset of the config (CsrDataset or Dataset); for the device-generated
    config a small host set of the same shape (CPU-only legs)."""
    import paper_2004_08771_b200 as hb

    s = shard_seed(seed, rank)
    n = cfg["n"] if n is None else n
    if cfg["kind"] == "csr":
        return hb.synthetic_csr(n, cfg["sizes"][0], cfg["nnz"], cfg["classes"], seed=s,
                                binary=cfg["binary"], normalize=cfg["normalize"])
    if cfg["kind"] == "blobs":
        means = hb.data.blob_means(cfg["sizes"][0], cfg["classes"], cfg["separation"], seed)
        rng = np.random.default_rng(s)
        y = rng.integers(0, cfg["classes"], size=n).astype(np.int64)
        return hb.Dataset(features=means[y] + rng.normal(size=(n, cfg["sizes"][0])), labels=y, name="blobs-host")
    return hb.synthetic_blobs(n, cfg["sizes"][0], cfg["classes"], 2.5, seed=s)


class Source:
    """Where a rank's rows live: a host dataset (staged once) or rows generated
    on the device (scaled).  rows(start, k) returns the exact float64 dense rows
    and labels the device trains on (for the CPU oracle / host batches)."""

    def __init__(self, cfg, seed, rank, world, ctx=None):
        self.cfg = cfg
        self.ctx = ctx
        if cfg["kind"] == "blobs":
            self.data = None
            self.n = cfg["n"] // world
            if ctx is not None:  # one dataset (one means draw), disjoint row ranges per rank
                ctx.stage_blobs(self.n, cfg["classes"], cfg["separation"], seed, row0=rank * self.n)
        else:
            self.data = make_data(cfg, seed, rank)
            self.n = self.data.n_examples
            if ctx is not None:
                if cfg["kind"] == "csr":
                    ctx.stage(self.data)
                else:
                    ctx.stage(self.data.features.astype(np.float32), self.data.labels)

    def rows(self, start, k):
        if self.data is None:
            x, y = self.ctx.read_staged(start, k)
            return x.astype(np.float64), y
        if self.cfg["kind"] == "csr":
            return self.data.dense(start, start + k), self.data.labels[start:start + k]
        return self.data.features[start:start + k].astype(np.float32).astype(np.float64), \
            self.data.labels[start:start + k]

    def host_batch(self, start, k):
        """(batch, labels) as the host-buffer replica call takes it."""
        if self.data is None:
            return self.ctx.read_staged(start, k)
        if self.cfg["kind"] == "csr":
            return self.data.rows(start, start + k), None
        return self.data.features[start:start + k].astype(np.float32), self.data.labels[start:start + k]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    """(hbm GB/s, dense TF32 TF/s, basis): HBM from MEASURED_PEAKS.json, TF32
    from the newest profiles/r*_tf32_peak.json (scripts/tf32_peak.py: fp32
    torch.matmul with TF32 tensor cores, 8192^3), else bf16/2 (stated)."""
    hbm, bf16, src = 6650.0, 1590.0, "fallback (B200_PROFILING.md)"
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        hbm, bf16, src = d.get("hbm_gbs", hbm), d.get("bf16_tflops", bf16), "MEASURED_PEAKS.json"
    files = sorted(ROOT.glob("profiles/r*_tf32_peak.json"))
    if files:
        t = json.loads(files[-1].read_text())
        return hbm, float(t["tf32_tflops_burst"]), f"measured dense TF32 {t['tf32_tflops_burst']} TF/s " \
                                                   f"(profiles/{files[-1].name}); HBM {src}"
    return hbm, bf16 / 2.0, f"TF32 = bf16/2 of {bf16} TF/s ({src}; no TF32 measurement found)"


def pcie_bandwidth(device):
    """Pinned host<->device copy rates in GB/s (256 MiB, best of 3), or None."""
    import torch

    try:
        n = 256 * 1024 * 1024
        host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        dev = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device}")
        out = {}
        for name, (dst, src) in (("h2d_gbs", (dev, host)), ("d2h_gbs", (host, dev))):
            best = 0.0
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                dst.copy_(src, non_blocking=True)
                e1.record()
                e1.synchronize()
                best = max(best, n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
            out[name] = round(best, 1)
        del host, dev
        return out
    except Exception:  # noqa: BLE001  (reporting only)
        return None


def l2_gather_ceiling(device, rows, cols):
    """GB/s at which the device gathers pseudo-random whole rows of an
    L2-resident (rows x cols) fp32 matrix (hb_probe_l2_gather), or None."""
    import ctypes as C

    import paper_2004_08771_b200 as hb

    if cols % 128 or cols > 1024:
        return None
    lib = hb.load_library()
    best = 0.0
    for unroll in (1, 2):
        v = C.c_double(0.0)
        if lib.hb_probe_l2_gather(int(device), int(rows), int(cols), 64, unroll, C.byref(v)) == 0:
            best = max(best, v.value)
    return best or None


def ncu_kernel_stats(config, kernel):
    """Per-launch ncu figures (DRAM / L2 bytes, cold-cache duration) of `kernel`
    for `config` from the newest profiles/r*_ncu_kernels.json (one `ncu --set
    full` capture per kernel, scripts/ncu_traffic.sh), or None."""
    for f in sorted(ROOT.glob("profiles/r*_ncu_kernels.json"), reverse=True):
        hit = json.loads(f.read_text()).get("kernels", {}).get(config, {}).get(kernel)
        if hit:
            return hit, f.name
    return None, None


def kernel_work(name, cfg, rows, dw_splits=None):
    """Algorithmic work of one launch of kernel `name` at `rows` batch rows:
    ("tensor", flops) for GEMMs, ("hbm", bytes) for the memory-bound kernels."""
    sizes = cfg["sizes"]
    base, _, l = name.rpartition("_l")
    l = int(l)
    if base.startswith(("gemm_fwd", "gemm_dx", "gemm_dw")):
        return "tensor", 2.0 * rows * sizes[l + 1] * sizes[l]
    if base == "spmm_sigmoid":
        nnz = cfg.get("nnz", 0)
        # gathered W0^T rows (unique rows touched ~ d_in at these batch sizes) + CSR + output write
        return "hbm", rows * (nnz * 8.0) + min(rows * nnz, sizes[0]) * sizes[1] * 4.0 + rows * sizes[1] * 4.0
    if base == "sparse_dw_sgd":
        nnz = cfg.get("nnz", 0)
        touched = min(rows * nnz, sizes[0])
        return "hbm", rows * sizes[1] * 4.0 + rows * nnz * 8.0 + 2.0 * touched * sizes[1] * 4.0
    if base == "head_small":
        d = sizes[-2]
        return "hbm", rows * d * 4.0 * 2 + rows * 8.0
    if base == "reduce_sgd":
        return "hbm", 3.0 * sizes[l + 1] * sizes[l] * 4.0 * (dw_splits or 1)
    return "hbm", 0.0


def choose_starts(cfg, n, b, count, seed, rank):
    """Batch starts of the timed steps.  The device-generated set draws full
    batches at random offsets over its whole row range (so the timed steps
    read rows from all of HBM); the others cycle through the epoch."""
    if cfg["kind"] == "blobs":
        rng = np.random.default_rng((seed, rank, 7))
        nb = n // b
        return [int(i) * b for i in rng.choice(nb, size=count, replace=count > nb)]
    return batch_starts(n, b, count)


# ---------------------------------------------------------------------------- CPU legs (oracle/)
def cpu_replica_rate(cfg, rows_fn, budget_s, max_steps, seed):
    """The reference's single-worker replica step (execute_batch_replica, float64
    NumPy + OpenBLAS on all host cores) at the full batch size, until the budget
    is spent (at least one step)."""
    from oracle import ref_nn

    w = ref_nn.init_weights(cfg["sizes"], seed)
    b = cfg["batch"]
    steps, t_total = 0, 0.0
    for i in range(max_steps):
        x, y = rows_fn(i * b, b)
        t0 = time.perf_counter()
        ref_nn.replica_step(w, x, y, cfg["eta"])
        t_total += time.perf_counter() - t0
        steps += 1
        if t_total > budget_s:
            break
    return dict(value=steps * b / t_total, unit=UNIT, seconds=round(t_total, 2), steps=steps, rows_per_step=b,
                sample=f"{steps} replica steps x {b} rows (float64 NumPy port of workers.py:126-138, oracle/ref_nn.py, "
                       f"OpenBLAS on all host cores)")


def cpu_hogbatch_run(cfg, rows_fn, budget_s, seed, threads=None, eval_fn=None):
    """The reference's host-CPU Hogbatch (execute_hogwild_sharded, workers.py:94-123):
    batches of threads*64 rows, one shard per thread updating the shared float64
    model, one BLAS thread per worker thread.  Learning rate per shard: the
    config's eta scaled by 64/b (the reference's proportional rule,
    policies.py:34-36)."""
    from oracle import ref_hogbatch, ref_nn

    threads = threads or os.cpu_count() or 1
    per = 64
    rows = threads * per
    w = ref_nn.init_weights(cfg["sizes"], seed)
    eta = cfg["eta"] * per / cfg["batch"]

    def batches():
        i = 0
        while True:
            yield rows_fn(i * rows, rows)
            i += 1

    r = ref_hogbatch.run_hogbatch(w, batches(), eta, budget_s, threads=threads, per_thread=per)
    r["value"] = r["samples"] / r["seconds"]
    r["eta_per_shard"] = eta
    r["loss"] = eval_fn(w) if eval_fn is not None else None
    r["cpu_model"] = ref_hogbatch.cpu_model()
    return r


# ---------------------------------------------------------------------------- time to target
def time_to_target(ctx, src, cfg, args, rank, world, dist, init_w, max_rows):
    """Time-to-target-loss (BASELINE metric), step-matched:
    batches i = 0, 1, ... are the contiguous rows [i*b, (i+1)*b) of each rank's
    data (epoch 0), the loss is evaluated on a fixed held-out slice (the last E
    rows of rank 0's data) and excluded from the training clock
    (engine.py:158-171).
      * replica target: the loss the reference's deterministic single-worker
        replica step (float64 oracle) reaches after K steps, K set by the CPU
        time budget; the CPU time is those K steps.
      * Hogbatch target: the loss the reference's host-CPU Hogbatch (all host
        cores) reaches within the same budget.
    The GPU side runs the same batches through the library (N>1: every rank
    its own batches, replicas averaged every step) until the eval loss is within
    1e-5 relative of each target.  CPU work runs on rank 0 only."""
    from oracle import ref_nn

    b, eta = cfg["batch"], cfg["eta"]
    E = min(8192, src.n // 8)
    e0 = src.n - E
    budget = args.ttt_budget_s
    out = None
    if rank == 0:
        ex, ey = src.rows(e0, E)

        def eval_fn(w):
            return ref_nn.loss_sum(w, ex, ey) / E

        w = ref_nn.init_weights(cfg["sizes"], args.seed)
        cpu_curve, cpu_s, k = [eval_fn(w)], 0.0, 0
        while (k + 1) * b <= min(e0, max_rows):
            x, y = src.rows(k * b, b)
            t0 = time.perf_counter()
            ref_nn.replica_step(w, x, y, eta)
            cpu_s += time.perf_counter() - t0
            k += 1
            cpu_curve.append(eval_fn(w))
            if cpu_s >= budget:
                break
        hog = cpu_hogbatch_run(cfg, lambda s, r: src.rows(s % max(1, e0 - r), r), budget, args.seed, eval_fn=eval_fn)
        out = {"eval_rows": E, "eval_slice": [e0, src.n], "replica": {"target_loss": cpu_curve[-1], "cpu_steps": k,
               "cpu_ms": round(cpu_s * 1000.0, 1), "cpu_curve": [round(v, 7) for v in cpu_curve]},
               "hogbatch": {"target_loss": hog["loss"], "cpu_ms": round(hog["seconds"] * 1000.0, 1),
                            "cpu_samples": hog["samples"], "threads": hog["threads"], "per_thread": 64,
                            "eta_per_shard": hog["eta_per_shard"]}}
    targets = [out["replica"]["target_loss"], out["hogbatch"]["target_loss"]] if rank == 0 else [0.0, 0.0]
    cpu_k = out["replica"]["cpu_steps"] if rank == 0 else 0
    if dist is not None:
        targets = [broadcast_float(dist, t) for t in targets]
        cpu_k = int(broadcast_float(dist, float(cpu_k)))
    # GPU run (every rank), eval by rank 0 outside the clock.  The CPU legs
    # leave BLAS / pool threads spinning for a while; let them settle and
    # warm the step's graph first, so the GPU leg's clock measures the GPU
    time.sleep(0.5)
    ctx.set_weights(init_w)
    for _ in range(2):
        ctx.step(0, b, eta, timed=True)
    ctx.set_weights(init_w)
    hit = [None, None]
    gpu_curve = []
    wall_s = dev_ms = 0.0
    step = 0
    # the replica target is step-matched (the same batches); the Hogbatch
    # target may need more passes over the training rows (the CPU pool made
    # many small updates): cycle through them, up to --ttt-max-steps
    limit = max(cpu_k + 3, 4)
    n_batches = max(1, e0 // b)
    loss = ctx.eval_loss_sum(e0, E) / E if rank == 0 else 0.0
    gpu_curve.append(loss)
    while step < max(limit, args.ttt_max_steps) and (step < limit or hit[0] is not None):
        if step >= limit and hit[1] is not None:
            break
        if dist is not None:
            barrier(dist)
        t0 = time.perf_counter()
        ctx.step((step % n_batches) * b, b, eta, timed=True, merge=dist is not None)
        wall_s += time.perf_counter() - t0
        dev_ms += ctx.last_step_ms
        step += 1
        if rank == 0:
            loss = ctx.eval_loss_sum(e0, E) / E
            gpu_curve.append(loss)
        done = 0.0
        if rank == 0:
            for j, t in enumerate(targets):
                if hit[j] is None and loss <= t * (1.0 + 1e-5):
                    hit[j] = (step, wall_s * 1000.0, dev_ms)
            done = 1.0 if all(h is not None for h in hit) else 0.0
        if dist is not None:
            done = broadcast_float(dist, done)
        if done:
            break
    if dist is not None:
        wall_s = max_over_ranks(dist, wall_s)
    if rank != 0:
        return None
    for j, key in enumerate(("replica", "hogbatch")):
        h = hit[j]
        out[key].update({"gpu_steps": None if h is None else h[0], "gpu_ms": None if h is None else round(h[1], 3),
                         "gpu_device_ms": None if h is None else round(h[2], 3),
                         "speedup": None if h is None else round(out[key]["cpu_ms"] / max(h[1], 1e-9), 1)})
    out["gpu_curve"] = [round(v, 7) for v in gpu_curve]
    out["n_gpus"] = world
    out["note"] = ("training clock (evaluation excluded); replica target: step-matched batches of epoch 0; Hogbatch "
                   "target: the GPU cycles over the training rows (up to --ttt-max-steps); GPU 'reached' = eval loss "
                   "within 1e-5 relative of the target (float64 vs the device's fp32 model); N>1: replicas averaged "
                   "every step, eval on rank 0")
    out["gpu_curve"] = out["gpu_curve"][:64]
    return out


# ---------------------------------------------------------------------------- our arm
def run_ours(args, cfg, rank, world, local_rank, dist):
    import torch

    import paper_2004_08771_b200 as hb
    from paper_2004_08771_b200.nn import Architecture, init_model

    distributed = dist is not None
    # HB_BENCH_SAME_DEVICE=1: every rank on cuda:0 (exercises the multi-rank
    # path, e.g. the CUDA-IPC peer merge, on a one-GPU box; not a bench number)
    device = 0 if os.environ.get("HB_BENCH_SAME_DEVICE") == "1" else local_rank
    sizes = cfg["sizes"]
    b = cfg["batch"]
    sparse = cfg["kind"] == "csr"
    torch.cuda.set_device(device)
    model = init_model(Architecture(sizes), seed=args.seed)
    ctx = hb.GpuReplica(sizes, b, device=device, sparse=sparse, precision=args.precision)
    ctx.set_weights(model.weights)
    t0 = time.perf_counter()
    src = Source(cfg, args.seed, rank, world, ctx)
    stage_s = time.perf_counter() - t0
    n = src.n
    comm = None
    if distributed:
        if args.transport == "peer":
            init_replica_peers(ctx, dist, rank, world)
            comm = {"nranks": world, "rank": rank,
                    "backend": "peer memory (hb_peer_attach: CUDA IPC exchange buffers, one-shot reduce kernel)"}
        else:
            init_replica_comm(ctx, dist, rank, world)
            comm = {"nranks": world, "rank": rank, "backend": "NCCL (library communicator, hb_comm_init)"}
        print(f"[bench] rank {rank}/{world}: {comm['backend']} up on cuda:{device}", file=sys.stderr)
    starts = choose_starts(cfg, n, b, args.warmup + args.steps, args.seed, rank)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{device}")

    def l2_flush():
        flush.zero_()
        torch.cuda.synchronize(device)

    def merge_due(i):
        return distributed and (i + 1) % args.merge_every == 0

    for i in range(args.warmup):
        ctx.step(starts[i], b, cfg["eta"], timed=True, merge=merge_due(i))
    # ---------------------------------------------------------- kernel breakdown
    # A separate instrumented pass (every launch bracketed by CUDA events) gives
    # the per-kernel shares and picks the dominant kernel.  Events around every
    # launch cost ~5 us each, so the timed region below brackets only that one.
    kernels, dom = {}, None
    if not args.no_prof:
        ctx.profile(True)
        for i in range(min(args.steps, 10)):
            l2_flush()
            ctx.step(starts[args.warmup + i], b, cfg["eta"], timed=True, merge=merge_due(i))
        prof = ctx.profile_read()
        ctx.profile(False)
        tot = sum(v[0] for v in prof.values()) or 1.0
        for name, (ms, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
            kernels[name] = {"avg_us": round(1000.0 * ms / cnt, 2), "launches": cnt, "share": round(ms / tot, 4)}
        dom = max(prof.items(), key=lambda kv: kv[1][0])[0] if prof else None
        ctx.profile_filter(dom)
        ctx.profile(True)
        for i in range(2):  # capture the singly-instrumented graph outside the timed region
            ctx.step(starts[i], b, cfg["eta"], timed=True, merge=merge_due(i))
        ctx.profile_read()
    # ---------------------------------------------------------- timed region
    if distributed:
        barrier(dist)
    torch.cuda.synchronize(device)
    step_ms, launches = [], 0
    with ClockSampler(device) as clocks:
        for i in range(args.warmup, args.warmup + args.steps):
            l2_flush()
            # distributed: the NCCL replica merge runs on the step's stream and
            # inside its CUDA-event bracket (HB_STEP_MERGE)
            ctx.step(starts[i], b, cfg["eta"], timed=True, merge=merge_due(i))
            step_ms.append(ctx.last_step_ms)
            launches += ctx.last_step_launches
        torch.cuda.synchronize(device)
    if distributed:
        barrier(dist)
    dom_live = ctx.profile_read() if dom else {}
    ctx.profile(False)
    ctx.profile_filter(None)
    total_ms = sum(step_ms)
    if distributed:
        total_ms = max_over_ranks(dist, total_ms)
    value = world * args.steps * b / (total_ms / 1000.0)

    # ---------------------------------------------------------- e2e (drop-in replica semantics)
    e2e = None
    if not args.skip_e2e:
        host_batches = []
        pool = []
        tstarts = starts[args.warmup:args.warmup + args.steps]
        if sparse:
            from paper_2004_08771_b200.data import CsrDataset

            subs = [src.data.rows(s, s + b) for s in tstarts]
            rp = np.concatenate([x.rowptr for x in subs])
            cl = np.concatenate([x.col for x in subs])
            vl = np.concatenate([x.val for x in subs]).astype(np.float32)
            lb = np.concatenate([x.labels for x in subs])
            pool = [rp, cl, vl, lb]
            o_rp = o_nz = 0
            for i, x in enumerate(subs):
                sub = CsrDataset.__new__(CsrDataset)  # views into the pinned pools, no copies
                sub.rowptr, sub.col = rp[o_rp:o_rp + b + 1], cl[o_nz:o_nz + x.nnz]
                sub.val, sub.labels = vl[o_nz:o_nz + x.nnz], lb[i * b:(i + 1) * b]
                sub.n_cols, sub.name = x.n_cols, x.name
                host_batches.append((sub, None))
                o_rp += b + 1
                o_nz += x.nnz
        else:
            parts = [src.host_batch(s, b) for s in tstarts]
            xs = np.concatenate([p[0] for p in parts])
            ys = np.concatenate([p[1] for p in parts])
            pool = [xs, ys]
            host_batches = [(xs[i * b:(i + 1) * b], ys[i * b:(i + 1) * b]) for i in range(len(parts))]
        ctx.pin_host(pool)
        host_model = [w.copy() for w in model.weights]
        ctx.pin_host(host_model)  # what execute_gpu_replica does for the shared model
        for i in range(max(3, min(args.warmup, len(host_batches)))):  # warm the host path (and its graph)
            xb, yb = host_batches[i % len(host_batches)]
            ctx.replica_step_host(host_model, xb, yb, cfg["eta"], sole_writer=True)
        def e2e_run(land_async):
            if distributed:
                barrier(dist)
            t0 = time.perf_counter()
            for i in range(args.steps):
                xb, yb = host_batches[i]
                # execute_batch_replica in one call: snapshot of the shared host model
                # (workers.py:132), batch H2D, the step, stale merge (workers.py:135), loss D2H
                # (a lone GPU replica is the host model's only writer: HB_STEP_SOLE_WRITER)
                ctx.replica_step_host(host_model, xb, yb, cfg["eta"], want_loss=True, sole_writer=True,
                                      land_async=land_async)
            ctx.landed()  # every step's merge is in the host model before the clock stops
            el = time.perf_counter() - t0
            return max_over_ranks(dist, el) if distributed else el

        el_seq = e2e_run(False)
        # PCIe bytes of the last call as the library issued them
        h2d, d2h = ctx.last_xfer_bytes
        el = e2e_run(True) if args.e2e_mode == "deferred" else el_seq
        e2e = {"value": world * args.steps * b / el, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "mode": args.e2e_mode,
               "path": "execute_gpu_replica semantics through the C ABI (hb_replica_step_host_*), per step: "
                       "batch H2D from pinned host memory, snapshot of the page-locked f64 host model (skipped while "
                       "the device-resident f64 mirror is current: the replica is the model's sole writer here), the "
                       "step, the f64 stale merge W_host += (-eta)*g per layer as soon as its gradient exists (run on "
                       "the device mirror, merged layers DMA'd back), loss D2H; the clock stops after hb_replica_landed "
                       "(every merge in the host model)" + (
                           ". deferred (HB_STEP_LAND_ASYNC): a call returns once its step and loss are done and its "
                           "write-backs land while the next call's batch copy and forward run" if args.e2e_mode ==
                           "deferred" else ""),
               "sequential": {"value": world * args.steps * b / el_seq, "unit": UNIT,
                              "note": "each call returns after its merge is in the host model (execute_batch_replica "
                                      "order, workers.py:126-138)"}}
        # PCIe roofline of the drop-in call: its bytes at the link's measured copy rate
        bw = pcie_bandwidth(device)
        if bw:
            t_link = max(h2d / (bw["h2d_gbs"] * 1e9), d2h / (bw["d2h_gbs"] * 1e9))
            e2e["pcie"] = {**bw, "link_bound_samples_s": round(world * b / t_link, 1),
                           "frac": round((world * args.steps * b / el) / (world * b / t_link), 4),
                           "note": "max(H2D, D2H bytes per step) at pinned cudaMemcpy rates (256 MiB, best of 3): "
                                   "the e2e ceiling the call's PCIe traffic allows, before any compute"}

    # ---------------------------------------------------------- CPU baselines (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        hog = cpu_hogbatch_run(cfg, lambda s, r: src.rows(s % max(1, n - r), r), args.cpu_budget_s, args.seed)
        rep = cpu_replica_rate(cfg, lambda s, r: src.rows(s % max(1, n - r), r), args.cpu_budget_s, 10, args.seed)
        from oracle import ref_hogbatch

        cpu = {"value": hog["value"], "unit": UNIT, "cores": hog["threads"], "kind": "port",
               "sample": f"host-CPU Hogbatch (execute_hogwild_sharded, workers.py:94-123; oracle/ref_hogbatch.py): "
                         f"{hog['batches']} batches x {hog['threads']} threads x 64 rows, one BLAS thread per thread, "
                         f"{hog['seconds']:.1f} s",
               "cpu_model": hog["cpu_model"], "blas": ref_hogbatch.blas_info(),
               "replica_step": {"value": rep["value"], "unit": UNIT, "sample": rep["sample"],
                                "seconds": rep["seconds"]}}

    # ---------------------------------------------------------- time to target
    # GPU loss evaluation (loss_sum, nn.py:139-146): the forward
    # plus the CE epilogue over staged rows, excluded from the training clock
    ev = None
    if rank == 0:
        er = min(n, 16 * b)
        ctx.eval_loss_sum(0, er)
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        for _ in range(3):
            ctx.eval_loss_sum(0, er)
        ev_s = (time.perf_counter() - t0) / 3
        ev = {"rows": er, "samples_s": round(er / ev_s, 1), "ms": round(ev_s * 1000.0, 3),
              "note": "hb_eval_loss_sum over staged rows in chunks of the context's max batch, host wall time"}
    ttt = None
    if args.ttt:
        ttt = time_to_target(ctx, src, cfg, args, rank, world, dist, model.weights, max_rows=n)
    ctx.close()

    # ---------------------------------------------------------- roofline of the dominant kernel
    hbm_peak, tf32_peak, peak_src = measured_peaks()
    roofline = None
    if dom and dom in dom_live:
        ms, cnt = dom_live[dom]
        bound, work = kernel_work(dom, cfg, b)
        avg_s = ms / cnt / 1000.0
        ncu, ncu_src = ncu_kernel_stats(args.config, dom)
        traffic = None if not ncu or "dram_bytes" not in ncu else ncu["dram_bytes"]
        if bound == "tensor":
            peak = tf32_peak / (3.0 if args.precision == "3xtf32" else 1.0)
            roofline = {"bound": "tensor", "kernel": dom, "achieved": round(work / avg_s / 1e12, 2),
                        "peak": round(peak, 1), "unit": "TFLOP/s", "frac": round(work / avg_s / 1e12 / peak, 4),
                        "traffic": traffic,
                        "peak_basis": ("3xTF32-effective = dense TF32 / 3; " if args.precision == "3xtf32" else "")
                        + peak_src,
                        "work_per_launch": work, "avg_launch_us": round(avg_s * 1e6, 2),
                        "raw_tf32_issue_frac": round(work * (3 if args.precision == "3xtf32" else 1) / avg_s / 1e12
                                                     / tf32_peak, 4),
                        "timing": "CUDA events around this kernel only, inside the timed region"}
        else:
            roofline = {"bound": "hbm", "kernel": dom, "achieved": round(work / avg_s / 1e9, 1),
                        "peak": hbm_peak, "unit": "GB/s", "frac": round(work / avg_s / 1e9 / hbm_peak, 4),
                        "traffic": traffic, "peak_basis": peak_src, "work_per_launch": work,
                        "avg_launch_us": round(avg_s * 1e6, 2),
                        "timing": "CUDA events around this kernel only, inside the timed region"}
            if dom.startswith(("spmm_sigmoid", "sparse_dw_sgd")):
                # the CSR kernels are L2-gather bound: one d1-wide row per nonzero,
                # against the gather ceiling measured live (hb_probe_l2_gather)
                gathered = b * cfg.get("nnz", 0) * sizes[1] * 4.0
                ceil = l2_gather_ceiling(device, sizes[0], sizes[1])
                roofline["l2"] = {"gathered_bytes_per_launch": gathered,
                                  "achieved_gbs": round(gathered / avg_s / 1e9, 1),
                                  "ceiling_gbs": None if ceil is None else round(ceil, 1),
                                  "frac": None if not ceil else round(gathered / avg_s / 1e9 / ceil, 4),
                                  "ceiling_basis": "hb_probe_l2_gather: pseudo-random whole rows of an L2-resident "
                                                   f"({sizes[0]} x {sizes[1]}) fp32 matrix, 64 warps/SM"}
                if ncu and "l2_bytes" in ncu:
                    roofline["l2"].update({"ncu_l2_bytes_per_launch": ncu["l2_bytes"],
                                           "ncu_l2_throughput_pct": round(ncu.get("l2_throughput_pct", 0.0), 1)})
        if roofline is not None and ncu:
            roofline["traffic_source"] = f"profiles/{ncu_src} ({args.config}/{dom}: dram read+write bytes of one launch)"
    # step-level tensor work: every GEMM of the step against the step time
    if roofline is not None:
        gemm_flops = dense_flops_per_sample(cfg["sizes"], sparse and hb_sparse_kernels(cfg)) * b
        step_s = (sum(step_ms) / len(step_ms)) / 1000.0
        peak = tf32_peak / (3.0 if args.precision == "3xtf32" else 1.0)
        roofline["step_tensor"] = {"gemm_flop_per_step": gemm_flops,
                                   "achieved_tflops": round(gemm_flops / step_s / 1e12, 2),
                                   "frac_of_peak": round(gemm_flops / step_s / 1e12 / peak, 4),
                                   "note": "all GEMM flops of the step / whole step time (non-GEMM kernels included)"}
        if roofline.get("kernel", "").startswith(("gemm_dx", "gemm_dw_partial", "reduce_sgd")):
            roofline["overlap_note"] = ("the backward's dX GEMM and the split-K dW partial GEMM of the same layer run "
                                        "concurrently on two streams, so this kernel's event-timed duration includes "
                                        "sharing the SMs with the other; step_tensor is the figure that adds up")
    return dict(value=value, total_ms=total_ms, e2e=e2e, roofline=roofline, kernels=kernels, clocks=clocks.summary(),
                launches=launches, cpu=cpu, ttt=ttt, comm=comm, stage_s=stage_s, rows_staged=n, eval=ev)


def config_block(args, cfg, world):
    return {"workload": cfg["desc"], "config": args.config, "arch": "-".join(map(str, cfg["sizes"])),
            "batch_per_gpu": cfg["batch"], "global_batch": cfg["batch"] * world, "precision": args.precision,
            "rows": cfg["n"], "rows_per_gpu": cfg["n"] // world if cfg["kind"] == "blobs" else cfg["n"],
            "parallelism": f"dp{world}" + (f" ({"peer-memory" if args.transport == "peer" else "NCCL"} replica averaging every {args.merge_every} step(s))"
                                           if world > 1 else ""),
            "l2": "flushed between timed steps (256 MiB write)", "data": "synthetic, resident in HBM"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="3xtf32", choices=["3xtf32", "tf32"])
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--merge-every", type=int, default=1, help="replica averaging cadence (N>1)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer"],
                    help="replica averaging over NCCL or over peer memory (CUDA IPC, hb_peer_attach)")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--e2e-mode", choices=["deferred", "sequential"], default="deferred",
                    help="e2e calls land their host-model write-backs in the background (HB_STEP_LAND_ASYNC) "
                         "or before returning")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--ttt-budget-s", type=float, default=20.0, help="CPU time budget of the time-to-target legs")
    ap.add_argument("--no-ttt", dest="ttt", action="store_false")
    ap.add_argument("--ttt-max-steps", type=int, default=256, help="GPU step cap of the Hogbatch time-to-target leg")
    ap.add_argument("--no-prof", action="store_true", help="no per-kernel events in the timed region")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.merge_every < 1:
        ap.error("--merge-every must be >= 1")
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        # the reference arm: host-CPU Hogbatch on this box's cores (rank 0 only)
        if rank != 0:
            return
        src = Source(cfg, args.seed, 0, 1, None) if cfg["kind"] != "blobs" else None
        host = make_data(cfg, args.seed, 0, n=min(cfg["n"], 65536)) if src is None else None

        def rows_fn(s, r):
            if src is not None:
                return src.rows(s % max(1, src.n - r), r)
            s = s % max(1, host.n_examples - r)
            return host.features[s:s + r], host.labels[s:s + r]

        budget = min(120.0, max(10.0, 3.0 * args.steps))
        hog = cpu_hogbatch_run(cfg, rows_fn, budget, args.seed)
        from oracle import ref_hogbatch

        line = {"impl": "reference", "metric": METRIC, "value": hog["value"], "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * hog["seconds"] / hog["batches"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": config_block(args, cfg, 1),
                "cpu_baseline": {"value": hog["value"], "unit": UNIT, "cores": hog["threads"], "kind": "port",
                                 "sample": f"host-CPU Hogbatch (execute_hogwild_sharded, workers.py:94-123; "
                                           f"oracle/ref_hogbatch.py): {hog['batches']} batches x {hog['threads']} "
                                           f"threads x 64 rows, one BLAS thread per thread, {hog['seconds']:.1f} s",
                                 "cpu_model": hog["cpu_model"], "blas": ref_hogbatch.blas_info()},
                "e2e": {"value": hog["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "note": "step = one coordinator batch of threads x 64 rows; the reference is pure Python/NumPy and "
                        "cannot travel to the GPU box, so this is its float64 restatement (oracle/, pinned to the "
                        "reference's golden vectors)"}
        print(json.dumps(line))
        return

    dist = None
    if world > 1 or os.environ.get("HB_BENCH_DIST") == "1":
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(0 if os.environ.get("HB_BENCH_SAME_DEVICE") == "1" else local_rank)
        init_process_group(dist)
    res = run_ours(args, cfg, rank, world, local_rank, dist)
    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["total_ms"] / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (3xTF32 tcgen05)" if args.precision == "3xtf32"
            else "f32 (TF32 tcgen05)", "data": "synthetic", "config": config_block(args, cfg, world),
            "e2e": res["e2e"], "roofline": res["roofline"], "cpu_baseline": res["cpu"],
            "clocks": res["clocks"], "gpu_launches": res["launches"], "kernels": res["kernels"],
            "kernels_note": "per-launch CUDA events on every kernel in a separate instrumented pass "
                            "(each bracket adds ~5 us); the timed region brackets only roofline.kernel",
            "time_to_target": res["ttt"], "eval": res["eval"], "comm": res["comm"],
            "staging": {"rows_per_gpu": res["rows_staged"], "seconds": round(res["stage_s"], 2)},
        }
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
