#!/usr/bin/env python
"""Benchmark of the B200 GPU replica step (Hogbatch / Adaptive Hogbatch MLP worker).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config w8a] [--impl ours|reference]

One "step" = one replica SGD step (forward, fused softmax-CE, backward, fused
SGD update) over one batch of the named BASELINE.json configuration.  The
default workload is configs[1], the w8a-shaped sparse MLP 300-512-512-512-2
at GPU batch 8192 (BASELINE.json).  N>1 (torchrun) runs one GPU worker per
rank on its own batch stream (weak scaling) and averages the replicas with
NCCL allreduce every step (the GPU-replica merge).

Prints ONE JSON line (rank 0).  `value` is device-timed throughput with the
epoch resident in HBM; `e2e` is the same metric through the drop-in replica
call (host float64 model snapshot H2D, CSR batch H2D from host memory, the
gradient D2H and float64 stale merge on the host, loss D2H) -- the exact
semantics of the reference's execute_batch_replica.  `--impl reference` times
the reference algorithm's CPU implementation (the float64 NumPy port in
oracle/, OpenBLAS on all host cores) on the same workload.
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

from paper_2004_08771_b200.parallel import barrier, batch_starts, init_process_group, init_replica_comm, max_over_ranks, shard_seed  # noqa: E402

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
    "scaled": dict(sizes=(1024, 4096, 4096, 4096, 1000), n=131072, kind="dense", classes=1000, batch=8192, eta=0.1,
                   desc="scaled synthetic dense 1024-d (131072 staged rows of the 10M-row set), "
                        "MLP 1024-4096-4096-4096-1000, GPU batch 8192"),
}


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


def make_data(cfg, seed, rank=0):
    import paper_2004_08771_b200 as hb

    s = shard_seed(seed, rank)
    if cfg["kind"] == "csr":
        return hb.synthetic_csr(cfg["n"], cfg["sizes"][0], cfg["nnz"], cfg["classes"], seed=s,
                                binary=cfg["binary"], normalize=cfg["normalize"])
    return hb.synthetic_blobs(cfg["n"], cfg["sizes"][0], cfg["classes"], 2.5, seed=s)


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
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def ncu_kernel_stats(config, kernel):
    """Per-launch ncu figures (DRAM / L2 bytes, cold-cache duration) of `kernel`
    for `config` from the newest profiles/r*_ncu_kernels.json (one `ncu --set
    full` capture per kernel, scripts/ncu_traffic.sh), or None."""
    files = sorted(ROOT.glob("profiles/r*_ncu_kernels.json"))
    if not files:
        return None, None
    d = json.loads(files[-1].read_text()).get("kernels", {})
    return d.get(config, {}).get(kernel), files[-1].name


def kernel_work(name, cfg, rows, dw_splits=None):
    """Algorithmic work of one launch of kernel `name` at `rows` batch rows:
    ("tensor", flops) for GEMMs, ("hbm", bytes) for the memory-bound kernels."""
    sizes = cfg["sizes"]
    base, _, l = name.rpartition("_l")
    l = int(l)
    if base.startswith("gemm_fwd"):
        return "tensor", 2.0 * rows * sizes[l + 1] * sizes[l]
    if base.startswith("gemm_dx"):
        return "tensor", 2.0 * rows * sizes[l + 1] * sizes[l]
    if base.startswith("gemm_dw"):
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


def run_ours(args, cfg, rank, world, local_rank, dist):
    import paper_2004_08771_b200 as hb

    # the multi-GPU code path (NCCL replica merge, max over ranks, barriers);
    # HB_BENCH_DIST=1 runs it even for one rank (a one-rank NCCL communicator)
    distributed = dist is not None
    from paper_2004_08771_b200.nn import Architecture, init_model

    device = local_rank
    sizes = cfg["sizes"]
    b = cfg["batch"]
    sparse = cfg["kind"] == "csr"
    data = make_data(cfg, args.seed, rank)
    n = data.n_examples
    model = init_model(Architecture(sizes), seed=args.seed)
    ctx = hb.GpuReplica(sizes, b, device=device, sparse=sparse, precision=args.precision)
    ctx.set_weights(model.weights)
    if sparse:
        ctx.stage(data)
    else:
        ctx.stage(data.features.astype(np.float32), data.labels)
    if distributed:
        init_replica_comm(ctx, dist, rank, world)
    starts = batch_starts(n, b, args.warmup + args.steps)

    import torch

    torch.cuda.set_device(device)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{device}")

    def l2_flush():
        flush.zero_()
        torch.cuda.synchronize(device)

    for i in range(args.warmup):
        ctx.step(starts[i], b, cfg["eta"], timed=True, merge=distributed)
    # ---------------------------------------------------------- kernel breakdown
    # A separate instrumented pass (every launch bracketed by CUDA events) gives
    # the per-kernel shares and picks the dominant kernel.  Events around every
    # launch cost ~5 us each, so the timed region below brackets only that one.
    kernels, dom = {}, None
    if not args.no_prof:
        ctx.profile(True)
        for i in range(min(args.steps, 10)):
            l2_flush()
            ctx.step(starts[args.warmup + i], b, cfg["eta"], timed=True, merge=distributed)
        prof = ctx.profile_read()
        ctx.profile(False)
        tot = sum(v[0] for v in prof.values()) or 1.0
        for name, (ms, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
            kernels[name] = {"avg_us": round(1000.0 * ms / cnt, 2), "launches": cnt, "share": round(ms / tot, 4)}
        dom = max(prof.items(), key=lambda kv: kv[1][0])[0] if prof else None
        ctx.profile_filter(dom)
        ctx.profile(True)
        for i in range(2):  # capture the singly-instrumented graph outside the timed region
            ctx.step(starts[i], b, cfg["eta"], timed=True)
        ctx.profile_read()
    # ---------------------------------------------------------- timed region
    if distributed:
        barrier(dist)
    torch.cuda.synchronize(device)
    step_ms, merge_ms, launches = [], [], 0
    with ClockSampler(device) as clocks:
        for i in range(args.warmup, args.warmup + args.steps):
            l2_flush()
            # distributed: the NCCL replica merge runs on the step's stream and
            # inside its CUDA-event bracket (HB_STEP_MERGE)
            ctx.step(starts[i], b, cfg["eta"], timed=True, merge=distributed)
            step_ms.append(ctx.last_step_ms)
            launches += ctx.last_step_launches
        torch.cuda.synchronize(device)
    if distributed:
        barrier(dist)
    dom_live = ctx.profile_read() if dom else {}
    ctx.profile(False)
    ctx.profile_filter(None)
    total_ms = sum(step_ms) + sum(merge_ms)
    if distributed:
        total_ms = max_over_ranks(dist, total_ms)
    value = world * args.steps * b / (total_ms / 1000.0)

    # ---------------------------------------------------------- e2e (drop-in replica semantics)
    e2e = None
    if not args.skip_e2e:
        # every step's batch lives in page-locked host memory (one registered
        # pool per array kind; each batch is a view into it)
        host_batches = []
        pool = []
        if sparse:
            from paper_2004_08771_b200.data import CsrDataset

            subs = [data.rows(starts[i], starts[i] + b) for i in range(args.steps)]
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
            xs = np.concatenate([data.features[starts[i]:starts[i] + b] for i in range(args.steps)]).astype(np.float32)
            ys = np.concatenate([data.labels[starts[i]:starts[i] + b] for i in range(args.steps)])
            pool = [xs, ys]
            host_batches = [(xs[i * b:(i + 1) * b], ys[i * b:(i + 1) * b]) for i in range(args.steps)]
        ctx.pin_host(pool)
        host_model = [w.copy() for w in model.weights]
        ctx.pin_host(host_model)  # what execute_gpu_replica does for the shared model
        for i in range(max(3, min(args.warmup, len(host_batches)))):  # warm the host path (and its graph)
            xb, yb = host_batches[i % len(host_batches)]
            ctx.replica_step_host(host_model, xb, yb, cfg["eta"])
        if distributed:
            barrier(dist)
        t0 = time.perf_counter()
        for i in range(args.steps):
            xb, yb = host_batches[i]
            # execute_batch_replica in one call: snapshot of the shared host model
            # (workers.py:132), batch H2D, the step, stale merge (workers.py:135), loss D2H
            ctx.replica_step_host(host_model, xb, yb, cfg["eta"], want_loss=True)
        el = time.perf_counter() - t0
        # PCIe bytes of the last call as the library issued them: batch, f64 snapshot, the merge by lane
        # (fp32 gradient D2H on the host lane, f64 rows both ways on the device lane), step record, loss
        h2d, d2h = ctx.last_xfer_bytes
        if distributed:
            el = max_over_ranks(dist, el)
        e2e = {"value": world * args.steps * b / el, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "path": "execute_gpu_replica semantics through the C ABI (hb_replica_step_host_*), per step: "
                       "batch H2D from pinned host memory (CSR rows are scattered into dense rows on the device "
                       "for narrow inputs), snapshot of the page-locked f64 host model (DMA H2D, layer l+1 in "
                       "flight while layer l computes), the step, the f64 stale merge W_host += (-eta)*g per layer as "
                       "soon as its gradient exists (fp32 gradient D2H + host float64 axpy, or on the device lane "
                       "for large split-K layers: f64 rows read, merged on the GPU, written back), loss D2H"}
    ctx.close()

    # ---------------------------------------------------------- roofline of the dominant kernel
    hbm_peak, bf16_peak, peak_src = measured_peaks()
    roofline = None
    if dom and dom in dom_live:
        ms, cnt = dom_live[dom]
        bound, work = kernel_work(dom, cfg, b)
        avg_s = ms / cnt / 1000.0
        ncu, ncu_src = ncu_kernel_stats(args.config, dom)
        traffic = None if not ncu or "dram_bytes" not in ncu else ncu["dram_bytes"]
        if bound == "tensor":
            tf32 = bf16_peak / 2.0
            peak = tf32 / (3.0 if args.precision == "3xtf32" else 1.0)
            roofline = {"bound": "tensor", "kernel": dom, "achieved": round(work / avg_s / 1e12, 2),
                        "peak": round(peak, 1), "unit": "TFLOP/s", "frac": round(work / avg_s / 1e12 / peak, 4),
                        "traffic": traffic,
                        "peak_basis": f"{'3xTF32-effective = ' if args.precision == '3xtf32' else ''}"
                                      f"TF32 dense = bf16/2 of {bf16_peak} TF/s {peak_src}",
                        "work_per_launch": work, "avg_launch_us": round(avg_s * 1e6, 2),
                        "timing": "CUDA events around this kernel only, inside the timed region"}
        else:
            roofline = {"bound": "hbm", "kernel": dom, "achieved": round(work / avg_s / 1e9, 1),
                        "peak": hbm_peak, "unit": "GB/s", "frac": round(work / avg_s / 1e9 / hbm_peak, 4),
                        "traffic": traffic, "peak_basis": peak_src, "work_per_launch": work,
                        "avg_launch_us": round(avg_s * 1e6, 2),
                        "timing": "CUDA events around this kernel only, inside the timed region"}
            if ncu and "l2_bytes" in ncu:
                # the gather kernels re-read W0^T / delta0 rows once per nonzero: their
                # real bound is the L2 -> SM gather traffic, not the unique HBM bytes
                roofline["l2"] = {"bytes_per_launch": ncu["l2_bytes"],
                                  "achieved_gbs": round(ncu["l2_bytes"] / avg_s / 1e9, 1),
                                  "ncu_l2_throughput_pct": round(ncu.get("l2_throughput_pct", 0.0), 1)}
        if roofline is not None and ncu:
            roofline["traffic_source"] = f"profiles/{ncu_src} ({args.config}/{dom}: dram read+write bytes of one launch)"
    # step-level tensor work: every GEMM of the step (dense layers; a sparse
    # first layer is gather work) against the step time -- with dX and the
    # split-K dW partials running concurrently, per-kernel event durations
    # overlap, so this is the figure that adds up
    if roofline is not None:
        gemm_flops = dense_flops_per_sample(cfg["sizes"], sparse and hb_sparse_kernels(cfg)) * b
        step_s = (sum(step_ms) / len(step_ms)) / 1000.0
        tf32 = bf16_peak / 2.0
        peak = tf32 / (3.0 if args.precision == "3xtf32" else 1.0)
        roofline["step_tensor"] = {"gemm_flop_per_step": gemm_flops,
                                   "achieved_tflops": round(gemm_flops / step_s / 1e12, 2),
                                   "frac_of_peak": round(gemm_flops / step_s / 1e12 / peak, 4),
                                   "note": "all GEMM flops of the step / whole step time (non-GEMM kernels included)"}
        if roofline.get("kernel", "").startswith(("gemm_dx", "gemm_dw_partial", "reduce_sgd")):
            roofline["overlap_note"] = ("the backward's dX GEMM and the split-K dW partial GEMM of the same layer run "
                                        "concurrently on two streams, so this kernel's event-timed duration includes "
                                        "sharing the SMs with the other; step_tensor is the figure that adds up")
    return dict(value=value, total_ms=total_ms, e2e=e2e, roofline=roofline, kernels=kernels,
                clocks=clocks.summary(), launches=launches, merge_ms=sum(merge_ms))


def cpu_reference_rate(cfg, seed, budget_s, max_steps):
    """The reference algorithm's CPU step (execute_batch_replica: deep copy,
    forward, backward, stale merge; float64 NumPy + OpenBLAS, all host cores)
    on the dense twin of the same batches -- the oracle port."""
    from oracle import ref_nn

    sizes, b = cfg["sizes"], cfg["batch"]
    data = make_data(dict(cfg, n=min(cfg["n"], 4 * b)), seed)
    w = ref_nn.init_weights(sizes, seed)
    nrow = data.n_examples

    def batch(i):
        s = (i * b) % max(1, nrow - b + 1)
        if cfg["kind"] == "csr":
            return data.dense(s, s + b), data.labels[s:s + b]
        return data.features[s:s + b], data.labels[s:s + b]

    x, y = batch(0)
    t0 = time.perf_counter()
    ref_nn.replica_step(w, x, y, cfg["eta"])  # warm-up + time estimate
    one = time.perf_counter() - t0
    rows = b
    if one * max_steps > budget_s:  # bounded sample: shrink the rows per step, same shapes otherwise
        rows = max(64, int(b * budget_s / (one * max_steps)))
    steps, t_total = 0, 0.0
    for i in range(max_steps):
        x, y = batch(i + 1)
        t0 = time.perf_counter()
        ref_nn.replica_step(w, x[:rows], y[:rows], cfg["eta"])
        t_total += time.perf_counter() - t0
        steps += 1
        if t_total > budget_s:
            break
    cores = os.cpu_count() or 1
    try:
        from threadpoolctl import threadpool_info

        blas = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        if blas:
            cores = int(blas[0])
    except Exception:
        pass
    return dict(value=steps * rows / t_total, unit=UNIT, cores=cores, kind="port",
                sample=f"{steps} replica steps x {rows} rows of the {cfg['desc']} workload "
                       f"(float64 NumPy port of workers.py:126-138, oracle/ref_nn.py)",
                seconds=round(t_total, 2))


def time_to_target(cfg, seed, epochs, device=0):
    """Time-to-target-loss (BASELINE metric): the target is the
    loss the reference algorithm reaches after `epochs` epochs of deterministic
    single-worker minibatch SGD (the float64 oracle, engine.py:175-316 with one
    replica worker); both sides are timed on the training clock (evaluation
    excluded, engine.py:158-171) on the same dataset, seed, eta and batch."""
    import paper_2004_08771_b200 as hb
    from oracle import ref_nn
    from paper_2004_08771_b200.nn import Architecture, init_model

    sizes, b, eta = cfg["sizes"], cfg["batch"], cfg["eta"]
    data = make_data(cfg, seed)
    n = data.n_examples
    dense = data.dense() if cfg["kind"] == "csr" else data.features
    labels = data.labels
    # reference (CPU) run
    w = ref_nn.init_weights(sizes, seed)
    cpu_s, curve = 0.0, [ref_nn.loss_sum(w, dense, labels) / n]
    for ep in range(epochs):
        perm = ref_nn.shuffle_epoch(n, (seed, ep))
        ex, ey = np.ascontiguousarray(dense[perm]), labels[perm]
        t0 = time.perf_counter()
        for st in range(0, n, b):
            xb, yb = ex[st:st + b], ey[st:st + b]
            ref_nn.apply_update(w, ref_nn.backward(w, ref_nn.forward(w, xb), yb), eta)
        cpu_s += time.perf_counter() - t0
        curve.append(ref_nn.loss_sum(w, dense, labels) / n)
    target = curve[-1]
    # GPU run until the target is reached (checked at epoch ends, like the reference's samples)
    model = init_model(Architecture(sizes), seed=seed)
    res = hb.train_gpu(data, model, b, eta, epochs + 2, seed, device=device, target_loss=target)
    return {"target_loss": target, "epochs": epochs, "cpu_ref_ms": round(cpu_s * 1000.0, 2),
            "gpu_ms": None if res.time_to_target_ms is None else round(res.time_to_target_ms, 3),
            "cpu_curve": [round(x, 6) for x in curve], "gpu_curve": [round(x, 6) for x in res.curve],
            "cpu_cores": os.cpu_count(),
            "note": "training clock, evaluation excluded; reference = float64 NumPy port of the reference step"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="w8a", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="3xtf32", choices=["3xtf32", "tf32"])
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--ttt-epochs", type=int, default=3, help="time-to-target epochs (0 disables)")
    ap.add_argument("--no-prof", action="store_true", help="no per-kernel events in the timed region")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    config = {"workload": cfg["desc"], "config": args.config, "arch": "-".join(map(str, cfg["sizes"])),
              "batch_per_gpu": cfg["batch"], "global_batch": cfg["batch"] * world, "precision": args.precision,
              "parallelism": f"dp{world}" + (" (NCCL replica averaging every step)" if world > 1 else ""),
              "l2": "flushed between timed steps (256 MiB write)", "data": "synthetic, resident in HBM"}

    if args.impl == "reference":
        if rank != 0:
            return
        cpu = cpu_reference_rate(cfg, args.seed, budget_s=min(120.0, 6.0 * args.steps), max_steps=args.steps)
        line = {"impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * cfg["batch"] / cpu["value"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": config,
                "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    dist = None
    if world > 1 or os.environ.get("HB_BENCH_DIST") == "1":
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        init_process_group(dist)
    res = run_ours(args, cfg, rank, world, local_rank, dist)
    if rank == 0:
        cpu = None
        if world == 1:
            cpu = cpu_reference_rate(cfg, args.seed, budget_s=args.cpu_budget_s, max_steps=10)
        ttt = None
        if world == 1 and args.ttt_epochs > 0 and cfg["n"] * cfg["sizes"][0] <= 64_000_000:
            ttt = time_to_target(cfg, args.seed, args.ttt_epochs, device=local_rank)
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["total_ms"] / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (3xTF32 tcgen05)" if args.precision == "3xtf32"
            else "f32 (TF32 tcgen05)", "data": "synthetic", "config": config,
            "e2e": res["e2e"], "roofline": res["roofline"],
            "cpu_baseline": None if cpu is None else {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "clocks": res["clocks"], "gpu_launches": res["launches"], "kernels": res["kernels"],
            "kernels_note": "per-launch CUDA events on every kernel in a separate instrumented pass "
                            "(each bracket adds ~5 us); the timed region brackets only roofline.kernel",
            "time_to_target": ttt,
        }
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
