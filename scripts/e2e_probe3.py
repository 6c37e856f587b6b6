"""Where the fused drop-in step (hb_replica_step_host_*) spends its time."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_08771_b200 as hb
from paper_2004_08771_b200.nn import Architecture, init_model
import bench
cfgname = sys.argv[1] if len(sys.argv) > 1 else "w8a"
cfg = bench.CONFIGS[cfgname]
sizes, b = cfg["sizes"], cfg["batch"]
sparse = cfg["kind"] == "csr"
data = bench.make_data(cfg, 1)
model = init_model(Architecture(sizes), seed=1)
ctx = hb.GpuReplica(sizes, b, sparse=sparse)
if sparse:
    sub = data.rows(0, b); sub.col = sub.col.copy(); sub.labels = sub.labels.copy(); sub.val = sub.val.astype(np.float32); xb, yb = sub, None
    ctx.pin_host([sub.rowptr, sub.col, sub.val, sub.labels])
else:
    xb = data.features[:b].astype(np.float32); yb = data.labels[:b].copy(); ctx.pin_host([xb, yb])
w = [x.copy() for x in model.weights]
ctx.pin_host(w)
def t(f, n=20):
    for _ in range(3): f()
    t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e3
print(cfgname)
print("step_host (batch H2D + step)      %.3f ms" % t(lambda: ctx.step_host(xb, yb, 0.1, emit_grad=True)))
print("step_host timed device ms         %.3f" % (ctx.step_host(xb, yb, 0.1, emit_grad=True, timed=True) and ctx.last_step_ms))
print("replica_step_host (fused)         %.3f ms" % t(lambda: ctx.replica_step_host(w, xb, yb, 0.1)))
ctx.replica_step_host(w, xb, yb, 0.1, timed=True); print("replica_step_host device ms       %.3f" % ctx.last_step_ms)
print("replica_step_host sole writer     %.3f ms" % t(lambda: ctx.replica_step_host(w, xb, yb, 0.1, sole_writer=True)))
ctx.replica_step_host(w, xb, yb, 0.1, timed=True, sole_writer=True); print("  ... device ms                   %.3f" % ctx.last_step_ms)
print("  ... PCIe bytes (h2d, d2h)       %s" % (ctx.last_xfer_bytes,))
print("set_weights                       %.3f ms" % t(lambda: ctx.set_weights(w)))
print("merge_grads_into                  %.3f ms" % t(lambda: ctx.merge_grads_into(w, 0.1)))
if not sparse:
    ctx.stage(data.features[: 4 * b].astype(np.float32), data.labels[: 4 * b])
else:
    ctx.stage(data.rows(0, 4 * b))
print("step staged                       %.3f ms" % t(lambda: ctx.step(0, b, 0.1, emit_grad=True)))
print("replica_step staged               %.3f ms" % t(lambda: ctx.replica_step(w, 0, b, 0.1)))
import torch
nbytes = sum(x.nbytes for x in w)
hbuf = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory(); dbuf = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
def h2d(): dbuf.copy_(hbuf, non_blocking=True); torch.cuda.synchronize()
def d2h(): hbuf.copy_(dbuf, non_blocking=True); torch.cuda.synchronize()
th, td = t(h2d), t(d2h)
print("raw H2D %d B: %.3f ms (%.1f GB/s); D2H %.3f ms (%.1f GB/s)" % (nbytes, th, nbytes / th / 1e6, td, nbytes / td / 1e6))
