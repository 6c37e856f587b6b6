"""Where the drop-in (replica-semantics) e2e step spends its time."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_08771_b200 as hb
from paper_2004_08771_b200.nn import Architecture, init_model
sizes = (300, 512, 512, 512, 2); b = 8192
data = hb.synthetic_csr(64700, 300, 12, 2, seed=1)
model = init_model(Architecture(sizes), seed=1)
ctx = hb.GpuReplica(sizes, b, sparse=True)
batches = []
for i in range(7):
    sub = data.rows(i * b, (i + 1) * b); sub.val = sub.val.astype(np.float32); batches.append(sub)
w = [x.copy() for x in model.weights]
ctx.pin_host(w)
T = {"set_weights": 0, "step_host": 0, "merge": 0}
for it in range(12):
    t0 = time.perf_counter(); ctx.set_weights(w); t1 = time.perf_counter()
    ctx.step_host(batches[it % 7], None, 0.5, emit_grad=True, want_loss=True); t2 = time.perf_counter()
    ctx.merge_grads_into(w, 0.5); t3 = time.perf_counter()
    if it >= 2:
        T["set_weights"] += t1 - t0; T["step_host"] += t2 - t1; T["merge"] += t3 - t2
for k, v in T.items(): print(f"{k:12s} {v / 10 * 1000:.3f} ms")
# device-only step for reference
ctx.stage(data)
for i in range(3): ctx.step(0, b, 0.5)
t0 = time.perf_counter()
for i in range(10): ctx.step((i % 7) * b, b, 0.5, blocking=False)
ctx.synchronize(); print(f"device step  {(time.perf_counter() - t0) / 10 * 1000:.3f} ms")
