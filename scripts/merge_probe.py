"""Host-model snapshot / merge timings through the C ABI (page-locked model)."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_08771_b200 as hb
sizes = (300, 512, 512, 512, 2); b = 8192
model = hb.init_model(hb.Architecture(sizes), seed=1)
ctx = hb.GpuReplica(sizes, b, sparse=True)
data = hb.synthetic_csr(2 * b, 300, 12, 2, seed=1)
ctx.stage(data)
w = [x.copy() for x in model.weights]
ctx.pin_host(w)
ctx.step(0, b, 0.5, emit_grad=True)
for name, fn in (("set_weights", lambda: ctx.set_weights(w)), ("merge", lambda: ctx.merge_grads_into(w, 0.5))):
    for _ in range(3): fn()
    t = time.perf_counter()
    for _ in range(20): fn()
    print(f"{name:12s} {(time.perf_counter() - t) / 20 * 1e3:.3f} ms")
