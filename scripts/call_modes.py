"""Per-call wall time of the drop-in replica call in its modes (sequential /
deferred landing, with and without the loss read) against the bare device
step, to locate the host-side cost of the e2e leg:
    python scripts/call_modes.py [config] [calls]"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2004_08771_b200 as hb  # noqa: E402
from paper_2004_08771_b200.nn import Architecture, init_model  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "covtype"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = bench.CONFIGS[name]
sizes, b = cfg["sizes"], cfg["batch"]
rng = np.random.default_rng(0)
xb = rng.standard_normal((b, sizes[0]), dtype=np.float32)
yb = rng.integers(0, sizes[-1], b).astype(np.int64)
w = [x.copy() for x in init_model(Architecture(sizes), seed=1).weights]
ctx = hb.GpuReplica(sizes, b)
ctx.pin_host([xb, yb])
ctx.pin_host(w)


def per_call(f):
    for _ in range(10):
        f()
    ctx.landed()
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(calls):
        f()
    ctx.landed()
    ctx.synchronize()
    return 1e6 * (time.perf_counter() - t0) / calls


res = {
    "replica seq +loss": per_call(lambda: ctx.replica_step_host(w, xb, yb, 1e-3, want_loss=True, sole_writer=True)),
    "replica deferred +loss": per_call(lambda: ctx.replica_step_host(w, xb, yb, 1e-3, want_loss=True, sole_writer=True,
                                                                      land_async=True)),
    "replica deferred": per_call(lambda: ctx.replica_step_host(w, xb, yb, 1e-3, want_loss=False, sole_writer=True,
                                                                land_async=True)),
    "replica shared +loss": per_call(lambda: ctx.replica_step_host(w, xb, yb, 1e-3, want_loss=True)),
    "step_host +loss (no exchange)": per_call(lambda: ctx.step_host(xb, yb, 1e-3)),
}
ctx.stage(xb, yb)
res["staged step +loss"] = per_call(lambda: ctx.step(0, b, 1e-3, want_loss=True))
res["staged step timed"] = per_call(lambda: ctx.step(0, b, 1e-3, timed=True))
res["device ms (last timed)"] = ctx.last_step_ms * 1e3
for k, v in res.items():
    print(f"{name:8s} {k:32s} {v:8.1f} us")
ctx.close()
