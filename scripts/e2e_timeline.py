"""Device timeline of the drop-in call with host buffers (bench.py's e2e leg):
    HB_DEBUG_XCHG=1 HB_NO_GRAPHS=1 python scripts/e2e_timeline.py [config] [calls]
prints the exchange's stream events of each call (relative to its first event)
and the wall time per call; without the env vars it only times the calls.
Also times raw pinned D2H into the registered float64 model vs a torch pinned
buffer of the same size (is the registered model as fast a DMA target?)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2004_08771_b200 as hb  # noqa: E402
from paper_2004_08771_b200.nn import Architecture, init_model  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "scaled"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 4
defer = len(sys.argv) > 3 and sys.argv[3] == "defer"  # HB_STEP_LAND_ASYNC calls
cfg = bench.CONFIGS[name]
sizes, b = cfg["sizes"], cfg["batch"]
rng = np.random.default_rng(0)
xb = rng.standard_normal((b, sizes[0]), dtype=np.float32)
yb = rng.integers(0, sizes[-1], b).astype(np.int64)
w = [x.copy() for x in init_model(Architecture(sizes), seed=1).weights]
ctx = hb.GpuReplica(sizes, b)
ctx.pin_host([xb, yb])
ctx.pin_host(w)
for i in range(calls):
    print("---- call", i, file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    ctx.replica_step_host(w, xb, yb, 0.01, sole_writer=True, land_async=defer)
    print("call %d wall %.3f ms" % (i, 1e3 * (time.perf_counter() - t0)), file=sys.stderr, flush=True)
t0 = time.perf_counter()
ctx.landed()
print("landed after %.3f ms" % (1e3 * (time.perf_counter() - t0)), file=sys.stderr)
print("bytes", ctx.last_xfer_bytes, file=sys.stderr)

dev = torch.empty(max(x.size for x in w), dtype=torch.float64, device="cuda")
pin = torch.empty(dev.numel(), dtype=torch.float64).pin_memory()
for arr in w:
    n = arr.size
    host = torch.from_numpy(arr.reshape(-1))
    for label, dst in (("registered model", host), ("torch pinned", pin[:n])):
        dst.copy_(dev[:n], non_blocking=True)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            dst.copy_(dev[:n], non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        print("D2H %-16s %9d B  %.3f ms  %.1f GB/s  pinned=%s" % (label, 8 * n, ms, 8 * n / ms / 1e6, dst.is_pinned()),
              file=sys.stderr)
ctx.close()
