import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_08771_b200 as hb
from paper_2004_08771_b200.nn import Architecture, init_model
import bench
cfg = bench.CONFIGS[sys.argv[1]]
sizes, b = cfg["sizes"], cfg["batch"]
sparse = cfg["kind"] == "csr"
data = bench.make_data(cfg, 1)
ctx = hb.GpuReplica(sizes, b, sparse=sparse)
w = [x.copy() for x in init_model(Architecture(sizes), seed=1).weights]
if sparse:
    sub = data.rows(0, b); sub.col = sub.col.copy(); sub.labels = sub.labels.copy(); sub.val = sub.val.astype(np.float32); xb, yb = sub, None
    ctx.pin_host([sub.rowptr, sub.col, sub.val, sub.labels])
else:
    xb = data.features[:b].astype(np.float32); yb = data.labels[:b].copy(); ctx.pin_host([xb, yb])
for i in range(6):
    t0 = time.perf_counter()
    ctx.replica_step_host(w, xb, yb, 0.1, want_loss=True)
    print(f"---- call {i}: {1e6*(time.perf_counter()-t0):.1f} us wall", file=sys.stderr, flush=True)
