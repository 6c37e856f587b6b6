"""Timeline of the fused replica step's exchange (HB_DEBUG_XCHG=1 HB_NO_GRAPHS=1)."""
import sys, os
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_08771_b200 as hb
from paper_2004_08771_b200.nn import Architecture, init_model
import bench
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "w8a"]
sizes, b = cfg["sizes"], cfg["batch"]
sparse = cfg["kind"] == "csr"
data = bench.make_data(cfg, 1)
ctx = hb.GpuReplica(sizes, b, sparse=sparse)
w = [x.copy() for x in init_model(Architecture(sizes), seed=1).weights]
if sparse:
    ctx.stage(data.rows(0, 2 * b))
else:
    ctx.stage(data.features[:2 * b].astype(np.float32), data.labels[:2 * b])
for i in range(3):
    print("---- call", i, file=sys.stderr, flush=True)
    ctx.replica_step(w, 0, b, 0.1)
