"""Timeline of the fused replica step's exchange (HB_DEBUG_XCHG=1 HB_NO_GRAPHS=1):
    python scripts/xchg_timeline.py <config> [sole]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2004_08771_b200 as hb  # noqa: E402
from paper_2004_08771_b200.nn import Architecture, init_model  # noqa: E402
from oracle import ref_nn  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "w8a"
sole = len(sys.argv) > 2 and sys.argv[2] == "sole"
cfg = bench.CONFIGS[name]
sizes, b = cfg["sizes"], cfg["batch"]
sparse = cfg["kind"] == "csr"
ctx = hb.GpuReplica(sizes, b, sparse=sparse)
w = [x.copy() for x in init_model(Architecture(sizes), seed=1).weights]
if sparse:
    ctx.stage(bench.make_data(cfg, 1).rows(0, 2 * b))
else:
    x, y = ref_nn.synthetic_blobs(2 * b, sizes[0], sizes[-1], 2.5, 1)
    ctx.stage(x.astype(np.float32), y)
for i in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    print("---- call", i, file=sys.stderr, flush=True)
    ctx.replica_step(w, 0, b, 0.1, sole_writer=sole)
