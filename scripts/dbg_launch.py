import sys, numpy as np
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_08771_b200 as hb
for sizes, b in [((2, 3, 2), 1), ((64, 96, 96, 10), 260), ((300, 512, 512, 2), 512), ((512, 512, 512, 2), 8192)]:
    try:
        ctx = hb.GpuReplica(sizes, b)
        rng = np.random.default_rng(0)
        ctx.set_weights([rng.normal(size=(sizes[l + 1], sizes[l])) for l in range(len(sizes) - 1)])
        ctx.stage(rng.normal(size=(b, sizes[0])), rng.integers(0, 2, b))
        ctx.step(0, b, 0.1)
        print(sizes, "ok")
    except Exception as e:
        print(sizes, "FAIL", e)
