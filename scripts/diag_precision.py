"""Per-case, per-layer parity diagnostics of the GPU step vs the golden vectors."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from conftest import load_cases, max_relative_error
from oracle import ref_nn
import paper_2004_08771_b200 as hb

for c in load_cases():
    for prec in ("3xtf32", "tf32"):
        ctx = hb.GpuReplica(c["sizes"], c["x"].shape[0], precision=prec)
        ctx.set_weights(c["w"]); ctx.stage(c["x"], c["y"])
        ctx.step(0, c["x"].shape[0], c["eta"], emit_grad=True)
        g = ctx.grads(); ctx.close()
        per = [max_relative_error([a], [b]) for a, b in zip(g, c["g"])]
        absd = [float(np.abs(a - b).max()) for a, b in zip(g, c["g"])]
        mag = [float(np.abs(b).max()) for b in c["g"]]
        print(f"{c['name']:16s} {prec:6s} rel/layer " + " ".join(f"{e:.1e}" for e in per)
              + " | maxabs " + " ".join(f"{e:.1e}" for e in absd) + " | gmax " + " ".join(f"{e:.1e}" for e in mag))
# isolated GEMM precision: 1-hidden-layer nets, compare the logits path
rng = np.random.default_rng(0)
for K in (24, 256, 983):
    x = rng.normal(size=(256, K)); W = rng.normal(size=(64, K)) / np.sqrt(K); W2 = rng.normal(size=(10, 64)) / 8
    y = rng.integers(0, 10, 256)
    ctx = hb.GpuReplica((K, 64, 10), 256); ctx.set_weights([W, W2]); ctx.stage(x, y)
    ctx.forward(0, 256); a = ctx.activation(1, 256); ctx.close()
    ref = ref_nn.sigmoid(x @ W.T)
    z = x @ W.T
    err = np.abs(a - ref) / (ref * (1 - ref))   # ~ abs error of z
    print(f"fwd K={K}: max |dz| {err.max():.2e}  rel-to-|z|row {float((err / np.abs(z).max()).max()):.2e}")
