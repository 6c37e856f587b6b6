"""Per-layer parity of one step at the BASELINE sizes (diagnostics)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent)); sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from oracle import ref_nn
import paper_2004_08771_b200 as hb
from test_gpu_parity import oracle_case, run_step
cases = {"delicious": ((500, 1024, 1024, 983), 8192, None, 0.5), "realsim": ((20958, 1024, 1024, 2), 2048, 52, 0.5),
         "scaled": ((1024, 4096, 4096, 4096, 1000), 8192, None, 0.1), "w8a": ((300, 512, 512, 512, 2), 8192, 12, 0.5)}
for name in sys.argv[1:] or list(cases):
    sizes, b, nnz, eta = cases[name]
    w, x, y = oracle_case(sizes, b, seed=7 + b, sparse_nnz=nnz)
    g = ref_nn.backward(w, ref_nn.forward(w, x), y)
    out = run_step(hb, sizes, w, x, y, eta, sparse=bool(nnz))
    for l, (a, r) in enumerate(zip(out["grads"], g)):
        d = np.maximum(np.maximum(np.abs(a), np.abs(r)), 1e-4)
        e = np.abs(a.astype(np.float64) - r) / d
        i = np.unravel_index(np.argmax(e), e.shape)
        print(f"{name} layer {l}: max rel {e.max():.2e} at {i} (gpu {a[i]:.6e} ref {r[i]:.6e}), |g| max {np.abs(r).max():.2e} median {np.median(np.abs(r)):.2e}, frac>1e-4 {np.mean(e > 1e-4):.2e}")
    upd = ref_nn.deep_copy(w)
    ref_nn.apply_update(upd, g, eta)
    for l, (a, r) in enumerate(zip(out["weights"], upd)):
        d = np.maximum(np.maximum(np.abs(a), np.abs(r)), 1e-4)
        e = np.abs(a - r) / d
        i = np.unravel_index(np.argmax(e), e.shape)
        print(f"{name} weights {l}: max rel {e.max():.2e} at {i} (gpu {a[i]:.8e} ref {r[i]:.8e})")
