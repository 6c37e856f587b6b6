"""Per-layer parity diagnostics of one step at a BASELINE shape (GPU vs the
float64 oracle): activations (max abs error and the mean *signed* error, a
bias indicator), gradients and updated weights under the reference's floored
metric, plus the same oracle run on fp32-rounded inputs/weights (the floor any
fp32 implementation starts from).

    python scripts/diag_layers.py realsim [b] [seeds...]
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from oracle import ref_nn  # noqa: E402
import paper_2004_08771_b200 as hb  # noqa: E402
from test_gpu_parity import oracle_case, run_step  # noqa: E402

CASES = {"delicious": ((500, 1024, 1024, 983), None, 0.5), "realsim": ((20958, 1024, 1024, 2), 52, 0.5),
         "scaled": ((1024, 4096, 4096, 4096, 1000), None, 0.1), "w8a": ((300, 512, 512, 512, 2), 12, 0.5),
         "covtype": ((54, 512, 512, 512, 2), None, 0.5)}


def rel(a, r):
    d = np.maximum(np.maximum(np.abs(a), np.abs(r)), 1e-4)
    return np.abs(a.astype(np.float64) - r) / d


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "realsim"
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    seeds = [int(s) for s in sys.argv[3:]] or [7 + b]
    sizes, nnz, eta = CASES[name]
    for seed in seeds:
        w, x, y = oracle_case(sizes, b, seed=seed, sparse_nnz=nnz)
        tape = ref_nn.forward(w, x)
        g = ref_nn.backward(w, tape, y)
        upd = ref_nn.deep_copy(w)
        ref_nn.apply_update(upd, g, eta)
        # fp32-input oracle
        w32 = [wi.astype(np.float32).astype(np.float64) for wi in w]
        x32 = x.astype(np.float32).astype(np.float64)
        g32 = ref_nn.backward(w32, ref_nn.forward(w32, x32), y)
        u32 = ref_nn.deep_copy(w32)
        ref_nn.apply_update(u32, g32, eta)
        for kern in ((False, True) if nnz else (False,)):
            out = run_step(hb, sizes, w, x, y, eta, sparse=bool(nnz), sparse_kernels=kern)
            tag = f"{name} b={b} seed={seed} {'csr-kernels' if kern else 'dense-l0'}"
            for l, a in enumerate(out["acts"]):
                r = tape[l + 1]
                dlt = a.astype(np.float64) - r
                print(f"{tag} A{l + 1}: max|err| {np.abs(dlt).max():.2e} mean err {dlt.mean():+.2e} "
                      f"mean|err| {np.abs(dlt).mean():.2e}")
            for l, (a, r) in enumerate(zip(out["grads"], g)):
                e = rel(a, r)
                e32 = rel(g32[l], r)
                i = np.unravel_index(np.argmax(e), e.shape)
                print(f"{tag} G{l}: max rel {e.max():.2e} at {i} (gpu {a[i]:.6e} ref {r[i]:.6e}) | fp32-oracle "
                      f"{e32.max():.2e} | |g| max {np.abs(r).max():.2e} | mean signed err "
                      f"{(a.astype(np.float64) - r).mean():+.2e}")
            for l, (a, r) in enumerate(zip(out["weights"], upd)):
                e = rel(a, r)
                e32 = rel(u32[l], r)
                i = np.unravel_index(np.argmax(e), e.shape)
                print(f"{tag} W{l}: max rel {e.max():.2e} at {i} (gpu {a[i]:.8e} ref {r[i]:.8e}) | fp32-oracle "
                      f"{e32.max():.2e}")
            sys.stdout.flush()


if __name__ == "__main__":
    main()
