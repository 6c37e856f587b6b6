"""Worst per-step error (gradients and updated weights, every layer, the
reference's floored metric) of the GPU step vs the float64 oracle over many
seeds at a BASELINE shape -- how much margin the 1e-4 bar has.

    python scripts/seed_sweep.py <config> <batch> <n_seeds>
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from conftest import max_relative_error  # noqa: E402
from oracle import ref_nn  # noqa: E402
import paper_2004_08771_b200 as hb  # noqa: E402
from test_gpu_parity import oracle_case, run_step  # noqa: E402

CASES = {"delicious": ((500, 1024, 1024, 983), None, 0.5), "realsim": ((20958, 1024, 1024, 2), 52, 0.5),
         "scaled": ((1024, 4096, 4096, 4096, 1000), None, 0.1), "w8a": ((300, 512, 512, 512, 2), 12, 0.5),
         "covtype": ((54, 512, 512, 512, 2), None, 0.5)}
name, b, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
sizes, nnz, eta = CASES[name]
worst = []
for seed in range(100, 100 + n):
    w, x, y = oracle_case(sizes, b, seed=seed, sparse_nnz=nnz)
    g = ref_nn.backward(w, ref_nn.forward(w, x), y)
    upd = ref_nn.deep_copy(w)
    ref_nn.apply_update(upd, g, eta)
    out = run_step(hb, sizes, w, x, y, eta, sparse=bool(nnz))
    worst.append(max(max_relative_error(out["grads"], g), max_relative_error(out["weights"], upd)))
worst.sort()
print(json.dumps({"config": name, "batch": b, "seeds": n, "max": worst[-1], "median": worst[n // 2],
                  "over_1e-4": sum(v > 1e-4 for v in worst)}))
