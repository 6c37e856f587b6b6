import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_cases():
    """Golden nn cases from tests/golden/nn_cases.npz (made by the reference)."""
    z = np.load(GOLDEN / "nn_cases.npz")
    cases = []
    for ci in range(int(z["n_cases"])):
        p = f"c{ci}_"
        sizes = tuple(int(s) for s in z[p + "sizes"])
        depth = len(sizes) - 1
        cases.append(
            dict(
                name=str(z[p + "name"]),
                sizes=sizes,
                x=z[p + "x"],
                y=z[p + "y"],
                eta=float(z[p + "eta"]),
                w=[z[p + f"w{l}"] for l in range(depth)],
                a=[z[p + f"a{l + 1}"] for l in range(depth)],
                g=[z[p + f"g{l}"] for l in range(depth)],
                u=[z[p + f"u{l}"] for l in range(depth)],
                ce=float(z[p + "ce"]),
                loss_sum=float(z[p + "loss_sum"]),
            )
        )
    return cases


def load_runs():
    z = np.load(GOLDEN / "sequential.npz")
    runs = []
    for i in range(int(z["n_runs"])):
        p = f"r{i}_"
        sizes = tuple(int(s) for s in z[p + "sizes"])
        b, epochs, seed = (int(v) for v in z[p + "meta"])
        runs.append(
            dict(
                name=str(z[p + "name"]), x=z[p + "x"], y=z[p + "y"], sizes=sizes,
                batch=b, epochs=epochs, seed=seed, eta=float(z[p + "eta"]),
                w=[z[p + f"w{l}"] for l in range(len(sizes) - 1)],
                final=[z[p + f"final{l}"] for l in range(len(sizes) - 1)],
                curve=z[p + "curve"], engine_curve=z[p + "engine_curve"],
                coverage=z[p + "coverage"],
            )
        )
    return runs


def max_relative_error(analytic, numeric, floor=1e-4):
    """Worst |a - n| / max(|a|, |n|, floor) over all layers -- the reference's
    own parity metric (pkg/tests/helpers.py:29-35)."""
    worst = 0.0
    for a, n in zip(analytic, numeric):
        a = np.asarray(a, dtype=np.float64)
        n = np.asarray(n, dtype=np.float64)
        denom = np.maximum(np.maximum(np.abs(a), np.abs(n)), floor)
        worst = max(worst, float((np.abs(a - n) / denom).max()))
    return worst


@pytest.fixture(scope="session")
def golden_cases():
    return load_cases()


@pytest.fixture(scope="session")
def golden_runs():
    return load_runs()
