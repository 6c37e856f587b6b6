"""Golden vectors for the native LIBSVM loader: texts run through the
REFERENCE's own `hogtrain.data.load_libsvm` (imported from
/root/reference/pkg/src), outputs committed to libsvm.npz.

Each case is a LIBSVM text plus either the reference's dense matrix and
labels, or the exception class name and message it raised.

    python tests/golden/make_libsvm_golden.py     # (build container only)
"""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def texts():
    rng = np.random.default_rng(2004)
    cases = {
        "basic": ("1 1:0.5 3:2.0\n", 4, "zero_one"),
        "pm": ("-1 2:1\n+1 1:3\n", 2, "plus_minus_one"),
        "multilabel": ("3,7,9 1:1\n0 1:2\n", 1, "zero_one"),
        "blank_lines_tabs": ("\n1\t2:1.5  4:-2e-3\n\n   \n0 1:1e10\r\n2 3:.25\n", 4, "zero_one"),
        "duplicate_and_zero": ("1 2:1 2:3 4:0 1:-0.5\n0 3:0.0\n", 4, "zero_one"),
        "unsorted": ("0 9:1 3:2 5:3\n1 1:1\n", 9, "zero_one"),
        "float_labels": ("1.7 1:1\n2e0 2:1\n0.0 1:3\n", 2, "zero_one"),
        "label_only": ("1\n0 1:1\n", 3, "zero_one"),
        "bad_token": ("1 1:0.5\n1 2:abc\n", 4, "zero_one"),
        "no_colon": ("1 1:0.5\n\n1 2\n", 4, "zero_one"),
        "oob": ("1 1:1\n1 5:1.0\n", 4, "zero_one"),
        "zero_index": ("1 0:1\n", 4, "zero_one"),
        "bad_label": ("x 1:1\n", 4, "zero_one"),
        "neg_label": ("-1 1:1\n", 4, "zero_one"),
        "pm_bad": ("1 1:1\n0 1:1\n", 4, "plus_minus_one"),
        "token_before_oob": ("1 2:q 9:1\n", 4, "zero_one"),
        "empty": ("\n\n", 4, "zero_one"),
    }
    # w8a-like binary rows and real-sim-like normalised rows (%.17g values)
    lines = []
    for r in range(300):
        cols = np.sort(rng.choice(300, size=rng.integers(1, 20), replace=False)) + 1
        lines.append(("+1" if rng.random() < 0.3 else "-1") + "".join(f" {c}:1" for c in cols))
    cases["w8a_like"] = ("\n".join(lines) + "\n", 300, "plus_minus_one")
    lines = []
    for r in range(200):
        cols = np.sort(rng.choice(2000, size=rng.integers(1, 60), replace=False)) + 1
        v = rng.random(len(cols))
        v /= np.linalg.norm(v)
        lines.append(str(int(rng.integers(0, 2))) + "".join(f" {c}:{x:.17g}" for c, x in zip(cols, v)))
    cases["realsim_like"] = ("\n".join(lines), 2000, "zero_one")  # no trailing newline
    return cases


def main():
    sys.path.insert(0, str(REF_SRC))
    from hogtrain.data import LabelMapping, load_libsvm

    out = {}
    meta = {}
    with tempfile.TemporaryDirectory() as td:
        for name, (text, dim, mapping) in texts().items():
            p = Path(td) / f"{name}.libsvm"
            p.write_bytes(text.encode())
            out[f"{name}__text"] = np.frombuffer(text.encode(), dtype=np.uint8)
            entry = {"dim": dim, "mapping": mapping}
            try:
                ds = load_libsvm(p, feature_dim=dim, label_mapping=LabelMapping(mapping))
                out[f"{name}__x"] = ds.features
                out[f"{name}__y"] = ds.labels
                entry["error"] = None
            except Exception as e:  # noqa: BLE001 -- the exception is the golden output
                entry["error"] = [type(e).__name__, str(e)]
            meta[name] = entry
    out["meta"] = np.frombuffer(json.dumps(meta, sort_keys=True).encode(), dtype=np.uint8)
    np.savez_compressed(OUT / "libsvm.npz", **out)
    print(f"wrote {len(meta)} cases to {OUT / 'libsvm.npz'}")


if __name__ == "__main__":
    main()
