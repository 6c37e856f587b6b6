"""Dataset / batch layouts of the drop-in surface, plus the sparse format.

Dense: `Dataset` and `BatchRef` mirror pkg/src/hogtrain/data.py:30-79 (a
BatchRef is a contiguous row range of a float64 (N, d) array, typically the
per-epoch shuffled copy, engine.py:214-221).  `synthetic_blobs`,
`shuffle_epoch` and `reorder` reproduce data.py:182-252 draw for draw so the
GPU runs on inputs identical to the reference's.

Sparse (new; the reference densifies LIBSVM, data.py:106-151): `CsrDataset`
holds CSR rows (int64 row pointer, int32 0-based column ids, float64 values)
and `CsrBatchRef` is the same contiguous-row-range view over it.
`synthetic_csr` generates the w8a-/real-sim-shaped inputs of BASELINE.json
 and `CsrDataset.dense()` is the exact dense twin the oracle
consumes.  `load_libsvm_csr` parses LIBSVM text natively (csrc/hb_libsvm.cpp)
straight to CSR with the reference loader's semantics and errors;
`load_libsvm` is the reference's dense signature on top of it.
"""

from __future__ import annotations

import gzip
from dataclasses import dataclass
from enum import Enum
from pathlib import Path

import numpy as np


@dataclass
class Dataset:  # data.py:30-54
    features: np.ndarray  # (N, d) float64, C-contiguous
    labels: np.ndarray  # (N,) int64
    name: str = ""

    def __post_init__(self):
        if self.features.ndim != 2 or self.features.shape[0] < 1:
            raise ValueError("features must be a non-empty 2-D matrix")
        if self.labels.shape != (self.features.shape[0],):
            raise ValueError("labels length must equal the number of feature rows")
        if self.labels.min() < 0:
            raise ValueError("labels must be non-negative class indices")

    @property
    def n_examples(self) -> int:
        return self.features.shape[0]

    @property
    def feature_dim(self) -> int:
        return self.features.shape[1]

    @property
    def class_count(self) -> int:
        return int(self.labels.max()) + 1


@dataclass(frozen=True)
class BatchRef:  # data.py:57-79
    features: np.ndarray
    labels: np.ndarray
    start: int
    length: int

    def __post_init__(self):
        if self.length < 1 or self.start < 0 or self.start + self.length > self.features.shape[0]:
            raise ValueError(
                f"batch range [{self.start}, {self.start + self.length}) out of bounds"
                f" for {self.features.shape[0]} rows"
            )

    @property
    def x(self):
        return self.features[self.start : self.start + self.length]

    @property
    def y(self):
        return self.labels[self.start : self.start + self.length]


@dataclass
class CsrDataset:
    """Sparse rows: row i holds col[rowptr[i]:rowptr[i+1]] / val[...]."""

    rowptr: np.ndarray  # (N+1,) int64, rowptr[0] == 0
    col: np.ndarray  # (nnz,) int32, 0-based
    val: np.ndarray  # (nnz,) float64
    labels: np.ndarray  # (N,) int64
    n_cols: int
    name: str = ""

    def __post_init__(self):
        self.rowptr = np.ascontiguousarray(self.rowptr, dtype=np.int64)
        self.col = np.ascontiguousarray(self.col, dtype=np.int32)
        self.val = np.ascontiguousarray(self.val, dtype=np.float64)
        self.labels = np.ascontiguousarray(self.labels, dtype=np.int64)
        n = self.labels.shape[0]
        if n < 1 or self.rowptr.shape != (n + 1,) or self.rowptr[0] != 0:
            raise ValueError("rowptr must have n_rows+1 entries starting at 0")
        if self.rowptr[-1] != self.col.shape[0] or self.col.shape != self.val.shape:
            raise ValueError("rowptr[-1] must equal nnz = len(col) = len(val)")
        if self.col.size and (self.col.min() < 0 or self.col.max() >= self.n_cols):
            raise ValueError(f"feature index outside [0, {self.n_cols})")

    @property
    def n_examples(self) -> int:
        return self.labels.shape[0]

    @property
    def feature_dim(self) -> int:
        return self.n_cols

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    @property
    def class_count(self) -> int:
        return int(self.labels.max()) + 1

    def rows(self, start: int, stop: int) -> "CsrDataset":
        """Rows [start, stop) as a standalone CSR (row pointer rebased to 0)."""
        e0, e1 = int(self.rowptr[start]), int(self.rowptr[stop])
        return CsrDataset(self.rowptr[start : stop + 1] - e0, self.col[e0:e1], self.val[e0:e1],
                          self.labels[start:stop], self.n_cols, self.name)

    def dense(self, start: int = 0, stop: int | None = None) -> np.ndarray:
        """Exact float64 dense twin of rows [start, stop) (what the reference's
        densifying loader would produce, data.py:128-140)."""
        stop = self.n_examples if stop is None else stop
        sub = self.rows(start, stop)
        out = np.zeros((stop - start, self.n_cols))
        r = np.repeat(np.arange(stop - start), np.diff(sub.rowptr))
        out[r, sub.col] = sub.val
        return out


@dataclass(frozen=True)
class CsrBatchRef:
    """Contiguous row range [start, start+length) of a CsrDataset."""

    data: CsrDataset
    start: int
    length: int

    def __post_init__(self):
        if self.length < 1 or self.start < 0 or self.start + self.length > self.data.n_examples:
            raise ValueError(f"batch range [{self.start}, {self.start + self.length}) out of bounds")

    @property
    def features(self):
        return self.data

    @property
    def y(self):
        return self.data.labels[self.start : self.start + self.length]

    @property
    def x(self):
        return self.data.dense(self.start, self.start + self.length)


def synthetic_blobs(n: int, dim: int, classes: int, separation: float, seed) -> Dataset:
    """Gaussian class clusters with minimum class-mean distance `separation`,
    rows shuffled (data.py:226-252, identical draws)."""
    if classes < 2:
        raise ValueError("need at least 2 classes")
    rng = np.random.default_rng(seed)
    raw = rng.normal(size=(classes, dim))
    raw -= raw.mean(axis=0)
    if separation > 0:
        # min pairwise distance, evaluated pair by pair with the same 1-D norm
        # as the reference so the means agree to the last bit
        best = min(np.linalg.norm(raw[i] - raw[j]) for i in range(classes) for j in range(i + 1, classes))
        means = raw * (separation / best)
    else:
        means = np.zeros_like(raw)
    labels = np.arange(n, dtype=np.int64) % classes
    features = means[labels] + rng.normal(size=(n, dim))
    perm = rng.permutation(n)
    return Dataset(features=np.ascontiguousarray(features[perm]), labels=labels[perm].copy(),
                   name=f"blobs(n={n},dim={dim},k={classes},sep={separation})")


def blob_means(dim: int, classes: int, separation: float, seed) -> np.ndarray:
    """The class means of synthetic_blobs (data.py:235-243) for datasets whose
    rows are generated on the device (GpuReplica.stage_blobs): same draw and
    centring, scaled so the closest pair of means is `separation` apart."""
    if classes < 2:
        raise ValueError("need at least 2 classes")
    rng = np.random.default_rng(seed)
    raw = rng.normal(size=(classes, dim))
    raw -= raw.mean(axis=0)
    if separation <= 0:
        return np.zeros_like(raw)
    best = min(float(np.linalg.norm(raw[i + 1:] - raw[i], axis=1).min()) for i in range(classes - 1))
    return raw * (separation / best)


def synthetic_csr(n: int, dim: int, nnz_per_row: int, classes: int, seed, binary: bool = True,
                  normalize: bool = False, name: str = "") -> CsrDataset:
    """Seeded sparse rows: `nnz_per_row` distinct uniform column draws per row,
    values 1.0 (binary, w8a-like) or |N(0,1)| L2-normalised (real-sim-like);
    labels planted as argmax over classes of the row's projection onto random
    class means plus unit noise."""
    if classes < 2:
        raise ValueError("need at least 2 classes")
    k = min(nnz_per_row, dim)
    rng = np.random.default_rng(seed)
    means = rng.normal(size=(classes, dim))
    # distinct columns per row: sort of k uniform keys over a (n, k*2) draw, deduplicated
    cols = np.empty((n, k), dtype=np.int64)
    chunk = 65536
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        m = r1 - r0
        cand = rng.integers(0, dim, size=(m, 3 * k + 8))
        cand.sort(axis=1)
        dup = np.zeros_like(cand, dtype=bool)
        dup[:, 1:] = cand[:, 1:] == cand[:, :-1]
        keys = np.where(dup, dim + 1, cand)  # push duplicates to the end
        # random subset of the distinct candidates: random priority, duplicates last
        prio = rng.random(size=cand.shape) + dup * 2.0
        pick = np.argsort(prio, axis=1)[:, :k]
        chosen = np.take_along_axis(keys, pick, axis=1)
        if (chosen > dim).any():  # vanishingly rare: redraw those rows exactly
            for i in np.nonzero((chosen > dim).any(axis=1))[0]:
                chosen[i] = rng.choice(dim, size=k, replace=False)
        chosen.sort(axis=1)
        cols[r0:r1] = chosen
    if binary:
        vals = np.ones((n, k))
    else:
        vals = np.abs(rng.normal(size=(n, k)))
    if normalize:
        vals /= np.linalg.norm(vals, axis=1, keepdims=True)
    score = np.einsum("nk,cnk->nc", vals, means[:, cols]) + rng.normal(size=(n, classes))
    labels = np.argmax(score, axis=1).astype(np.int64)
    rowptr = np.arange(0, n * k + 1, k, dtype=np.int64)
    return CsrDataset(rowptr, cols.reshape(-1).astype(np.int32), vals.reshape(-1), labels, dim,
                      name or f"csr(n={n},dim={dim},nnz={k},k={classes})")


def shuffle_epoch(n_examples: int, seed) -> np.ndarray:
    """Deterministic permutation for the epoch seed (run_seed, epoch)
    (data.py:182-184, engine.py:74-76)."""
    return np.random.default_rng(seed).permutation(n_examples)


def epoch_shuffle_seed(run_seed: int, epoch: int) -> tuple:
    return (run_seed, epoch)


def reorder(ds, perm: np.ndarray):
    """Row-permuted contiguous copy (data.py:187-193); CSR datasets permute rows."""
    if isinstance(ds, CsrDataset):
        lengths = np.diff(ds.rowptr)[perm]
        rowptr = np.zeros(ds.n_examples + 1, dtype=np.int64)
        np.cumsum(lengths, out=rowptr[1:])
        starts = ds.rowptr[perm]
        idx = np.repeat(starts - rowptr[:-1], lengths) + np.arange(rowptr[-1])
        return CsrDataset(rowptr, ds.col[idx], ds.val[idx], ds.labels[perm].copy(), ds.n_cols, ds.name)
    return Dataset(features=np.ascontiguousarray(ds.features[perm]), labels=ds.labels[perm].copy(), name=ds.name)


class LabelMapping(Enum):  # data.py:21-23
    ZERO_ONE = "zero_one"
    PLUS_MINUS_ONE = "plus_minus_one"


class LibsvmParseError(ValueError):  # data.py:26-27
    """Malformed LIBSVM input; message carries the 1-based line number."""


def _read_text_bytes(path: Path) -> bytes:
    # data.py:80-83: gzip is detected by the .gz extension
    if path.suffix == ".gz":
        with gzip.open(path, "rb") as fh:
            return fh.read()
    return path.read_bytes()


def load_libsvm_csr(path, feature_dim: int, label_mapping: LabelMapping = LabelMapping.ZERO_ONE,
                    minmax_scale: bool = False, name: str | None = None) -> CsrDataset:
    """LIBSVM text -> CsrDataset without densifying (the reference's
    load_libsvm, data.py:106-151, builds an (N, feature_dim) float64 matrix).
    Rows, labels and values equal the nonzeros of the reference's matrix;
    errors are LibsvmParseError / ValueError with the same line numbers.
    minmax_scale (data.py:167-171) is applied when it keeps the data sparse
    (every column's minimum is 0, true for non-negative features); otherwise
    it would densify and ValueError says to use load_libsvm."""
    import ctypes as C

    from . import _native as N

    path = Path(path)
    buf = _read_text_bytes(path)
    lib = N.load()
    mode = 1 if label_mapping is LabelMapping.PLUS_MINUS_ONE else 0
    n_rows, nnz = C.c_int64(0), C.c_int64(0)
    _libsvm_check(N, lib.hb_libsvm_scan(buf, len(buf), int(feature_dim), mode, C.byref(n_rows), C.byref(nnz)))
    if n_rows.value == 0:
        raise ValueError(f"{path}: no examples")
    rowptr = np.empty(n_rows.value + 1, dtype=np.int64)
    col = np.empty(max(nnz.value, 1), dtype=np.int32)
    val = np.empty(max(nnz.value, 1), dtype=np.float64)
    labels = np.empty(n_rows.value, dtype=np.int64)
    _libsvm_check(N, lib.hb_libsvm_fill(buf, len(buf), int(feature_dim), mode, N.ptr(rowptr, C.c_int64),
                                        N.ptr(col, C.c_int32), N.ptr(val, C.c_double), N.ptr(labels, C.c_int64)))
    ds = CsrDataset(rowptr, col[: nnz.value], val[: nnz.value], labels, int(feature_dim), name or path.stem)
    if minmax_scale:
        ds = _minmax_scale_csr(ds)
    return ds


def _libsvm_check(N, rc: int) -> None:
    if rc == N.HB_EPARSE:
        raise LibsvmParseError(N.last_error())
    N.check(rc)


def _minmax_scale_csr(ds: CsrDataset) -> CsrDataset:
    n, d = ds.n_examples, ds.n_cols
    count = np.bincount(ds.col, minlength=d)
    lo = np.full(d, np.inf)
    hi = np.full(d, -np.inf)
    np.minimum.at(lo, ds.col, ds.val)
    np.maximum.at(hi, ds.col, ds.val)
    implicit_zero = count < n  # a column with a missing entry has a 0.0 in the dense matrix
    lo = np.where(implicit_zero, np.minimum(lo, 0.0), lo)
    hi = np.where(implicit_zero, np.maximum(hi, 0.0), hi)
    if np.any(lo != 0.0):
        raise ValueError("minmax_scale would shift zeros (a column minimum is not 0); use load_libsvm (dense)")
    span = hi - lo
    span[span == 0.0] = 1.0
    # (x - 0.0) / span == x / span exactly: same values as data.py:167-171
    return CsrDataset(ds.rowptr, ds.col, ds.val / span[ds.col], ds.labels, d, ds.name)


def load_libsvm(path, feature_dim: int, label_mapping: LabelMapping = LabelMapping.ZERO_ONE,
                minmax_scale: bool = False, name: str | None = None) -> Dataset:
    """The reference's dense loader (data.py:106-151) on the native parser."""
    csr = load_libsvm_csr(path, feature_dim, label_mapping, False, name)
    features = np.ascontiguousarray(csr.dense())
    if minmax_scale:  # data.py:167-171
        lo = features.min(axis=0)
        span = features.max(axis=0) - lo
        span[span == 0.0] = 1.0
        features = (features - lo) / span
    return Dataset(features=features, labels=csr.labels, name=csr.name)
