"""Native LIBSVM -> CSR loader (csrc/hb_libsvm.cpp) against the reference's
own loader (golden outputs of hogtrain.data.load_libsvm, make_libsvm_golden.py)
and the reference's test_data.py cases.  Host code only: no GPU needed."""

import gzip
import json

import numpy as np
import pytest

import paper_2004_08771_b200 as hb
from conftest import GOLDEN

Z = np.load(GOLDEN / "libsvm.npz")
META = json.loads(bytes(Z["meta"]))


@pytest.mark.parametrize("name", sorted(META))
def test_matches_reference_loader(tmp_path, name):
    m = META[name]
    p = tmp_path / f"{name}.libsvm"
    p.write_bytes(bytes(Z[f"{name}__text"]))
    mapping = hb.LabelMapping(m["mapping"])
    if m["error"] is None:
        ds = hb.load_libsvm(p, m["dim"], mapping)
        assert np.array_equal(ds.features, Z[f"{name}__x"])  # bit-exact values
        assert np.array_equal(ds.labels, Z[f"{name}__y"])
        csr = hb.load_libsvm_csr(p, m["dim"], mapping)
        assert np.array_equal(csr.dense(), Z[f"{name}__x"])
        for r in range(csr.n_examples):  # ascending, distinct, no explicit zeros
            c = csr.col[csr.rowptr[r]:csr.rowptr[r + 1]]
            assert np.all(np.diff(c) > 0)
        assert np.all(csr.val != 0.0)
    else:
        kind, msg = m["error"]
        exc = hb.LibsvmParseError if kind == "LibsvmParseError" else ValueError
        with pytest.raises(exc) as ei:
            hb.load_libsvm_csr(p, m["dim"], mapping)
        if kind == "LibsvmParseError":
            assert isinstance(ei.value, hb.LibsvmParseError)
            assert str(ei.value) == msg
        elif "no examples" in msg:
            assert "no examples" in str(ei.value)
        else:
            assert str(ei.value) == msg
            assert not isinstance(ei.value, hb.LibsvmParseError)


def test_gzip_and_large_multithreaded(tmp_path):
    """A multi-MiB file parses in several chunks; the result is independent
    of the chunking and equals the plain-text parse; .gz is detected."""
    d = hb.synthetic_csr(60000, 300, 12, 2, seed=9, binary=False)
    lines = []
    for r in range(d.n_examples):
        s, e = d.rowptr[r], d.rowptr[r + 1]
        lines.append(str(int(d.labels[r])) + "".join(f" {c + 1}:{v:.17g}" for c, v in zip(d.col[s:e], d.val[s:e])))
    text = ("\n".join(lines) + "\n").encode()
    assert len(text) > 4 << 20
    p = tmp_path / "big.libsvm"
    p.write_bytes(text)
    back = hb.load_libsvm_csr(p, 300)
    assert np.array_equal(back.rowptr, d.rowptr) and np.array_equal(back.col, d.col)
    assert np.array_equal(back.val, d.val) and np.array_equal(back.labels, d.labels)
    g = tmp_path / "big.libsvm.gz"
    with gzip.open(g, "wb") as fh:
        fh.write(text)
    back_gz = hb.load_libsvm_csr(g, 300)
    assert np.array_equal(back_gz.val, d.val)
    # an error deep in the file reports its global line number
    bad = text + b"1 1:1\n1 3:zz\n"
    p.write_bytes(bad)
    with pytest.raises(hb.LibsvmParseError, match=f"line {d.n_examples + 2}:"):
        hb.load_libsvm_csr(p, 300)


def test_minmax(tmp_path):
    p = tmp_path / "scale.libsvm"
    p.write_text("0 1:2 2:10\n1 1:4 2:30\n0 1:6 2:20\n")  # test_data.py:64-68
    ds = hb.load_libsvm(p, 2, minmax_scale=True)
    assert ds.features.min() == 0.0 and ds.features.max() == 1.0
    lo = np.array([2.0, 10.0])
    ref = (np.array([[2, 10], [4, 30], [6, 20.0]]) - lo) / np.array([4.0, 20.0])
    assert np.array_equal(ds.features, ref)
    with pytest.raises(ValueError, match="minmax_scale"):
        hb.load_libsvm_csr(p, 2, minmax_scale=True)  # column minimum 2: would densify
    q = tmp_path / "sparse.libsvm"
    q.write_text("0 1:2\n1 2:4\n0 1:1 2:1\n")
    csr = hb.load_libsvm_csr(q, 2, minmax_scale=True)
    assert np.array_equal(csr.dense(), hb.load_libsvm(q, 2, minmax_scale=True).features)
