"""Host cost of the Python layer around the drop-in call: GpuReplica.replica_step_host
vs the same C entry called with pre-built ctypes arguments (covtype / w8a shapes).

    python scripts/call_overhead.py [config]
"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import ref_nn  # noqa: E402
import paper_2004_08771_b200 as hb  # noqa: E402
from paper_2004_08771_b200 import _native as N  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "covtype"
sizes, b = {"covtype": ((54, 512, 512, 512, 2), 512), "w8a": ((300, 512, 512, 512, 2), 8192)}[name]
x, y = ref_nn.synthetic_blobs(b, sizes[0], 2, 2.5, 1)
x = x.astype(np.float32)
w = ref_nn.init_weights(sizes, 2)
ctx = hb.GpuReplica(sizes, b)
ctx.pin_host([x, y])
for _ in range(5):
    ctx.replica_step_host(w, x, y, 0.01, sole_writer=True)


def t(f, n=300):
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    return (time.perf_counter() - t0) / n * 1e6


py_us = t(lambda: ctx.replica_step_host(w, x, y, 0.01, sole_writer=True))
table = ctx._model_table(w)
lib, h = ctx._lib, ctx._h
loss = C.c_double()
args = (h, table, x.ctypes.data, x.strides[0] // 4, y.ctypes.data, b, 0.01, N.HB_STEP_SOLE_WRITER, C.byref(loss))
c_us = t(lambda: lib.hb_replica_step_host_dense(*args))
print(f"{name}: replica_step_host {py_us:.1f} us/call, bare C call {c_us:.1f} us/call, Python layer {py_us - c_us:.1f} us")
