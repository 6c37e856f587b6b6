"""Pipeline timeline of the N-th GEMM launch of a training step (-DHB_TRACE build, HB_TRACE_LAUNCH=N)."""
import ctypes as C, os, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_08771_b200 as hb
from paper_2004_08771_b200 import _native as N
lib = N.load()
sizes = tuple(int(x) for x in os.environ.get("SIZES", "512,512,512,512,2").split(","))
b = int(os.environ.get("ROWS", "8192"))
ctx = hb.GpuReplica(sizes, b)
rng = np.random.default_rng(0)
ctx.set_weights([rng.normal(size=(sizes[l + 1], sizes[l])) / 20 for l in range(len(sizes) - 1)])
ctx.stage(rng.normal(size=(b, sizes[0])).astype(np.float32), rng.integers(0, 2, b))
buf = (C.c_ulonglong * 4096)()
lib.hb_trace_read.argtypes = [C.c_void_p, C.c_int]
os.environ["HB_NO_GRAPHS"] = "1"
ctx.step(0, b, 0.1)
lib.hb_trace_read(buf, 4096)
a = np.array(buf, dtype=np.int64)
t0 = a[6 * 512 + 2]
rel = lambda x: (x - t0) / 1000.0 if x else float('nan')
print(f"CTA start 0, epilogue start {rel(a[6*512]):.2f} us, end {rel(a[6*512+1]):.2f} us")
for i in range(64):
    if not a[0 * 512 + i] and not a[1 * 512 + i]: break
    print(f"kb {i:2d}: tma_issue {rel(a[i]):7.2f}  mma_start {rel(a[512+i]):7.2f}  mma_issued {rel(a[1024+i]):7.2f}")
for c in range(8):
    t0_, t1_ = a[7 * 512 + 4 * c], a[7 * 512 + 4 * c + 1]
    if t0_: print(f"epi chunk {c}: tmem loaded {rel(t0_):.2f}  transposed {rel(t1_):.2f}")
