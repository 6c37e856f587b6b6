"""Per-CTA timeline of every GEMM in one training step (HB_TRACE build):
entry skew, setup, mainloop, epilogue and the gaps between launches."""
import ctypes as C, os, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("HOGBATCH_B200_LIB", str(Path(__file__).resolve().parent.parent / "build_variants/trace.so"))
import paper_2004_08771_b200 as hb
from paper_2004_08771_b200 import _native as N
lib = N.load()
sizes = tuple(int(x) for x in os.environ.get("SIZES", "300,512,512,512,2").split(","))
b = int(os.environ.get("ROWS", "8192"))
sparse = os.environ.get("SPARSE", "0") == "1"
ctx = hb.GpuReplica(sizes, b, sparse=sparse)
w = hb.init_model(hb.Architecture(sizes), seed=1).weights
ctx.set_weights(w)
d = hb.synthetic_csr(2 * b, sizes[0], 12, 2, seed=1)
if sparse:
    ctx.stage(d)
else:
    ctx.stage(d.dense().astype(np.float32), d.labels)
buf = (C.c_ulonglong * (8 * 1024 * 4))()
lib.hb_trace_cta_read.argtypes = [C.c_void_p]
for it in range(4):
    lib.hb_trace_cta_read(buf)  # resets the launch counter
    ctx.step(0, b, 0.1)
lib.hb_trace_cta_read(buf)
a = np.array(buf, dtype=np.int64).reshape(8, 1024, 4)
used = [s for s in range(8) if a[s, 0, 0]]
t0 = min(a[s][a[s][:, 0] > 0][:, 0].min() for s in used)
prev_end = None
for s in used:
    r = a[s][a[s][:, 0] > 0]
    r = (r - t0) / 1000.0
    e, su, ep, en = r[:, 0], r[:, 1], r[:, 2], r[:, 3]
    gap = f"gap {e.min() - prev_end:6.2f}" if prev_end is not None else " " * 10
    print(f"gemm {s}: ctas {len(r):4d} {gap} entry {e.min():7.2f}..{e.max():7.2f}  setup {np.median(su - e):5.2f}"
          f"  mainloop {np.median(ep - su):6.2f} (max epi start {ep.max():7.2f})  epilogue {np.median(en - ep):5.2f}"
          f"  end {en.min():7.2f}..{en.max():7.2f}  span {en.max() - e.min():6.2f}")
    prev_end = en.max()
