import time, torch, numpy as np
n = 5_400_000 // 8 * 8
for pinned in (False, True):
    h = torch.empty(n // 8, dtype=torch.float64, pin_memory=pinned)
    d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
    for _ in range(3): d.copy_(h); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
    print(f"H2D pinned={pinned}: {n/dt/1e9:.1f} GB/s ({dt*1e3:.3f} ms for {n/1e6:.1f} MB)")
    t = time.perf_counter()
    for _ in range(20): h.copy_(d, non_blocking=True)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
    print(f"D2H pinned={pinned}: {n/dt/1e9:.1f} GB/s")
a = np.random.rand(n // 8); b = np.random.rand(n // 8)
t = time.perf_counter()
for _ in range(20): np.add(a, 0.5 * b, out=a)
print(f"host axpy numpy: {(time.perf_counter()-t)/20*1e3:.3f} ms for {n/8/1e6:.2f} M doubles")
import os; print("cpus", os.cpu_count())
# bidirectional: H2D on one stream while D2H on another
h1 = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n // 8, dtype=torch.float64, device="cuda")
d2 = torch.empty(n // 8, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
print(f"bidirectional: {2*n/dt/1e9:.1f} GB/s total ({dt*1e3:.3f} ms per pair)")
for chunk in (1 << 18, 1 << 20, 1 << 22):
    t = time.perf_counter()
    for _ in range(5):
        for o in range(0, n // 8, chunk // 8):
            d1[o:o + chunk // 8].copy_(h1[o:o + chunk // 8], non_blocking=True)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
    print(f"H2D in {chunk>>10} KiB chunks: {n/dt/1e9:.1f} GB/s")
# registered (cudaHostRegister) numpy memory through our library
import sys
sys.path.insert(0, ".")
import ctypes as C
from paper_2004_08771_b200 import _native as N
lib = N.load()
a = np.random.rand(n // 8)
N.check(lib.hb_host_register(C.c_void_p(a.ctypes.data), a.nbytes))
ta = torch.from_numpy(a)
print("registered is_pinned:", ta.is_pinned())
for _ in range(3): d1.copy_(ta, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20): d1.copy_(ta, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
print(f"H2D registered: {n/dt/1e9:.1f} GB/s")
t = time.perf_counter()
for _ in range(20): ta.copy_(d1, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
print(f"D2H registered: {n/dt/1e9:.1f} GB/s")
b2 = np.random.rand(n // 8)
N.check(lib.hb_host_register(C.c_void_p(b2.ctypes.data), b2.nbytes))
tb = torch.from_numpy(b2)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    with torch.cuda.stream(s1):
        d1.copy_(ta, non_blocking=True)
    with torch.cuda.stream(s2):
        tb.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
print(f"bidirectional registered: {2*n/dt/1e9:.1f} GB/s total ({dt*1e3:.3f} ms per pair)")
