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
