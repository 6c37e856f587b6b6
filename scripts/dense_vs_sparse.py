"""w8a shape: sparse kernels vs the dense GEMM path on the densified batch."""
import numpy as np, torch
import paper_2004_08771_b200 as hb

sizes, b, n = (300, 512, 512, 512, 2), 8192, 64700
d = hb.synthetic_csr(n, 300, 12, 2, seed=1)
w = hb.init_model(hb.Architecture(sizes), seed=1).weights
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for sparse in (True, False):
    ctx = hb.GpuReplica(sizes, b, sparse=sparse)
    ctx.set_weights(w)
    if sparse:
        ctx.stage(d)
    else:
        ctx.stage(d.dense().astype(np.float32), d.labels)
    starts = [(i * b) % (n - b) for i in range(40)]
    for s in starts[:5]:
        ctx.step(s, b, 0.1)
    ms = []
    for s in starts[5:25]:
        flush.zero_(); torch.cuda.synchronize()
        ctx.step(s, b, 0.1, timed=True)
        ms.append(ctx.last_step_ms)
    ctx.profile(True)
    for s in starts[25:35]:
        flush.zero_(); torch.cuda.synchronize()
        ctx.step(s, b, 0.1, timed=True)
    prof = ctx.profile_read()
    ctx.profile(False)
    print("sparse" if sparse else "dense ", "ms/step %.4f" % np.median(ms))
    print("   ", " ".join("%s=%.1f" % (k, v[0] / v[1] * 1e3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])))
    ctx.close()
