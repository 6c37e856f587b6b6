import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_08771_b200 as hb
from paper_2004_08771_b200.nn import Architecture, init_model
sizes = (300, 512, 512, 512, 2); b = 8192
model = init_model(Architecture(sizes), seed=1)
def t(f, n=20):
    f(); f()
    t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e3
for pin in (False, True):
    ctx = hb.GpuReplica(sizes, b, sparse=True)
    w = [x.copy() for x in model.weights]
    if pin: ctx.pin_host(w)
    print("pin", pin, "set_weights %.3f ms" % t(lambda: ctx.set_weights(w)))
    data = hb.synthetic_csr(8192, 300, 12, 2, seed=1); ctx.stage(data)
    ctx.step(0, b, 0.1, emit_grad=True)
    print("pin", pin, "merge %.3f ms" % t(lambda: ctx.merge_grads_into(w, 0.0)))
    print("pin", pin, "sync %.3f ms" % t(lambda: ctx.synchronize()))
    ctx.close()
