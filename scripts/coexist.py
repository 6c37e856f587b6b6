"""CPU+GPU Hogbatch coexistence (configs C2-C4: a CPU Hogwild pool and a GPU
replica writing one shared float64 model): throughput of the host-CPU Hogbatch
pool (oracle/ref_hogbatch.py, threads = host cores, 64 rows per thread, one
BLAS thread each) alone and with a GPU replica worker running
execute_gpu_replica-style calls on the same model in another thread -- with
the library's default merge pool, and with the pool shrunk and not spinning
(install(cpu_pool_threads=...) -> hb_host_merge_threads).

    python scripts/coexist.py [config] [seconds]
"""
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import ref_hogbatch, ref_nn  # noqa: E402
import paper_2004_08771_b200 as hb  # noqa: E402
from paper_2004_08771_b200 import workers as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "w8a"
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 8.0
sizes = {"w8a": (300, 512, 512, 512, 2), "covtype": (54, 512, 512, 512, 2),
         "delicious": (500, 1024, 1024, 983)}[name]
classes = sizes[-1]
threads = os.cpu_count() or 8
x, y = ref_nn.synthetic_blobs(65536, sizes[0], classes, 2.5, 1)
xg, yg = x[:8192].astype(np.float32), y[:8192]


def run(mode):
    model = ref_nn.init_weights(sizes, 2)
    stop = threading.Event()
    gpu = {"steps": 0, "ms": 0.0}

    def gpu_loop():
        ctx = hb.GpuReplica(sizes, 8192)
        try:
            while not stop.is_set():
                t0 = time.perf_counter()
                ctx.replica_step_host(model, xg, yg, 0.01)  # shared model, not sole writer
                gpu["ms"] += 1000 * (time.perf_counter() - t0)
                gpu["steps"] += 1
        finally:
            ctx.close()

    if mode == "shrunk":
        W.set_host_merge_threads(2, spin=0)
    elif mode == "gpu_default":
        W.set_host_merge_threads(min(12, max(1, threads * 3 // 4)), spin=20000)
    t = None
    if mode != "cpu_alone":
        t = threading.Thread(target=gpu_loop)
        t.start()
        time.sleep(1.0)  # GPU warm (graph captured, model pinned)

    def batches():
        i = 0
        while True:
            s = (i * threads * 64) % (x.shape[0] - threads * 64)
            yield x[s:s + threads * 64], y[s:s + threads * 64]
            i += 1

    res = ref_hogbatch.run_hogbatch(model, batches(), 0.0005, secs, threads=threads)
    stop.set()
    if t is not None:
        t.join()
    out = {"mode": mode, "cpu_samples_s": res["samples"] / res["seconds"], "threads": threads}
    if gpu["steps"]:
        out["gpu_samples_s"] = gpu["steps"] * 8192 / (gpu["ms"] / 1000.0)
    return out


results = [run(m) for m in ("cpu_alone", "gpu_default", "shrunk")]
base = results[0]["cpu_samples_s"]
for r in results:
    r["cpu_vs_alone"] = round(r["cpu_samples_s"] / base, 3)
print(json.dumps({"config": name, "seconds": secs, "results": results}))
