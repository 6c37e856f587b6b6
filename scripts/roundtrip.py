"""Coordinator round trip vs the pipelined GPU worker on a B200.

The reference engine cannot travel to the GPU box, so this stands in for its
protocol: a coordinator thread serves one batch per request through a
Condition-guarded queue (the shape of messaging.py:24-67 / engine.py:278-316:
one message each way per batch), a GPU worker thread runs the drop-in replica
step.  Sequential: the worker replies after execute_gpu_replica returns (the
reference's WorkerThread._execute).  Pipelined: it replies after
execute_gpu_replica_begin and lands the merge with execute_gpu_replica_end
while the coordinator serves the next batch (feed.pipelined).

    python scripts/roundtrip.py [config] [steps]
"""
import collections
import json
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import ref_nn  # noqa: E402
import paper_2004_08771_b200 as hb  # noqa: E402
from paper_2004_08771_b200 import workers as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "w8a"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
sizes, b = {"w8a": ((300, 512, 512, 512, 2), 8192), "covtype": ((54, 512, 512, 512, 2), 512),
            "delicious": ((500, 1024, 1024, 983), 8192)}[name]
n = 8 * b
x, y = ref_nn.synthetic_blobs(n, sizes[0], sizes[-1], 2.5, 1)


class Queue:  # a Condition-guarded FIFO, one message at a time
    def __init__(self):
        self.cv = threading.Condition()
        self.items = collections.deque()

    def send(self, m):
        with self.cv:
            self.items.append(m)
            self.cv.notify()

    def receive(self):
        with self.cv:
            while not self.items:
                self.cv.wait()
            return self.items.popleft()


def run(pipelined):
    model = hb.Model(hb.Architecture(sizes), ref_nn.init_weights(sizes, 2))
    to_worker, to_coord = Queue(), Queue()
    W.set_sole_writer(True)

    def worker():
        to_coord.send(("schedule", 0))
        while True:
            m = to_worker.receive()
            if m is None:
                break
            batch, eta = m
            if pipelined:
                W.execute_gpu_replica_begin(model, batch, eta)
                to_coord.send(("schedule", 1))
                W.execute_gpu_replica_end()
            else:
                W.execute_gpu_replica(model, batch, eta)
                to_coord.send(("schedule", 1))
        W.release_thread_contexts()

    t = threading.Thread(target=worker, name="worker-gpu0")
    t.start()
    served, cursor, t0 = 0, 0, None
    while served < steps + 5:
        to_coord.receive()
        if served == 5:
            t0 = time.perf_counter()  # after warm-up (staging, graph capture)
        batch = hb.BatchRef(x, y, cursor, b)
        cursor = (cursor + b) % n
        to_worker.send((batch, 0.05))
        served += 1
    to_coord.receive()
    el = time.perf_counter() - t0
    to_worker.send(None)
    t.join()
    W.set_sole_writer(False)
    return {"pipelined": pipelined, "samples_s": round(steps * b / el, 1), "ms_per_batch": round(1000 * el / steps, 4)}


res = [run(False), run(True)]
print(json.dumps({"config": name, "batch": b, "steps": steps, "results": res,
                  "speedup": round(res[1]["samples_s"] / res[0]["samples_s"], 3)}))
