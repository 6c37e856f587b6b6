"""Generate the golden vectors that pin the oracle (and the GPU path).

Runs the REFERENCE itself -- `hogtrain` imported from
/root/reference/pkg/src -- on small seeded inputs and commits the inputs and
outputs as .npz fixtures next to this script.  /root/reference does not
exist on the GPU box, so nothing at test/bench time imports it; the fixtures
travel instead.

    python tests/golden/make_golden.py        # (build container only)
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
OUT = Path(__file__).resolve().parent


def _import_reference():
    sys.path.insert(0, str(REF_SRC))
    sys.path.insert(0, str(REF_TESTS))
    import hogtrain  # noqa: F401
    return hogtrain


def nn_cases(h):
    from hogtrain import nn
    from hogtrain.data import BatchRef, synthetic_blobs
    from hogtrain.linalg import as_matrix
    from hogtrain.workers import execute_batch_replica
    from helpers import random_small_net

    cases = []
    # 1. the hand-computed 2-3-2 net of test_nn.py:76-97
    w1 = as_matrix([[0.1, -0.2], [0.3, 0.4], [-0.5, 0.6]])
    w2 = as_matrix([[0.7, -0.8, 0.9], [-1.0, 1.1, -1.2]])
    cases.append(("hand232", nn.Model(nn.Architecture((2, 3, 2)), [w1, w2]),
                  as_matrix([[0.5, -1.5]]), np.array([1]), 0.25))
    # 2. helpers.random_small_net draws (widths <= 8, batch <= 8)
    rng = np.random.default_rng(99)
    for i in range(6):
        m, x, y = random_small_net(rng)
        cases.append((f"small{i}", m, x, y, 0.1 * (i + 1)))
    # 3. shapes that stress the device kernels: K=54 tail, wide softmax,
    #    several hidden layers, odd batch tails
    shapes = [
        ("covtype_like", (54, 40, 40, 40, 2), 37, 2, 0.5),
        ("delicious_like", (20, 24, 983), 19, 983, 0.3),
        ("deep_odd", (13, 33, 17, 65, 5), 130, 5, 0.05),
        ("wide_batch", (64, 96, 96, 10), 260, 10, 1.0),
    ]
    for name, sizes, b, k, eta in shapes:
        arch = nn.Architecture(sizes)
        m = nn.init_model(arch, seed=len(name))
        ds = synthetic_blobs(b, sizes[0], k, 2.5, seed=len(name) + 1)
        cases.append((name, m, ds.features, ds.labels, eta))
    # 4. a sparse (w8a-like binary) input, densified
    rs = np.random.default_rng(5)
    b, d = 50, 300
    x = np.zeros((b, d))
    for r in range(b):
        x[r, rs.choice(d, size=12, replace=False)] = 1.0
    y = rs.integers(0, 2, size=b)
    cases.append(("sparse_w8a_like", nn.init_model(nn.Architecture((300, 64, 64, 2)), seed=3), x, y, 0.7))

    out = {}
    for ci, (name, model, x, y, eta) in enumerate(cases):
        p = f"c{ci}_"
        out[p + "name"] = np.array(name)
        out[p + "sizes"] = np.array(model.arch.layer_sizes, dtype=np.int64)
        out[p + "x"] = np.ascontiguousarray(x, dtype=np.float64)
        out[p + "y"] = np.asarray(y, dtype=np.int64)
        out[p + "eta"] = np.array(eta)
        for l, w in enumerate(model.weights):
            out[p + f"w{l}"] = w.copy()
        tape = nn.forward(model, out[p + "x"])
        for l, a in enumerate(tape.per_layer[1:]):
            out[p + f"a{l + 1}"] = a
        grads = nn.backward(model, tape, out[p + "y"])
        for l, g in enumerate(grads):
            out[p + f"g{l}"] = g
        out[p + "ce"] = np.array(nn.cross_entropy_loss(tape, out[p + "y"]))
        out[p + "loss_sum"] = np.array(nn.loss_sum(model, out[p + "x"], out[p + "y"]))
        # the replica step itself (workers.py:126-138) on a copy
        merged = nn.deep_copy(model)
        batch = BatchRef(out[p + "x"], out[p + "y"], 0, out[p + "x"].shape[0])
        assert execute_batch_replica(merged, batch, eta) == 1.0
        for l, w in enumerate(merged.weights):
            out[p + f"u{l}"] = w
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(OUT / "nn_cases.npz", **out)
    return len(cases)


def data_and_init(h):
    from hogtrain.data import shuffle_epoch, synthetic_blobs
    from hogtrain.engine import epoch_shuffle_seed
    from hogtrain.nn import Architecture, InitScheme, init_model

    ds = synthetic_blobs(50, 5, 3, 2.5, seed=7)
    m = init_model(Architecture((5, 7, 3)), seed=11)
    m2 = init_model(Architecture((4, 6, 2)), seed=11, scheme=InitScheme.FAN_IN_STD)
    perm = shuffle_epoch(ds, epoch_shuffle_seed(42, 1))
    np.savez_compressed(
        OUT / "data_init.npz",
        blobs_x=ds.features, blobs_y=ds.labels,
        init_w0=m.weights[0], init_w1=m.weights[1],
        fan_w0=m2.weights[0], fan_w1=m2.weights[1],
        perm_42_1=perm,
    )


def sequential_runs(h):
    from hogtrain.data import synthetic_blobs
    from hogtrain.engine import run_training
    from hogtrain.nn import Architecture, deep_copy, init_model
    from hogtrain.policies import UniformHogbatch
    from hogtrain.workers import WorkerConfig, WorkerMode
    from helpers import sequential_minibatch_sgd

    out = {}
    runs = [
        ("blobs2", 300, 6, 2, (6, 10, 10, 2), 64, 0.5, 3, 3),
        ("blobs983", 120, 10, 983, (10, 16, 983), 32, 2.0, 2, 5),
        ("covtype_small", 1000, 54, 2, (54, 32, 32, 32, 2), 100, 0.5, 3, 42),
    ]
    for i, (name, n, dim, k, sizes, b, eta, epochs, seed) in enumerate(runs):
        p = f"r{i}_"
        ds = synthetic_blobs(n, dim, k, 2.5, seed=seed)
        model = init_model(Architecture(sizes), seed=seed)
        out[p + "name"] = np.array(name)
        out[p + "x"] = ds.features
        out[p + "y"] = ds.labels
        out[p + "sizes"] = np.array(sizes, dtype=np.int64)
        out[p + "meta"] = np.array([b, epochs, seed], dtype=np.int64)
        out[p + "eta"] = np.array(eta)
        for l, w in enumerate(model.weights):
            out[p + f"w{l}"] = w.copy()
        seq_model = deep_copy(model)
        curve = sequential_minibatch_sgd(ds, seq_model, b, eta, epochs, seed)
        out[p + "curve"] = np.array(curve)
        for l, w in enumerate(seq_model.weights):
            out[p + f"final{l}"] = w
        # the engine itself in deterministic single-worker mode
        eng_model = deep_copy(model)
        metrics = run_training(
            ds, eng_model, [WorkerConfig("w0", WorkerMode.BATCH_REPLICA, min_batch=b, max_batch=b)],
            UniformHogbatch(b, eta), epochs=epochs, seed=seed,
        )
        out[p + "engine_curve"] = np.array([s.loss for s in metrics.samples])
        out[p + "coverage"] = np.array([[c.epoch, c.start, c.length] for c in metrics.coverage])
    out["n_runs"] = np.array(len(runs))
    np.savez_compressed(OUT / "sequential.npz", **out)


def adaptive_sequences(h):
    from hogtrain.policies import AdaptiveHogbatch, FixedHeterogeneous, UniformHogbatch
    from hogtrain.workers import WorkerConfig, WorkerMode

    rng = np.random.default_rng(20240003)
    rows = []  # seq, strict, alpha, base_eta, wid_index, reported_u, batch, lr
    rosters = []
    for seq in range(200):
        alpha = float(rng.choice([1.5, 2.0, 4.0]))
        strict = bool(rng.integers(0, 2))
        base_eta = float(rng.choice([0.01, 0.02, 0.5]))
        roster = []
        for w in range(3):
            min_b = int(rng.integers(1, 64))
            max_b = min_b * int(rng.integers(1, 256))
            mode = WorkerMode.HOGWILD_SHARDED if w == 0 else WorkerMode.BATCH_REPLICA
            threads = int(rng.integers(1, 16)) if w == 0 else 1
            roster.append(WorkerConfig(f"w{w}", mode, threads=threads, min_batch=min_b, max_batch=max_b))
            rosters.append([seq, w, int(mode is WorkerMode.BATCH_REPLICA), threads, min_b, max_b])
        pol = AdaptiveHogbatch(base_eta=base_eta, alpha=alpha, strict_thresholds=strict)
        first = pol.prepare(roster)
        for w, cfg in enumerate(roster):
            d = first[cfg.worker_id]
            rows.append([seq, int(strict), alpha, base_eta, w, -1.0, d.batch_size, d.learning_rate])
        counts = [0.0, 0.0, 0.0]
        for _ in range(60):
            w = int(rng.integers(0, 3))
            counts[w] += float(rng.integers(0, 8)) * (0.25 if w == 0 else 1.0)
            d = pol.decide(f"w{w}", counts[w])
            rows.append([seq, int(strict), alpha, base_eta, w, counts[w], d.batch_size, d.learning_rate])
    # fixed heterogeneous / uniform decisions for one roster
    roster = [WorkerConfig("cpu", WorkerMode.HOGWILD_SHARDED, threads=8, min_batch=8, max_batch=8),
              WorkerConfig("gpu", WorkerMode.BATCH_REPLICA, min_batch=64, max_batch=8192)]
    fh = FixedHeterogeneous(base_eta=0.02, cpu_batch_per_thread=1, gpu_batch=8192).prepare(roster)
    un = UniformHogbatch(512, 0.1).prepare(roster)
    np.savez_compressed(
        OUT / "adaptive.npz",
        rows=np.array(rows, dtype=np.float64),
        rosters=np.array(rosters, dtype=np.int64),
        fixed=np.array([[fh["cpu"].batch_size, fh["cpu"].learning_rate],
                        [fh["gpu"].batch_size, fh["gpu"].learning_rate]]),
        uniform=np.array([[un["cpu"].batch_size, un["cpu"].learning_rate],
                          [un["gpu"].batch_size, un["gpu"].learning_rate]]),
    )


def main():
    h = _import_reference()
    n = nn_cases(h)
    data_and_init(h)
    sequential_runs(h)
    adaptive_sequences(h)
    for f in sorted(OUT.glob("*.npz")):
        print(f"{f.name}: {f.stat().st_size / 1024:.1f} KiB")
    print(f"{n} nn cases")


if __name__ == "__main__":
    main()
