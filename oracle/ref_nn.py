"""Float64 NumPy restatement of the reference MLP math (test oracle only).

Each function cites the reference line range it restates.  Layout is the
reference's: a batch is (examples x features); weights[l] is (d_{l+1}, d_l)
(`nn.py:3-7`, `nn.py:70-78`); no bias (`SPEC.md:89`).
"""

from __future__ import annotations

import numpy as np

PROB_FLOOR = 1e-12  # nn.py:26


# ---------------------------------------------------------------- linalg.py
def gemm(a, b, transpose_a=False, transpose_b=False):
    """op(a) @ op(b) with the reference's shape check (linalg.py:31-45)."""
    lhs = a.T if transpose_a else a
    rhs = b.T if transpose_b else b
    if lhs.shape[1] != rhs.shape[0]:
        raise ValueError(f"gemm dimension mismatch: {lhs.shape} x {rhs.shape}")
    return lhs @ rhs


def sigmoid(m):
    """Two-branch stable logistic (linalg.py:48-55)."""
    out = np.empty_like(m, dtype=np.float64)
    pos = m >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-m[pos]))
    e = np.exp(m[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def sigmoid_deriv_from_output(s):
    """s * (1 - s) (linalg.py:58-60)."""
    return s * (1.0 - s)


def softmax_rows(m):
    """Row-max-shifted softmax (linalg.py:63-67)."""
    shifted = m - m.max(axis=1, keepdims=True)
    e = np.exp(shifted)
    return e / e.sum(axis=1, keepdims=True)


def axpy_in_place(target, source, scale):
    """target += scale * source, in place (linalg.py:70-79)."""
    if target.shape != source.shape:
        raise ValueError(f"axpy shape mismatch: {target.shape} vs {source.shape}")
    np.add(target, scale * source, out=target)


# -------------------------------------------------------------------- nn.py
def init_weights(layer_sizes, seed, fan_in_std=False):
    """Gaussian init, std 1/sqrt(fan_in) (or fan_in) (nn.py:96-105)."""
    rng = np.random.default_rng(seed)
    weights = []
    for l in range(len(layer_sizes) - 1):
        fan_in, fan_out = layer_sizes[l], layer_sizes[l + 1]
        std = float(fan_in) if fan_in_std else 1.0 / np.sqrt(fan_in)
        weights.append(rng.normal(0.0, std, size=(fan_out, fan_in)))
    return weights


def forward(weights, x):
    """Per layer z = state @ W^T; sigmoid hidden, softmax last (nn.py:108-121).

    Returns the activation tape [x, A_1, ..., P]."""
    if x.ndim != 2 or x.shape[1] != weights[0].shape[1]:
        raise ValueError(f"batch shape {x.shape} incompatible with input dim {weights[0].shape[1]}")
    layers = [x]
    state = x
    last = len(weights) - 1
    for l, w in enumerate(weights):
        z = gemm(state, w, transpose_b=True)
        state = softmax_rows(z) if l == last else sigmoid(z)
        layers.append(state)
    return layers


def cross_entropy_loss(tape, labels):
    """Mean -log max(p_y, 1e-12) (nn.py:124-136)."""
    probs = tape[-1]
    labels = np.asarray(labels)
    if labels.shape[0] != probs.shape[0]:
        raise ValueError("label count does not match batch size")
    if labels.min() < 0 or labels.max() >= probs.shape[1]:
        raise ValueError("labels out of range")
    picked = probs[np.arange(probs.shape[0]), labels]
    return float(-np.log(np.maximum(picked, PROB_FLOOR)).mean())


def loss_sum(weights, features, labels, chunk=4096):
    """Sum of per-example CE over a slice, in chunks of 4096 (nn.py:139-146)."""
    total = 0.0
    for start in range(0, features.shape[0], chunk):
        stop = min(start + chunk, features.shape[0])
        tape = forward(weights, features[start:stop])
        total += cross_entropy_loss(tape, labels[start:stop]) * (stop - start)
    return total


def output_delta(probs, labels):
    """delta = (P - onehot(y)) / n, the fused softmax/CE error (nn.py:162-164)."""
    n = probs.shape[0]
    delta = probs.copy()
    delta[np.arange(n), np.asarray(labels)] -= 1.0
    delta /= n
    return delta


def backward(weights, tape, labels):
    """Mean-CE gradient for every layer (nn.py:149-171).

    dW_l = delta_l^T A_l; for l > 0, delta_{l-1} = (delta_l W_l) * A_l (1 - A_l);
    no input gradient for l = 0 (nn.py:169)."""
    labels = np.asarray(labels)
    if labels.shape[0] != tape[-1].shape[0]:
        raise ValueError("label count does not match batch size")
    delta = output_delta(tape[-1], labels)
    grads = [None] * len(weights)
    for l in range(len(weights) - 1, -1, -1):
        grads[l] = gemm(delta, tape[l], transpose_a=True)
        if l > 0:
            delta = gemm(delta, weights[l]) * sigmoid_deriv_from_output(tape[l])
    return grads


def backward_deltas(weights, tape, labels):
    """The per-layer error signals backward() walks through (nn.py:162-170):
    deltas[l] is the error at the output of layer l (shape (b, d_{l+1}))."""
    delta = output_delta(tape[-1], labels)
    deltas = [None] * len(weights)
    for l in range(len(weights) - 1, -1, -1):
        deltas[l] = delta
        if l > 0:
            delta = gemm(delta, weights[l]) * sigmoid_deriv_from_output(tape[l])
    return deltas


def apply_update(weights, grads, eta):
    """W^l -= eta * g^l in place (nn.py:174-179)."""
    if len(grads) != len(weights):
        raise ValueError("gradient layer count does not match model")
    for w, g in zip(weights, grads):
        axpy_in_place(w, g, -eta)


def deep_copy(weights):
    """Independent snapshot (nn.py:182-184)."""
    return [np.array(w, copy=True) for w in weights]


def replica_step(weights, x, y, eta):
    """execute_batch_replica without the sleep (workers.py:126-138): gradient
    on a deep-copied snapshot, then a stale merge into `weights` in place.
    Returns the gradients (for per-step parity checks)."""
    replica = deep_copy(weights)
    tape = forward(replica, x)
    grads = backward(replica, tape, y)
    apply_update(weights, grads, eta)
    return grads


# ----------------------------------------------------- data.py / engine.py
def synthetic_blobs(n, dim, classes, separation, seed):
    """Gaussian class clusters, rows shuffled (data.py:226-252).
    Returns (features float64 (n, dim), labels int64 (n,))."""
    if classes < 2:
        raise ValueError("need at least 2 classes")
    rng = np.random.default_rng(seed)
    raw = rng.normal(size=(classes, dim))
    raw -= raw.mean(axis=0)
    if separation > 0:
        dists = [np.linalg.norm(raw[i] - raw[j]) for i in range(classes) for j in range(i + 1, classes)]
        means = raw * (separation / min(dists))
    else:
        means = np.zeros_like(raw)
    labels = np.arange(n, dtype=np.int64) % classes
    features = means[labels] + rng.normal(size=(n, dim))
    perm = rng.permutation(n)
    return np.ascontiguousarray(features[perm]), labels[perm].copy()


def shuffle_epoch(n, seed):
    """Per-epoch permutation (data.py:182-184), seeded (run_seed, epoch)
    (engine.py:74-76)."""
    return np.random.default_rng(seed).permutation(n)


def sequential_minibatch_sgd(features, labels, weights, batch_size, eta, epochs, run_seed):
    """Deterministic single-worker schedule (tests/helpers.py:54-74, which
    mirrors engine.py:214-316 with one replica worker and drain_tail):
    per-epoch reshuffle, contiguous batches, short tail, loss sampled before
    training and after each epoch.  Mutates `weights`; returns the curve."""
    n = features.shape[0]
    losses = [loss_sum(weights, features, labels) / n]
    for epoch in range(epochs):
        perm = shuffle_epoch(n, (run_seed, epoch))
        ex = np.ascontiguousarray(features[perm])
        ey = labels[perm].copy()
        for start in range(0, n, batch_size):
            stop = min(start + batch_size, n)
            tape = forward(weights, ex[start:stop])
            grads = backward(weights, tape, ey[start:stop])
            apply_update(weights, grads, eta)
        losses.append(loss_sum(weights, features, labels) / n)
    return losses
