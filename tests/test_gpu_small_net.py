"""The persistent small-net step (csrc/hb_small.cuh) against the float64 oracle.

With HB_SMALL_NET=1, small dense nets with a small head (covtype-class,
BASELINE configs[0]) run the whole training step as one cooperative kernel
(opt-in: the per-layer tcgen05 path is faster).  Bar: gradients and updated weights within 1e-4 under
the reference's floored metric (pkg/tests/helpers.py:29-35), loss to 1e-5.
"""

import os

import numpy as np
import pytest

from conftest import max_relative_error
from oracle import ref_nn

pytestmark = pytest.mark.gpu

STEP_TOL = 1e-4


@pytest.fixture(scope="module")
def hb():
    import paper_2004_08771_b200 as hb

    if hb.device_count() < 1:
        pytest.fail("GPU tests need a CUDA device")
    return hb


def case(sizes, b, seed, classes=None):
    rng = np.random.default_rng(seed)
    w = ref_nn.init_weights(sizes, seed)
    x, _ = ref_nn.synthetic_blobs(b, sizes[0], 2, 2.5, seed)
    y = rng.integers(0, classes or sizes[-1], size=b)
    return w, x, y


def make_ctx(hb, sizes, b, small=True):
    """A context with the fused step switched on (HB_SMALL_NET=1, read at creation) or off."""
    old = os.environ.get("HB_SMALL_NET")
    os.environ["HB_SMALL_NET"] = "1" if small else "0"
    try:
        return hb.GpuReplica(sizes, b)
    finally:
        if old is None:
            del os.environ["HB_SMALL_NET"]
        else:
            os.environ["HB_SMALL_NET"] = old


def step(hb, sizes, w, x, y, eta, small=True, bias=None, profile=False):
    ctx = make_ctx(hb, sizes, max(x.shape[0], 1), small)
    try:
        ctx.set_weights(w)
        if bias is not None:
            for l, bl in enumerate(bias):
                ctx.set_bias(l, bl)
        ctx.stage(x, y)
        if profile:
            ctx.profile(True)
        loss = ctx.step(0, x.shape[0], eta, emit_grad=True, want_loss=True)
        names = set(ctx.profile_read()) if profile else set()
        return dict(grads=ctx.grads(), weights=ctx.get_weights(), loss=loss, kernels=names)
    finally:
        ctx.close()


def oracle(w, x, y, eta, bias=None):
    if bias is None:
        tape = ref_nn.forward(w, x)
    else:  # forward with a fixed per-unit offset on the hidden layers
        tape = [x]
        s = x
        for l, wl in enumerate(w):
            z = s @ wl.T
            if l < len(w) - 1:
                s = ref_nn.sigmoid(z + bias[l])
            else:
                s = ref_nn.softmax_rows(z)
            tape.append(s)
    g = ref_nn.backward(w, tape, y)
    u = ref_nn.deep_copy(w)
    ref_nn.apply_update(u, g, eta)
    return g, u, ref_nn.cross_entropy_loss(tape, y)


@pytest.mark.parametrize("seed", range(5))
def test_covtype_config_step(hb, seed):
    sizes, b = (54, 512, 512, 512, 2), 512
    w, x, y = case(sizes, b, 100 + seed)
    g, u, ce = oracle(w, x, y, 0.5)
    out = step(hb, sizes, w, x, y, 0.5, profile=True)
    assert "small_net_step_l0" in out["kernels"], out["kernels"]
    assert max_relative_error(out["grads"], g) <= STEP_TOL
    assert max_relative_error(out["weights"], u) <= STEP_TOL
    assert out["loss"] == pytest.approx(ce, rel=1e-5)


@pytest.mark.parametrize(
    "sizes,b,eta",
    [
        ((54, 128, 2), 300, 0.5),          # one hidden layer (head dW beside nothing)
        ((37, 96, 3), 129, 0.1),           # odd widths, 3 classes
        ((300, 256, 256, 4), 1024, 0.3),   # 4 classes, the largest fused batch
        ((54, 512, 512, 512, 2), 1, 0.5),  # one-row batch
        ((54, 512, 512, 512, 2), 65, 0.5), # M tail
        ((1000, 1024, 1024, 2), 256, 0.2), # widest fused layers
        ((20, 33, 17, 9, 5, 7, 11, 3), 77, 0.4),  # deep and ragged
    ],
)
def test_shapes(hb, sizes, b, eta):
    w, x, y = case(sizes, b, sum(sizes) + b)
    g, u, ce = oracle(w, x, y, eta)
    out = step(hb, sizes, w, x, y, eta, profile=True)
    assert "small_net_step_l0" in out["kernels"]
    assert max_relative_error(out["grads"], g) <= STEP_TOL
    assert max_relative_error(out["weights"], u) <= STEP_TOL
    assert out["loss"] == pytest.approx(ce, rel=1e-5)


def test_bias(hb):
    sizes, b = (54, 256, 256, 2), 400
    w, x, y = case(sizes, b, 5)
    rng = np.random.default_rng(6)
    bias = [rng.normal(0, 0.3, size=sizes[l + 1]) for l in range(len(sizes) - 2)]
    g, u, ce = oracle(w, x, y, 0.3, bias=bias)
    out = step(hb, sizes, w, x, y, 0.3, bias=bias, profile=True)
    assert "small_net_step_l0" in out["kernels"]
    assert max_relative_error(out["grads"], g) <= STEP_TOL
    assert max_relative_error(out["weights"], u) <= STEP_TOL


def test_per_layer_path_agrees_and_is_switchable(hb):
    sizes, b = (54, 512, 512, 512, 2), 512
    w, x, y = case(sizes, b, 77)
    fused = step(hb, sizes, w, x, y, 0.5, small=True, profile=True)
    layered = step(hb, sizes, w, x, y, 0.5, small=False, profile=True)
    assert "small_net_step_l0" in fused["kernels"]
    assert "small_net_step_l0" not in layered["kernels"]
    assert max_relative_error(fused["grads"], layered["grads"]) <= STEP_TOL
    assert fused["loss"] == pytest.approx(layered["loss"], rel=1e-5)


def test_deterministic_and_graph_replay(hb):
    """Eager first step, graph-replayed steps after: every step bit-identical
    to a fresh context's, and a chain of steps tracks the oracle."""
    sizes, b, eta = (54, 512, 512, 512, 2), 512, 0.5
    w, x, y = case(sizes, 4 * b, 9)
    ctx = make_ctx(hb, sizes, b)
    ctx.set_weights(w)
    ctx.stage(x, y)
    ref = ref_nn.deep_copy(w)
    for i in range(4):
        ctx.step(i * b, b, eta)
        tape = ref_nn.forward(ref, x[i * b:(i + 1) * b])
        ref_nn.apply_update(ref, ref_nn.backward(ref, tape, y[i * b:(i + 1) * b]), eta)
    got = ctx.get_weights()
    ctx.close()
    assert max_relative_error(got, ref) <= STEP_TOL
    ctx = make_ctx(hb, sizes, b)
    ctx.set_weights(w)
    ctx.stage(x, y)
    for i in range(4):
        ctx.step(i * b, b, eta)
    again = ctx.get_weights()
    ctx.close()
    for p, q in zip(got, again):
        assert np.array_equal(p, q)


def test_replica_step_through_the_fused_kernel(hb):
    """execute_gpu_replica semantics (snapshot, step, float64 stale merge into
    the host model) with the fused step inside."""
    sizes, b, eta = (54, 256, 256, 2), 300, 0.3
    w, x, y = case(sizes, b, 21)
    host = [np.array(a, dtype=np.float64, order="C") for a in w]
    g = ref_nn.backward(w, ref_nn.forward(w, x), y)
    ctx = make_ctx(hb, sizes, b)
    ctx.stage(x, y)
    ctx.profile(True)
    ctx.replica_step(host, 0, b, eta)
    names = set(ctx.profile_read())
    ctx.close()
    assert "small_net_step_l0" in names
    assert max_relative_error(host, [a - eta * gl for a, gl in zip(w, g)]) <= STEP_TOL
