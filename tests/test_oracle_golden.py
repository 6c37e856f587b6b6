"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz)
and the reference's inline known-answer tests."""

import math

import numpy as np
import pytest

from conftest import GOLDEN, load_runs
from oracle import ref_nn, ref_policies


class TestKnownAnswers:
    """Inline KATs of pkg/tests/test_linalg.py and test_nn.py."""

    def test_sigmoid_values(self):
        assert ref_nn.sigmoid(np.array([[0.0]]))[0, 0] == 0.5  # test_linalg.py:63
        v = ref_nn.sigmoid(np.array([[-100.0]]))[0, 0]
        assert 0.0 < v <= 1e-40  # test_linalg.py:67-70
        assert ref_nn.sigmoid(np.array([[1.0]]))[0, 0] == pytest.approx(0.7310585786, abs=1e-10)

    def test_deriv_and_softmax(self):
        assert ref_nn.sigmoid_deriv_from_output(np.array([[0.7310585786]]))[0, 0] == pytest.approx(
            0.1966119332, abs=1e-10)
        out = ref_nn.softmax_rows(np.array([[1.0, 2.0, 3.0]]))
        assert np.abs(out[0] - [0.09003057, 0.24472847, 0.66524096]).max() <= 1e-8

    def test_gemm_and_ce(self):
        assert np.array_equal(ref_nn.gemm(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[5.0], [6.0]])),
                              [[17.0], [39.0]])
        with pytest.raises(ValueError, match="dimension mismatch"):
            ref_nn.gemm(np.ones((2, 3)), np.ones((4, 2)))
        tape = [None, np.array([[0.7, 0.3]])]
        assert ref_nn.cross_entropy_loss(tape, np.array([0])) == pytest.approx(0.356675, abs=1e-6)
        tape = [None, np.array([[1.0, 0.0]])]
        assert ref_nn.cross_entropy_loss(tape, np.array([1])) == pytest.approx(-math.log(1e-12), rel=1e-9)


class TestGoldenNN:
    def test_forward_backward_update_bitwise(self, golden_cases):
        for c in golden_cases:
            tape = ref_nn.forward(c["w"], c["x"])
            for l, a in enumerate(c["a"]):
                assert np.abs(tape[l + 1] - a).max() <= 1e-12, (c["name"], l)
            grads = ref_nn.backward(c["w"], tape, c["y"])
            for l, g in enumerate(c["g"]):
                assert np.abs(grads[l] - g).max() <= 1e-12, (c["name"], l)
            w = ref_nn.deep_copy(c["w"])
            ref_nn.replica_step(w, c["x"], c["y"], c["eta"])
            for l, u in enumerate(c["u"]):
                assert np.abs(w[l] - u).max() <= 1e-12, (c["name"], l)
            assert ref_nn.cross_entropy_loss(tape, c["y"]) == pytest.approx(c["ce"], abs=1e-12)
            assert ref_nn.loss_sum(c["w"], c["x"], c["y"]) == pytest.approx(c["loss_sum"], abs=1e-10)

    def test_hand_case_present(self, golden_cases):
        assert golden_cases[0]["name"] == "hand232"
        assert len(golden_cases) >= 10


class TestGoldenData:
    def test_blobs_init_shuffle(self):
        z = np.load(GOLDEN / "data_init.npz")
        x, y = ref_nn.synthetic_blobs(50, 5, 3, 2.5, seed=7)
        assert np.array_equal(x, z["blobs_x"]) and np.array_equal(y, z["blobs_y"])
        w = ref_nn.init_weights((5, 7, 3), seed=11)
        assert np.array_equal(w[0], z["init_w0"]) and np.array_equal(w[1], z["init_w1"])
        w = ref_nn.init_weights((4, 6, 2), seed=11, fan_in_std=True)
        assert np.array_equal(w[0], z["fan_w0"])
        assert np.array_equal(ref_nn.shuffle_epoch(50, (42, 1)), z["perm_42_1"])


class TestGoldenSequential:
    def test_curves_bitwise(self):
        for r in load_runs():
            x, y = ref_nn.synthetic_blobs(r["x"].shape[0], r["x"].shape[1], int(r["sizes"][-1]), 2.5, seed=r["seed"])
            assert np.array_equal(x, r["x"])
            w = ref_nn.deep_copy(r["w"])
            curve = ref_nn.sequential_minibatch_sgd(r["x"], r["y"], w, r["batch"], r["eta"], r["epochs"], r["seed"])
            assert np.array_equal(np.array(curve), r["curve"]), r["name"]
            # the engine's single-worker mode equals the sequential oracle (test_engine.py:160-185)
            assert np.array_equal(r["curve"], r["engine_curve"]), r["name"]
            for a, b in zip(w, r["final"]):
                assert np.array_equal(a, b)


class TestGoldenAdaptive:
    def test_sequences(self):
        z = np.load(GOLDEN / "adaptive.npz")
        rows, rosters = z["rows"], z["rosters"]
        by_seq = {}
        for r in rosters:
            by_seq.setdefault(int(r[0]), []).append(r)
        states = {}
        for row in rows:
            seq, strict, alpha, base_eta, w, u, batch, lr = row
            seq, w = int(seq), int(w)
            roster = by_seq[seq]
            if seq not in states:
                st = ref_policies.OracleAdaptive(alpha)
                ref_b = min(int(r[4]) for r in roster)
                for r in roster:
                    b0 = ref_policies.initial_batch_size(bool(r[2]), int(r[3]), int(r[4]), int(r[5]))
                    st.register(f"w{int(r[1])}", b0, int(r[4]), int(r[5]))
                states[seq] = (st, ref_b)
            st, ref_b = states[seq]
            if u < 0:  # prepare() decision
                got = st.slots[f"w{w}"][0]
            else:
                got = st.update(f"w{w}", u, strict=bool(strict))
            assert got == int(batch)
            assert ref_policies.scaled_learning_rate(base_eta, got, ref_b) == lr
