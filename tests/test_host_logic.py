"""Host-side logic of the drop-in surface (no GPU): data layouts and
generators, model layout, worker config, the batch-size controller, bench
work accounting.  Pinned to the reference's golden vectors where they exist."""

import numpy as np
import pytest

import paper_2004_08771_b200 as hb
from conftest import GOLDEN, load_runs
from oracle import ref_nn
from paper_2004_08771_b200 import policies as P


class TestGeneratorsMatchReference:
    def test_blobs_init_shuffle_identical_draws(self):
        z = np.load(GOLDEN / "data_init.npz")
        ds = hb.synthetic_blobs(50, 5, 3, 2.5, seed=7)
        assert np.array_equal(ds.features, z["blobs_x"]) and np.array_equal(ds.labels, z["blobs_y"])
        m = hb.init_model(hb.Architecture((5, 7, 3)), seed=11)
        assert np.array_equal(m.weights[0], z["init_w0"]) and np.array_equal(m.weights[1], z["init_w1"])
        m2 = hb.init_model(hb.Architecture((4, 6, 2)), seed=11, scheme=hb.InitScheme.FAN_IN_STD)
        assert np.array_equal(m2.weights[0], z["fan_w0"])
        assert np.array_equal(hb.shuffle_epoch(50, hb.epoch_shuffle_seed(42, 1)), z["perm_42_1"])

    def test_blobs_runs(self):
        for r in load_runs():
            ds = hb.synthetic_blobs(r["x"].shape[0], r["x"].shape[1], r["sizes"][-1], 2.5, seed=r["seed"])
            assert np.array_equal(ds.features, r["x"]) and np.array_equal(ds.labels, r["y"])


class TestModelLayout:
    def test_validation_mirrors_reference(self):
        with pytest.raises(ValueError):
            hb.Architecture((5,))
        with pytest.raises(ValueError):
            hb.Architecture((5, 0, 2))
        arch = hb.Architecture((3, 4, 2))
        with pytest.raises(ValueError):
            hb.Model(arch, [np.zeros((4, 3))])
        with pytest.raises(ValueError):
            hb.Model(arch, [np.zeros((3, 4)), np.zeros((2, 4))])
        m = hb.Model(arch, [np.zeros((4, 3)), np.zeros((2, 4))])
        c = hb.deep_copy(m)
        c.weights[0][0, 0] = 1.0
        assert m.weights[0][0, 0] == 0.0

    def test_batchref_bounds(self):
        x = np.zeros((10, 3))
        y = np.zeros(10, dtype=np.int64)
        b = hb.BatchRef(x, y, 4, 6)
        assert b.x.shape == (6, 3) and np.shares_memory(b.x, x)
        with pytest.raises(ValueError):
            hb.BatchRef(x, y, 5, 6)
        with pytest.raises(ValueError):
            hb.BatchRef(x, y, 0, 0)


class TestCsr:
    def test_w8a_shape_generator(self):
        d = hb.synthetic_csr(2000, 300, 12, 2, seed=1)
        assert d.nnz == 2000 * 12 and d.col.dtype == np.int32 and d.rowptr.dtype == np.int64
        for r in range(0, 2000, 97):
            cols = d.col[d.rowptr[r]:d.rowptr[r + 1]]
            assert np.all(np.diff(cols) > 0)  # sorted, distinct
        assert set(np.unique(d.val)) == {1.0}
        assert 0.2 < d.labels.mean() < 0.8
        again = hb.synthetic_csr(2000, 300, 12, 2, seed=1)
        assert np.array_equal(again.col, d.col) and np.array_equal(again.labels, d.labels)

    def test_realsim_shape_generator_normalised(self):
        d = hb.synthetic_csr(500, 20958, 52, 2, seed=2, binary=False, normalize=True)
        norms = np.sqrt(np.add.reduceat(d.val ** 2, d.rowptr[:-1]))
        assert np.allclose(norms, 1.0)
        assert d.col.max() < 20958

    def test_reorder_and_dense_twin(self):
        d = hb.synthetic_csr(300, 50, 5, 3, seed=3, binary=False)
        perm = hb.shuffle_epoch(300, (7, 0))
        r = hb.reorder(d, perm)
        assert np.array_equal(r.dense(), d.dense()[perm])
        assert np.array_equal(r.labels, d.labels[perm])
        sub = r.rows(10, 40)
        assert np.array_equal(sub.dense(), r.dense(10, 40))
        b = hb.CsrBatchRef(r, 10, 30)
        assert np.array_equal(b.x, r.dense()[10:40]) and np.array_equal(b.y, r.labels[10:40])

    def test_validation(self):
        with pytest.raises(ValueError):
            hb.CsrDataset(np.array([0, 2]), np.array([0, 5]), np.ones(2), np.array([0]), 5)
        with pytest.raises(ValueError):
            hb.CsrDataset(np.array([1, 2]), np.array([0]), np.ones(1), np.array([0]), 5)


class TestWorkerConfig:
    def test_gpu_mode_and_invariants(self):
        cfg = hb.WorkerConfig("gpu0", hb.WorkerMode.GPU_REPLICA, min_batch=64, max_batch=8192, device=3)
        assert cfg.replica_mode.value == "deep_copy" and cfg.device == 3
        with pytest.raises(ValueError):
            hb.WorkerConfig("g", hb.WorkerMode.GPU_REPLICA, min_batch=10, max_batch=5)
        with pytest.raises(ValueError):
            hb.WorkerConfig("g", hb.WorkerMode.GPU_REPLICA, device=-1)
        assert hb.WorkerMode("gpu_replica") is hb.WorkerMode.GPU_REPLICA


class TestController:
    def test_adaptive_matches_reference_sequences(self):
        z = np.load(GOLDEN / "adaptive.npz")
        rows, rosters = z["rows"], z["rosters"]
        by_seq = {}
        for r in rosters:
            by_seq.setdefault(int(r[0]), []).append(r)
        pols = {}
        for row in rows:
            seq, strict, alpha, base_eta, w, u, batch, lr = row
            seq, w = int(seq), int(w)
            if seq not in pols:
                roster = [hb.WorkerConfig(f"w{int(r[1])}",
                                          hb.WorkerMode.BATCH_REPLICA if r[2] else hb.WorkerMode.HOGWILD_SHARDED,
                                          threads=int(r[3]), min_batch=int(r[4]), max_batch=int(r[5]))
                          for r in by_seq[seq]]
                pol = hb.AdaptiveHogbatch(base_eta=base_eta, alpha=alpha, strict_thresholds=bool(strict))
                pols[seq] = (pol, pol.prepare(roster))
            pol, first = pols[seq]
            d = first[f"w{w}"] if u < 0 else pol.decide(f"w{w}", u)
            assert d.batch_size == int(batch) and d.learning_rate == lr

    def test_fixed_and_uniform(self):
        z = np.load(GOLDEN / "adaptive.npz")
        roster = [hb.WorkerConfig("cpu", hb.WorkerMode.HOGWILD_SHARDED, threads=8, min_batch=8, max_batch=8),
                  hb.WorkerConfig("gpu", hb.WorkerMode.GPU_REPLICA, min_batch=64, max_batch=8192)]
        fh = hb.FixedHeterogeneous(base_eta=0.02, cpu_batch_per_thread=1, gpu_batch=8192).prepare(roster)
        assert [[fh["cpu"].batch_size, fh["cpu"].learning_rate], [fh["gpu"].batch_size, fh["gpu"].learning_rate]] \
            == z["fixed"].tolist()
        un = hb.UniformHogbatch(512, 0.1).prepare(roster)
        assert un["gpu"].batch_size == 512 and un["cpu"].learning_rate == 0.1

    def test_device_speed_feed(self):
        feed = hb.DeviceSpeedFeed()
        assert feed.eval_slices(["a", "b"], 10) == [("a", 0, 5), ("b", 5, 5)]
        feed.record("a", 8192, 1.0)  # 8.192M ex/s
        feed.record("b", 100, 1.0)  # 0.1M ex/s
        feed.record("a", 8192, 2.0)  # EWMA 0.5/0.5 (engine.py:318-328)
        assert feed.speed["a"] == pytest.approx(0.5 * 8192e3 + 0.5 * 4096e3)
        sl = feed.eval_slices(["a", "b"], 1000)
        assert sum(s[2] for s in sl) == 1000 and sl[0][2] > 900

    def test_policy_errors(self):
        with pytest.raises(ValueError):
            hb.UniformHogbatch(0, 0.1)
        st = hb.AdaptiveState(alpha=2.0)
        with pytest.raises(ValueError):
            hb.AdaptiveState(alpha=1.0)
        st.register(hb.WorkerConfig("g", hb.WorkerMode.GPU_REPLICA, min_batch=64, max_batch=8192))
        assert st.workers["g"].batch_size == 8192
        hb.adaptive_update(st, "g", 5.0)
        with pytest.raises(ValueError, match="backwards"):
            hb.adaptive_update(st, "g", 4.0)


class TestBenchAccounting:
    def test_flops_per_sample_match_survey(self):
        import bench

        # MFLOP/sample
        assert bench.dense_flops_per_sample((54, 512, 512, 512, 2), False) / 1e6 == pytest.approx(3.262, abs=1e-3)
        assert bench.dense_flops_per_sample((500, 1024, 1024, 983), False) / 1e6 == pytest.approx(14.379, abs=1e-3)
        assert bench.dense_flops_per_sample((1024, 4096, 4096, 4096, 1000), False) / 1e6 == pytest.approx(
            242.680, abs=1e-3)
        assert bench.dense_flops_per_sample((300, 512, 512, 512, 2), True) / 1e6 == pytest.approx(3.152, abs=2e-3)

    def test_cpu_legs_run(self):
        import bench

        cfg = dict(bench.CONFIGS["w8a"], n=2048, batch=128)
        data = bench.make_data(cfg, 1, n=2048)

        def rows_fn(s, r):
            s = s % max(1, data.n_examples - r)
            return data.dense(s, s + r), data.labels[s:s + r]

        r = bench.cpu_replica_rate(cfg, rows_fn, budget_s=0.5, max_steps=2, seed=1)
        assert r["value"] > 0 and r["steps"] >= 1 and r["rows_per_step"] == 128
        h = bench.cpu_hogbatch_run(cfg, rows_fn, budget_s=0.3, seed=1, threads=2)
        assert h["value"] > 0 and h["threads"] == 2 and h["samples"] % 128 == 0
        assert h["eta_per_shard"] == pytest.approx(cfg["eta"] * 64 / 128)

    def test_hogbatch_port_matches_reference_split(self):
        from oracle import ref_hogbatch

        # workers.py:80-91: remainder one-extra on the leading shards
        assert ref_hogbatch.split_batch(10, 3) == [(0, 4), (4, 3), (7, 3)]
        assert ref_hogbatch.split_batch(2, 4) == [(0, 1), (1, 1)]
        # one shard == one sequential step on the shared model
        w1 = ref_nn.init_weights((6, 5, 2), 3)
        w2 = ref_nn.deep_copy(w1)
        x, y = ref_nn.synthetic_blobs(16, 6, 2, 2.0, 4)
        assert ref_hogbatch.execute_hogwild_sharded(w1, x, y, 1, 0.1) == 1.0
        ref_nn.apply_update(w2, ref_nn.backward(w2, ref_nn.forward(w2, x), y), 0.1)
        for a, b in zip(w1, w2):
            np.testing.assert_array_equal(a, b)

    def test_bench_defaults_to_headline_config(self):
        import bench

        # BASELINE.json configs[4]: the 1/2/4/8-GPU scaled config at its full 10M rows
        assert bench.DEFAULT_CONFIG == "scaled"
        c = bench.CONFIGS["scaled"]
        assert c["n"] == 10_000_000 and c["sizes"] == (1024, 4096, 4096, 4096, 1000) and c["batch"] == 8192

    def test_oracle_replica_step_is_the_reference(self):
        # the CPU baseline times exactly the pinned oracle step
        w = ref_nn.init_weights((6, 5, 2), 1)
        x, y = ref_nn.synthetic_blobs(20, 6, 2, 2.0, 2)
        g = ref_nn.replica_step(w, x, y, 0.1)
        assert len(g) == 2
