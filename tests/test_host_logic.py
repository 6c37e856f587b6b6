"""Host-side logic of the drop-in surface (no GPU): data layouts and
generators, model layout, worker config, the batch-size controller, bench
work accounting.  Pinned to the reference's golden vectors where they exist."""

from pathlib import Path

import numpy as np
import pytest

import paper_2004_08771_b200 as hb
from conftest import GOLDEN, load_runs
from oracle import ref_nn


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
    def test_device_speed_feed(self):
        feed = hb.DeviceSpeedFeed()
        assert feed.eval_slices(["a", "b"], 10) == [("a", 0, 5), ("b", 5, 5)]
        feed.record("a", 8192, 1.0)  # 8.192M ex/s
        feed.record("b", 100, 1.0)  # 0.1M ex/s
        feed.record("a", 8192, 2.0)  # EWMA 0.5/0.5 (engine.py:318-328)
        assert feed.speed["a"] == pytest.approx(0.5 * 8192e3 + 0.5 * 4096e3)
        sl = feed.eval_slices(["a", "b"], 1000)
        assert sum(s[2] for s in sl) == 1000 and sl[0][2] > 900

    def test_seam_routes_by_worker_thread(self):
        """install(devices=...) maps the reference's worker threads
        ("worker-<id>", workers.py:154) to GPUs, and only GPU worker threads
        evaluate on the GPU (CPU Hogwild workers keep the reference loss_sum)."""
        import threading

        from paper_2004_08771_b200 import workers as W

        seen = {}

        def probe():
            seen[threading.current_thread().name] = (W._thread_device(), W.is_gpu_thread())

        W.set_worker_devices({"gpu0": 0, "gpu1": 1})
        try:
            for name in ("worker-gpu0", "worker-gpu1", "worker-cpu", "main-ish"):
                t = threading.Thread(target=probe, name=name)
                t.start()
                t.join()
            calls = []
            routed = W.routed_loss_sum(lambda m, x, y: calls.append(threading.current_thread().name) or 1.5)
            t = threading.Thread(target=lambda: calls.append(routed(None, None, None)), name="worker-cpu")
            t.start()
            t.join()
        finally:
            W.set_worker_devices({})
        assert seen == {"worker-gpu0": (0, True), "worker-gpu1": (1, True), "worker-cpu": (None, False),
                        "main-ish": (None, False)}
        assert calls == ["worker-cpu", 1.5]


class TestReferenceEngineSeam:
    """The device-timed accounting wrapped around the reference's own engine
    (imported from /root/reference in this container; skipped elsewhere)."""

    def test_device_timed_busy_and_speed(self, monkeypatch):
        ref_src = Path("/root/reference/pkg/src")
        if not ref_src.exists():
            pytest.skip("reference package not present")
        monkeypatch.syspath_prepend(str(ref_src))
        import hogtrain
        import hogtrain.engine as E
        import hogtrain.workers as RW

        from paper_2004_08771_b200 import workers as W

        monkeypatch.setattr(RW.WorkerThread, "_execute", RW.WorkerThread._execute)
        monkeypatch.setattr(E._Coordinator, "_update_speed", E._Coordinator._update_speed)
        ref_step = RW.execute_batch_replica
        feed = hb.DeviceSpeedFeed()
        monkeypatch.setattr(W, "_speed_feed", feed)

        def device_step(model, batch, eta, speed_factor=0.0):
            # the reference's own CPU step, booked as a 2 ms device step: the
            # booking is what execute_gpu_replica does after hb_replica_step
            out = ref_step(model, batch, eta, speed_factor)
            W.book_device_step(batch.length, 2.0)
            return out

        monkeypatch.setattr(RW, "execute_batch_replica", device_step)
        hb.device_timed(RW, E, feed)
        hb.device_timed(RW, E, feed)  # idempotent
        speeds = []
        wrapped = E._Coordinator._update_speed

        def spy(self, wid):
            wrapped(self, wid)
            speeds.append(self.speed.get(wid))

        monkeypatch.setattr(E._Coordinator, "_update_speed", spy)
        ds = hogtrain.data.synthetic_blobs(600, 6, 2, 2.5, seed=1)
        model = hogtrain.nn.init_model(hogtrain.nn.Architecture((6, 8, 2)), seed=2)
        roster = [RW.WorkerConfig("gpu0", RW.WorkerMode.BATCH_REPLICA, min_batch=50, max_batch=100)]
        m = hogtrain.run_training(ds, model, roster, hogtrain.policies.UniformHogbatch(100, 0.1), epochs=2, seed=3)
        steps = m.per_worker_updates["gpu0"]
        assert steps == 12
        assert m.per_worker_busy_ms["gpu0"] == pytest.approx(2.0 * steps)
        assert feed.speed["gpu0"] == pytest.approx(100 / 2e-3)
        assert speeds[-1] == pytest.approx(100 / 2e-3)


    def test_pipelined_worker_keeps_the_reference_curve(self, monkeypatch):
        """feed.pipelined answers the coordinator while the step runs and lands
        the merge afterwards.  With a deterministic single worker
        the loss curve and final model must equal the reference's own run
        bit for bit -- including evaluations the coordinator starts right after
        the early reply (it waits for in-flight merges first)."""
        import threading
        import time as _time

        ref_src = Path("/root/reference/pkg/src")
        if not ref_src.exists():
            pytest.skip("reference package not present")
        monkeypatch.syspath_prepend(str(ref_src))
        import hogtrain
        import hogtrain.engine as E
        import hogtrain.workers as RW

        from paper_2004_08771_b200 import workers as W

        def run():
            ds = hogtrain.data.synthetic_blobs(900, 6, 2, 2.5, seed=1)
            model = hogtrain.nn.init_model(hogtrain.nn.Architecture((6, 8, 2)), seed=2)
            roster = [RW.WorkerConfig("gpu0", RW.WorkerMode.BATCH_REPLICA, min_batch=64, max_batch=64)]
            m = hogtrain.run_training(ds, model, roster, hogtrain.policies.UniformHogbatch(64, 0.3), epochs=3,
                                      seed=3, loss_every_batches=4)
            return [s.loss for s in m.samples], model.weights, m

        ref_curve, ref_w, _ = run()
        ref_step = RW.execute_batch_replica
        tls = threading.local()

        def begin(model, batch, eta):
            tls.args = (model, batch, eta)

        def end():
            _time.sleep(0.003)  # the merge lands well after the early reply
            ref_step(*tls.args)
            W.book_device_step(tls.args[1].length, 1.0)
            return 1e-3

        monkeypatch.setattr(RW.WorkerThread, "_execute", RW.WorkerThread._execute)
        monkeypatch.setattr(E._Coordinator, "_evaluate_and_sample", E._Coordinator._evaluate_and_sample)
        monkeypatch.setattr(RW, "execute_batch_replica", W.execute_gpu_replica)
        monkeypatch.setattr(W, "execute_gpu_replica_begin", begin)
        monkeypatch.setattr(W, "execute_gpu_replica_end", end)
        inflight = {"n": 0}
        orig_begin = begin

        def counting_begin(model, batch, eta):
            with W._inflight:
                W._inflight_n += 1
            inflight["n"] += 1
            orig_begin(model, batch, eta)

        def counting_end():
            try:
                return end()
            finally:
                with W._inflight:
                    W._inflight_n -= 1
                    W._inflight.notify_all()

        monkeypatch.setattr(W, "execute_gpu_replica_begin", counting_begin)
        monkeypatch.setattr(W, "execute_gpu_replica_end", counting_end)
        hb.pipelined(RW, E)
        hb.pipelined(RW, E)  # idempotent
        curve, w, m = run()
        assert inflight["n"] == m.per_worker_updates["gpu0"] > 0
        assert curve == ref_curve
        for a, b in zip(w, ref_w):
            assert np.array_equal(a, b)
        assert m.per_worker_busy_ms["gpu0"] == pytest.approx(1.0 * m.per_worker_updates["gpu0"])


    def test_share_host_sizes_the_merge_pool_from_the_roster(self, monkeypatch):
        """feed.share_host reads the coordinator's roster: a CPU Hogwild pool
        gets the host threads, the merge pool shrinks and stops spinning."""
        ref_src = Path("/root/reference/pkg/src")
        if not ref_src.exists():
            pytest.skip("reference package not present")
        monkeypatch.syspath_prepend(str(ref_src))
        import os

        import hogtrain
        import hogtrain.engine as E
        import hogtrain.workers as RW

        from paper_2004_08771_b200 import feed

        monkeypatch.setattr(E._Coordinator, "__init__", E._Coordinator.__init__)
        hb.share_host(E)
        hb.share_host(E)  # idempotent
        ds = hogtrain.data.synthetic_blobs(300, 6, 2, 2.5, seed=1)
        model = hogtrain.nn.init_model(hogtrain.nn.Architecture((6, 8, 2)), seed=2)
        hw = os.cpu_count() or 4
        roster = [RW.WorkerConfig("cpu", RW.WorkerMode.HOGWILD_SHARDED, threads=3, min_batch=3, max_batch=30),
                  RW.WorkerConfig("gpu0", RW.WorkerMode.BATCH_REPLICA, min_batch=50, max_batch=100)]
        hogtrain.run_training(ds, model, roster, hogtrain.policies.UniformHogbatch(30, 0.1), epochs=1, seed=3)
        assert feed.last_host_share == (max(2, min(12, hw - 3)), 0)
        roster = roster[1:]
        hogtrain.run_training(ds, model, roster, hogtrain.policies.UniformHogbatch(50, 0.1), epochs=1, seed=3)
        assert feed.last_host_share == (max(2, min(12, hw * 3 // 4)), 20000)


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
