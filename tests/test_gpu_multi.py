"""The GPU-replica merge with more than one rank, on one GPU:
two replicas (threads of one process, or two processes over CUDA IPC) average
their models over peer memory (hb_peer_attach + hb_merge_allreduce).  The
result must be the model average of parallel.average_models_host, rounded as
fp32 (w_0 + w_1) * 0.5, with the lo twins rewritten so the next step equals a
fresh replica holding the averaged model."""

import os
import socket
import threading

import numpy as np
import pytest

from oracle import ref_nn

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hb():
    import paper_2004_08771_b200 as hb

    if hb.device_count() < 1:
        pytest.fail("GPU tests need a CUDA device")
    return hb


def _case(sizes, b, seed, sparse):
    w = ref_nn.init_weights(sizes, seed)
    if sparse:
        import paper_2004_08771_b200 as hb

        data = hb.synthetic_csr(b, sizes[0], 9, sizes[-1], seed=seed + 1)
        return w, data, None
    x, y = ref_nn.synthetic_blobs(b, sizes[0], sizes[-1], 2.5, seed + 1)
    return w, x.astype(np.float32), y


def _merge_all(reps):
    errs = []

    def run(r):
        try:
            r.merge_allreduce()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=run, args=(r,)) for r in reps]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


@pytest.mark.parametrize("sparse", [False, True])
def test_peer_merge_two_replicas_in_process(hb, sparse):
    from paper_2004_08771_b200.parallel import average_models_host, local_peer_group

    sizes = (300, 128, 64, 3) if sparse else (40, 128, 96, 5)
    b = 256
    reps = [hb.GpuReplica(sizes, b, sparse=sparse, sparse_kernels=sparse) for _ in range(2)]
    fresh = hb.GpuReplica(sizes, b, sparse=sparse, sparse_kernels=sparse)
    try:
        for k, r in enumerate(reps):  # different models and data per rank
            w, x, y = _case(sizes, b, 10 + k, sparse)
            r.set_weights(w)
            r.stage(x, y)
            r.step(0, b, 0.4)
        before = [r.get_weights() for r in reps]
        local_peer_group(reps)
        for rounds in range(3):  # repeated merges: the flag generations advance
            _merge_all(reps)
            after = [r.get_weights() for r in reps]
            want = [((a.astype(np.float32) + c.astype(np.float32)) * np.float32(0.5)).astype(np.float64)
                    for a, c in zip(*before)]
            for a0, a1, wnt, avg in zip(after[0], after[1], want, average_models_host(before)):
                assert np.array_equal(a0, a1) and np.array_equal(a0, wnt)
                assert np.abs(a0 - avg).max() <= 1e-7 * max(1.0, np.abs(avg).max())
            before = after
        # lo twins rewritten: the next step equals a fresh replica holding the average
        w, x, y = _case(sizes, b, 99, sparse)
        fresh.set_weights(after[0])
        fresh.stage(x, y)
        fresh.step(0, b, 0.4, emit_grad=True)
        for r in reps:
            r.stage(x, y)
            r.step(0, b, 0.4, emit_grad=True)
            for g, gf in zip(r.grads(), fresh.grads()):
                assert np.array_equal(g, gf)
    finally:
        for r in reps + [fresh]:
            r.close()


def test_peer_merge_inside_the_step(hb):
    """HB_STEP_MERGE with a peer group: step + merge in one call per rank
    (concurrent threads), equal to step then merge."""
    from paper_2004_08771_b200.parallel import local_peer_group

    sizes = (40, 128, 96, 5)
    b = 256
    a = [hb.GpuReplica(sizes, b) for _ in range(2)]
    s = [hb.GpuReplica(sizes, b) for _ in range(2)]
    try:
        for k in range(2):
            w, x, y = _case(sizes, b, 20 + k, False)
            for r in (a[k], s[k]):
                r.set_weights(w)
                r.stage(x, y)
        local_peer_group(a)
        local_peer_group(s)
        for it in range(4):
            ts = [threading.Thread(target=a[k].step, args=(0, b, 0.3), kwargs=dict(merge=True)) for k in range(2)]
            for t in ts:
                t.start()
            for t in ts:
                t.join()
            for r in s:
                r.step(0, b, 0.3)
            _merge_all(s)
            for k in range(2):
                for wa, ws in zip(a[k].get_weights(), s[k].get_weights()):
                    assert np.array_equal(wa, ws), it
    finally:
        for r in a + s:
            r.close()


def test_peer_merge_times_out_instead_of_hanging(hb, monkeypatch):
    from paper_2004_08771_b200.parallel import local_peer_group

    monkeypatch.setenv("HB_PEER_TIMEOUT_S", "0.5")
    sizes = (16, 32, 2)
    reps = [hb.GpuReplica(sizes, 32) for _ in range(2)]
    try:
        local_peer_group(reps)
        with pytest.raises(RuntimeError, match="never signalled"):
            reps[0].merge_allreduce()  # rank 1 never merges
    finally:
        for r in reps:
            r.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0")
    import torch
    import torch.distributed as dist

    import paper_2004_08771_b200 as hb
    from paper_2004_08771_b200 import parallel as P

    dist.init_process_group("gloo")
    sizes = (40, 128, 96, 5)
    b = 256
    w, x, y = _case(sizes, b, 30 + rank, False)
    r = hb.GpuReplica(sizes, b)
    shadow = hb.GpuReplica(sizes, b)  # the same step without the merge
    for c in (r, shadow):
        c.set_weights(w)
        c.stage(x, y)
    worker = P.DataParallelWorker(r, dist, merge_every=2, transport="peer")
    trail, worst = [], 0.0
    for it in range(6):
        shadow.set_weights(r.get_weights())
        worker.step(0, b, 0.3)
        shadow.step(0, b, 0.3)
        got = r.get_weights()
        if it % 2 == 1:  # merged inside the backward, layer by layer: the fp32 average of both ranks' local steps
            mine = [torch.from_numpy(a.astype(np.float32)) for a in shadow.get_weights()]
            both = [[torch.zeros_like(t) for _ in range(world)] for t in mine]
            for t, out in zip(mine, both):
                dist.all_gather(out, t)
            for g, parts in zip(got, both):
                want = ((parts[0] + parts[1]) * 0.5).numpy().astype(np.float64)
                worst = max(worst, float(np.abs(g - want).max()))
        trail.append([a.copy() for a in got])
    q.put((rank, trail, worst, r.last_step_launches))
    P.barrier(dist)
    r.close()
    shadow.close()
    dist.destroy_process_group()


def test_peer_merge_two_processes_over_ipc(hb):
    """Two processes (torchrun-style ranks) on one GPU: the exchange buffers
    are shared with CUDA IPC, handles all-gathered over gloo; every 2nd step
    (DataParallelWorker's cadence) averages the replicas inside the backward,
    layer by layer as each update lands (flag kernels, capture-safe
    generations), and the result is the exact fp32 average of both ranks'
    local steps."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = {}
    for _ in ps:
        rank, trail, worst, launches = q.get(timeout=300)
        got[rank] = (trail, worst)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (t0, w0), (t1, w1) = got[0], got[1]
    assert w0 == 0.0 and w1 == 0.0  # bit-exact fp32 average, eager and graph-replayed merges
    for it in range(6):
        same = all(np.array_equal(a, c) for a, c in zip(t0[it], t1[it]))
        assert same == (it % 2 == 1), it  # merged on steps 2, 4, 6 only
