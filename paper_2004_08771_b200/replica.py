"""GpuReplica: one device context of the C library, owned by one worker thread.

This is the B200 replacement for the state `execute_batch_replica` rebuilds
on every call (workers.py:126-138): instead of `deep_copy` + NumPy tape, the
context keeps the fp32 model mirror, the activation tape, the staged epoch
and TMA descriptors resident on the GPU, and exchanges only the model
snapshot (H2D) and the gradient for the stale merge (D2H).
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _native as N
from .data import CsrDataset


class GpuReplica:
    """Device context for layer sizes `sizes` and batches of <= max_batch rows."""

    def __init__(self, sizes, max_batch: int, device: int = 0, sparse: bool = False, precision: str = "3xtf32",
                 sparse_kernels: bool = False):
        """sparse: the replica takes CSR input.  Inputs at most
        HB_DENSIFY_MAX_DIN wide are scattered into dense rows on the device and
        layer 0 runs as a tensor-core GEMM; sparse_kernels=True (or a wider
        input) keeps the CSR-gather SpMM / CSC-slice dW kernels."""
        self._lib = N.load()
        self.sizes = tuple(int(s) for s in sizes)
        self.depth = len(self.sizes) - 1
        self.max_batch = int(max_batch)
        self.device = int(device)
        self.sparse = bool(sparse)
        if precision not in ("3xtf32", "tf32"):
            raise ValueError(f"precision must be '3xtf32' or 'tf32', got {precision!r}")
        self.precision = precision
        flags = (N.HB_SPARSE_INPUT if sparse else 0) | (N.HB_PRECISION_TF32 if precision == "tf32" else 0)
        if sparse and sparse_kernels:
            flags |= N.HB_SPARSE_KERNELS
        self.sparse_kernels = bool(sparse) and (bool(sparse_kernels) or self.sizes[0] > N.HB_DENSIFY_MAX_DIN)
        arr = (C.c_int * len(self.sizes))(*self.sizes)
        h = C.c_void_p()
        N.check(self._lib.hb_ctx_create(C.byref(h), self.device, self.depth, arr, self.max_batch, flags))
        self._h = h
        self._staged_key = None
        self._staged_ref = None
        self._keep = None
        self._pinned = {}  # data address -> array kept alive while page-locked
        self._tbl_key = None  # _model_table cache: ids of the last host model's arrays
        self._tbl = self._tbl_arrays = self._tbl_shapes = None
        self._fin = weakref.finalize(self, GpuReplica._destroy, self._lib, h, self._pinned)

    @staticmethod
    def _destroy(lib, h, pinned):
        if h:
            lib.hb_ctx_destroy(h)
        for addr in list(pinned):
            lib.hb_host_unregister(C.c_void_p(addr))
        pinned.clear()

    def pin_host(self, arrays) -> None:
        """Page-lock host arrays exchanged every step (the shared float64 model)
        so the snapshot / merge copies run at full link speed.  The arrays are
        kept referenced until close()."""
        for a in arrays:
            addr = a.__array_interface__["data"][0]
            if addr not in self._pinned and a.nbytes > 0:
                N.check(self._lib.hb_host_register(C.c_void_p(addr), a.nbytes))
                self._pinned[addr] = a

    def close(self):
        self._fin()

    # ----------------------------------------------------------- model
    def set_weights(self, weights) -> None:
        """Snapshot a host float64 model into the device mirror (deep_copy, nn.py:182)."""
        if len(weights) != self.depth:
            raise ValueError("weight count does not match architecture")
        arrs = []
        for l, w in enumerate(weights):
            want = (self.sizes[l + 1], self.sizes[l])
            if w.shape != want:
                raise ValueError(f"weights[{l}] has shape {w.shape}, expected {want}")
            arrs.append(np.ascontiguousarray(w, dtype=np.float64))
        table = (C.POINTER(C.c_double) * self.depth)(*[N.ptr(a, C.c_double) for a in arrs])
        N.check(self._lib.hb_set_weights_all_f64(self._h, table))

    def set_bias(self, layer: int, bias) -> None:
        """Optional fixed per-unit offset of hidden layer `layer`, fused into the
        forward epilogue (A = sigmoid(Z + b)); None removes it.  The reference
        MLP has no bias; it is not trained."""
        if bias is None:
            N.check(self._lib.hb_set_bias_f64(self._h, int(layer), None))
            return
        b = np.ascontiguousarray(bias, dtype=np.float64)
        if b.shape != (self.sizes[layer + 1],):
            raise ValueError(f"bias of layer {layer} must have shape ({self.sizes[layer + 1]},)")
        N.check(self._lib.hb_set_bias_f64(self._h, int(layer), N.ptr(b, C.c_double)))

    def get_weights(self) -> list:
        out = []
        for l in range(self.depth):
            w = np.empty((self.sizes[l + 1], self.sizes[l]), dtype=np.float64)
            N.check(self._lib.hb_get_weights_f64(self._h, l, N.ptr(w, C.c_double)))
            out.append(w)
        return out

    def write_weights_into(self, weights) -> None:
        """Copy the device model into existing host float64 arrays in place."""
        for l, w in enumerate(self.get_weights()):
            np.copyto(weights[l], w)

    def grads(self) -> list:
        """Raw mean gradients of the last step run with emit_grad=True."""
        out = []
        for l in range(self.depth):
            g = np.empty((self.sizes[l + 1], self.sizes[l]), dtype=np.float32)
            N.check(self._lib.hb_get_grad_f32(self._h, l, N.ptr(g, C.c_float)))
            out.append(g)
        return out

    def merge_grads_into(self, weights, eta: float) -> None:
        """Stale merge W_global -= eta * g (workers.py:135 -> linalg.py:79) with
        the gradient of the last emit_grad step, in place on host float64 arrays."""
        if len(weights) != self.depth:
            raise ValueError("weight count does not match architecture")
        for l, w in enumerate(weights):
            if not (w.flags.c_contiguous and w.dtype == np.float64):
                raise ValueError("host weights must be C-contiguous float64 (Model layout, nn.py:75)")
            if w.shape != (self.sizes[l + 1], self.sizes[l]):
                raise ValueError(f"weights[{l}] has shape {w.shape}")
        table = (C.POINTER(C.c_double) * self.depth)(*[N.ptr(w, C.c_double) for w in weights])
        N.check(self._lib.hb_merge_grads_all_into_f64(self._h, table, float(eta)))

    # ------------------------------------------------------------ data
    @staticmethod
    def key_of(data) -> tuple:
        """Identity of a host dataset: its buffer address and shape.  The
        staged array is kept referenced, so the address cannot be recycled by
        a different array while it is staged."""
        if isinstance(data, CsrDataset):
            return ("csr", data.rowptr.__array_interface__["data"][0], data.col.__array_interface__["data"][0],
                    data.n_examples)
        return ("dense", data.__array_interface__["data"][0], data.shape, data.dtype.str)

    def stage(self, data, labels=None) -> None:
        """Stage a dataset (dense (N, d) float array + labels, or CsrDataset) on
        the device; steps then index it by (start, rows)."""
        key = self.key_of(data)
        if isinstance(data, CsrDataset):
            if not self.sparse:
                raise ValueError("dense context cannot stage CSR data")
            if data.n_cols != self.sizes[0]:
                raise ValueError(f"CSR has {data.n_cols} columns, model input is {self.sizes[0]}")
            val32 = np.ascontiguousarray(data.val, dtype=np.float32)
            N.check(self._lib.hb_stage_csr(self._h, N.ptr(data.rowptr, C.c_int64), N.ptr(data.col, C.c_int32),
                                           N.ptr(val32, C.c_float), data.n_examples, N.ptr(data.labels, C.c_int64)))
            self._staged_key = key
            self._keep = data
            return
        x = data
        if x.ndim != 2 or x.shape[1] != self.sizes[0]:
            raise ValueError(f"batch shape {x.shape} incompatible with input dim {self.sizes[0]}")
        y = np.ascontiguousarray(labels, dtype=np.int64)
        if y.shape != (x.shape[0],):
            raise ValueError("labels length must equal the number of feature rows")
        if self.sparse:
            # the densified epoch copy of sparse data (data.py:128-140): staged
            # as CSR, its zeros dropped on the host
            x = x if (x.dtype == np.float64 and x.strides[1] == 8) else np.ascontiguousarray(x, dtype=np.float64)
            N.check(self._lib.hb_stage_dense_as_csr_f64(self._h, N.ptr(x, C.c_double), x.shape[0],
                                                        x.strides[0] // 8, N.ptr(y, C.c_int64)))
            self._staged_key = key
            self._keep = (data, x, y)
            return
        if x.dtype == np.float32 and x.strides[1] == 4:
            N.check(self._lib.hb_stage_dense_f32(self._h, N.ptr(x, C.c_float), x.shape[0], x.strides[0] // 4,
                                                 N.ptr(y, C.c_int64)))
        else:
            x = x if (x.dtype == np.float64 and x.strides[1] == 8) else np.ascontiguousarray(x, dtype=np.float64)
            N.check(self._lib.hb_stage_dense_f64(self._h, N.ptr(x, C.c_double), x.shape[0], x.strides[0] // 8,
                                                 N.ptr(y, C.c_int64)))
        self._staged_key = key
        self._keep = (data, x, y)

    def stage_blobs(self, n_rows: int, classes: int, separation: float, seed: int, row0: int = 0) -> None:
        """Stage n_rows Gaussian-blob rows generated on the device (means from
        data.blob_means(seed); rows row0.. of a Philox stream keyed by seed) --
        datasets larger than host memory, e.g. the 10M x 1024 scaled config."""
        from .data import blob_means

        if self.sparse:
            raise ValueError("blob staging needs a dense context")
        means = np.ascontiguousarray(blob_means(self.sizes[0], classes, separation, seed), dtype=np.float64)
        N.check(self._lib.hb_stage_blobs(self._h, int(n_rows), int(row0), int(classes), N.ptr(means, C.c_double),
                                         int(seed) & 0xFFFFFFFFFFFFFFFF))
        self._staged_key = ("blobs", int(n_rows), int(row0), int(classes), float(separation), int(seed))
        self._keep = None

    def read_staged(self, start: int, rows: int):
        """(x fp32 (rows, d0), labels int64) of staged dense rows [start, start+rows)."""
        x = np.empty((rows, self.sizes[0]), dtype=np.float32)
        y = np.empty(rows, dtype=np.int64)
        N.check(self._lib.hb_read_staged(self._h, int(start), int(rows), N.ptr(x, C.c_float), N.ptr(y, C.c_int64)))
        return x, y

    def permute_epoch(self, perm) -> None:
        """Make the staged rows base[perm] on the device, base being the data
        as staged (reorder, data.py:187-192, without a re-stage).  The staged
        key is dropped: the rows no longer match the staged array."""
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        N.check(self._lib.hb_permute_epoch(self._h, N.ptr(perm, C.c_int64), perm.shape[0]))
        self._staged_key = None

    def is_staged(self, key) -> bool:
        return self._staged_key == key

    @property
    def staged_rows(self) -> int:
        return int(self._lib.hb_staged_rows(self._h))

    # ------------------------------------------------------------ steps
    def step(self, start: int, rows: int, eta: float, emit_grad: bool = False, timed: bool = False,
             want_loss: bool = False, blocking: bool = True, merge: bool = False):
        """One SGD step on staged rows [start, start+rows); returns the mean
        training loss of the batch when want_loss.  blocking=False returns as
        soon as the step is enqueued (synchronize() waits).  merge=True then
        averages the replicas over the communicator (comm_init) on the same
        stream, inside the step's timing bracket."""
        flags = (N.HB_STEP_EMIT_GRAD if emit_grad else 0) | (N.HB_STEP_TIMED if timed else 0) | (
            N.HB_STEP_MERGE if merge else 0)
        if not blocking and not want_loss:
            flags |= N.HB_STEP_ASYNC
        loss = C.c_double(0.0)
        N.check(self._lib.hb_train_step(self._h, int(start), int(rows), float(eta), flags,
                                        C.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def step_host(self, batch, labels, eta: float, emit_grad: bool = False, timed: bool = False,
                  want_loss: bool = True):
        """One SGD step on a batch held in host memory (copied H2D in the call).
        batch: float32 (rows, d) array, or a CsrDataset of the batch rows."""
        flags = (N.HB_STEP_EMIT_GRAD if emit_grad else 0) | (N.HB_STEP_TIMED if timed else 0)
        loss = C.c_double(0.0)
        lp = C.byref(loss) if want_loss else None
        if isinstance(batch, CsrDataset):
            val32 = batch.val if batch.val.dtype == np.float32 else np.ascontiguousarray(batch.val, dtype=np.float32)
            y = batch.labels if labels is None else np.ascontiguousarray(labels, dtype=np.int64)
            N.check(self._lib.hb_train_step_host_csr(self._h, N.ptr(batch.rowptr, C.c_int64),
                                                     N.ptr(batch.col, C.c_int32), N.ptr(val32, C.c_float),
                                                     N.ptr(y, C.c_int64), batch.n_examples, float(eta), flags, lp))
        else:
            x = batch if (batch.dtype == np.float32 and batch.strides[1] == 4) else np.ascontiguousarray(
                batch, dtype=np.float32)
            y = np.ascontiguousarray(labels, dtype=np.int64)
            N.check(self._lib.hb_train_step_host_dense(self._h, N.ptr(x, C.c_float), x.strides[0] // 4,
                                                       N.ptr(y, C.c_int64), x.shape[0], float(eta), flags, lp))
        return loss.value if want_loss else None

    # ------------------------------------------- fused drop-in replica step
    def _model_table(self, weights):
        """Pointer table of the shared host model (Model layout, nn.py:75),
        page-locked on first use (it is exchanged every call)."""
        key = tuple(map(id, weights))
        if key == self._tbl_key and all(w.shape == s and w.dtype == np.float64
                                        for w, s in zip(weights, self._tbl_shapes)):
            return self._tbl  # same array objects (kept alive by _tbl_arrays): same addresses
        if len(weights) != self.depth:
            raise ValueError("weight count does not match architecture")
        for l, w in enumerate(weights):
            if not (isinstance(w, np.ndarray) and w.flags.c_contiguous and w.dtype == np.float64):
                raise ValueError("host weights must be C-contiguous float64 (Model layout, nn.py:75)")
            if w.shape != (self.sizes[l + 1], self.sizes[l]):
                raise ValueError(f"weights[{l}] has shape {w.shape}, expected {(self.sizes[l + 1], self.sizes[l])}")
        self.pin_host(weights)
        self._tbl = (C.POINTER(C.c_double) * self.depth)(*[N.ptr(w, C.c_double) for w in weights])
        self._tbl_arrays = list(weights)
        self._tbl_shapes = [w.shape for w in weights]
        self._tbl_key = key
        return self._tbl

    @staticmethod
    def _replica_flags(timed: bool, sole_writer: bool, land_async: bool) -> int:
        if land_async and not sole_writer:
            raise ValueError("land_async needs sole_writer=True")
        return ((N.HB_STEP_TIMED if timed else 0) | (N.HB_STEP_SOLE_WRITER if sole_writer else 0)
                | (N.HB_STEP_LAND_ASYNC if land_async else 0))

    def landed(self) -> None:
        """Wait until the write-backs of land_async calls are in the host model."""
        N.check(self._lib.hb_replica_landed(self._h))

    def replica_step(self, weights, start: int, rows: int, eta: float, timed: bool = False,
                     want_loss: bool = False, sole_writer: bool = False, land_async: bool = False):
        """execute_batch_replica (workers.py:126-138) on staged rows in one call:
        snapshot of the shared float64 `weights`, the step, and the stale merge
        weights[l] -= eta * g_l, with the snapshot / merge DMAs overlapped with
        the compute layer by layer.  Returns the batch's mean loss if want_loss.
        sole_writer=True promises that no other thread writes `weights` during
        the call, which lets the largest layers merge on the device lane.
        land_async=True (sole writers) returns before the merged layers have
        landed in `weights`: the next call overlaps them; landed() (or any call
        on another model) waits -- do not read `weights` in between."""
        table = self._model_table(weights)
        flags = self._replica_flags(timed, sole_writer, land_async)
        loss = C.c_double(0.0)
        N.check(self._lib.hb_replica_step(self._h, table, int(start), int(rows), float(eta), flags,
                                          C.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def replica_begin(self, weights, start: int, rows: int, eta: float, timed: bool = False,
                      sole_writer: bool = False, land_async: bool = False) -> None:
        """First half of replica_step: enqueue snapshot, step and gradient
        copies and return; replica_end applies the stale merge and waits."""
        table = self._model_table(weights)
        flags = self._replica_flags(timed, sole_writer, land_async)
        N.check(self._lib.hb_replica_begin(self._h, table, int(start), int(rows), float(eta), flags))

    def replica_end(self, want_loss: bool = False):
        loss = C.c_double(0.0)
        N.check(self._lib.hb_replica_end(self._h, C.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def replica_step_host(self, weights, batch, labels, eta: float, timed: bool = False, want_loss: bool = True,
                          sole_writer: bool = False, land_async: bool = False):
        """replica_step on a batch held in host memory (float32 rows or a CsrDataset)."""
        table = self._model_table(weights)
        flags = self._replica_flags(timed, sole_writer, land_async)
        loss = C.c_double(0.0)
        lp = C.byref(loss) if want_loss else None
        if isinstance(batch, CsrDataset):
            val32 = batch.val if batch.val.dtype == np.float32 else np.ascontiguousarray(batch.val, dtype=np.float32)
            y = batch.labels if labels is None else np.ascontiguousarray(labels, dtype=np.int64)
            N.check(self._lib.hb_replica_step_host_csr(self._h, table, batch.rowptr.ctypes.data, batch.col.ctypes.data,
                                                       val32.ctypes.data, y.ctypes.data, batch.n_examples,
                                                       float(eta), flags, lp))
        else:
            x = batch if (batch.dtype == np.float32 and batch.strides[1] == 4) else np.ascontiguousarray(
                batch, dtype=np.float32)
            y = np.ascontiguousarray(labels, dtype=np.int64)
            N.check(self._lib.hb_replica_step_host_dense(self._h, table, x.ctypes.data, x.strides[0] // 4,
                                                         y.ctypes.data, x.shape[0], float(eta), flags, lp))
        return loss.value if want_loss else None

    def eval_loss_sum(self, start: int, rows: int) -> float:
        """Sum of per-example cross-entropy over staged rows (loss_sum, nn.py:139-146)."""
        out = C.c_double(0.0)
        N.check(self._lib.hb_eval_loss_sum(self._h, int(start), int(rows), C.byref(out)))
        return out.value

    def forward(self, start: int, rows: int) -> None:
        N.check(self._lib.hb_forward(self._h, int(start), int(rows)))

    def activation(self, layer: int, rows: int) -> np.ndarray:
        out = np.empty((rows, self.sizes[layer]), dtype=np.float32)
        N.check(self._lib.hb_get_activation_f32(self._h, int(layer), int(rows), N.ptr(out, C.c_float)))
        return out

    @property
    def last_step_ms(self) -> float:
        v = C.c_float(0.0)
        N.check(self._lib.hb_last_step_ms(self._h, C.byref(v)))
        return float(v.value)

    @property
    def last_step_launches(self) -> int:
        v = C.c_int(0)
        N.check(self._lib.hb_last_step_launches(self._h, C.byref(v)))
        return int(v.value)

    @property
    def last_xfer_bytes(self) -> tuple:
        """(host->device, device->host) bytes of the last replica_step* call."""
        h, d = C.c_int64(0), C.c_int64(0)
        N.check(self._lib.hb_last_xfer_bytes(self._h, C.byref(h), C.byref(d)))
        return int(h.value), int(d.value)

    def profile(self, on: bool) -> None:
        """Bracket every kernel launch with CUDA events on the step stream."""
        N.check(self._lib.hb_profile_enable(self._h, 1 if on else 0))

    def profile_filter(self, name: str | None) -> None:
        """Bracket only launches named `name` (e.g. "gemm_dx_dsig_l1"); None: all."""
        N.check(self._lib.hb_profile_filter(self._h, name.encode() if name else None))

    def profile_read(self) -> dict:
        """{kernel name: (total ms, launches)} since profile(True) / the last read."""
        cap = 256
        names = C.create_string_buffer(64 * cap)
        tot = (C.c_double * cap)()
        cnt = (C.c_int * cap)()
        n = C.c_int(0)
        N.check(self._lib.hb_profile_read(self._h, cap, names, tot, cnt, C.byref(n)))
        raw = names.raw
        return {raw[64 * i: 64 * i + 64].split(b"\0")[0].decode(): (tot[i], cnt[i]) for i in range(n.value)}

    def synchronize(self) -> None:
        N.check(self._lib.hb_synchronize(self._h))

    # ------------------------------------------------- multi-GPU merge
    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = N.load()
        buf = (C.c_char * 128)()
        N.check(lib.hb_nccl_unique_id(buf))
        return bytes(buf)

    def comm_init(self, uid: bytes, nranks: int, rank: int) -> None:
        buf = (C.c_char * 128).from_buffer_copy(uid)
        N.check(self._lib.hb_comm_init(self._h, buf, int(nranks), int(rank)))

    def peer_handle(self) -> bytes:
        """This replica's exchange-buffer handle for a peer-memory merge group."""
        buf = (C.c_char * N.HB_PEER_HANDLE_BYTES)()
        N.check(self._lib.hb_peer_handle(self._h, buf))
        return bytes(buf)

    def peer_attach(self, handles, rank: int) -> None:
        """Join the merge group whose ranks' handles are `handles` (rank order);
        merges then average over peer memory (NVLink P2P / CUDA IPC)."""
        blob = b"".join(handles)
        if len(blob) != N.HB_PEER_HANDLE_BYTES * len(handles):
            raise ValueError("every peer handle must be HB_PEER_HANDLE_BYTES long")
        buf = (C.c_char * len(blob)).from_buffer_copy(blob)
        N.check(self._lib.hb_peer_attach(self._h, len(handles), int(rank), buf))

    def merge_allreduce(self) -> None:
        """Average the device models of all ranks (NCCL allreduce over NVLink)."""
        N.check(self._lib.hb_merge_allreduce(self._h))
