/*
 * hogbatch_b200.h -- C ABI of the B200-native GPU replica worker for the
 * heterogeneous CPU+GPU Hogbatch / Adaptive Hogbatch SGD of
 * arXiv:2004.08771 (reference package: /root/reference/pkg, `hogtrain`).
 *
 * The reference's GPU worker is `execute_batch_replica(model, batch, eta,
 * speed_factor)` (pkg/src/hogtrain/workers.py:126-138), called from
 * `WorkerThread._execute` (workers.py:193-210), plus the evaluation call
 * `loss_sum(eval_model, x, y)` (nn.py:139-146, from workers.py:212-222).
 * Everything below is what a binding of that seam needs: a device context
 * per (worker, device), the model layout of nn.py:63-78, the batch layout of
 * data.py:30-79, one training step, the stale merge back into the host
 * model, loss evaluation, device timing for the batch-size controller
 * (policies.py:84-129 fed from engine.py:318-328), and the NCCL merge between
 * GPU replicas.
 *
 * Conventions
 *  - Every function returns HB_OK (0) or an HB_E* code; hb_last_error()
 *    returns a thread-local message for the last failure on the calling
 *    thread.  Argument/shape errors are HB_EINVAL (the reference raises
 *    ValueError there: linalg.py:40-44, nn.py:110-113); CUDA/NCCL failures
 *    are HB_ECUDA / HB_ENCCL.
 *  - Plain pointers and sizes only.  "host" pointers are ordinary (pageable
 *    or pinned) CPU memory; nothing here retains a host pointer after return.
 *  - A context is affine to one device and must be used from one thread at a
 *    time (the reference's worker thread).  Calls block until the device work
 *    they enqueue is complete unless stated otherwise.
 *  - Layer l weight: row-major (d_{l+1}, d_l) float64 on the host, exactly
 *    `Model.weights[l]` (nn.py:75).  The device keeps an fp32 mirror; for a
 *    sparse first layer it stores W_0 transposed, which is invisible here.
 */
#ifndef HOGBATCH_B200_H
#define HOGBATCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_OK 0
#define HB_EINVAL 1
#define HB_ECUDA 2
#define HB_ENCCL 3
#define HB_ESTATE 4
#define HB_EPARSE 5 /* malformed LIBSVM text (the reference's LibsvmParseError, data.py:26) */

/* hb_ctx_create flags */
#define HB_SPARSE_INPUT 1u  /* first layer consumes CSR input (CSR-gather SpMM) */
#define HB_PRECISION_TF32 2u /* 1-pass TF32 GEMMs (fast mode); default is 3xTF32 */
/* CSR contexts with a narrow input layer (d_0 <= HB_DENSIFY_MAX_DIN) scatter
 * the CSR rows into a dense device copy once at staging (per step for host
 * batches) and run layer 0 as a tensor-core GEMM, like every other layer --
 * the reference's own dense formulation (data.py:128-141).  This flag keeps
 * the CSR-gather SpMM / CSC-slice dW kernels instead. */
#define HB_SPARSE_KERNELS 4u
#define HB_DENSIFY_MAX_DIN 512

/* hb_train_step flags */
#define HB_STEP_EMIT_GRAD 1u /* keep the raw mean gradient of every layer (for the host merge / parity) */
#define HB_STEP_TIMED 2u     /* bracket the step with CUDA events (hb_last_step_ms) */
#define HB_STEP_ASYNC 4u     /* return once the step is enqueued (no out_loss); hb_synchronize() waits */
#define HB_STEP_MERGE 8u     /* average the replicas within the step (NCCL or a cross-process peer group:
                                * each layer as soon as its update lands, overlapping the rest of the
                                * backward; an in-process peer group: the whole model after the step) */
/* hb_replica_step*: the caller guarantees no other thread writes the host
 * model during the call (a lone GPU replica, no CPU Hogwild pool).  Lets the
 * largest split-K layers merge on the device (host rows read while the dW
 * partial GEMM runs, written back after the reduce); without it every layer
 * merges on the host with per-element read-modify-writes, as np.add does. */
#define HB_STEP_SOLE_WRITER 16u
/* hb_replica_step* / hb_replica_begin with HB_STEP_SOLE_WRITER: return once the
 * step and its loss are done and let the merged layers' write-backs into the
 * host model finish in the background -- the next call's batch copy and
 * forward overlap them.  Consecutive deferred calls on the same host arrays
 * chain on the device copy; hb_replica_landed (or any call that reads or
 * writes the host model through the context: another replica call without the
 * flag or on other arrays, set_weights, merge_grads, hb_synchronize,
 * hb_ctx_destroy) waits until every write-back is in host memory.  The caller
 * must not read ws in between (the reference's coordinator snapshot waits,
 * feed.pipelined). */
#define HB_STEP_LAND_ASYNC 32u

typedef struct hb_ctx hb_ctx;

/* Thread-local message describing the last error on this thread. */
const char* hb_last_error(void);
/* Library build identification (arch, precision modes). */
const char* hb_version(void);
int hb_device_count(int* out);

/* Device context for one GPU replica worker.  Replaces the per-call
 * deep_copy + numpy state of execute_batch_replica (workers.py:131-135) with
 * resident device buffers.  layer_sizes[0..n_layers] as Architecture.layer_sizes
 * (nn.py:38-60).  max_batch bounds every step's row count (WorkerConfig.max_batch,
 * workers.py:61-62). */
int hb_ctx_create(hb_ctx** out, int device, int n_layers, const int* layer_sizes, int max_batch, uint32_t flags);
int hb_ctx_destroy(hb_ctx* ctx);

/* Model snapshot H2D (deep_copy, nn.py:182-184): host float64 (d_{l+1}, d_l). */
int hb_set_weights_f64(hb_ctx* ctx, int layer, const double* w);
/* Optional fixed per-unit offset of hidden layer `layer` (0..n_layers-2),
 * d_{layer+1} float64 values, fused into the forward epilogue before the
 * sigmoid (A = sigmoid(Z + b)); null removes it.  The reference MLP has no
 * bias (nn.py:63-78), so parity runs without one; the offset is not trained. */
int hb_set_bias_f64(hb_ctx* ctx, int layer, const double* bias);
/* Device model D2H into host float64 (d_{l+1}, d_l). */
int hb_get_weights_f64(hb_ctx* ctx, int layer, double* w);
int hb_get_weights_f32(hb_ctx* ctx, int layer, float* w);

/* Stale merge (workers.py:135 -> nn.py:174-179 -> linalg.py:70-79):
 * host_w -= eta * g_l for the gradient kept by the last HB_STEP_EMIT_GRAD
 * step, element by element with aligned 8-byte stores.  */
int hb_merge_grad_into_f64(hb_ctx* ctx, int layer, double* host_w, double eta);
/* Whole-model forms of the two calls above (one transfer each way, one sync):
 * ws[l] points at layer l's host float64 (d_{l+1}, d_l) array. */
int hb_set_weights_all_f64(hb_ctx* ctx, const double* const* ws);
int hb_merge_grads_all_into_f64(hb_ctx* ctx, double* const* ws, double eta);
/* Page-lock (and later release) a host range used for repeated exchanges, e.g.
 * the shared float64 model, so its copies run at full link speed.  Counted per
 * base address: contexts of several worker threads may register the same
 * shared model, and only the last release unregisters it. */
int hb_host_register(const void* p, size_t bytes);
int hb_host_unregister(const void* p);
/* Raw mean gradient of the last HB_STEP_EMIT_GRAD step, (d_{l+1}, d_l) fp32. */
int hb_get_grad_f32(hb_ctx* ctx, int layer, float* g);

/* Host threads (caller included) that apply the float64 stale merges, and how
 * long (pause iterations, ~25 ns each) they spin for the next layer before
 * sleeping.  Default: 3/4 of the host threads (at most 12), 20000 spins.  A
 * process that also runs the reference's CPU Hogwild pool
 * (execute_hogwild_sharded, workers.py:94-123) gives its cores back with e.g.
 * hb_host_merge_threads(2, 0).  Process-wide. */
int hb_host_merge_threads(int threads, int spin);
/* Self-test of that pool (host only, no device): `jobs` back-to-back jobs of
 * varying part counts; out_errors = parts not run exactly once. */
int hb_host_pool_selftest(int jobs, int64_t* out_errors);

/* Stage one epoch's (or any dataset's) rows on the device so steps can index
 * them by (start, rows) -- the per-epoch shuffled copy that BatchRef views
 * (engine.py:214-221, data.py:57-79).  Dense: features (n_rows, n_cols) with
 * row stride ld (elements); labels int64 class indices. */
int hb_stage_dense_f64(hb_ctx* ctx, const double* x, int64_t n_rows, int64_t ld, const int64_t* labels);
int hb_stage_dense_f32(hb_ctx* ctx, const float* x, int64_t n_rows, int64_t ld, const int64_t* labels);
/* Sparse (HB_SPARSE_INPUT contexts): CSR with int64 row pointer (n_rows+1),
 * int32 0-based column ids, fp32 values.  The column-sorted (CSC) copy used
 * by the sparse dW kernel is built once here. */
int hb_stage_csr(hb_ctx* ctx, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n_rows,
                 const int64_t* labels);
/* Sparse-input contexts: stage a dense float64 (n_rows, d_0) array (row
 * stride ld) whose rows are mostly zero -- the densified epoch copy the
 * reference's LIBSVM loader produces (data.py:128-140) and BatchRef views --
 * as CSR: the nonzeros are gathered on the host (values to fp32) and staged
 * like hb_stage_csr, so layer 0 runs on the CSR kernels. */
int hb_stage_dense_as_csr_f64(hb_ctx* ctx, const double* x, int64_t n_rows, int64_t ld, const int64_t* labels);
int64_t hb_staged_rows(hb_ctx* ctx);
/* Stage n_rows synthetic Gaussian-blob rows generated on the device (the
 * shape of synthetic_blobs, data.py:226-252: row = means[label] + N(0, I)),
 * for datasets too large for host memory (the 10M x 1024 scaled config,
 * 41 GB fp32).  means: (n_classes, d_0) float64 from the host generator;
 * row r's label (uniform over n_classes) and noise are a pure function of
 * (seed, row0 + r) (counter-based Philox4x32-10), so results do not depend on
 * the launch shape and data-parallel ranks stage disjoint row ranges of one
 * dataset (row0 = rank * n_rows).  Replaces hb_stage_dense_* for this context. */
int hb_stage_blobs(hb_ctx* ctx, int64_t n_rows, int64_t row0, int n_classes, const double* means, uint64_t seed);
/* Copy staged dense rows [start, start+rows) back: x (rows, d_0) fp32
 * contiguous and labels (either may be null) -- the exact values the device
 * trains on, for the CPU oracle and the host-buffer (e2e) path. */
int hb_read_staged(hb_ctx* ctx, int64_t start, int64_t rows, float* x, int64_t* labels);
/* Replace the staged rows by base[perm] on the device (perm: n_rows distinct
 * indices in [0, n_rows)), where base is the data as first staged -- the
 * per-epoch reshuffle of engine.py:214-221 (shuffle_epoch + reorder,
 * data.py:182-192) without re-staging: dense rows, labels and the CSR/CSC
 * copies come out identical to staging the host-reordered dataset. */
int hb_permute_epoch(hb_ctx* ctx, const int64_t* perm, int64_t n_rows);

/* LIBSVM text -> CSR, natively (the reference's loader, data.py:106-151,
 * densifies to (N, feature_dim) float64 in Python).  buf/len hold the whole
 * (decompressed) text.  scan validates every line and counts rows / nonzeros;
 * fill writes rowptr (n_rows+1), col (nnz, 0-based, ascending per row), val
 * (nnz) and labels (n_rows).  label_mapping: 0 = ZERO_ONE, 1 = PLUS_MINUS_ONE
 * (data.py:21-23, 86-103).  Bad tokens/labels return HB_EPARSE, an index
 * outside [1, feature_dim] HB_EINVAL, both with "line N: ..." messages.  A
 * repeated index keeps the last value and explicit zeros are dropped. */
int hb_libsvm_scan(const char* buf, size_t len, int64_t feature_dim, int label_mapping, int64_t* n_rows,
                   int64_t* nnz);
int hb_libsvm_fill(const char* buf, size_t len, int64_t feature_dim, int label_mapping, int64_t* rowptr,
                   int32_t* col, double* val, int64_t* labels);

/* One replica SGD step over staged rows [start, start+rows): forward
 * (nn.py:108-121), fused softmax/CE error (nn.py:162-164), backward
 * (nn.py:149-171) and the SGD update W -= eta * g fused into the dW epilogues
 * (nn.py:174-179), all on the device.  out_loss (nullable) receives the mean
 * training cross-entropy of the batch (nn.py:124-136), a by-product. */
int hb_train_step(hb_ctx* ctx, int64_t start, int rows, double eta, uint32_t flags, double* out_loss);
/* Same step on a batch held in host memory (copied H2D inside the call):
 * dense (rows, d0) with row stride ld, or CSR (rows+1 row pointer starting at 0). */
int hb_train_step_host_dense(hb_ctx* ctx, const float* x, int64_t ld, const int64_t* labels, int rows, double eta,
                             uint32_t flags, double* out_loss);
int hb_train_step_host_csr(hb_ctx* ctx, const int64_t* rowptr, const int32_t* col, const float* val,
                           const int64_t* labels, int rows, double eta, uint32_t flags, double* out_loss);

/* The whole drop-in replica step, execute_batch_replica(model, batch, eta)
 * (workers.py:126-138), in one call with the host-model exchange overlapped
 * with the compute: the snapshot of the shared float64 model ws[l]
 * (deep_copy, workers.py:132) is DMA'd layer by layer so layer l computes
 * while layer l+1 is in flight, and the stale merge ws[l] -= eta * g_l
 * (apply_update into the *current* shared model, workers.py:135 ->
 * nn.py:174-179 -> linalg.py:70-79, float64, aligned 8-byte stores) is a
 * chunked DMA read-modify-write issued as soon as layer l's gradient exists,
 * overlapping the rest of the backward pass.  ws[l] must be page-locked
 * (hb_host_register).  Returns once the host model holds the merge.  The
 * three forms take the batch like hb_train_step / _host_dense / _host_csr. */
int hb_replica_step(hb_ctx* ctx, double* const* ws, int64_t start, int rows, double eta, uint32_t flags,
                    double* out_loss);
int hb_replica_step_host_dense(hb_ctx* ctx, double* const* ws, const float* x, int64_t ld, const int64_t* labels,
                               int rows, double eta, uint32_t flags, double* out_loss);
int hb_replica_step_host_csr(hb_ctx* ctx, double* const* ws, const int64_t* rowptr, const int32_t* col,
                             const float* val, const int64_t* labels, int rows, double eta, uint32_t flags,
                             double* out_loss);

/* hb_replica_step on staged rows split in two: begin enqueues the snapshot,
 * the step and the gradient copies and returns; end applies the stale merge
 * into ws as the gradients land and waits for the step (out_loss as in
 * hb_replica_step).  The calling thread may do host work in between -- the
 * GPU worker answers the coordinator (SCHEDULE_WORK, workers.py:209) while
 * its step runs, so the coordinator round trip (engine.py:278-316) overlaps
 * the device instead of following it.  No other call on the context may
 * come in between; ws must stay valid until end. */
int hb_replica_begin(hb_ctx* ctx, double* const* ws, int64_t start, int rows, double eta, uint32_t flags);
int hb_replica_end(hb_ctx* ctx, double* out_loss);
/* Block until the write-backs of HB_STEP_LAND_ASYNC calls are in the host model. */
int hb_replica_landed(hb_ctx* ctx);

/* Sum over staged rows [start, start+rows) of -log max(p_y, 1e-12)
 * (loss_sum, nn.py:139-146), evaluated in chunks of at most max_batch rows. */
int hb_eval_loss_sum(hb_ctx* ctx, int64_t start, int64_t rows, double* out_sum);

/* Forward only over staged rows (tests): then read layer activations
 * A_l (rows, d_l), l = 1..n_layers-1, or the output probabilities. */
int hb_forward(hb_ctx* ctx, int64_t start, int rows);
int hb_get_activation_f32(hb_ctx* ctx, int layer, int rows, float* out);

/* Device time of the last HB_STEP_TIMED step (CUDA events on the step stream). */
int hb_last_step_ms(hb_ctx* ctx, float* ms);
/* Kernel launches issued by the last step. */
int hb_last_step_launches(hb_ctx* ctx, int* n);

/* PCIe bytes moved by the last hb_replica_step* call on this context: the
 * batch (host entry points), the model snapshot and the stale merge by lane
 * (fp32 gradient D2H on the host lane, float64 rows both ways on the device
 * lane / HB_XCHG_MERGE=dma), the step record and the loss.  Reporting only;
 * no reference counterpart (bench.py's e2e h2d/d2h_bytes_per_step). */
int hb_last_xfer_bytes(hb_ctx* ctx, int64_t* h2d_bytes, int64_t* d2h_bytes);
int hb_synchronize(hb_ctx* ctx);
/* Per-launch CUDA-event profiling on the step stream (off by default):
 * enable, run steps, then read per-kernel totals.  names receives
 * max_entries NUL-terminated 64-byte slots ("gemm_fwd_sigmoid_l1", ...). */
int hb_profile_enable(hb_ctx* ctx, int on);
int hb_profile_read(hb_ctx* ctx, int max_entries, char* names, double* total_ms, int* counts, int* n_out);
/* Restrict profiling to launches named `name` (null/empty: all launches). */
int hb_profile_filter(hb_ctx* ctx, const char* name);

/* Measurement only (bench.py's "l2" ceiling of the CSR kernels): rate in GB/s
 * at which the device gathers pseudo-random whole rows of an L2-resident
 * (rows x cols) fp32 matrix, `unroll` rows in flight per warp lane -- the
 * access pattern of one W0^T row per nonzero.  No reference counterpart. */
int hb_probe_l2_gather(int device, int64_t rows, int cols, int per_warp, int unroll, double* out_gbps);

/* NCCL merge between GPU replicas (one communicator per process/device). */
int hb_nccl_unique_id(void* out_128_bytes);
int hb_comm_init(hb_ctx* ctx, const void* id_128_bytes, int nranks, int rank);
/* Average the device models of all ranks in place (allreduce-sum / nranks). */
int hb_merge_allreduce(hb_ctx* ctx);
int hb_comm_destroy(hb_ctx* ctx);

/* The same merge over peer memory instead of NCCL: each rank's context
 * exports an exchange buffer (hb_peer_handle: HB_PEER_HANDLE_BYTES, carrying a
 * CUDA IPC handle), the handles of all ranks are exchanged by the caller (any
 * transport: torch.distributed, a shared list between threads), and
 * hb_peer_attach maps every peer (same process: direct NVLink peer access;
 * another process: CUDA IPC).  hb_merge_allreduce / HB_STEP_MERGE then run a
 * one-shot reduce-scatter + all-gather kernel that reads and writes the peers'
 * buffers directly (no collective library), with flag-based waits bounded by
 * a timeout (HB_ESTATE "never signalled" instead of a hang).  Every rank must
 * issue the same sequence of merges.  At most 8 ranks. */
#define HB_PEER_HANDLE_BYTES 128
int hb_peer_handle(hb_ctx* ctx, void* out_handle);
int hb_peer_attach(hb_ctx* ctx, int nranks, int rank, const void* handles);

#ifdef __cplusplus
}
#endif
#endif /* HOGBATCH_B200_H */
