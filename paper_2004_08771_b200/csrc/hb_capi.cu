// hb_capi.cu -- device context and the C ABI of include/hogbatch_b200.h.
//
// A context owns, on one B200:
//   * the fp32 model mirror W_l (row-major (d_{l+1}, d_l), W_0 transposed for
//     sparse input), laid out with 16-byte-aligned row strides for TMA;
//   * the activation tape A_l and error signals D_l for up to max_batch rows;
//   * the staged epoch (dense fp32 rows or CSR + its column-sorted twin);
//   * split-K / per-block reduction workspaces, TMA tensor maps, one stream.
// A training step is a fixed sequence of kernel launches on that stream:
//   forward  : [SpMM+sigmoid | GEMM+sigmoid] per hidden layer
//   head     : fused small softmax-CE head (classes <= 4) or
//              GEMM logits -> softmax_delta (wide heads)
//   backward : per layer dX GEMM (x s(1-s) epilogue) then dW GEMM whose
//              epilogue applies W -= eta*g (split-K: deterministic reduce+SGD)
//   sparse L0: CSC-slice gather dW + in-place update of active rows
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <dlfcn.h>
#include <unistd.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <tuple>
#include <vector>
#include <atomic>
#if defined(__x86_64__)
#include <immintrin.h>
#endif
#include <chrono>
#include <condition_variable>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "../../include/hogbatch_b200.h"
#include "hb_gemm.cuh"
#include "hb_kernels.cuh"
#include "hb_peer.cuh"
#include "hb_small.cuh"

using namespace hb;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define HB_CUDA(expr)                                                                                   \
  do {                                                                                                  \
    cudaError_t e_ = (expr);                                                                            \
    if (e_ != cudaSuccess) return fail(HB_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                             \
  } while (0)
#define HB_TRY(expr)          \
  do {                        \
    int r_ = (expr);          \
    if (r_ != HB_OK) return r_; \
  } while (0)

inline long long round_up(long long x, long long m) { return (x + m - 1) / m * m; }
inline int cdiv(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// ---------------------------------------------------------------- TMA maps
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled g_encode = nullptr;

int get_encoder() {
  if (g_encode) return HB_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  HB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (fn == nullptr || q != cudaDriverEntryPointSuccess) return fail(HB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<PFN_encodeTiled>(fn);
  return HB_OK;
}

// fp32 2-D map over (rows, inner) with row stride ld (elements).
//   K-major operand tiles: box {32, box_rows}, SWIZZLE_128B.
//   MN-major operand tiles: box {32, 32}, SWIZZLE_128B_ATOM_32B.
int make_map(CUtensorMap* m, const float* base, long long inner, long long rows, long long ld, int box_rows,
             bool mn_major) {
  HB_TRY(get_encoder());
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(std::max<long long>(rows, 1))};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  cuuint32_t box[2] = {32, static_cast<cuuint32_t>(mn_major ? 32 : box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(HB_ECUDA, "cuTensorMapEncodeTiled failed (%d): inner=%lld rows=%lld ld=%lld box_rows=%d mn=%d",
                static_cast<int>(r), inner, rows, ld, box_rows, static_cast<int>(mn_major));
  return HB_OK;
}

std::atomic<long long> g_pin_epoch{0};  // bumped whenever a host range is unregistered
std::mutex g_host_mu;
std::map<uintptr_t, std::pair<size_t, void*>> g_host_ranges;  // host base -> (bytes, device alias)
std::map<uintptr_t, int> g_host_refs;  // registrations per base: contexts of several worker threads can share
                                       // one host model (engine.py:131-134); the last release unregisters

// ------------------------------------------------ programmatic dependent launch
// Every kernel of the step is launched with programmatic stream serialization
// (HB_NO_PDL=1 turns it off): it may be scheduled while its predecessor
// finishes and waits in-kernel (pdl_wait) before touching step buffers, which
// hides the launch gap and the setup (barriers, TMEM, descriptor prefetch).
bool pdl_enabled() {
  static const bool on = !(getenv("HB_NO_PDL") && getenv("HB_NO_PDL")[0] == '1');
  return on;
}
// The next launch on this stream is issued without the programmatic attribute
// (set where a merge kernel forks off the step: an early-launched successor
// would hold every SM and keep the merge -- and the copy behind it -- waiting
// for a whole GEMM).
thread_local cudaStream_t t_no_pdl_once = nullptr;
bool pdl_for(cudaStream_t st) {
  if (st != nullptr && st == t_no_pdl_once) {
    t_no_pdl_once = nullptr;
    return false;
  }
  return pdl_enabled();
}
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_for(st) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// launch_k with an optional L2 access-policy window: [base, base + bytes) is kept
// resident (persisting) in L2 while the kernel runs -- the operand a gather
// kernel re-reads row by row (W0^T for the CSR SpMM: every nonzero pulls one
// 4 KB row, 426 K rows per real-sim batch against 86 MB of unique bytes).
// The device's persisting carve-out is set once, to at most what it allows.
template <typename... KArgs, typename... Args>
cudaError_t launch_k_l2(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                        const void* base, size_t bytes, Args&&... args) {
  // measured on real-sim (b = 8192): no faster (0.655 vs 0.625 ms/step, the
  // carve-out shrinks the L2 every other kernel sees), so opt-in: HB_L2_WINDOW=1
  static const bool off = !(getenv("HB_L2_WINDOW") && getenv("HB_L2_WINDOW")[0] == '1');
  static size_t carve[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  size_t max_persist = 0;
  if (!off && dev < 64) {
    if (carve[dev] == 0) {
      cudaDeviceProp prop{};
      if (cudaGetDeviceProperties(&prop, dev) == cudaSuccess && prop.persistingL2CacheMaxSize > 0 &&
          cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prop.persistingL2CacheMaxSize) == cudaSuccess)
        carve[dev] = prop.persistingL2CacheMaxSize;
      else
        carve[dev] = 1;  // unsupported: remember, launch without the window
      cudaGetLastError();
    }
    max_persist = carve[dev] > 1 ? carve[dev] : 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_for(st) ? 1 : 0;
  int n = 1;
  if (max_persist > 0 && bytes > 0) {
    attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[1].val.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    attr[1].val.accessPolicyWindow.num_bytes = bytes;
    attr[1].val.accessPolicyWindow.hitRatio =
        static_cast<float>(std::min(1.0, static_cast<double>(max_persist) / static_cast<double>(bytes)));
    attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    n = 2;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ------------------------------------------------------------ GEMM launch
constexpr int kTileSyncTiles = 4096;
[[maybe_unused]] int g_trace_launch_no = 0;  // HB_TRACE builds: index of the GEMM launch being issued
// A GEMM operand: the fp32 tensor's map and its 3xTF32 lo twin's map.
struct Operand {
  const CUtensorMap* hi;
  const CUtensorMap* lo;
};

template <int BN, bool A_MN, bool B_MN, int EPI, int PASSES>
int launch_gemm_t(const Operand& ta, const Operand& tb, const GemmArgs& a, int m_tiles, int n_tiles, int splits,
                  cudaStream_t st) {
  using C = GemmCfg<BN, PASSES>;
  auto kern = gemm_tf32_kernel<BN, A_MN, B_MN, EPI, PASSES>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    HB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    configured = true;
  }
  // CTA pairs (cta_group::2) along M for the 3xTF32 kernels: grid.y padded to even
#ifdef HB_TRACE
  {
    const int target = getenv("HB_TRACE_LAUNCH") ? atoi(getenv("HB_TRACE_LAUNCH")) : -1;
    const_cast<GemmArgs&>(a).trace = (target < 0 || g_trace_launch_no == target) ? 1 : 0;
    const_cast<GemmArgs&>(a).trace_slot = 1 + g_trace_launch_no % 8;
    ++g_trace_launch_no;
  }
#endif
  const int cm = C::PAIR ? 2 : 1;
  const int gy = (m_tiles + cm - 1) / cm * cm;  // M tiles (padded to whole pairs) along grid.x
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(gy, n_tiles, splits);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cm;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_for(st) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t le = cudaLaunchKernelEx(&cfg, kern, *ta.hi, *tb.hi, *ta.lo, *tb.lo, a);
  if (le != cudaSuccess)
    return fail(HB_ECUDA, "gemm launch failed: %s (BN=%d pair=%d passes=%d grid=%d,%d,%d smem=%d)",
                cudaGetErrorString(le), BN, static_cast<int>(C::PAIR), PASSES, gy, n_tiles, splits, C::SMEM);
  return HB_OK;
}

enum GemmKind { G_FWD = 0, G_DX = 1, G_DW = 2 };

template <int PASSES>
int launch_gemm_p(GemmKind kind, int epi, int bn, const Operand& ta, const Operand& tb, const GemmArgs& a,
                  int m_tiles, int n_tiles, int splits, cudaStream_t st) {
#define HB_L(BN_, AMN_, BMN_, EPI_) \
  return launch_gemm_t<BN_, AMN_, BMN_, EPI_, PASSES>(ta, tb, a, m_tiles, n_tiles, splits, st)
#define HB_BN(AMN_, BMN_, EPI_)                    \
  do {                                             \
    if (bn == 32) HB_L(32, AMN_, BMN_, EPI_);      \
    if (bn == 64) HB_L(64, AMN_, BMN_, EPI_);      \
    if (bn == 256) HB_L(256, AMN_, BMN_, EPI_);    \
    HB_L(128, AMN_, BMN_, EPI_);                   \
  } while (0)
  if (kind == G_FWD) {
    if (epi == EPI_SIGMOID) HB_BN(false, false, EPI_SIGMOID);
    if (epi == EPI_PARTIAL) HB_BN(false, false, EPI_PARTIAL);
    HB_BN(false, false, EPI_STORE);
  }
  if (kind == G_DX) {
    if (epi == EPI_PARTIAL) HB_BN(false, true, EPI_PARTIAL);
    HB_BN(false, true, EPI_DSIG);
  }
  if (epi == EPI_SGD) HB_BN(true, true, EPI_SGD);
  if (epi == EPI_SPLIT_SGD) HB_BN(true, true, EPI_SPLIT_SGD);
  HB_BN(true, true, EPI_PARTIAL);
#undef HB_BN
#undef HB_L
}

// CTAs of the fused split-K dW kernel that can be resident at once (its split
// CTAs wait for each other, so a launch must never exceed this).
template <int BN, int PASSES>
int split_sgd_capacity_t() {
  using C = GemmCfg<BN, PASSES>;
  auto kern = gemm_tf32_kernel<BN, true, true, EPI_SPLIT_SGD, PASSES>;
  static int cap = -1;
  if (cap >= 0) return cap;
  cap = 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) != cudaSuccess) return cap;
  if (C::PAIR) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2, 1, 1);
    cfg.blockDim = dim3(C::THREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) == cudaSuccess) cap = 2 * clusters;
  } else {
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM) == cudaSuccess)
      cap = per_sm * sms;
  }
  cudaGetLastError();
  return cap;
}

int split_sgd_capacity(int passes, int bn) {
#define HB_C(P_)                                       \
  do {                                                 \
    if (bn == 32) return split_sgd_capacity_t<32, P_>();   \
    if (bn == 64) return split_sgd_capacity_t<64, P_>();   \
    if (bn == 256) return split_sgd_capacity_t<256, P_>(); \
    return split_sgd_capacity_t<128, P_>();                \
  } while (0)
  if (passes == 3) HB_C(3);
  HB_C(1);
#undef HB_C
}

int launch_gemm(int passes, GemmKind kind, int epi, int bn, const Operand& ta, const Operand& tb,
                const GemmArgs& a, int m_tiles, int n_tiles, int splits, cudaStream_t st) {
  if (passes == 3) return launch_gemm_p<3>(kind, epi, bn, ta, tb, a, m_tiles, n_tiles, splits, st);
  return launch_gemm_p<1>(kind, epi, bn, ta, tb, a, m_tiles, n_tiles, splits, st);
}

// ---------------------------------------------------------------- NCCL (dlopen)
typedef struct {
  char internal[128];
} nccl_uid_t;
typedef void* nccl_comm_t;
struct NcclApi {
  void* h = nullptr;
  int (*getUniqueId)(nccl_uid_t*) = nullptr;
  int (*commInitRank)(nccl_comm_t*, int, nccl_uid_t, int) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*commDestroy)(nccl_comm_t) = nullptr;
  const char* (*errStr)(int) = nullptr;
};
NcclApi g_nccl;
int load_nccl() {
  if (g_nccl.h) return HB_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail(HB_ENCCL, "cannot dlopen libnccl.so.2: %s", dlerror());
  g_nccl.getUniqueId = reinterpret_cast<int (*)(nccl_uid_t*)>(dlsym(h, "ncclGetUniqueId"));
  g_nccl.commInitRank = reinterpret_cast<int (*)(nccl_comm_t*, int, nccl_uid_t, int)>(dlsym(h, "ncclCommInitRank"));
  g_nccl.allReduce =
      reinterpret_cast<int (*)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t)>(dlsym(h, "ncclAllReduce"));
  g_nccl.commDestroy = reinterpret_cast<int (*)(nccl_comm_t)>(dlsym(h, "ncclCommDestroy"));
  g_nccl.errStr = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
  if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.allReduce || !g_nccl.commDestroy)
    return fail(HB_ENCCL, "libnccl is missing required symbols");
  g_nccl.h = h;
  return HB_OK;
}
constexpr int kNcclFloat32 = 7;  // ncclFloat32
constexpr int kNcclSum = 0;      // ncclSum

}  // namespace

// ======================================================================
struct DataView {
  // dense
  const float* x = nullptr;
  long long ldx = 0;
  long long n_rows = 0;
  const float* x_lo = nullptr;  // 3xTF32 lo twin of x (same layout)
  bool x_lo_zero = false;        // every x is exact in TF32 (lo twin all zero): layer-0 GEMMs skip it
  CUtensorMap tm_fwd, tm_fwd_lo;  // K-major A operand of the first forward GEMM
  CUtensorMap tm_dw, tm_dw_lo;    // MN-major B operand of the first dW GEMM
  Operand fwd() const { return {&tm_fwd, x_lo ? &tm_fwd_lo : &tm_fwd}; }
  Operand dw() const { return {&tm_dw, x_lo ? &tm_dw_lo : &tm_dw}; }
  // sparse
  const int64_t* rowptr = nullptr;
  const int32_t* col = nullptr;
  const float* val = nullptr;
  const int64_t* colptr = nullptr;
  const int32_t* rowidx = nullptr;
  const float* cval = nullptr;
  const int64_t* labels = nullptr;
};

struct Mark {
  std::string name;
  cudaEvent_t e0, e1;
};
struct StepGraph {
  cudaGraphExec_t exec = nullptr;
  std::vector<char> xdma_used;  // device-lane merges inside this graph
  std::vector<char> d2h_defer;  // deferred-landing graphs: layers whose D2H follows the launch
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> events;
  int launches = 0;
};

// Host->device batch bytes issued by the calling thread since the last reset
// (hb_replica_step*: reported by hb_last_xfer_bytes with the exchange bytes).
static thread_local long long t_h2d_bytes = 0;

// Ranks of a peer-merge group that live in one process (one GPU worker
// thread each, as the reference engine runs its roster).  They order their
// merges with events and a host barrier instead of device-side flag waits: two
// streams of one process can share a hardware queue, where a spinning wait
// kernel queued ahead of a peer's pack kernel would never let it run.
struct LocalGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long phase = 0;
  std::vector<cudaEvent_t> ev_pack, ev_red;  // per rank, created on that rank's device
  bool broken = false;
  // every rank arrives (bounded wait: a rank that never merges is an error, not a hang)
  bool barrier(double timeout_s) {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long my = phase;
    if (++arrived == n) {
      arrived = 0;
      ++phase;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return phase != my || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

struct hb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int L = 0;
  std::vector<int> d;          // layer sizes, L+1 entries
  std::vector<long long> ld;   // padded row stride of a width-d_l buffer
  int cap = 0;                 // row capacity (max_batch rounded up to 128)
  int max_batch = 0;
  bool csr_in = false;  // the context takes CSR input (HB_SPARSE_INPUT)
  bool sparse = false;  // ... and runs layer 0 on the CSR kernels (else: densified rows + GEMM)
  int passes = 3;
  bool small_head = false;
  int head_nct = 0, head_maxt = 0;

  std::vector<float*> W, G;    // W[l]; G[l] raw gradient (EMIT_GRAD)
  std::vector<float*> bias;    // optional fixed per-unit offset of hidden layer l (hb_set_bias_f64), or null
  std::vector<float*> W_lo, A_lo, D_lo;  // 3xTF32 lo twins of the GEMM operands (3-pass only)
  std::vector<long long> ldw;  // row stride of W[l] (in its device layout)
  std::vector<float*> A;       // A[l] l=1..L-1 activations (cap, ld[l])
  std::vector<float*> D;       // D[l] error at the output of layer l (cap, ld[l+1])
  std::vector<int> bn_fwd, bn_dx, bn_dw;
  std::vector<CUtensorMap> tmW_k, tmW_mn, tmA_k, tmA_mn, tmD_k, tmD_mn;
  std::vector<CUtensorMap> tmW_k_lo, tmW_mn_lo, tmA_k_lo, tmA_mn_lo, tmD_k_lo, tmD_mn_lo;
  bool need_lo() const { return passes == 3; }
  Operand opW_k(int l) const { return {&tmW_k[l], need_lo() ? &tmW_k_lo[l] : &tmW_k[l]}; }
  Operand opW_mn(int l) const { return {&tmW_mn[l], need_lo() ? &tmW_mn_lo[l] : &tmW_mn[l]}; }
  Operand opA_k(int l) const { return {&tmA_k[l], need_lo() ? &tmA_k_lo[l] : &tmA_k[l]}; }
  Operand opA_mn(int l) const { return {&tmA_mn[l], need_lo() ? &tmA_mn_lo[l] : &tmA_mn[l]}; }
  Operand opD_k(int l) const { return {&tmD_k[l], need_lo() ? &tmD_k_lo[l] : &tmD_k[l]}; }
  Operand opD_mn(int l) const { return {&tmD_mn[l], need_lo() ? &tmD_mn_lo[l] : &tmD_mn[l]}; }

  // staged epoch / host batch slot
  float* ex = nullptr;
  float* ex_lo = nullptr;
  int64_t* elabels = nullptr;
  int64_t *erowptr = nullptr, *ecolptr = nullptr;
  int32_t *ecol = nullptr, *erowidx = nullptr;
  float *eval_ = nullptr, *ecval = nullptr;
  long long e_rows = 0, e_nnz = 0;
  DataView epoch;
  bool staged = false;

  // unpermuted base copy kept on the device by hb_permute_epoch (the epoch
  // buffers above then hold base[perm]); gather/sort scratch reused per epoch
  bool has_base = false;
  float *px = nullptr, *px_lo = nullptr;
  int64_t *plabels = nullptr, *prowptr = nullptr, *pcolptr = nullptr;
  int32_t *pcol = nullptr, *prowidx = nullptr;
  float *pval = nullptr, *pcval = nullptr;
  int64_t *d_perm = nullptr, *d_inv = nullptr, *d_rowlen = nullptr;
  uint64_t* p_keys = nullptr;
  int32_t* p_idx = nullptr;
  void* p_temp = nullptr;
  size_t p_temp_bytes = 0;

  float* bx = nullptr;  // batch slot (dense rows) for host-buffer steps
  float* bx_lo = nullptr;
  float* bx_stage = nullptr;  // contiguous landing slot of a host batch whose device rows are padded
  int64_t* blabels = nullptr;
  int64_t *browptr = nullptr, *bcolptr = nullptr;
  int32_t *bcol = nullptr, *browidx = nullptr;
  float *bval = nullptr, *bcval = nullptr;
  long long b_nnz_cap = 0;
  DataView batch;
  std::vector<int64_t> h_colptr;  // host scratch for the per-batch CSC
  std::vector<int32_t> h_rowidx;
  std::vector<float> h_cval;
  void* pinned = nullptr;  // pinned host staging
  size_t pinned_bytes = 0;

  long long *csc_lo = nullptr, *csc_hi = nullptr;  // per-feature batch slices (sparse dW)
  uint32_t* csc_keys = nullptr;  // device batch-CSC build scratch (host-buffer steps)
  int32_t* csc_idx = nullptr;
  int* csc_counts = nullptr;
  void* csc_temp = nullptr;
  size_t csc_temp_bytes = 0;
  long long csc_cap = 0;
  double nnz_per_row = 0.0;
  float* ws = nullptr;  // split-K partials / head partials
  size_t ws_floats = 0;
  double* ws_loss = nullptr;
  int ws_loss_n = 0;
  double* d_loss = nullptr;
  double* h_loss = nullptr;  // mapped pinned: the loss read back by a kernel store, not a copy-engine D2H
  double* stage64 = nullptr;  // f64 staging for the weight exchange
  size_t stage64_n = 0;
  float* stage32 = nullptr;  // fp32 staging (grad transpose)
  double* stage_all = nullptr;  // whole-model f64 staging (set_weights_all)
  float* grad_all = nullptr;    // whole-model gradient gather
  float* grad_host = nullptr;   // pinned host copy of grad_all
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  float last_ms = 0.f;
  int last_launches = 0;
  cudaStream_t xfer = nullptr;                  // H2D stream of the pipelined host-model merge
  std::vector<cudaEvent_t> xfer_ev;             // one per merge chunk
  cudaEvent_t snap_ev = nullptr;                // snapshot DMA landed
  cudaEvent_t merge_ev = nullptr;               // merge: the step stream's prior work is done
  int* tile_sync = nullptr;  // split-K rendezvous counters (2 per output tile), zero between launches
  int pre_launches = 0;  // kernels a host-buffer step enqueued before do_step (densify / batch CSC)
  bool grads_valid = false;
  // per-launch CUDA-event profiling (bench.py reads it live; off by default)
  bool prof_on = false;
  std::vector<cudaEvent_t> evpool;
  size_t ev_used = 0;
  std::pair<cudaEvent_t, cudaEvent_t> pending;
  bool pending_active = false;
  std::string prof_filter;  // empty: every launch
  std::vector<Mark> step_marks;
  std::map<std::string, std::pair<double, int>> prof_acc;
  // CUDA graphs of the step, one per (rows, flags, data view generation)
  bool use_graphs = true;
  bool capturing = false;
  std::vector<cudaEvent_t> cap_events;
  std::map<std::tuple<int, uint32_t, long long, bool, long long>, StepGraph> graphs;
  std::map<std::tuple<int, uint32_t, long long, bool, long long>, int> graph_seen;
  DevStep* d_step = nullptr;  // device copy of the per-step scalars
  long long view_gen = 1;     // bumped whenever staged buffers / maps change
  // Overlapped host-model exchange of the fused replica step (hb_replica_step*):
  // while armed, the step itself snapshots the host float64 model layer by
  // layer (DMA on xh2d, layer l+1 in flight while layer l computes) and merges
  // W_host -= eta*g_l as a chunked DMA read-modify-write (H2D on xh2d, update
  // + D2H on xmrg) as soon as layer l's gradient exists.
  std::vector<double*> xw;          // armed host model (page-locked); empty: no exchange
  // Resident mirror (sole-writer calls): after a HB_STEP_SOLE_WRITER call the
  // f64 staging buffer holds exactly the host model (the device applies the
  // same f64 merge, rounding like np.add), so the next sole-writer call on the
  // same arrays skips the snapshot DMA -- unless a sampled fingerprint of the
  // host model shows another write in between.
  bool mirror_valid = false;   // stage_all == host model (as of the last call)
  long long mirror_gen = 0;    // pointer-set key the mirror belongs to
  bool xmirror = false;        // the call being enqueued uses (and keeps) the mirror
  bool xsole = false;          // the call being enqueued is a sole-writer call
  std::vector<double> fp_vals; // sampled host values after the last sole-writer call
  std::vector<double*> xw_prev;     // pointer set of the last armed call (graph key)
  long long pin_epoch = -1;         // g_pin_epoch when that set's page-lock was last checked
  long long xgen = 0;               // graph key of the armed pointer set (hash)
  cudaStream_t xh2d = nullptr, xmrg = nullptr;
  std::vector<cudaEvent_t> xsnap_ev, xgrad_ev, xchunk_ev;
  cudaEvent_t xstart_ev = nullptr, xdone_ev = nullptr;
  int xchunk_used = 0;
  // concurrent backward: split-K dW partial GEMMs and their reduce+SGD run on
  // `side` while the dX GEMMs run on `stream` (the partials never touch W)
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> bev;   // fork / join events of one backward pass
  cudaEvent_t bev_loss = nullptr; // fork of the loss reduction
  float* ws_dw = nullptr;         // per-layer split-K slabs of the concurrent dW partials
  double* ws_head = nullptr;      // the small head's per-block dW partials (float64)
  bool side_pending = false;      // the forward left work on `side` (joined by the backward)
  bool ranges_early = false;      // this step's CSC batch ranges were launched on `side` by the forward
  std::vector<size_t> ws_dw_off;
  bool conc_bwd = false;
  cudaStream_t prof_st = nullptr;  // stream the profiling marks go on (null: stream)
  // merge strategy: 0 = host (gradient D2H as fp32, float64 axpy on host
  // threads as each layer's gradient lands -- the reference's own np.add on
  // the host model); 1 = DMA read-modify-write through device memory
  int xmode = 0;       // this call: 0 = host / mirror merge, 1 = chunked device read-modify-write
  int xmode_env = 0;   // HB_XCHG_MERGE=dma: the DMA merge for sole-writer calls (its per-chunk window
                       // would drop a concurrent writer's updates; shared-model calls keep the host merge)
  // host mode: "layer l's gradient is in grad_host" flags.  Event syncs do
  // not survive graph capture, so the merge stream copies the call's sequence
  // number (read from pinned memory when the step runs) into xflags[l] after
  // the gradient D2H, and the calling thread polls it.
  float* xgrad_host = nullptr;    // pinned landing zone of the fp32 gradients
  int32_t* xseq_host = nullptr;  // pinned: [0] = this call's sequence number, [1 + l] = layer flags
  int32_t* d_xseq = nullptr;
  int32_t xseq = 0;
  // device lane of the host merge: layers whose stale merge is done by their
  // split-K reduce kernel on a float64 copy of the host rows DMA'd in just
  // before it and DMA'd back (splits the merge between PCIe and host DRAM)
  std::vector<char> xdma;       // planned per layer
  std::vector<char> xml;        // sole-writer calls: layers merged on the mirror lane (planned per layer)
  // one merge stream per layer: a layer's merge / copy-back starts as soon as
  // its gradient exists, not behind a later-finishing layer's (the backward's
  // two streams can finish layers out of order)
  std::vector<cudaStream_t> xmrg_l;
  std::vector<cudaEvent_t> xmdone_ev;
  std::vector<char> xmrg_used;  // this call's layers whose merge stream carried work (joined at the end)
  long long last_h2d = 0, last_d2h = 0;  // PCIe bytes of the last hb_replica_step* call
  std::vector<char> xdma_used;  // taken by the step just enqueued (rows decide whether the split-K path runs)
  std::vector<cudaEvent_t> xread_ev;
  void* comm = nullptr;
  int nranks = 1;
  float* flat = nullptr;  // contiguous model copy for allreduce
  size_t n_params = 0;
  // replica merge over peer memory (hb_peer_handle / hb_peer_attach): own
  // exchange buffer (flags + flat model), every rank's buffer mapped
  char* xbuf = nullptr;
  PeerTable peers{};                // peers.n == 0: not attached
  std::vector<void*> ipc_opened;    // peer buffers opened through CUDA IPC
  unsigned long long peer_gen = 0;  // merges issued (the flag value of the last one)
  // per-layer merge inside the backward (HB_STEP_MERGE with NCCL or a
  // cross-process peer group): layer l is averaged on comm_st as soon as its
  // update lands, overlapping the rest of the backward
  bool merge_layers = false;
  cudaStream_t comm_st = nullptr;
  std::vector<cudaEvent_t> mev;  // per layer: update done; mev[L]: comm stream joined
  std::vector<long long> flat_off;  // segment start of layer l in the packed model (multiple of 4)
  long long flat_n = 0;             // packed model length incl. segment padding
  std::shared_ptr<LocalGroup> local;  // all ranks in this process: event + host-barrier ordering
  // hb_replica_begin / hb_replica_end: the replica step in flight between them
  bool pend_active = false;
  int pend_rows = 0;
  double pend_eta = 0.0;
  uint32_t pend_flags = 0;
  // HB_STEP_LAND_ASYNC (sole writer): the call returns once the step and its
  // loss are done; the merged layers' write-backs land in the host model in the
  // background (the next call's batch copy and forward overlap them)
  bool xland = false;                  // this call defers its write-backs
  bool land_pending = false;           // write-backs of a deferred call may be in flight
  std::vector<double*> land_ws;        // the host model they land in
  std::vector<cudaEvent_t> xmerged_ev;  // layer l's merged float64 values are on the device
  std::vector<char> xmerged_rec;       // ... recorded by the pending call
  // deferred calls replayed from the step graph (every layer on the mirror
  // lane): the graph ends after the merge kernels; each merged layer's D2H is
  // issued after the graph launch, on the layer's merge stream, behind an
  // external event the graph records (xd2h_ready_ev), and the next graph's
  // merge of that layer waits for xd2h_done_ev before it rewrites the rows
  std::vector<cudaEvent_t> xd2h_ready_ev, xd2h_done_ev;
  std::vector<char> xd2h_defer;        // layers whose D2H the graph being captured leaves to its launcher
  // small nets (hb_small.cuh): the whole training step as one persistent kernel
  bool sn_ok = false;          // shape qualifies (dense, small head, widths <= kSnMaxWidth) and HB_SMALL_NET=1
  int sn_grid = 0;             // CTAs of the cooperative launch (all co-resident)
  float* sn_hd = nullptr;      // (kSnMaxRows, 4) output error signal
  double* sn_loss = nullptr;   // (kSnMaxRows) per-row loss
  unsigned* sn_bar = nullptr;  // grid barrier counter
};

extern "C" {
static int land_wait(hb_ctx* c);  // (defined in the extern "C" block below)
}

namespace {

int enqueue_layer_merge(hb_ctx* c, int l, cudaStream_t src, const DevStep* ds);
const float* layer_bias(const hb_ctx* c, int l);

const float* layer_bias(const hb_ctx* c, int l) {
  return l < static_cast<int>(c->bias.size()) ? c->bias[l] : nullptr;
}

int ctx_check(hb_ctx* c) {
  if (c == nullptr) return fail(HB_EINVAL, "null context");
  HB_CUDA(cudaSetDevice(c->device));
  return HB_OK;
}


// Profiling marks: (kernel name, begin event, end event) on the step stream.
// Eager steps take events from a reusable pool; a captured graph owns its
// events (they become event-record nodes) and re-reads them after every launch.
static void prof_name(char (&name)[64], const char* kind, int layer) {
  if (layer >= 0)
    snprintf(name, sizeof name, "%s_l%d", kind, layer);
  else
    snprintf(name, sizeof name, "%s", kind);
}
// A launch is bracketed when profiling is on and it passes the filter (the
// bench instruments only the dominant kernel inside its timed region).
// HB_NVTX=1: every step launch also sits in an NVTX range of the same name, so
// `ncu --nvtx --nvtx-include "gemm_dx_dsig_l2/"` captures exactly that kernel
// (eager steps, HB_NO_GRAPHS=1) -- how profiles/ ties traffic to bench names.
static bool nvtx_on() {
  static const bool on = getenv("HB_NVTX") && getenv("HB_NVTX")[0] == '1';
  return on;
}
void prof_begin(hb_ctx* c, const char* kind, int layer) {
  c->pending_active = false;
  char name[64];
  if (nvtx_on()) {
    prof_name(name, kind, layer);
    nvtxRangePushA(name);
  }
  if (!c->prof_on) return;
  prof_name(name, kind, layer);
  if (!c->prof_filter.empty() && c->prof_filter != name) return;
  cudaEvent_t e0, e1;
  if (c->capturing) {
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return;
    c->cap_events.push_back(e0);
    c->cap_events.push_back(e1);
  } else {
    while (c->evpool.size() < c->ev_used + 2) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return;
      c->evpool.push_back(e);
    }
    e0 = c->evpool[c->ev_used];
    e1 = c->evpool[c->ev_used + 1];
    c->ev_used += 2;
  }
  c->pending = {e0, e1};
  c->pending_active = true;
  // inside stream capture a plain record is only a dependency marker; the
  // External flag makes it a real event-record node of the graph
  if (c->capturing)
    cudaEventRecordWithFlags(e0, c->prof_st ? c->prof_st : c->stream, cudaEventRecordExternal);
  else
    cudaEventRecord(e0, c->prof_st ? c->prof_st : c->stream);
}
void prof_end(hb_ctx* c, const char* kind, int layer) {
  if (nvtx_on()) nvtxRangePop();
  if (!c->prof_on || !c->pending_active) return;
  c->pending_active = false;
  if (c->capturing)
    cudaEventRecordWithFlags(c->pending.second, c->prof_st ? c->prof_st : c->stream, cudaEventRecordExternal);
  else
    cudaEventRecord(c->pending.second, c->prof_st ? c->prof_st : c->stream);
  char name[64];
  prof_name(name, kind, layer);
  c->step_marks.push_back({name, c->pending.first, c->pending.second});
}
// fold the marks of a completed step into the per-kernel totals
int prof_resolve(hb_ctx* c, const std::vector<Mark>& marks) {
  for (auto& m : marks) {
    float ms = 0.f;
    HB_CUDA(cudaEventElapsedTime(&ms, m.e0, m.e1));
    auto& acc = c->prof_acc[m.name];
    acc.first += ms;
    acc.second += 1;
  }
  return HB_OK;
}

int build_data_maps(hb_ctx* c, DataView& v) {
  if (c->sparse) return HB_OK;
  HB_TRY(make_map(&v.tm_fwd, v.x, c->d[0], v.n_rows, v.ldx, 128, false));
  HB_TRY(make_map(&v.tm_dw, v.x, c->d[0], v.n_rows, v.ldx, 32, true));
  if (v.x_lo != nullptr) {
    HB_TRY(make_map(&v.tm_fwd_lo, v.x_lo, c->d[0], v.n_rows, v.ldx, 128, false));
    HB_TRY(make_map(&v.tm_dw_lo, v.x_lo, c->d[0], v.n_rows, v.ldx, 32, true));
  }
  return HB_OK;
}

long long env_long(const char* name, long long dflt) {
  const char* v = getenv(name);
  return v != nullptr && v[0] != 0 ? atoll(v) : dflt;
}

int choose_bn(long long m_tiles, long long n, bool batch_rows = false) {
  // narrow outputs get narrow tiles: less wasted MMA work and more TMEM
  // accumulators to rotate over (hb_gemm.cuh, GemmCfg::NBIG)
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  if (m_tiles * cdiv(n, 256) >= 120) return 256;
  // forward / dX GEMMs of a small batch (covtype's b = 512): 64-wide tiles give more CTAs to
  // spread the latency-bound k-loop over (measured covtype 0.084 -> 0.080 ms/step; on w8a's dW
  // GEMMs -- few M tiles but a long K -- it measured 20% slower, hence batch rows only)
  if (batch_rows && m_tiles * cdiv(n, 128) < 32 && env_long("HB_SMALL_BN64", 1) != 0) return 64;
  return 128;
}


// Accumulator drain (hb_gemm.cuh "Drain mode") per GEMM: D k-blocks per
// fresh accumulator, 0 = rotating accumulators.  The precision-critical GEMMs
// are the ones the output layer's cancelling dW sum depends on -- the forward
// GEMM that produces A_{L-1} and, for a wide softmax head, its logits and dW
// GEMMs: the truncating tensor-core accumulation over a whole K biases them
// enough to miss the per-step 1e-4 weight bar at near-cancelling output
// weights (real-sim 8.6e-4, delicious 1.1e-4; 4.6e-5 / 8e-6 drained every
// k-block).  Measured at b = 8192 (seed 1, worst weight error / step time):
//   small head (real-sim)  D=1 4.6e-5 / 0.630 ms  D=2 1.03e-4  D=3 1.44e-4   rotation 8.6e-4 / 0.602 ms
//   wide head (delicious)  D=1 7e-6 / 0.727 ms    D=2 2.1e-5 / 0.645 ms      rotation 1.1e-4 / 0.626 ms
//   wide head (scaled)     D=2 6e-6 / 8.25 ms     D=3 9.6e-6 / 8.18 ms       rotation 3.9e-5 / 8.36 ms
// (the drained head GEMMs also keep their 256-wide tiles, which the rotation
// had to give up for precision).  Others keep the rotation (HB_DRAIN_KB: their
// D, 0 = off); HB_DRAIN_KB_CRIT overrides the critical ones' D.
enum GemmRole { R_FWD = 0, R_LOGITS = 1, R_DX = 2, R_DW = 3 };
// (small heads need D=1 even at K = 512: w8a with D=2 measured 1.21e-4 on one of five seeds)
int crit_drain_default(const hb_ctx* c, int) { return c->small_head ? 1 : 2; }
int drain_kb(const hb_ctx* c, GemmRole role, int l) {
  if (c->passes != 3 || !HB_GEMM_DRAIN) return 0;
  const int L = c->L;
  const bool crit = (role == R_FWD && l == L - 2) || (!c->small_head && l == L - 1 && (role == R_LOGITS || role == R_DW));
  if (crit) return static_cast<int>(env_long("HB_DRAIN_KB_CRIT", crit_drain_default(c, l)));
  // small heads: the other forward GEMMs feed the critical one; D=3 (the drain hides under three k-blocks
  // of MMAs) lifts w8a's worst of 20 seeds from 9.8e-5 to 7.2e-5 at no measured cost.  Wide heads have the
  // margin without it (and the scaled config's power-capped GEMMs measured ~3% slower with it).
  if (role == R_FWD)
    return static_cast<int>(env_long("HB_DRAIN_KB_FWD", env_long("HB_DRAIN_KB", c->small_head ? 3 : 0)));
  return static_cast<int>(env_long("HB_DRAIN_KB", 0));
}

// Split-K plan for a forward / dX GEMM: when its output tiles cannot fill
// the SMs (small batches, e.g. covtype's b=512 gives 8-16 CTAs) K is split so
// the launch covers about one wave; splitk_epi_kernel sums the slabs and
// applies the fused op.  Returns the split count (1 = no split).
constexpr int kSplitSlabFloats = 148 * kBM * 256;  // bound on S * M * N of any such split
int fx_plan(const hb_ctx* c, int m_tiles, int n_tiles, int bn, int kb_total, int* kb_per) {
  *kb_per = kb_total;
  if (getenv("HB_NO_FX_SPLIT") && getenv("HB_NO_FX_SPLIT")[0] == '1') return 1;
  const int ctas = (c->passes == 3 && bn >= 64 ? (m_tiles + 1) / 2 * 2 : m_tiles) * n_tiles;
  if (ctas >= 64 || kb_total < 4) return 1;
  const int want = std::min(148 / ctas, kb_total / 2);
  if (want < 2) return 1;
  *kb_per = cdiv(kb_total, want);
  return cdiv(kb_total, *kb_per);
}

// split-K plan for the dW GEMM of layer l at `rows` batch rows
void dw_plan(const hb_ctx* c, int l, int rows, int* splits, int* kb_per, int* kb_total) {
  const int M = c->d[l + 1], N = c->d[l];
  // CTAs per split: M tiles padded to whole CTA pairs (3xTF32 kernels run in pairs)
  const int mt = cdiv(M, kBM);
  const int tiles = (c->passes == 3 && c->bn_dw[l] >= 64 ? (mt + 1) / 2 * 2 : mt) * cdiv(N, c->bn_dw[l]);
  *kb_total = std::max(1, cdiv(rows, kBK));
  // one wave: as many K splits as fit on the 148 SMs (1 CTA / SM)
  int want = std::max(1, 148 / tiles);
  if (l == c->L - 1 && !c->small_head && c->passes == 3 && !(drain_kb(c, R_DW, l) > 0 && c->bn_dw[l] >= 64)) {
    // precision: at most 16 k-blocks per rotating hi*hi accumulator for the
    // softmax head's cancelling dW sum (measured: 1e-4 bar missed at 1024
    // MMAs per accumulator on the 1000-class scaled config)
    const int nbig = std::min(15, std::max(1, 512 / c->bn_dw[l] - 1));
    want = std::max(want, cdiv(*kb_total, 16 * nbig));
  }
  want = std::min(want, *kb_total);
  *kb_per = cdiv(*kb_total, want);
  *splits = cdiv(*kb_total, *kb_per);
}

// debug (HB_DEBUG_XFER=1): host-side phase timings of the host-model exchange
static bool xfer_debug() {
  static const bool on = getenv("HB_DEBUG_XFER") && getenv("HB_DEBUG_XFER")[0] == '1';
  return on;
}
struct XferClock {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  const char* what;
  explicit XferClock(const char* w) : what(w) {}
  void mark(const char* phase) const {
    if (!xfer_debug()) return;
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "[xfer] %s %s %.1f us\n", what, phase, us);
  }
};

static std::chrono::steady_clock::time_point g_call_t0;
static void xmark(const char* what, int l = -1) {
  if (!xfer_debug()) return;
  const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - g_call_t0).count();
  fprintf(stderr, "[xfer] %8.1f us  %s %d\n", us, what, l);
}

// split-K forward / dX: partial slabs into c->ws, then the fused finish
int launch_fx_split(hb_ctx* c, GemmKind kind, int mode, int bn, const Operand& ta, const Operand& tb, GemmArgs a,
                    int m_tiles, int n_tiles, int splits, int kb_per, cudaStream_t st) {
  float* out = a.out;
  float* out_lo = a.out_lo;
  const long long ldo = a.ldo;
  a.out = c->ws;
  a.out_lo = nullptr;
  a.ldo = a.N;
  a.split_stride = static_cast<long long>(a.M) * a.N;
  a.kb_per_split = kb_per;
  {
    GemmArgs pa = a;
    pa.bias = nullptr;  // the slabs are raw partial sums; the finish adds the bias once
    HB_TRY(launch_gemm(c->passes, kind, EPI_PARTIAL, bn, ta, tb, pa, m_tiles, n_tiles, splits, st));
  }
  const bool vec = (a.N % 4 == 0) && (ldo % 4 == 0);
  const int rows_total = mode == SPLIT_DSIG ? std::max(a.M, a.m_zero_rows) : a.M;
  const long long items = static_cast<long long>(rows_total) * (vec ? a.N / 4 : a.N);
  const dim3 grid(static_cast<int>(std::min<long long>(cdiv(items, 256), 148 * 8)));
#define HB_SE(MODE_, VEC_)                                                                                  \
  HB_CUDA(launch_k(splitk_epi_kernel<MODE_, VEC_>, grid, dim3(256), 0, st, out, out_lo, ldo, c->ws, splits, a.M, \
                   a.N, a.aux, a.ld_aux, a.m_zero_rows, a.bias))
  if (mode == SPLIT_SIGMOID) {
    if (vec) HB_SE(SPLIT_SIGMOID, true); else HB_SE(SPLIT_SIGMOID, false);
  } else if (mode == SPLIT_STORE) {
    if (vec) HB_SE(SPLIT_STORE, true); else HB_SE(SPLIT_STORE, false);
  } else {
    if (vec) HB_SE(SPLIT_DSIG, true); else HB_SE(SPLIT_DSIG, false);
  }
#undef HB_SE
  c->last_launches++;
  return HB_OK;
}

// ---------------------------------------------- overlapped host-model exchange
// (armed by hb_replica_step*; every call below is a no-op otherwise).  All of
// it is plain stream/event work, so it is captured into the step's CUDA graph
// like the kernels (the graph key carries the armed pointer set).
// debug (HB_DEBUG_XCHG=1, eager steps): timeline of the exchange on its streams
static bool xchg_debug() {
  static const bool on = getenv("HB_DEBUG_XCHG") && getenv("HB_DEBUG_XCHG")[0] == '1';
  return on;
}
// (capture-safe: events are external record nodes of the step graph, reused by label)
static std::vector<std::pair<std::string, cudaEvent_t>> g_xtl;
static cudaError_t record_ev(hb_ctx* c, cudaEvent_t e, cudaStream_t s) {
  return c->capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s);
}
static void xtl(hb_ctx* c, cudaStream_t s, const char* fmt, int a = 0, int b = 0) {
  if (!xchg_debug()) return;
  char buf[96];
  snprintf(buf, sizeof buf, fmt, a, b);
  static const char* only = getenv("HB_XTL_ONLY");  // record only labels containing this (and begin / end)
  if (only && !strstr(buf, only) && strcmp(buf, "begin") != 0 && strcmp(buf, "end") != 0) return;
  cudaEvent_t e = nullptr;
  for (auto& p : g_xtl)
    if (p.first == buf) e = p.second;
  if (e == nullptr) {
    cudaEventCreate(&e);
    g_xtl.emplace_back(buf, e);
  }
  cudaError_t er = record_ev(c, e, s);
  if (er != cudaSuccess) fprintf(stderr, "[xchg] event %s: %s\n", buf, cudaGetErrorString(er));
}
static void xtl_dump() {
  if (g_xtl.empty()) return;
  cudaDeviceSynchronize();
  for (auto& p : g_xtl) {
    float ms = 0.f;
    cudaError_t er = cudaEventElapsedTime(&ms, g_xtl.front().second, p.second);
    fprintf(stderr, "[xchg] %8.1f us  %s %s\n", ms * 1000.f, p.first.c_str(),
            er == cudaSuccess ? "" : cudaGetErrorString(er));
  }
  cudaGetLastError();
}

// Small persistent pool for the host side of the merge: run(n, fn) calls
// fn(0..n-1) on up to n threads (the caller included) and returns when done.
// Workers spin briefly after each job (a merge is a burst of one job per
// layer, tens of microseconds apart) before sleeping on the condition variable.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool p;
    return p;
  }
  int size() const { return static_cast<int>(threads_.size()) + 1; }
  void run(int n, const std::function<void(int)>& fn) {
    if (n <= 1 || threads_.empty()) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    // one job at a time: several replica worker threads (one per GPU, as the
    // reference engine runs them) may merge concurrently
    std::lock_guard<std::mutex> job(run_mu_);
    const uint64_t jid = ++job_;
    fn_.store(&fn, std::memory_order_relaxed);
    done_.store(0, std::memory_order_relaxed);
    // a ticket is (job, n, index): whoever takes one knows which job and how
    // many parts it has without reading shared fields that the next job may
    // already have replaced, so a late worker can never run a part twice or
    // run a stale part with the next job's function
    next_.store(ticket(jid, n, 0), std::memory_order_release);
    {
      std::lock_guard<std::mutex> lk(mu_);
      gen_.fetch_add(1, std::memory_order_acq_rel);
    }
    cv_.notify_all();
    work();
    while (done_.load(std::memory_order_acquire) < n) pause();
    next_.store(ticket(jid, 0, 0), std::memory_order_release);  // late workers find nothing to take
  }

 private:
  static constexpr int kIdxBits = 20;
  static constexpr uint64_t kIdxMask = (uint64_t(1) << kIdxBits) - 1;
  static uint64_t ticket(uint64_t jid, int n, int i) {
    return (jid << (2 * kIdxBits)) | (static_cast<uint64_t>(n) << kIdxBits) | static_cast<uint64_t>(i);
  }
  static void pause() {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  void work() {
    for (;;) {
      // index overflow into the n field is impossible: at most n + (threads)
      // tickets are ever taken per job, far below 2^20
      const uint64_t t = next_.fetch_add(1, std::memory_order_acq_rel);
      const int i = static_cast<int>(t & kIdxMask), n = static_cast<int>((t >> kIdxBits) & kIdxMask);
      if (i >= n) return;
      // a valid ticket of job J: J cannot finish (done_ < n) before this part
      // is counted, so fn_ still holds J's function (published before next_)
      (*fn_.load(std::memory_order_acquire))(i);
      done_.fetch_add(1, std::memory_order_acq_rel);
    }
  }
  HostPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    // merge threads (caller included): 3/4 of the host threads, at most 12 -- e2e on a 16-thread B200 host,
    // w8a / covtype / delicious: 8 threads 1.46e7 / 1.36e6 / 4.71e6, 12 threads 1.54e7 / 1.36e6 / 4.87e6
    int t = static_cast<int>(std::min(12u, std::max(1u, hw * 3 / 4)));
    if (const char* e = getenv("HB_HOST_MERGE_THREADS")) t = std::max(1, atoi(e));
    spins_ = getenv("HB_POOL_SPIN") ? atoi(getenv("HB_POOL_SPIN")) : 20000;
    next_.store(ticket(0, 0, 0));
    start(t);
  }
  ~HostPool() { stop(); }

 public:
  // Resize the pool (threads, caller included) and its post-job spin: a CPU
  // Hogwild pool in the same process wants the cores back (hb_host_merge_threads)
  void configure(int threads, int spins) {
    std::lock_guard<std::mutex> job(run_mu_);  // no job in flight
    stop();
    spins_ = std::max(0, spins);
    start(std::max(1, threads));
  }

 private:
  void start(int threads) {
    stop_ = false;
    // the generation a worker starts from is read here, not in the new
    // thread: a stop() racing its start-up must still wake it
    const unsigned long long g0 = gen_.load();
    for (int i = 0; i < threads - 1; ++i) threads_.emplace_back([this, g0] { loop(g0); });
  }
  void stop() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
    threads_.clear();
  }
  void loop(unsigned long long seen) {
    for (;;) {
      // spin ~0.5 ms for the next job (a merge is a burst of one job per
      // layer), then sleep; spin 0 yields the cores at once
      const int spins = spins_;
      for (int k = 0; k < spins && gen_.load(std::memory_order_acquire) == seen; ++k) pause();
      if (gen_.load(std::memory_order_acquire) == seen) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_.load() != seen; });
      }
      if (stop_) return;
      seen = gen_.load(std::memory_order_acquire);
      work();
    }
  }
  std::vector<std::thread> threads_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_;
  std::atomic<const std::function<void(int)>*> fn_{nullptr};
  std::atomic<uint64_t> next_{0};
  std::atomic<int> done_{0};
  std::atomic<unsigned long long> gen_{0};
  uint64_t job_ = 0;
  std::atomic<bool> stop_{false};
  std::atomic<int> spins_{20000};
};

#if defined(__x86_64__)
// One part of the merge.  Measured on the B200 host: device DMA into or out of
// host lines that sit in some core's private cache is slow (it snoops them
// out), so the merge leaves none behind -- w is written with streaming
// (non-temporal) stores and the gradient lines it read are flushed -- which is
// what lets several threads share the merge without slowing the next call's
// snapshot DMA or the next gradient DMA.
__attribute__((target("sse4.1,clflushopt"))) static void axpy_part(double* w, const float* g, size_t a, size_t b,
                                                                    double scale) {
  size_t i = a;
  for (; i < b && (reinterpret_cast<uintptr_t>(w + i) & 15) != 0; ++i) w[i] = w[i] + scale * static_cast<double>(g[i]);
  const __m128d sc = _mm_set1_pd(scale);
  for (; i + 2 <= b; i += 2) {
    const __m128d gv = _mm_cvtps_pd(_mm_castpd_ps(_mm_load_sd(reinterpret_cast<const double*>(g + i))));
    _mm_stream_pd(w + i, _mm_add_pd(_mm_load_pd(w + i), _mm_mul_pd(sc, gv)));
  }
  for (; i < b; ++i) w[i] = w[i] + scale * static_cast<double>(g[i]);
  _mm_sfence();
  const uintptr_t g0 = reinterpret_cast<uintptr_t>(g + a) & ~uintptr_t(63), g1 = reinterpret_cast<uintptr_t>(g + b);
  for (uintptr_t p = g0; p < g1; p += 64) _mm_clflushopt(reinterpret_cast<void*>(p));
}
#else
static void axpy_part(double* w, const float* g, size_t a, size_t b, double scale) {
  for (size_t i = a; i < b; ++i) w[i] = w[i] + scale * static_cast<double>(g[i]);
}
#endif

// w[i] = w[i] + (-eta) * g[i]: linalg.py:79 np.add(target, scale*source,
// out=target) in float64, product and sum rounded separately (the library's
// host code is built with -ffp-contract=off), every double written whole
// (no torn scalars for concurrent host readers, linalg.py:3-7)
static void host_axpy_f64(double* w, const float* g, size_t n, double eta) {
  const double scale = -eta;
  HostPool& pool = HostPool::get();
  static const int max_parts = getenv("HB_MERGE_PARTS") ? atoi(getenv("HB_MERGE_PARTS")) : 64;
  static const size_t part_elems = getenv("HB_MERGE_PART_ELEMS") ? atoll(getenv("HB_MERGE_PART_ELEMS")) : (1 << 15);
  const int parts = static_cast<int>(
      std::min<size_t>(std::min(pool.size(), max_parts), std::max<size_t>(1, n / part_elems)));
  if (xfer_debug()) fprintf(stderr, "[xfer] axpy n=%zu parts=%d pool=%d\n", n, parts, pool.size());
  pool.run(parts, [&](int t) {
    // part boundaries on 16-element multiples keep the parts' cache lines apart
    const size_t a = (n * t / parts) & ~size_t(15), b = t + 1 == parts ? n : (n * (t + 1) / parts) & ~size_t(15);
    axpy_part(w, g, a, b, scale);
  });
}

size_t layer_offset(const hb_ctx* c, int l) {
  size_t off = 0;
  for (int i = 0; i < l; ++i) off += static_cast<size_t>(c->d[i + 1]) * c->d[i];
  return off;
}

// snapshot DMA of every layer (deep_copy, workers.py:132), layer 0 first
int xchg_begin(hb_ctx* c) {
  if (c->xw.empty()) return HB_OK;
  c->xchunk_used = 0;
  xtl(c, c->stream, "begin");
  if (c->xmode == 0)  // the sequence number the layer flags will carry (read at run time)
    HB_CUDA(cudaMemcpyAsync(c->d_xseq, c->xseq_host, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
  HB_CUDA(cudaEventRecord(c->xstart_ev, c->stream));
  HB_CUDA(cudaStreamWaitEvent(c->xh2d, c->xstart_ev, 0));  // earlier users of the staging buffer are done
  for (int l = 0; l < c->L; ++l) {
    const size_t n = static_cast<size_t>(c->d[l + 1]) * c->d[l];
    if (!c->xmirror)  // resident mirror: the staging buffer already holds the host model
      HB_CUDA(cudaMemcpyAsync(c->stage_all + layer_offset(c, l), c->xw[l], n * sizeof(double),
                              cudaMemcpyHostToDevice, c->xh2d));
    HB_CUDA(cudaEventRecord(c->xsnap_ev[l], c->xh2d));
    xtl(c, c->xh2d, "h2d: snapshot layer %d landed", l);
  }
  return HB_OK;
}

// before the first kernel that reads W_l: wait for its bytes, convert to the
// fp32 (+ lo twin) device layout
int xchg_use(hb_ctx* c, int l) {
  if (c->xw.empty()) return HB_OK;
  xtl(c, c->stream, "step: ready for W%d", l);
  HB_CUDA(cudaStreamWaitEvent(c->stream, c->xsnap_ev[l], 0));
  xtl(c, c->stream, "step: W%d snapshot available", l);
  const int rows = c->d[l + 1], cols = c->d[l];
  const size_t n = static_cast<size_t>(rows) * cols;
  const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 4096));
  const double* src = c->stage_all + layer_offset(c, l);
  if (l == 0 && c->sparse)
    HB_CUDA(launch_k(f64_to_f32_kernel<true>, dim3(blocks), dim3(256), 0, c->stream, c->W[0], c->ldw[0], src, cols, rows, cols, nullptr));
  else
    HB_CUDA(launch_k(f64_to_f32_kernel<false>, dim3(blocks), dim3(256), 0, c->stream, c->W[l], c->ldw[l], src, cols, rows, cols,
                                                            c->need_lo() ? c->W_lo[l] : nullptr));
  HB_CUDA(cudaGetLastError());
  c->last_launches++;
  return HB_OK;
}

// after the last kernel that writes G_l: stale merge of layer l into the host
// model (workers.py:135 -> nn.py:174-179 -> linalg.py:79, w += -eta*g in
// float64), chunk k read H2D while chunk k-1 is updated and written back D2H.
// Each chunk is read just before it is written, so the window in which a
// concurrent host writer's update could be overwritten stays one chunk long.
// deferred calls: "layer l's merged values (and every read of its gradient)
// are done" -- the next step waits for this before it converts or rewrites them
static int record_merged(hb_ctx* c, int l, cudaStream_t ms) {
  if (!c->xland) return HB_OK;
  HB_CUDA(c->capturing ? cudaEventRecordWithFlags(c->xmerged_ev[l], ms, cudaEventRecordExternal)
                       : cudaEventRecord(c->xmerged_ev[l], ms));
  c->xmerged_rec[l] = 1;
  return HB_OK;
}

int xchg_merge(hb_ctx* c, int l, double eta, const DevStep* ds, cudaStream_t src = nullptr) {
  if (c->xw.empty()) return HB_OK;
  if (src == nullptr) src = c->stream;
  xtl(c, src, "step: G%d done", l);
  cudaStream_t ms = c->xmrg;
  if (c->xmode == 0 && l < static_cast<int>(c->xmrg_l.size())) {
    ms = c->xmrg_l[l];
    c->xmrg_used[l] = 1;
  }
  HB_CUDA(cudaEventRecord(c->xgrad_ev[l], src));
  const int rows = c->d[l + 1], cols = c->d[l];
  const bool tr = (l == 0 && c->sparse);
  if (c->xmode == 0 && l < static_cast<int>(c->xdma_used.size()) && c->xdma_used[l] && src == c->side) {
    // device lane: the reduce kernel already merged the freshly read host
    // rows; write them back
    HB_CUDA(cudaStreamWaitEvent(ms, c->xgrad_ev[l], 0));
    HB_TRY(record_merged(c, l, ms));
    HB_CUDA(cudaMemcpyAsync(c->xw[l], c->stage_all + layer_offset(c, l),
                            static_cast<size_t>(rows) * cols * sizeof(double), cudaMemcpyDeviceToHost, ms));
    xtl(c, ms, "mrg: layer %d written back (device lane)", l);
    return HB_OK;
  }
  if (c->xmode == 0 && c->xsole && l < static_cast<int>(c->xml.size()) && c->xml[l]) {
    // mirror lane (sole writer): the device staging copy equals the host model
    // (snapshot or resident mirror), so the float64 merge runs on the device
    // (w + (-eta) * g, NumPy's rounding) and the merged layer goes D2H in place
    // of the gradient -- no host read-modify-write, no merge read
    HB_CUDA(cudaStreamWaitEvent(ms, c->xgrad_ev[l], 0));
    static const bool keep_pdl = getenv("HB_XCHG_KEEP_PDL") && getenv("HB_XCHG_KEEP_PDL")[0] == '1';
    if (!keep_pdl) t_no_pdl_once = src;
    const size_t n = static_cast<size_t>(rows) * cols;
    const size_t off = layer_offset(c, l);
    const bool defer_d2h = c->xland && c->capturing;
    if (defer_d2h)  // the previous call's copy of these rows was issued outside any graph
      HB_CUDA(cudaStreamWaitEvent(ms, c->xd2h_done_ev[l], cudaEventWaitExternal));
    merge_host_f64_kernel<<<static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 4)), 256, 0, ms>>>(
        c->stage_all + off, c->G[l], tr ? c->ldw[0] : cols, rows, cols, tr ? 1 : 0, eta, ds);
    HB_CUDA(cudaGetLastError());
    c->last_launches++;
    HB_TRY(record_merged(c, l, ms));
    if (defer_d2h) {
      HB_CUDA(cudaEventRecordWithFlags(c->xd2h_ready_ev[l], ms, cudaEventRecordExternal));
      c->xd2h_defer[l] = 1;
      if (l < static_cast<int>(c->xdma_used.size())) c->xdma_used[l] = 2;
      return HB_OK;
    }
    HB_CUDA(cudaMemcpyAsync(c->xw[l], c->stage_all + off, n * sizeof(double), cudaMemcpyDeviceToHost, ms));
    if (c->xland) HB_CUDA(cudaEventRecord(c->xd2h_done_ev[l], ms));
    if (l < static_cast<int>(c->xdma_used.size())) c->xdma_used[l] = 2;  // merged on the device (no host pass)
    xtl(c, ms, "mrg: layer %d written back (mirror lane)", l);
    return HB_OK;
  }
  if (c->xmode == 0) {
    // host mode: the fp32 gradient goes D2H on the merge stream; the calling
    // thread applies it (hb_replica_step*, xchg_host_merges)
    HB_CUDA(cudaStreamWaitEvent(ms, c->xgrad_ev[l], 0));
    const size_t n = static_cast<size_t>(rows) * cols;
    const size_t off = layer_offset(c, l);
    const float* src = c->G[l];
    if (tr) {
      transpose_f32_kernel<<<static_cast<int>(std::min<size_t>((n + 255) / 256, 1024)), 256, 0, ms>>>(
          c->grad_all + off, c->G[0], c->ldw[0], rows, cols);
      HB_CUDA(cudaGetLastError());
      c->last_launches++;
      src = c->grad_all + off;
    }
    HB_CUDA(cudaMemcpyAsync(c->xgrad_host + off, src, n * sizeof(float), cudaMemcpyDeviceToHost, ms));
    HB_CUDA(cudaMemcpyAsync(c->xseq_host + 1 + l, c->d_xseq, sizeof(int32_t), cudaMemcpyDeviceToHost, ms));
    if (c->xsole) {
      // the same f64 merge on the device copy (w + (-eta) * g, product and sum
      // rounded like the host's): the staging buffer stays equal to the host model
      merge_host_f64_kernel<<<static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 4)), 256, 0, ms>>>(
          c->stage_all + off, c->G[l], tr ? c->ldw[0] : cols, rows, cols, tr ? 1 : 0, eta, ds);
      HB_CUDA(cudaGetLastError());
      c->last_launches++;
    }
    HB_TRY(record_merged(c, l, ms));
    xtl(c, ms, "mrg: gradient %d on host", l);
    return HB_OK;
  }
  HB_CUDA(cudaStreamWaitEvent(c->xh2d, c->xgrad_ev[l], 0));
  const size_t kChunk = size_t(1) << 17;  // doubles (1 MiB)
  const int rows_per = static_cast<int>(std::max<size_t>(1, kChunk / std::max(1, cols)));
  double* base = c->stage_all + layer_offset(c, l);
  for (int r0 = 0; r0 < rows; r0 += rows_per) {
    const int nr = std::min(rows_per, rows - r0);
    const size_t e0 = static_cast<size_t>(r0) * cols, ne = static_cast<size_t>(nr) * cols;
    if (c->xchunk_used >= static_cast<int>(c->xchunk_ev.size())) {
      cudaEvent_t e;
      HB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->xchunk_ev.push_back(e);
    }
    cudaEvent_t ev = c->xchunk_ev[c->xchunk_used++];
    HB_CUDA(cudaMemcpyAsync(base + e0, c->xw[l] + e0, ne * sizeof(double), cudaMemcpyHostToDevice, c->xh2d));
    HB_CUDA(cudaEventRecord(ev, c->xh2d));
    xtl(c, c->xh2d, "h2d: merge read layer %d row %d", l, r0);
    HB_CUDA(cudaStreamWaitEvent(c->xmrg, ev, 0));
    const float* g = tr ? c->G[0] + r0 : c->G[l] + static_cast<size_t>(r0) * cols;
    // a few CTAs on the high-priority merge stream: they fit beside (or right
    // after) the step's GEMM CTAs instead of queueing behind a whole wave
    merge_host_f64_kernel<<<static_cast<int>(std::min<size_t>((ne + 255) / 256, 16)), 256, 0, c->xmrg>>>(
        base + e0, g, tr ? c->ldw[0] : cols, nr, cols, tr ? 1 : 0, eta, ds);
    HB_CUDA(cudaGetLastError());
    c->last_launches++;
    xtl(c, c->xmrg, "mrg: updated layer %d row %d", l, r0);
    HB_CUDA(cudaMemcpyAsync(c->xw[l] + e0, base + e0, ne * sizeof(double), cudaMemcpyDeviceToHost, c->xmrg));
    xtl(c, c->xmrg, "mrg: written back layer %d row %d", l, r0);
  }
  return HB_OK;
}

// host mode, on the calling thread after the step is enqueued: apply each
// layer's gradient as soon as it has landed, in the order the backward pass
// produces them (last layer first), overlapping the rest of the device work
int xchg_host_merges(hb_ctx* c, double eta) {
  if (c->xw.empty() || c->xmode != 0) return HB_OK;
  const int32_t seq = c->xseq;
  xmark("enqueued");
  for (int l = c->L - 1; l >= 0; --l) {
    if (l < static_cast<int>(c->xdma_used.size()) && c->xdma_used[l]) continue;  // merged on the device lane
    volatile int32_t* flag = c->xseq_host + 1 + l;
    // spin on the flag (pinned host memory, no driver calls); the stream is
    // queried only every ~2^18 spins to surface a failed step
    for (long long spin = 1; *flag != seq; ++spin) {
#if defined(__x86_64__)
      __builtin_ia32_pause();
#endif
      if ((spin & ((1 << 18) - 1)) == 0) {
        const cudaError_t e = cudaStreamQuery(c->stream);
        if (e == cudaSuccess && *flag != seq) return fail(HB_ECUDA, "merge of layer %d never signalled", l);
        if (e != cudaSuccess && e != cudaErrorNotReady)
          return fail(HB_ECUDA, "step failed during the merge: %s", cudaGetErrorString(e));
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    xmark("flag seen", l);
    host_axpy_f64(c->xw[l], c->xgrad_host + layer_offset(c, l), static_cast<size_t>(c->d[l + 1]) * c->d[l], eta);
    xmark("axpy done", l);
  }
  return HB_OK;
}

// join: the step stream waits for the last write-back
int xchg_end(hb_ctx* c) {
  if (c->xw.empty()) return HB_OK;
  for (size_t l = 0; l < c->xmrg_l.size(); ++l) {  // every layer's merge stream this call used
    if (!c->xmrg_used[l]) continue;
    c->xmrg_used[l] = 0;
    if (c->xland && !c->capturing) continue;  // deferred: lands in the background (land_wait / the next step's waits)
    // (a captured deferred step joins its merge streams: they hold only the merge kernels, the D2H follows the launch)
    HB_CUDA(cudaEventRecord(c->xmdone_ev[l], c->xmrg_l[l]));
    HB_CUDA(cudaStreamWaitEvent(c->stream, c->xmdone_ev[l], 0));
  }
  if (c->xmode != 0) {  // the DMA merge's chunks run on the shared merge stream
    HB_CUDA(cudaEventRecord(c->xdone_ev, c->xmrg));
    HB_CUDA(cudaStreamWaitEvent(c->stream, c->xdone_ev, 0));
  }
  xtl(c, c->stream, "end");
  // the H2D stream must rejoin too (its last reads feed xmrg, but a capture
  // needs every forked stream joined)
  HB_CUDA(cudaEventRecord(c->xstart_ev, c->xh2d));
  HB_CUDA(cudaStreamWaitEvent(c->stream, c->xstart_ev, 0));
  return HB_OK;
}

// `ds` != null: graph mode -- kernels read the batch start and eta from
// device memory (the by-value start/eta are then 0 and ignored).
// The batch loss is only read after the step (out_loss): in training steps
// with the concurrent backward its reduction runs on the side stream, off the
// forward -> backward critical path.
int launch_loss_reduce(hb_ctx* c, bool train, int n_partials) {
  cudaStream_t s = c->stream;
  if (train && c->conc_bwd) {
    HB_CUDA(cudaEventRecord(c->bev_loss, c->stream));
    HB_CUDA(cudaStreamWaitEvent(c->side, c->bev_loss, 0));
    s = c->side;
    c->side_pending = true;
  }
  HB_CUDA(launch_k(loss_reduce_kernel, dim3(1), dim3(32), 0, s, c->ws_loss, n_partials, c->d_loss, 0));
  return HB_OK;
}

// per-feature batch slices of the CSC (sparse dW of layer 0); depends only on
// the batch, so with the concurrent backward it runs on the side stream under
// the forward pass
int launch_csc_ranges(hb_ctx* c, const DataView& v, long long start, int rows, const DevStep* ds, cudaStream_t s) {
  if (v.n_rows > 0 && static_cast<double>(c->e_nnz) / std::max(1, c->d[0]) <= 1024.0)
    HB_CUDA(launch_k(csc_batch_ranges_warp_kernel, dim3(static_cast<int>(std::min<long long>(cdiv(c->d[0], 8), 148 * 16))),
                     dim3(256), 0, s, v.colptr, v.rowidx, c->d[0], start, rows, ds, c->csc_lo, c->csc_hi));
  else
    HB_CUDA(launch_k(csc_batch_ranges_kernel, dim3(cdiv(c->d[0], 256)), dim3(256), 0, s, v.colptr, v.rowidx, c->d[0],
                     start, rows, ds, c->csc_lo, c->csc_hi));
  c->last_launches++;
  return HB_OK;
}

int run_forward(hb_ctx* c, const DataView& v, long long start, int rows, bool train, uint32_t flags, double eta,
                const DevStep* ds) {
  cudaStream_t st = c->stream;
  c->ranges_early = false;
  if (train && c->sparse && c->conc_bwd) {
    HB_CUDA(cudaEventRecord(c->bev[0], st));  // the batch (CSC view) is in place
    HB_CUDA(cudaStreamWaitEvent(c->side, c->bev[0], 0));
    HB_TRY(launch_csc_ranges(c, v, start, rows, ds, c->side));
    HB_CUDA(cudaEventRecord(c->bev[1], c->side));
    c->side_pending = true;
    c->ranges_early = true;
  }
  const int L = c->L;
  const int m_tiles = cdiv(rows, kBM);
  const int zrows = std::min<long long>(round_up(rows, kBM), c->cap);
  // hidden layers
  for (int l = 0; l < L - 1; ++l) {
    HB_TRY(xchg_use(c, l));
    if (l == 0 && c->sparse) {
      SpmmArgs p{v.rowptr, v.col, v.val, ds, start, rows, c->W[0], c->ldw[0], c->d[0], c->d[1], c->A[1], c->ld[1],
                 (c->need_lo() && !(c->small_head && L == 2)) ? c->A_lo[1] : nullptr, layer_bias(c, 0)};
      prof_begin(c, "spmm_sigmoid", 0);
      const int blocks = cdiv(static_cast<long long>(rows) * 32, 256);
      const size_t w0t_bytes = static_cast<size_t>(c->d[0]) * c->ldw[0] * sizeof(float);
      if (c->d[1] % 128 == 0)
        HB_CUDA(launch_k_l2(spmm_sigmoid_kernel<true>, dim3(blocks), dim3(256), 0, st, c->W[0], w0t_bytes, p));
      else
        HB_CUDA(launch_k_l2(spmm_sigmoid_kernel<false>, dim3(blocks), dim3(256), 0, st, c->W[0], w0t_bytes, p));
      HB_CUDA(cudaGetLastError());
      prof_end(c, "spmm_sigmoid", 0);
      c->last_launches++;
      continue;
    }
    GemmArgs a{};
    a.M = rows;
    a.N = c->d[l + 1];
    a.a_off = l == 0 ? static_cast<int>(start) : 0;
    a.a_start = (l == 0) ? 1 : 0;
    a.a_lo_zero = (l == 0 && v.x_lo_zero) ? 1 : 0;
    a.ds = ds;
    a.kb_total = cdiv(c->d[l], kBK);
    a.kb_per_split = a.kb_total;
    a.out = c->A[l + 1];
    // the last hidden activation feeds only the CUDA-core head (its forward and
    // its dW), never a tensor-core GEMM: no lo twin to write
    a.out_lo = (c->need_lo() && !(c->small_head && l + 1 == L - 1)) ? c->A_lo[l + 1] : nullptr;
    a.ldo = c->ld[l + 1];
    a.drain_kb = drain_kb(c, R_FWD, l);
    a.bias = layer_bias(c, l);
    const Operand ta = l == 0 ? v.fwd() : c->opA_k(l);
    prof_begin(c, "gemm_fwd_sigmoid", l);
    int kb_per = a.kb_total;
    const int fsplit = fx_plan(c, m_tiles, cdiv(a.N, c->bn_fwd[l]), c->bn_fwd[l], a.kb_total, &kb_per);
    if (fsplit > 1)
      HB_TRY(launch_fx_split(c, G_FWD, SPLIT_SIGMOID, c->bn_fwd[l], ta, c->opW_k(l), a, m_tiles,
                             cdiv(a.N, c->bn_fwd[l]), fsplit, kb_per, st));
    else
      HB_TRY(launch_gemm(c->passes, G_FWD, EPI_SIGMOID, c->bn_fwd[l], ta, c->opW_k(l), a, m_tiles,
                         cdiv(a.N, c->bn_fwd[l]), 1, st));
    prof_end(c, "gemm_fwd_sigmoid", l);
    c->last_launches++;
  }
  // output layer
  const int l = L - 1;
  const float inv_n = 1.0f / static_cast<float>(rows);
  HB_TRY(xchg_use(c, l));
  if (c->small_head) {
    HeadArgs h{};
    if (L == 1) {
      h.a = v.x;
      h.lda = v.ldx;
      h.a_input = 1;
    } else {
      h.a = c->A[L - 1];
      h.lda = c->ld[L - 1];
    }
    h.w = c->W[l];
    h.ldw = c->ldw[l];
    h.labels = v.labels;
    h.start = start;
    h.ds = ds;
    h.rows = rows;
    h.d = c->d[l];
    h.nc = c->d[L];
    h.zero_rows = zrows;
    h.inv_n = inv_n;
    h.train = train ? 1 : 0;
    h.delta_prev = (train && L >= 2) ? c->D[L - 2] : nullptr;
    h.delta_prev_lo = (train && L >= 2 && c->need_lo()) ? c->D_lo[L - 2] : nullptr;
    h.ld_dp = L >= 2 ? c->ld[L - 1] : 0;
    h.delta_out = nullptr;
    h.ws_dw = c->ws_head;
    h.ws_loss = c->ws_loss;
    const bool vec = (h.d % 4 == 0) && (h.lda % 4 == 0) && (h.ld_dp % 4 == 0) &&
                     (h.d <= 1024 && (c->head_nct == 2 || h.d <= 512));
    // the vectorised head walks several 16-row passes per block: at most two
    // blocks per SM, so the per-block dW partials (reduced below) stay few
    const int passes_total = cdiv(std::max(rows, zrows), kHeadRowsPerBlock);
    // (the scalar kernel covers one 16-row pass per block, zero-fill rows included)
    const int grid = vec ? std::min(passes_total, 2 * 148) : passes_total;
    h.rows_per_block = cdiv(passes_total, grid) * kHeadRowsPerBlock;
    const int threads = kHeadWarps * 32;
    prof_begin(c, "head_small", l);
#define HB_HEAD(NCT_, MAXT_) HB_CUDA(launch_k(head_small_kernel<NCT_, MAXT_>, dim3(grid), dim3(threads), 0, st, h))
#define HB_HEADV(NCT_, VPL_) HB_CUDA(launch_k(head_small_vec_kernel<NCT_, VPL_>, dim3(grid), dim3(threads), 0, st, h))
    if (vec) {
      const int vpl = h.d <= 256 ? 2 : (h.d <= 512 ? 4 : 8);
      if (c->head_nct == 2) {
        if (vpl == 2) HB_HEADV(2, 2); else if (vpl == 4) HB_HEADV(2, 4); else HB_HEADV(2, 8);
      } else {
        if (vpl == 2) HB_HEADV(4, 2); else HB_HEADV(4, 4);
      }
    } else if (c->head_nct == 2) {
      if (c->head_maxt == 8)
        HB_HEAD(2, 8);
      else if (c->head_maxt == 16)
        HB_HEAD(2, 16);
      else
        HB_HEAD(2, 32);
    } else {
      if (c->head_maxt == 8)
        HB_HEAD(4, 8);
      else if (c->head_maxt == 16)
        HB_HEAD(4, 16);
      else
        HB_HEAD(4, 32);
    }
#undef HB_HEAD
#undef HB_HEADV
    HB_CUDA(cudaGetLastError());
    prof_end(c, "head_small", l);
    HB_TRY(launch_loss_reduce(c, train, grid));
    c->last_launches += 2;
    if (train) {
      // the output layer's reduce + SGD only needs the head's partials: with
      // the concurrent backward it runs on the side stream beside dX_{L-2}
      // (nothing later reads W_{L-1}; the head kernel already has)
      cudaStream_t rs = st;
      if (c->conc_bwd && L >= 2) {
        HB_CUDA(cudaEventRecord(c->bev[2 * l], st));
        HB_CUDA(cudaStreamWaitEvent(c->side, c->bev[2 * l], 0));
        rs = c->side;
        c->side_pending = true;
      }
      const long long n = static_cast<long long>(c->d[L]) * c->d[l];
      c->prof_st = rs;
      prof_begin(c, "reduce_sgd", l);
      HB_CUDA(launch_k(reduce_sgd_f64p_kernel, dim3(cdiv(n, 32)), dim3(256), 0, rs, c->W[l], c->ldw[l], c->ws_head, grid, n,
                       c->d[L], c->d[l], static_cast<float>(eta), (flags & HB_STEP_EMIT_GRAD) ? c->G[l] : nullptr,
                       c->d[l], ds, c->need_lo() ? c->W_lo[l] : nullptr));
      prof_end(c, "reduce_sgd", l);
      c->prof_st = nullptr;
      c->last_launches++;
      HB_TRY(xchg_merge(c, l, eta, ds, rs));
      if (c->merge_layers) HB_TRY(enqueue_layer_merge(c, l, rs, ds));
    }
    return HB_OK;
  }
  // wide head: logits GEMM then softmax -> delta in place
  GemmArgs a{};
  a.M = rows;
  a.N = c->d[L];
  a.a_off = l == 0 ? static_cast<int>(start) : 0;
  a.a_start = (l == 0) ? 1 : 0;
  a.a_lo_zero = (l == 0 && v.x_lo_zero) ? 1 : 0;
  a.ds = ds;
  a.kb_total = cdiv(c->d[l], kBK);
  a.kb_per_split = a.kb_total;
  a.out = c->D[l];
  a.ldo = c->ld[L];
  a.drain_kb = drain_kb(c, R_LOGITS, l);
  const Operand ta = l == 0 ? v.fwd() : c->opA_k(l);
  prof_begin(c, "gemm_fwd_logits", l);
  {
    int kb_per = a.kb_total;
    const int fsplit = fx_plan(c, m_tiles, cdiv(a.N, c->bn_fwd[l]), c->bn_fwd[l], a.kb_total, &kb_per);
    if (fsplit > 1)
      HB_TRY(launch_fx_split(c, G_FWD, SPLIT_STORE, c->bn_fwd[l], ta, c->opW_k(l), a, m_tiles,
                             cdiv(a.N, c->bn_fwd[l]), fsplit, kb_per, st));
    else
      HB_TRY(launch_gemm(c->passes, G_FWD, EPI_STORE, c->bn_fwd[l], ta, c->opW_k(l), a, m_tiles,
                         cdiv(a.N, c->bn_fwd[l]), 1, st));
  }
  prof_end(c, "gemm_fwd_logits", l);
  SoftmaxArgs sm{c->D[l], c->need_lo() ? c->D_lo[l] : nullptr, c->ld[L], v.labels, start, ds, rows, c->d[L],
                 zrows, inv_n, train ? 1 : 0, c->ws_loss};
  const int grid = cdiv(std::max(rows, zrows), 8);
  prof_begin(c, "softmax_delta", l);
  HB_CUDA(launch_k(softmax_delta_kernel, dim3(grid), dim3(256), 0, st, sm));
  HB_CUDA(cudaGetLastError());
  prof_end(c, "softmax_delta", l);
  HB_TRY(launch_loss_reduce(c, train, grid));
  c->last_launches += 3;
  return HB_OK;
}

int run_backward(hb_ctx* c, const DataView& v, long long start, int rows, uint32_t flags, double eta,
                 const DevStep* ds) {
  cudaStream_t st = c->stream;
  const int L = c->L;
  const int zrows = std::min<long long>(round_up(rows, kBM), c->cap);
  const bool emit = (flags & HB_STEP_EMIT_GRAD) != 0;
  // with the small head the output layer is already done (dW + delta_{L-2})
  const int top = c->small_head ? L - 2 : L - 1;
  bool used_side = false;
  for (int l = top; l >= 0; --l) {
    // dX: D[l-1] = (D[l] . W[l]) * A[l] (1 - A[l])   -- must precede W[l]'s update
    auto do_dx = [&]() -> int {
    if (l >= 1) {
      GemmArgs a{};
      a.M = rows;
      a.N = c->d[l];
      a.m_zero_rows = zrows;
      a.kb_total = cdiv(c->d[l + 1], kBK);
      a.kb_per_split = a.kb_total;
      a.out = c->D[l - 1];
      a.out_lo = c->need_lo() ? c->D_lo[l - 1] : nullptr;
      a.ldo = c->ld[l];
      a.aux = c->A[l];
      a.ld_aux = c->ld[l];
      a.ds = ds;
      a.drain_kb = drain_kb(c, R_DX, l);
      prof_begin(c, "gemm_dx_dsig", l);
      int kb_per = a.kb_total;
      const int fsplit = fx_plan(c, cdiv(zrows, kBM), cdiv(a.N, c->bn_dx[l]), c->bn_dx[l], a.kb_total, &kb_per);
      if (fsplit > 1)
        HB_TRY(launch_fx_split(c, G_DX, SPLIT_DSIG, c->bn_dx[l], c->opD_k(l), c->opW_mn(l), a, cdiv(zrows, kBM),
                               cdiv(a.N, c->bn_dx[l]), fsplit, kb_per, st));
      else
        HB_TRY(launch_gemm(c->passes, G_DX, EPI_DSIG, c->bn_dx[l], c->opD_k(l), c->opW_mn(l), a,
                           cdiv(zrows, kBM), cdiv(a.N, c->bn_dx[l]), 1, st));
      prof_end(c, "gemm_dx_dsig", l);
      c->last_launches++;
    }
    return HB_OK;
    };
    // dW + SGD
    if (l == 0 && c->sparse) {
      HB_TRY(do_dx());
      SparseDwArgs p{v.colptr, v.rowidx, v.cval, ds, start, rows, c->d[0], c->d[1], c->D[0], c->ld[1],
                     c->W[0], c->ldw[0], static_cast<float>(eta), emit ? c->G[0] : nullptr, c->ldw[0],
                     c->csc_lo, c->csc_hi};
      prof_begin(c, "sparse_dw_sgd", 0);
      if (c->ranges_early)
        HB_CUDA(cudaStreamWaitEvent(st, c->bev[1], 0));  // computed on the side stream under the forward
      else
        HB_TRY(launch_csc_ranges(c, v, start, rows, ds, st));
      // batch entries per feature decide the parallelisation
      const double per_feature = static_cast<double>(rows) * c->nnz_per_row / std::max(1, c->d[0]);
      if (per_feature < 48.0 && c->d[1] % 4 == 0) {
        // the gathered operand here is delta_0 (rows x d1): one row per nonzero of each feature's CSC slice
        HB_CUDA(launch_k_l2(sparse_dw_warp_kernel, dim3(cdiv(static_cast<long long>(c->d[0]) * 32, 256)), dim3(256), 0,
                            st, c->D[0], static_cast<size_t>(rows) * c->ld[1] * sizeof(float), p));
      } else {
        const dim3 blocks(c->d[0], cdiv(c->d[1], 128));
        if (c->d[1] % 4 == 0)
          HB_CUDA(launch_k(sparse_dw_kernel<true>, dim3(blocks), dim3(256), 0, st, p));
        else
          HB_CUDA(launch_k(sparse_dw_kernel<false>, dim3(blocks), dim3(256), 0, st, p));
      }
      HB_CUDA(cudaGetLastError());
      c->last_launches++;
      prof_end(c, "sparse_dw_sgd", 0);
      HB_TRY(xchg_merge(c, 0, eta, ds));
      if (c->merge_layers) HB_TRY(enqueue_layer_merge(c, 0, st, ds));
      continue;
    }
    int splits, kb_per, kb_total;
    dw_plan(c, l, rows, &splits, &kb_per, &kb_total);
    GemmArgs a{};
    a.M = c->d[l + 1];
    a.N = c->d[l];
    a.b_off = l == 0 ? static_cast<int>(start) : 0;
    a.b_start = (l == 0) ? 1 : 0;
    a.b_lo_zero = (l == 0 && v.x_lo_zero) ? 1 : 0;
    a.ds = ds;
    a.kb_total = kb_total;
    a.kb_per_split = kb_per;
    a.eta = static_cast<float>(eta);
    a.drain_kb = drain_kb(c, R_DW, l);
    const Operand tb = l == 0 ? v.dw() : c->opA_mn(l);
    const int mt = cdiv(a.M, kBM), nt = cdiv(a.N, c->bn_dw[l]);
    if (c->conc_bwd && l >= 1 && splits > 1) {
      // concurrent: the split-K dW partial GEMM (reads D_l, A_l; never W_l)
      // runs on the side stream beside dX_l; its reduce + SGD waits for dX_l,
      // which is the last reader of W_l.  The idle SMs of one kernel's wave
      // and its epilogue tail are filled by the other's CTAs.
      const long long slab = static_cast<long long>(a.M) * a.N;
      float* wsb = c->ws_dw + c->ws_dw_off[l];
      a.out = wsb;
      a.ldo = a.N;
      a.split_stride = slab;
      HB_CUDA(cudaEventRecord(c->bev[2 * l], st));  // D_l and A_l are complete
      HB_CUDA(cudaStreamWaitEvent(c->side, c->bev[2 * l], 0));
      // device lane of the merge: the host rows of W_l come in while the
      // partial GEMM runs (the merge read), the reduce applies both updates
      // Only when the caller declares the replica the host model's sole writer
      // (HB_STEP_SOLE_WRITER): the lane reads a whole layer when the partial GEMM
      // starts and writes it back after the reduce, so a concurrent host writer's
      // updates to that layer inside the window would be overwritten -- wider
      // than the per-element race of the reference's np.add (linalg.py:79).
      const bool dev_lane = (flags & HB_STEP_SOLE_WRITER) != 0 && !c->xw.empty() && c->xmode == 0 &&
                            l < static_cast<int>(c->xdma.size()) && c->xdma[l];
      double* host_rows = dev_lane ? c->stage_all + layer_offset(c, l) : nullptr;
      if (dev_lane) {
        c->xdma_used[l] = 1;
        HB_CUDA(cudaStreamWaitEvent(c->xh2d, c->bev[2 * l], 0));
        if (!c->xmirror)  // (a resident mirror already holds these rows)
          HB_CUDA(cudaMemcpyAsync(host_rows, c->xw[l], static_cast<size_t>(a.M) * a.N * sizeof(double),
                                  cudaMemcpyHostToDevice, c->xh2d));
        HB_CUDA(cudaEventRecord(c->xread_ev[l], c->xh2d));
      }
      c->prof_st = c->side;
      prof_begin(c, "gemm_dw_partial", l);
      HB_TRY(launch_gemm(c->passes, G_DW, EPI_PARTIAL, c->bn_dw[l], c->opD_mn(l), tb, a, mt, nt, splits, c->side));
      prof_end(c, "gemm_dw_partial", l);
      c->prof_st = nullptr;
      HB_TRY(do_dx());
      HB_CUDA(cudaEventRecord(c->bev[2 * l + 1], st));  // dX_l has read W_l
      HB_CUDA(cudaStreamWaitEvent(c->side, c->bev[2 * l + 1], 0));
      if (dev_lane) HB_CUDA(cudaStreamWaitEvent(c->side, c->xread_ev[l], 0));
      c->prof_st = c->side;
      prof_begin(c, "reduce_sgd", l);
      if (dev_lane || (a.N % 4 == 0 && c->ldw[l] % 4 == 0 && (slab / 4) >= 148 * 256))
        HB_CUDA(launch_k(reduce_sgd_vec_kernel, dim3(static_cast<int>(std::min<long long>(cdiv(slab / 4, 256), 148 * 8))),
                         dim3(256), 0, c->side, c->W[l], c->ldw[l], wsb, splits, slab, a.M, a.N,
                         static_cast<float>(eta), emit ? c->G[l] : nullptr, c->d[l], ds,
                         c->need_lo() ? c->W_lo[l] : nullptr, host_rows, eta));
      else
        HB_CUDA(launch_k(reduce_sgd_kernel, dim3(cdiv(slab, 32)), dim3(256), 0, c->side, c->W[l], c->ldw[l], wsb,
                         splits, slab, a.M, a.N, static_cast<float>(eta), emit ? c->G[l] : nullptr, c->d[l], ds,
                         c->need_lo() ? c->W_lo[l] : nullptr));
      prof_end(c, "reduce_sgd", l);
      c->prof_st = nullptr;
      c->last_launches += 2;
      HB_TRY(xchg_merge(c, l, eta, ds, c->side));
      if (c->merge_layers) HB_TRY(enqueue_layer_merge(c, l, c->side, ds));
      used_side = true;
      continue;
    }
    if (splits == 1 && l >= 1 && c->xsole && c->xmode == 0 && l < static_cast<int>(c->xml.size()) && c->xml[l] &&
        !(getenv("HB_NO_DW_FIRST") && getenv("HB_NO_DW_FIRST")[0] == '1')) {
      // sole-writer mirror lane: the host copy of W_l is PCIe-bound (8 B per
      // weight), so start it as early as possible -- dW first (the gradient
      // into G_l, W_l untouched), the float64 merge + D2H on the merge stream
      // from here, then dX (the last reader of the old W_l), then the SGD update
      a.out = c->G[l];
      a.ldo = c->d[l];
      a.split_stride = 0;
      prof_begin(c, "gemm_dw_first", l);
      HB_TRY(launch_gemm(c->passes, G_DW, EPI_PARTIAL, c->bn_dw[l], c->opD_mn(l), tb, a, mt, nt, 1, st));
      prof_end(c, "gemm_dw_first", l);
      HB_TRY(xchg_merge(c, l, eta, ds));
      HB_TRY(do_dx());
      const long long slab = static_cast<long long>(a.M) * a.N;
      prof_begin(c, "sgd_update", l);
      if (a.N % 4 == 0 && c->ldw[l] % 4 == 0 && (slab / 4) >= 148 * 256)
        HB_CUDA(launch_k(reduce_sgd_vec_kernel, dim3(static_cast<int>(std::min<long long>(cdiv(slab / 4, 256), 148 * 8))),
                         dim3(256), 0, st, c->W[l], c->ldw[l], c->G[l], 1, slab, a.M, a.N, static_cast<float>(eta),
                         nullptr, c->d[l], ds, c->need_lo() ? c->W_lo[l] : nullptr, nullptr, 0.0));
      else
        HB_CUDA(launch_k(reduce_sgd_kernel, dim3(cdiv(slab, 32)), dim3(256), 0, st, c->W[l], c->ldw[l], c->G[l], 1, slab,
                         a.M, a.N, static_cast<float>(eta), nullptr, c->d[l], ds, c->need_lo() ? c->W_lo[l] : nullptr));
      HB_CUDA(cudaGetLastError());
      prof_end(c, "sgd_update", l);
      c->last_launches += 2;
      if (c->merge_layers) HB_TRY(enqueue_layer_merge(c, l, st, ds));
      continue;
    }
    HB_TRY(do_dx());
    if (splits == 1) {
      a.out = c->W[l];
      a.out_lo = c->need_lo() ? c->W_lo[l] : nullptr;
      a.ldo = c->ldw[l];
      a.grad = emit ? c->G[l] : nullptr;
      a.ld_grad = c->d[l];
      prof_begin(c, "gemm_dw_sgd", l);
      HB_TRY(launch_gemm(c->passes, G_DW, EPI_SGD, c->bn_dw[l], c->opD_mn(l), tb, a, mt, nt, 1, st));
      prof_end(c, "gemm_dw_sgd", l);
      c->last_launches++;
    } else if (c->tile_sync != nullptr && a.N % 4 == 0 && c->ldw[l] % 4 == 0 &&
               static_cast<long long>(mt + (c->passes == 3 && c->bn_dw[l] >= 64 ? mt % 2 : 0)) * nt * splits <=
                   split_sgd_capacity(c->passes, c->bn_dw[l]) &&
               static_cast<long long>(mt + 1) * nt <= kTileSyncTiles) {
      // split-K partials reduced and applied inside the GEMM (no reduce kernel)
      a.out = c->ws;
      a.ldo = a.N;
      a.split_stride = static_cast<long long>(a.M) * a.N;
      a.w = c->W[l];
      a.w_lo = c->need_lo() ? c->W_lo[l] : nullptr;
      a.ldw = c->ldw[l];
      a.grad = emit ? c->G[l] : nullptr;
      a.ld_grad = c->d[l];
      a.tile_sync = c->tile_sync;
      prof_begin(c, "gemm_dw_splitk_sgd", l);
      HB_TRY(launch_gemm(c->passes, G_DW, EPI_SPLIT_SGD, c->bn_dw[l], c->opD_mn(l), tb, a, mt, nt, splits, st));
      prof_end(c, "gemm_dw_splitk_sgd", l);
      c->last_launches++;
    } else {
      const long long slab = static_cast<long long>(a.M) * a.N;
      a.out = c->ws;
      a.ldo = a.N;
      a.split_stride = slab;
      prof_begin(c, "gemm_dw_partial", l);
      HB_TRY(launch_gemm(c->passes, G_DW, EPI_PARTIAL, c->bn_dw[l], c->opD_mn(l), tb, a, mt, nt, splits, st));
      prof_end(c, "gemm_dw_partial", l);
      prof_begin(c, "reduce_sgd", l);
      if (a.N % 4 == 0 && c->ldw[l] % 4 == 0 && (slab / 4) >= 148 * 256)
        HB_CUDA(launch_k(reduce_sgd_vec_kernel, dim3(static_cast<int>(std::min<long long>(cdiv(slab / 4, 256), 148 * 8))), dim3(256), 0, st, 
            c->W[l], c->ldw[l], c->ws, splits, slab, a.M, a.N, static_cast<float>(eta), emit ? c->G[l] : nullptr,
            c->d[l], ds, c->need_lo() ? c->W_lo[l] : nullptr, nullptr, 0.0));
      else
        HB_CUDA(launch_k(reduce_sgd_kernel, dim3(cdiv(slab, 32)), dim3(256), 0, st, c->W[l], c->ldw[l], c->ws, splits, slab, a.M, a.N,
                                                          static_cast<float>(eta), emit ? c->G[l] : nullptr, c->d[l],
                                                          ds, c->need_lo() ? c->W_lo[l] : nullptr));
      HB_CUDA(cudaGetLastError());
      prof_end(c, "reduce_sgd", l);
      c->last_launches += 2;
    }
    HB_TRY(xchg_merge(c, l, eta, ds));
    if (c->merge_layers) HB_TRY(enqueue_layer_merge(c, l, st, ds));
  }
  if (c->merge_layers) {  // join the merge stream: every layer averaged before the step ends
    HB_CUDA(cudaEventRecord(c->mev[c->L], c->comm_st));
    HB_CUDA(cudaStreamWaitEvent(st, c->mev[c->L], 0));
  }
  if (used_side || c->side_pending) {  // join the side stream
    HB_CUDA(cudaEventRecord(c->bev.back(), c->side));
    HB_CUDA(cudaStreamWaitEvent(st, c->bev.back(), 0));
    c->side_pending = false;
  }
  return HB_OK;
}

// Enqueue one step.  Eager the first time a (rows, flags, data view) shape is
// seen; from the second time on, the whole step is a captured CUDA graph that
// reads (start, eta) from c->d_step, so a step costs one graph launch.
// phase 0: whole step; 1: forward (incl. the fused head and its update); 2: backward
int run_small_net(hb_ctx* c, const DataView& v, long long start, int rows, uint32_t flags, double eta,
                  const DevStep* ds);

int run_phase(hb_ctx* c, const DataView& v, long long start, int rows, uint32_t flags, double eta, const DevStep* ds,
              int phase) {
  if (phase == 0 && c->sn_ok && rows <= kSnMaxRows && !c->merge_layers && v.x != nullptr)
    return run_small_net(c, v, start, rows, flags, eta, ds);
  if (phase != 2) c->xdma_used.assign(c->L, 0);
  if (phase != 2) HB_TRY(xchg_begin(c));
  if (phase != 2) HB_TRY(run_forward(c, v, start, rows, true, flags, eta, ds));
  if (phase != 1) HB_TRY(run_backward(c, v, start, rows, flags, eta, ds));
  if (phase != 1) HB_TRY(xchg_end(c));
  return HB_OK;
}

// A deferred (HB_STEP_LAND_ASYNC) call can replay the step graph when every
// layer merges on the mirror lane (no device lane, no host lane): the graph
// then carries the merge kernels and leaves the write-backs to its launcher.
bool land_graph_ok(const hb_ctx* c) {
  if (c->xmode != 0 || !c->xsole || static_cast<int>(c->xml.size()) < c->L) return false;
  if (getenv("HB_LAND_EAGER") && getenv("HB_LAND_EAGER")[0] == '1') return false;
  for (int l = 0; l < c->L; ++l) {
    if (!c->xml[l]) return false;
    if (l < static_cast<int>(c->xdma.size()) && c->xdma[l]) return false;
  }
  return true;
}

// The whole step of a small net (hb_small.cuh): the snapshot conversions, one
// cooperative launch, then every layer's stale merge (top layer first, as the
// backward produces them).
int run_small_net(hb_ctx* c, const DataView& v, long long start, int rows, uint32_t flags, double eta,
                  const DevStep* ds) {
  const int L = c->L;
  c->xdma_used.assign(L, 0);
  HB_TRY(xchg_begin(c));
  for (int l = 0; l < L; ++l) HB_TRY(xchg_use(c, l));
  SmallNetArgs p{};
  p.L = L;
  p.rows = rows;
  p.train = 1;
  for (int l = 0; l <= L; ++l) {
    p.d[l] = c->d[l];
    p.ld[l] = c->ld[l];
  }
  p.x = v.x;
  p.ldx = v.ldx;
  p.start = start;
  p.labels = v.labels;
  p.ds = ds;
  p.eta = static_cast<float>(eta);
  const bool emit = (flags & HB_STEP_EMIT_GRAD) != 0;
  for (int l = 0; l < L; ++l) {
    p.W[l] = c->W[l];
    p.W_lo[l] = c->need_lo() ? c->W_lo[l] : nullptr;
    p.ldw[l] = c->ldw[l];
    p.bias[l] = l < L - 1 ? layer_bias(c, l) : nullptr;
    p.A[l] = c->A[l];
    p.D[l] = c->D[l];
    p.G[l] = emit ? c->G[l] : nullptr;
  }
  p.hd = c->sn_hd;
  p.row_loss = c->sn_loss;
  p.loss_out = c->d_loss;
  p.bar = c->sn_bar;
  cudaStream_t st = c->stream;
  HB_CUDA(cudaMemsetAsync(c->sn_bar, 0, sizeof(unsigned), st));
  prof_begin(c, "small_net_step", 0);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c->sn_grid);
  cfg.blockDim = dim3(kSnThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HB_CUDA(cudaLaunchKernelEx(&cfg, small_net_step_kernel, p));
  prof_end(c, "small_net_step", 0);
  c->last_launches++;
  for (int l = L - 1; l >= 0; --l) HB_TRY(xchg_merge(c, l, eta, ds));
  HB_TRY(xchg_end(c));
  return HB_OK;
}

int enqueue_step(hb_ctx* c, const DataView& v, long long start, int rows, double eta, uint32_t flags, bool graph_ok,
                 int phase = 0) {
  const uint32_t gflags = (flags & (HB_STEP_EMIT_GRAD | HB_STEP_SOLE_WRITER)) | (static_cast<uint32_t>(phase) << 8) |
                          (c->merge_layers ? (1u << 18) : 0u) | (c->xland ? (1u << 19) : 0u) |
                          (v.x_lo_zero ? (1u << 16) : 0u) | (c->xmirror ? (1u << 17) : 0u);
  const bool view_epoch = (&v == &c->epoch);
  if (!c->use_graphs || !graph_ok || (c->xland && !land_graph_ok(c)))
    return run_phase(c, v, start, rows, flags, eta, nullptr, phase);
  const auto key = std::make_tuple(rows, gflags, view_epoch ? c->view_gen : -c->view_gen, c->prof_on,
                                   c->xw.empty() ? 0LL : c->xgen);
  DevStep hs{start, static_cast<float>(eta), 0, eta, c->peer_gen};
  auto it = c->graphs.find(key);
  if (it == c->graphs.end()) {
    if (c->graph_seen[key]++ == 0)  // first sighting: run eagerly (also configures kernel attributes)
      return run_phase(c, v, start, rows, flags, eta, nullptr, phase);
    StepGraph g;
    c->capturing = true;
    c->cap_events.clear();
    c->step_marks.clear();
    HB_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const int launches0 = c->last_launches;
    c->xd2h_defer.assign(c->L, 0);
    int rc = run_phase(c, v, 0, rows, flags, 0.0, c->d_step, phase);
    cudaGraph_t graph = nullptr;
    cudaError_t ce = cudaStreamEndCapture(c->stream, &graph);
    c->capturing = false;
    if (rc != HB_OK) return rc;
    if (ce != cudaSuccess) return fail(HB_ECUDA, "graph capture failed: %s", cudaGetErrorString(ce));
    ce = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) return fail(HB_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(ce));
    g.marks = c->step_marks;
    g.events = c->cap_events;
    g.xdma_used = c->xdma_used;
    g.d2h_defer = c->xd2h_defer;
    g.launches = c->last_launches - launches0;
    c->step_marks.clear();
    c->cap_events.clear();
    it = c->graphs.emplace(key, std::move(g)).first;
    c->last_launches = 0;
  }
  if (phase != 2) {
    HB_CUDA(cudaMemcpyAsync(c->d_step, &hs, sizeof hs, cudaMemcpyHostToDevice, c->stream));
    t_h2d_bytes += static_cast<long long>(sizeof hs);
  }
  xmark("graph launch");
  c->xdma_used = it->second.xdma_used;
  HB_CUDA(cudaGraphLaunch(it->second.exec, c->stream));
  // deferred landing: each merged layer's D2H, once the graph has merged it
  const std::vector<char>& dd = it->second.d2h_defer;
  for (int l = 0; l < static_cast<int>(dd.size()) && l < c->L; ++l) {
    if (!dd[l]) continue;
    cudaStream_t ms = c->xmrg_l[l];
    HB_CUDA(cudaStreamWaitEvent(ms, c->xd2h_ready_ev[l], 0));
    HB_CUDA(cudaMemcpyAsync(c->xw[l], c->stage_all + layer_offset(c, l),
                            static_cast<size_t>(c->d[l + 1]) * c->d[l] * sizeof(double), cudaMemcpyDeviceToHost, ms));
    HB_CUDA(cudaEventRecord(c->xd2h_done_ev[l], ms));
  }
  xmark("graph launched");
  c->last_launches += it->second.launches;
  if (c->prof_on) c->step_marks.insert(c->step_marks.end(), it->second.marks.begin(), it->second.marks.end());
  return HB_OK;
}

void drop_graphs(hb_ctx* c) {
  for (auto& kv : c->graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    for (auto e : kv.second.events) cudaEventDestroy(e);
  }
  c->graphs.clear();
  c->graph_seen.clear();
}

// peer-memory merge (hb_peer.cuh): pack, signal, wait, one-shot reduce of
// this rank's slice across every rank's flat, signal, wait, unpack
double peer_timeout_s() { return getenv("HB_PEER_TIMEOUT_S") ? atof(getenv("HB_PEER_TIMEOUT_S")) : 30.0; }

// packed-model layout: layer l's (rows, cols) block at flat_off[l], padded to 4 floats
void ensure_flat_layout(hb_ctx* c) {
  if (!c->flat_off.empty()) return;
  c->flat_off.assign(c->L + 1, 0);
  long long off = 0;
  for (int l = 0; l < c->L; ++l) {
    c->flat_off[l] = off;
    off += round_up(static_cast<long long>(c->d[l + 1]) * c->d[l], 4);
  }
  c->flat_off[c->L] = off;
  c->flat_n = off;
}

// layers [l0, l1) of the packed model; offsets relative to flat_off[l0]
ModelLayout merge_layout(const hb_ctx* c, int l0, int l1) {
  ModelLayout m{};
  m.n = l1 - l0;
  for (int l = l0; l < l1; ++l) {
    const bool tr = l == 0 && c->sparse;  // W0^T (d_in, d_out) on the device: averaged in that layout
    const long long rows = tr ? c->d[0] : c->d[l + 1], cols = tr ? c->d[1] : c->d[l];
    const int i = l - l0;
    m.w[i] = c->W[l];
    m.w_lo[i] = (c->need_lo() && !tr) ? c->W_lo[l] : nullptr;
    m.ld[i] = c->ldw[l];
    m.cols[i] = static_cast<int>(cols);
    m.off[i] = c->flat_off[l] - c->flat_off[l0];
    m.size[i] = rows * cols;
  }
  m.off[m.n] = c->flat_off[l1] - c->flat_off[l0];
  return m;
}

bool layerwise_merge_ok(const hb_ctx* c) {
  if (getenv("HB_NO_LAYER_MERGE") && getenv("HB_NO_LAYER_MERGE")[0] == '1') return false;
  if (c->L > kMaxMergeLayers) return false;
  if (c->peers.n > 0) return !c->local;  // in-process groups order merges on the host
  return c->comm != nullptr;
}

// Average layer l across the replicas on comm_st once its update (enqueued on
// `src`) is done; the step joins comm_st at the end of the backward.
int enqueue_layer_merge(hb_ctx* c, int l, cudaStream_t src, const DevStep* ds) {
  HB_CUDA(cudaEventRecord(c->mev[l], src));
  HB_CUDA(cudaStreamWaitEvent(c->comm_st, c->mev[l], 0));
  const ModelLayout m = merge_layout(c, l, l + 1);
  const long long n = m.off[1], base = c->flat_off[l];
  const dim3 grid(static_cast<int>(std::min<long long>(cdiv(n, 256), 148 * 4)));
  if (c->peers.n > 0) {
    const int r = c->peers.rank;
    const unsigned long long g = c->peer_gen;  // eager value; graphs read the step record
    const unsigned long long timeout_ns = static_cast<unsigned long long>(peer_timeout_s() * 1e9);
    unsigned long long* own = reinterpret_cast<unsigned long long*>(c->xbuf);
    pack_model_kernel<<<grid, 256, 0, c->comm_st>>>(c->peers.flat[r] + base, m);
    peer_signal_kernel<<<1, 1, 0, c->comm_st>>>(own, 2 + 2 * l, g, ds);
    peer_wait_kernel<<<1, 32, 0, c->comm_st>>>(c->peers, 2 + 2 * l, g, timeout_ns, ds);
    peer_reduce_kernel<<<grid, 256, 0, c->comm_st>>>(c->peers, n, 1.0f / static_cast<float>(c->peers.n), base);
    peer_signal_kernel<<<1, 1, 0, c->comm_st>>>(own, 3 + 2 * l, g, ds);
    peer_wait_kernel<<<1, 32, 0, c->comm_st>>>(c->peers, 3 + 2 * l, g, timeout_ns, ds);
    unpack_model_kernel<<<grid, 256, 0, c->comm_st>>>(c->peers.flat[r] + base, 1.0f, m);
    c->last_launches += 7;
  } else {
    pack_model_kernel<<<grid, 256, 0, c->comm_st>>>(c->flat + base, m);
    const int rc = g_nccl.allReduce(c->flat + base, c->flat + base, static_cast<size_t>(n), kNcclFloat32, kNcclSum,
                                    c->comm, c->comm_st);
    if (rc != 0) return fail(HB_ENCCL, "ncclAllReduce: %s", g_nccl.errStr ? g_nccl.errStr(rc) : "error");
    unpack_model_kernel<<<grid, 256, 0, c->comm_st>>>(c->flat + base, 1.0f / static_cast<float>(c->nranks), m);
    c->last_launches += 2;
  }
  HB_CUDA(cudaGetLastError());
  return HB_OK;
}

int ensure_comm_stream(hb_ctx* c) {
  if (c->comm_st) return HB_OK;
  int lo_prio = 0, hi_prio = 0;
  HB_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  HB_CUDA(cudaStreamCreateWithPriority(&c->comm_st, cudaStreamNonBlocking, hi_prio));
  c->mev.resize(c->L + 1);
  for (auto& e : c->mev) HB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return HB_OK;
}

int enqueue_peer_merge(hb_ctx* c, const ModelLayout& m, long long n_elems, const dim3 grid, bool bump) {
  const unsigned long long g = bump ? ++c->peer_gen : c->peer_gen;
  const int r = c->peers.rank;
  if (c->local) {
    // in-process group: every rank's pack is enqueued before anyone waits on it
    LocalGroup& lg = *c->local;
    HB_CUDA(launch_k(pack_model_kernel, grid, dim3(256), 0, c->stream, c->peers.flat[r], m));
    HB_CUDA(cudaEventRecord(lg.ev_pack[r], c->stream));
    if (!lg.barrier(peer_timeout_s())) return fail(HB_ESTATE, "peer merge: a rank never signalled (timeout)");
    for (int q = 0; q < lg.n; ++q)
      if (q != r) HB_CUDA(cudaStreamWaitEvent(c->stream, lg.ev_pack[q], 0));
    peer_reduce_kernel<<<grid, 256, 0, c->stream>>>(c->peers, n_elems, 1.0f / static_cast<float>(c->peers.n));
    HB_CUDA(cudaEventRecord(lg.ev_red[r], c->stream));
    if (!lg.barrier(peer_timeout_s())) return fail(HB_ESTATE, "peer merge: a rank never signalled (timeout)");
    for (int q = 0; q < lg.n; ++q)
      if (q != r) HB_CUDA(cudaStreamWaitEvent(c->stream, lg.ev_red[q], 0));
    unpack_model_kernel<<<grid, 256, 0, c->stream>>>(c->peers.flat[r], 1.0f, m);
    HB_CUDA(cudaGetLastError());
    c->last_launches += 3;
    return HB_OK;
  }
  unsigned long long* own = reinterpret_cast<unsigned long long*>(c->xbuf);
  const unsigned long long timeout_ns = static_cast<unsigned long long>(peer_timeout_s() * 1e9);
  HB_CUDA(launch_k(pack_model_kernel, grid, dim3(256), 0, c->stream, c->peers.flat[c->peers.rank], m));
  peer_signal_kernel<<<1, 1, 0, c->stream>>>(own, 0, g);
  peer_wait_kernel<<<1, 32, 0, c->stream>>>(c->peers, 0, g, timeout_ns);
  peer_reduce_kernel<<<grid, 256, 0, c->stream>>>(c->peers, n_elems, 1.0f / static_cast<float>(c->peers.n));
  peer_signal_kernel<<<1, 1, 0, c->stream>>>(own, 1, g);
  peer_wait_kernel<<<1, 32, 0, c->stream>>>(c->peers, 1, g, timeout_ns);
  unpack_model_kernel<<<grid, 256, 0, c->stream>>>(c->peers.flat[c->peers.rank], 1.0f, m);
  HB_CUDA(cudaGetLastError());
  c->last_launches += 7;
  return HB_OK;
}

// error word of the peer merge (a peer that never signalled within the timeout)
int peer_check(hb_ctx* c) {
  if (c->peers.n == 0) return HB_OK;
  unsigned err = 0;
  HB_CUDA(cudaMemcpyAsync(&err, c->xbuf + 8 * kPeerErrWord, sizeof err, cudaMemcpyDeviceToHost, c->stream));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  if (err != 0) return fail(HB_ESTATE, "peer merge: rank %u never signalled (timeout)", err - 1);
  return HB_OK;
}

// pack -> allreduce(sum) -> unpack x 1/nranks (+ lo twins), enqueued on the
// step stream: inside a step's CUDA-event bracket when HB_STEP_MERGE asks.
// Peer-attached contexts average over peer memory instead of NCCL.
int enqueue_merge(hb_ctx* c, bool bump = true) {
  if (!c->comm && c->peers.n == 0) return fail(HB_ESTATE, "communicator not initialised");
  if (c->L > kMaxMergeLayers) return fail(HB_EINVAL, "merge supports up to %d layers", kMaxMergeLayers);
  ensure_flat_layout(c);
  const ModelLayout m = merge_layout(c, 0, c->L);
  const long long off = c->flat_n;
  const dim3 grid(static_cast<int>(std::min<long long>(cdiv(off, 256), 148 * 8)));
  if (c->peers.n > 0) return enqueue_peer_merge(c, m, off, grid, bump);
  HB_CUDA(launch_k(pack_model_kernel, grid, dim3(256), 0, c->stream, c->flat, m));
  int r = g_nccl.allReduce(c->flat, c->flat, static_cast<size_t>(off), kNcclFloat32, kNcclSum, c->comm, c->stream);
  if (r != 0) return fail(HB_ENCCL, "ncclAllReduce: %s", g_nccl.errStr ? g_nccl.errStr(r) : "error");
  unpack_model_kernel<<<grid, 256, 0, c->stream>>>(c->flat, 1.0f / static_cast<float>(c->nranks), m);
  HB_CUDA(cudaGetLastError());
  c->last_launches += 2;
  return HB_OK;
}

// `mid` (optional): host work run between the enqueued forward and backward
// phases (the host-buffer CSR step builds the batch CSC there, overlapping the
// device forward pass).
// The step's loss sum to the host: a one-thread kernel stores it into mapped
// pinned memory.  A D2H copy would queue on the copy engine behind the merged
// layers a replica call writes back (tens to hundreds of MB), so a deferred
// call (HB_STEP_LAND_ASYNC) would still wait for them.
__global__ void store_loss_kernel(const double* d, volatile double* h) { *h = *d; }
int read_loss(hb_ctx* c, double* out) {
  *reinterpret_cast<volatile double*>(c->h_loss) = 0.0;
  store_loss_kernel<<<1, 1, 0, c->stream>>>(c->d_loss, c->h_loss);
  HB_CUDA(cudaGetLastError());
  c->last_launches++;
  HB_CUDA(cudaStreamSynchronize(c->stream));
  *out = *reinterpret_cast<volatile double*>(c->h_loss);
  return HB_OK;
}

int do_step(hb_ctx* c, const DataView& v, long long start, int rows, double eta, uint32_t flags, double* out_loss,
            bool graph_ok = true, const std::function<int()>& mid = nullptr) {
  if (c->pend_active) return fail(HB_ESTATE, "a replica step is in flight (hb_replica_end first)");
  if (rows < 1 || rows > c->max_batch) return fail(HB_EINVAL, "rows=%d outside [1, %d]", rows, c->max_batch);
  c->last_launches = c->pre_launches;
  c->pre_launches = 0;
  c->ev_used = 0;
  c->step_marks.clear();
  const bool timed = (flags & HB_STEP_TIMED) != 0;
  const bool merge = (flags & HB_STEP_MERGE) != 0;
  if (merge && !c->comm && c->peers.n == 0) return fail(HB_ESTATE, "communicator not initialised");
  // the replica merge: per layer inside the backward where the transport
  // allows (NCCL, cross-process peers), else the whole model after the step
  c->merge_layers = merge && layerwise_merge_ok(c);
  if (merge) {
    ++c->peer_gen;
    ensure_flat_layout(c);
    if (c->merge_layers) HB_TRY(ensure_comm_stream(c));
  }
  if (c->land_pending) {
    // a deferred call's merges read G_l and write the float64 copy this step
    // converts: wait for them (its write-backs keep running)
    for (int l = 0; l < c->L && l < static_cast<int>(c->xmerged_rec.size()); ++l)
      if (c->xmerged_rec[l]) HB_CUDA(cudaStreamWaitEvent(c->stream, c->xmerged_ev[l], 0));
  }
  std::fill(c->xmerged_rec.begin(), c->xmerged_rec.end(), 0);
  if (timed) HB_CUDA(cudaEventRecord(c->ev0, c->stream));
  if (mid) {
    HB_TRY(enqueue_step(c, v, start, rows, eta, flags, graph_ok, 1));
    HB_TRY(mid());
    HB_TRY(enqueue_step(c, v, start, rows, eta, flags, graph_ok, 2));
  } else {
    HB_TRY(enqueue_step(c, v, start, rows, eta, flags, graph_ok));
  }
  if (merge && !c->merge_layers) HB_TRY(enqueue_merge(c, false));  // the replica merge, inside the timed bracket
  c->merge_layers = false;
  if (timed) HB_CUDA(cudaEventRecord(c->ev1, c->stream));
  c->grads_valid = (flags & HB_STEP_EMIT_GRAD) != 0;
  if (out_loss != nullptr) {
    double s = 0.0;
    HB_TRY(read_loss(c, &s));
    *out_loss = s / rows;
  } else if (!(flags & HB_STEP_ASYNC) || c->prof_on) {
    HB_CUDA(cudaStreamSynchronize(c->stream));
  }
  if (timed) {
    HB_CUDA(cudaEventSynchronize(c->ev1));
    HB_CUDA(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
  }
  if (c->prof_on) {
    HB_TRY(prof_resolve(c, c->step_marks));
    c->step_marks.clear();
  }
  if ((flags & HB_STEP_MERGE) && !(flags & HB_STEP_ASYNC)) HB_TRY(peer_check(c));
  return HB_OK;
}

// stable counting sort of CSR entries by column -> CSC with ascending rows
void build_csc(const int64_t* rowptr, const int32_t* col, const float* val, long long n_rows, int n_cols,
               std::vector<int64_t>& colptr, std::vector<int32_t>& rowidx, std::vector<float>& cval,
               long long row_base) {
  const long long nnz = rowptr[n_rows] - rowptr[0];
  colptr.assign(n_cols + 1, 0);
  for (long long e = rowptr[0]; e < rowptr[n_rows]; ++e) colptr[col[e] + 1]++;
  for (int j = 0; j < n_cols; ++j) colptr[j + 1] += colptr[j];
  rowidx.resize(nnz);
  cval.resize(nnz);
  std::vector<int64_t> cur(colptr.begin(), colptr.end() - 1);
  for (long long r = 0; r < n_rows; ++r)
    for (long long e = rowptr[r]; e < rowptr[r + 1]; ++e) {
      const long long k = cur[col[e]]++;
      rowidx[k] = static_cast<int32_t>(r + row_base);
      cval[k] = val[e];
    }
}

// ------------------------------------------------ batch CSC on the device
// keys[e] = col[e] * rows + row(e): sorting the (unique) keys orders entries by
// feature and, within a feature, by row -- the same order as the host counting
// sort, so results stay bit-identical to the staged-epoch path.
__global__ void csc_keys_kernel(const int64_t* rowptr, const int32_t* col, int rows, uint32_t* keys, int32_t* idx,
                                int* counts) {
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  for (long long e = rowptr[r] + lane; e < rowptr[r + 1]; e += 32) {
    const int f = col[e];
    keys[e] = static_cast<uint32_t>(f) * static_cast<uint32_t>(rows) + static_cast<uint32_t>(r);
    idx[e] = static_cast<int32_t>(e);
    atomicAdd(&counts[f + 1], 1);  // integer counts: order-independent
  }
}
__global__ void csc_gather_kernel(const uint32_t* keys_sorted, const int32_t* idx_sorted, const float* val,
                                  long long nnz, int rows, int32_t* rowidx, float* cval) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    rowidx[k] = static_cast<int32_t>(keys_sorted[k] % static_cast<uint32_t>(rows));
    cval[k] = val[idx_sorted[k]];
  }
}
__global__ void counts_to_colptr_kernel(const int* counts, int64_t* colptr, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) colptr[i] = counts[i];
}

// Same stable counting sort writing straight into (pinned) output arrays.
void build_csc_into(const int64_t* rowptr, const int32_t* col, const float* val, long long n_rows, int n_cols,
                    int64_t* colptr, int32_t* rowidx, float* cval, std::vector<int64_t>& cur) {
  std::memset(colptr, 0, (n_cols + 1) * sizeof(int64_t));
  for (long long e = rowptr[0]; e < rowptr[n_rows]; ++e) colptr[col[e] + 1]++;
  for (int j = 0; j < n_cols; ++j) colptr[j + 1] += colptr[j];
  cur.assign(colptr, colptr + n_cols);
  for (long long r = 0; r < n_rows; ++r)
    for (long long e = rowptr[r]; e < rowptr[r + 1]; ++e) {
      const long long k = cur[col[e]]++;
      rowidx[k] = static_cast<int32_t>(r);
      cval[k] = val[e];
    }
}

int ensure_pinned(hb_ctx* c, size_t bytes) {
  if (c->pinned_bytes >= bytes) return HB_OK;
  if (c->pinned) cudaFreeHost(c->pinned);
  c->pinned = nullptr;
  HB_CUDA(cudaMallocHost(&c->pinned, bytes));
  c->pinned_bytes = bytes;
  return HB_OK;
}

int free_epoch(hb_ctx* c) {
  cudaFree(c->ex);
  cudaFree(c->ex_lo);
  c->ex_lo = nullptr;
  cudaFree(c->elabels);
  cudaFree(c->erowptr);
  cudaFree(c->ecol);
  cudaFree(c->eval_);
  cudaFree(c->ecolptr);
  cudaFree(c->erowidx);
  cudaFree(c->ecval);
  c->ex = nullptr;
  c->elabels = nullptr;
  c->erowptr = nullptr;
  c->ecol = nullptr;
  c->eval_ = nullptr;
  c->ecolptr = nullptr;
  c->erowidx = nullptr;
  c->ecval = nullptr;
  for (void* q : {static_cast<void*>(c->px), static_cast<void*>(c->px_lo), static_cast<void*>(c->plabels),
                  static_cast<void*>(c->prowptr), static_cast<void*>(c->pcolptr), static_cast<void*>(c->pcol),
                  static_cast<void*>(c->prowidx), static_cast<void*>(c->pval), static_cast<void*>(c->pcval),
                  static_cast<void*>(c->d_perm), static_cast<void*>(c->d_inv), static_cast<void*>(c->d_rowlen),
                  static_cast<void*>(c->p_keys), static_cast<void*>(c->p_idx), c->p_temp})
    cudaFree(q);
  c->px = c->px_lo = c->pval = c->pcval = nullptr;
  c->plabels = c->prowptr = c->pcolptr = c->d_perm = c->d_inv = c->d_rowlen = nullptr;
  c->pcol = c->prowidx = c->p_idx = nullptr;
  c->p_keys = nullptr;
  c->p_temp = nullptr;
  c->p_temp_bytes = 0;
  c->has_base = false;
  c->staged = false;
  c->e_rows = 0;
  c->view_gen++;  // captured graphs baked the old buffers / tensor maps
  return HB_OK;
}

}  // namespace

// ======================================================================
namespace hb {
// error slot shared with the other translation units of the library
int set_error(int code, const char* msg) {
  g_err = msg;
  return code;
}
}  // namespace hb

extern "C" {

const char* hb_last_error(void) { return g_err.c_str(); }

const char* hb_version(void) {
  return "hogbatch_b200 0.1 sm_100a tcgen05 kind::tf32 (3xTF32 / TF32), TMA SW128, CSR SpMM";
}

int hb_device_count(int* out) {
  if (!out) return fail(HB_EINVAL, "null out");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) n = 0;
  *out = n;
  return HB_OK;
}

int hb_ctx_create(hb_ctx** out, int device, int n_layers, const int* sizes, int max_batch, uint32_t flags) {
  if (!out || !sizes) return fail(HB_EINVAL, "null argument");
  *out = nullptr;
  if (n_layers < 1) return fail(HB_EINVAL, "architecture needs at least input and output layers");
  for (int i = 0; i <= n_layers; ++i)
    if (sizes[i] < 1) return fail(HB_EINVAL, "layer sizes must be >= 1, got %d at %d", sizes[i], i);
  if (sizes[n_layers] < 2) return fail(HB_EINVAL, "softmax output needs >= 2 classes");
  if (max_batch < 1) return fail(HB_EINVAL, "max_batch must be >= 1");
  if ((flags & HB_SPARSE_INPUT) && n_layers < 2)
    return fail(HB_EINVAL, "sparse input needs at least one hidden layer");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(HB_ECUDA, "no CUDA device available");
  if (device < 0 || device >= ndev) return fail(HB_EINVAL, "device %d out of range [0, %d)", device, ndev);
  HB_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  HB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(HB_ECUDA, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major, prop.minor);

  hb_ctx* c = new hb_ctx();
  c->device = device;
  c->L = n_layers;
  c->d.assign(sizes, sizes + n_layers + 1);
  c->csr_in = (flags & HB_SPARSE_INPUT) != 0;
  c->sparse = c->csr_in && ((flags & HB_SPARSE_KERNELS) || sizes[0] > HB_DENSIFY_MAX_DIN);
  c->passes = (flags & HB_PRECISION_TF32) ? 1 : 3;
  c->max_batch = max_batch;
  c->cap = static_cast<int>(round_up(max_batch, kBM));
  const int L = c->L;
  c->ld.resize(L + 1);
  for (int l = 0; l <= L; ++l) c->ld[l] = round_up(c->d[l], 4);
  const int nc = c->d[L], dlast = c->d[L - 1];
  c->small_head = nc <= 4 && dlast <= 1024 && !(c->sparse && L == 1);
  if (c->small_head) {
    c->head_nct = nc <= 2 ? 2 : 4;
    c->head_maxt = dlast <= 256 ? 8 : (dlast <= 512 ? 16 : 32);
  }
  auto bail = [&](int code) {
    hb_ctx_destroy(c);
    return code;
  };
#define HB_CK(expr)                                                                                       \
  do {                                                                                                    \
    cudaError_t e_ = (expr);                                                                              \
    if (e_ != cudaSuccess) return bail(fail(HB_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e_))); \
  } while (0)
  HB_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  HB_CK(cudaEventCreate(&c->ev0));
  HB_CK(cudaEventCreate(&c->ev1));
  c->W.assign(L, nullptr);
  c->G.assign(L, nullptr);
  c->ldw.assign(L, 0);
  c->A.assign(L + 1, nullptr);
  c->D.assign(L, nullptr);
  c->W_lo.assign(L, nullptr);
  c->A_lo.assign(L + 1, nullptr);
  c->D_lo.assign(L, nullptr);
  const bool lo = c->need_lo();
  c->bn_fwd.assign(L, 128);
  c->bn_dx.assign(L, 128);
  c->bn_dw.assign(L, 128);
  const int m_tiles = cdiv(c->cap, kBM);
  size_t n_params = 0;
  for (int l = 0; l < L; ++l) {
    const bool tr = (l == 0 && c->sparse);
    c->ldw[l] = tr ? c->ld[1] : c->ld[l];
    const long long rows = tr ? c->d[0] : c->d[l + 1];
    HB_CK(cudaMalloc(&c->W[l], rows * c->ldw[l] * sizeof(float)));
    HB_CK(cudaMemset(c->W[l], 0, rows * c->ldw[l] * sizeof(float)));
    HB_CK(cudaMalloc(&c->G[l], static_cast<size_t>(c->d[l + 1]) * c->d[l] * sizeof(float)));
    HB_CK(cudaMalloc(&c->D[l], static_cast<size_t>(c->cap) * c->ld[l + 1] * sizeof(float)));
    HB_CK(cudaMemset(c->D[l], 0, static_cast<size_t>(c->cap) * c->ld[l + 1] * sizeof(float)));
    if (lo) {
      if (!tr) {
        HB_CK(cudaMalloc(&c->W_lo[l], rows * c->ldw[l] * sizeof(float)));
        HB_CK(cudaMemset(c->W_lo[l], 0, rows * c->ldw[l] * sizeof(float)));
      }
      HB_CK(cudaMalloc(&c->D_lo[l], static_cast<size_t>(c->cap) * c->ld[l + 1] * sizeof(float)));
      HB_CK(cudaMemset(c->D_lo[l], 0, static_cast<size_t>(c->cap) * c->ld[l + 1] * sizeof(float)));
    }
    c->bn_fwd[l] = choose_bn(m_tiles, c->d[l + 1], true);
    c->bn_dx[l] = choose_bn(m_tiles, c->d[l], true);
    // precision: the wide softmax head's logits GEMM with a long contraction
    // (K > 1024) rotates the hi*hi term over >= 3 accumulators (BN <= 128; a
    // 256-wide tile has room for only one): the biased round-toward-zero
    // accumulation of K = 4096 logits reached the head's cancelling dW sum
    // (scaled config: 1.6e-4 -> 8e-5).  HB_BN_LONG_FROM=0 applies it to every
    // long-K forward GEMM (measured ~15% slower steps, no further gain needed)
    const int max_bn_long = static_cast<int>(env_long("HB_BN_LONG_K", 128));
    const int long_from = static_cast<int>(env_long("HB_BN_LONG_FROM", c->small_head ? L : L - 1));
    // (with the accumulator drain every k-block starts a fresh accumulator, so
    // neither cap is needed: HB_GEMM_DRAIN builds keep the wide tiles)
    const bool crit_drain = HB_GEMM_DRAIN && env_long("HB_DRAIN_KB_CRIT", 1) > 0;
    if (c->passes == 3 && cdiv(c->d[l], kBK) > 32 && l >= long_from && !crit_drain)
      c->bn_fwd[l] = std::min(c->bn_fwd[l], max_bn_long);
    c->bn_dw[l] = choose_bn(cdiv(c->d[l + 1], kBM), c->d[l]);
    // experiments: cap the tile width (more rotating accumulators, shorter MMA chains)
    c->bn_fwd[l] = std::min<int>(c->bn_fwd[l], static_cast<int>(env_long("HB_FWD_BN_MAX", 256)));
    c->bn_dx[l] = std::min<int>(c->bn_dx[l], static_cast<int>(env_long("HB_DX_BN_MAX", 256)));
    c->bn_dw[l] = std::min<int>(c->bn_dw[l], static_cast<int>(env_long("HB_DW_BN_MAX", 256)));
    // the wide softmax head's dW sums error signals of both signs over the
    // whole batch (a cancelling sum): 128-wide tiles give 3 rotating hi*hi
    // accumulators, and dw_plan bounds the chain per accumulator
    if (l == L - 1 && !c->small_head && c->passes == 3 && c->d[l] >= 64 && !crit_drain)
      c->bn_dw[l] = static_cast<int>(env_long("HB_HEAD_DW_BN", 128));
    n_params += static_cast<size_t>(c->d[l + 1]) * c->d[l];
  }
  c->n_params = n_params;
  for (int l = 1; l < L; ++l) {
    HB_CK(cudaMalloc(&c->A[l], static_cast<size_t>(c->cap) * c->ld[l] * sizeof(float)));
    HB_CK(cudaMemset(c->A[l], 0, static_cast<size_t>(c->cap) * c->ld[l] * sizeof(float)));
    if (lo) {
      HB_CK(cudaMalloc(&c->A_lo[l], static_cast<size_t>(c->cap) * c->ld[l] * sizeof(float)));
      HB_CK(cudaMemset(c->A_lo[l], 0, static_cast<size_t>(c->cap) * c->ld[l] * sizeof(float)));
    }
  }
  // tensor maps
  c->tmW_k.resize(L);
  c->tmW_mn.resize(L);
  c->tmA_k.resize(L + 1);
  c->tmA_mn.resize(L + 1);
  c->tmD_k.resize(L);
  c->tmD_mn.resize(L);
  c->tmW_k_lo.resize(L);
  c->tmW_mn_lo.resize(L);
  c->tmA_k_lo.resize(L + 1);
  c->tmA_mn_lo.resize(L + 1);
  c->tmD_k_lo.resize(L);
  c->tmD_mn_lo.resize(L);
  int rc = HB_OK;
  for (int l = 0; l < L && rc == HB_OK; ++l) {
    for (int h = 0; h < (lo ? 2 : 1) && rc == HB_OK; ++h) {
      if (!(l == 0 && c->sparse)) {
        float* w = h ? c->W_lo[l] : c->W[l];
        rc = make_map(h ? &c->tmW_k_lo[l] : &c->tmW_k[l], w, c->d[l], c->d[l + 1], c->ldw[l], 32, false);
        if (rc == HB_OK)
          rc = make_map(h ? &c->tmW_mn_lo[l] : &c->tmW_mn[l], w, c->d[l], c->d[l + 1], c->ldw[l], 32, true);
      }
      float* dd = h ? c->D_lo[l] : c->D[l];
      if (rc == HB_OK)
        rc = make_map(h ? &c->tmD_k_lo[l] : &c->tmD_k[l], dd, c->d[l + 1], c->cap, c->ld[l + 1], 128, false);
      if (rc == HB_OK)
        rc = make_map(h ? &c->tmD_mn_lo[l] : &c->tmD_mn[l], dd, c->d[l + 1], c->cap, c->ld[l + 1], 32, true);
    }
  }
  for (int l = 1; l < L && rc == HB_OK; ++l) {
    for (int h = 0; h < (lo ? 2 : 1) && rc == HB_OK; ++h) {
      float* aa = h ? c->A_lo[l] : c->A[l];
      rc = make_map(h ? &c->tmA_k_lo[l] : &c->tmA_k[l], aa, c->d[l], c->cap, c->ld[l], 128, false);
      if (rc == HB_OK) rc = make_map(h ? &c->tmA_mn_lo[l] : &c->tmA_mn[l], aa, c->d[l], c->cap, c->ld[l], 32, true);
    }
  }
  if (rc != HB_OK) return bail(rc);
  // workspaces: split-K partial slabs and head partials
  size_t ws = 0;
  for (int l = 0; l < L; ++l) {
    int splits, kb_per, kb_total;
    dw_plan(c, l, c->cap, &splits, &kb_per, &kb_total);
    if (splits > 1) ws = std::max(ws, static_cast<size_t>(splits) * c->d[l + 1] * c->d[l]);
  }
  if (c->small_head)
    HB_CK(cudaMalloc(&c->ws_head, static_cast<size_t>(cdiv(c->cap, kHeadRowsPerBlock)) * nc * dlast * sizeof(double)));
  ws = std::max(ws, static_cast<size_t>(kSplitSlabFloats));  // split-K forward / dX slabs
  c->ws_floats = std::max<size_t>(ws, 1);
  HB_CK(cudaMalloc(&c->ws, c->ws_floats * sizeof(float)));
  // concurrent backward: per-layer split-K slabs (layers >= 1) + fork/join events
  c->conc_bwd = !(getenv("HB_SPLITK_FUSION") && getenv("HB_SPLITK_FUSION")[0] == '1') &&
                !(getenv("HB_NO_CONC_BWD") && getenv("HB_NO_CONC_BWD")[0] == '1');
  if (c->conc_bwd) {
    size_t tot = 0;
    c->ws_dw_off.assign(L, 0);
    for (int l = 1; l < L; ++l) {
      int splits, kb_per, kb_total;
      dw_plan(c, l, c->cap, &splits, &kb_per, &kb_total);
      c->ws_dw_off[l] = tot;
      if (splits > 1) tot += round_up(static_cast<long long>(splits) * c->d[l + 1] * c->d[l], 64);
    }
    HB_CK(cudaMalloc(&c->ws_dw, std::max<size_t>(tot, 1) * sizeof(float)));
    int lo_prio = 0, hi_prio = 0;
    HB_CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    HB_CK(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, lo_prio));
    c->bev.resize(2 * L + 1);
    for (auto& e : c->bev) HB_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    HB_CK(cudaEventCreateWithFlags(&c->bev_loss, cudaEventDisableTiming));
  }
  c->ws_loss_n = std::max(cdiv(c->cap, kHeadRowsPerBlock), cdiv(c->cap, 8)) + 1;
  HB_CK(cudaMalloc(&c->ws_loss, c->ws_loss_n * sizeof(double)));
  HB_CK(cudaMalloc(&c->d_loss, sizeof(double)));
  HB_CK(cudaHostAlloc(&c->h_loss, sizeof(double), cudaHostAllocMapped));
  HB_CK(cudaMalloc(&c->d_step, sizeof(DevStep)));
  if (c->sparse) {
    HB_CK(cudaMalloc(&c->csc_lo, static_cast<size_t>(c->d[0]) * sizeof(long long)));
    HB_CK(cudaMalloc(&c->csc_hi, static_cast<size_t>(c->d[0]) * sizeof(long long)));
  }
  HB_CK(cudaMemset(c->d_step, 0, sizeof(DevStep)));
  // experimental: split-K dW reduced inside the GEMM (measured no faster than
  // GEMM + reduce kernel at w8a shapes: the rendezvous waits for the slowest split)
  if (getenv("HB_SPLITK_FUSION") && getenv("HB_SPLITK_FUSION")[0] == '1') {
    HB_CK(cudaMalloc(&c->tile_sync, 2 * kTileSyncTiles * sizeof(int)));
    HB_CK(cudaMemset(c->tile_sync, 0, 2 * kTileSyncTiles * sizeof(int)));
  }
  if (const char* g = getenv("HB_NO_GRAPHS")) c->use_graphs = g[0] == '0';
  size_t maxw = 0;
  for (int l = 0; l < L; ++l) maxw = std::max(maxw, static_cast<size_t>(c->d[l + 1]) * c->d[l]);
  c->stage64_n = std::max<size_t>(maxw, size_t(4) << 20);
  HB_CK(cudaMalloc(&c->stage64, c->stage64_n * sizeof(double)));
  HB_CK(cudaMalloc(&c->stage32, maxw * sizeof(float)));
  // batch slot for host-buffer steps
  HB_CK(cudaMalloc(&c->blabels, static_cast<size_t>(c->cap) * sizeof(int64_t)));
  if (c->csr_in) HB_CK(cudaMalloc(&c->browptr, static_cast<size_t>(c->cap + 1) * sizeof(int64_t)));
  if (c->sparse) {
    HB_CK(cudaMalloc(&c->bcolptr, static_cast<size_t>(c->d[0] + 1) * sizeof(int64_t)));
  } else {
    HB_CK(cudaMalloc(&c->bx, static_cast<size_t>(c->cap) * c->ld[0] * sizeof(float)));
    HB_CK(cudaMemset(c->bx, 0, static_cast<size_t>(c->cap) * c->ld[0] * sizeof(float)));
    if (lo) {
      HB_CK(cudaMalloc(&c->bx_lo, static_cast<size_t>(c->cap) * c->ld[0] * sizeof(float)));
      HB_CK(cudaMemset(c->bx_lo, 0, static_cast<size_t>(c->cap) * c->ld[0] * sizeof(float)));
    }
    c->batch.x = c->bx;
    c->batch.x_lo = c->bx_lo;
    c->batch.ldx = c->ld[0];
    c->batch.n_rows = c->cap;
    rc = build_data_maps(c, c->batch);
    if (rc != HB_OK) return bail(rc);
  }
  c->batch.labels = c->blabels;
  {
    const char* e = getenv("HB_SMALL_NET");
    // opt-in (HB_SMALL_NET=1): measured slower than the per-layer tcgen05 path at
    // the covtype config (0.23 vs 0.092 ms/step, profiles/r02_small_net.txt)
    bool ok = !c->sparse && c->passes == 3 && c->small_head && L >= 2 && L <= kSnMaxL && (e && e[0] == '1');
    for (int l = 0; l < L; ++l) ok = ok && c->d[l] <= kSnMaxWidth;
    if (ok) {
      int sms = 0, per_sm = 0;
      HB_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
      HB_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, small_net_step_kernel, kSnThreads, 0));
      if (per_sm >= 1) {
        c->sn_grid = sms * std::min(per_sm, 2);  // two CTAs per SM: a B phase's dX and dW tiles in one wave
        HB_CK(cudaMalloc(&c->sn_hd, kSnMaxRows * 4 * sizeof(float)));
        HB_CK(cudaMalloc(&c->sn_loss, kSnMaxRows * sizeof(double)));
        HB_CK(cudaMalloc(&c->sn_bar, sizeof(unsigned)));
        c->sn_ok = true;
      }
    }
  }
#undef HB_CK
  *out = c;
  return HB_OK;
}

int hb_ctx_destroy(hb_ctx* c) {
  if (!c) return HB_OK;
  cudaSetDevice(c->device);
  land_wait(c);
  if (c->stream) cudaStreamSynchronize(c->stream);
  hb_comm_destroy(c);
  drop_graphs(c);
  cudaFree(c->d_step);
  cudaFree(c->csc_lo);
  cudaFree(c->csc_keys);
  cudaFree(c->csc_idx);
  cudaFree(c->csc_counts);
  cudaFree(c->csc_temp);
  cudaFree(c->csc_hi);
  for (auto p : c->W) cudaFree(p);
  for (auto p : c->G) cudaFree(p);
  for (auto p : c->A) cudaFree(p);
  for (auto p : c->D) cudaFree(p);
  for (auto p : c->W_lo) cudaFree(p);
  for (auto p : c->A_lo) cudaFree(p);
  for (auto p : c->D_lo) cudaFree(p);
  cudaFree(c->bx_lo);
  cudaFree(c->bx_stage);
  free_epoch(c);
  cudaFree(c->bx);
  cudaFree(c->blabels);
  cudaFree(c->browptr);
  cudaFree(c->bcol);
  cudaFree(c->bval);
  cudaFree(c->bcolptr);
  cudaFree(c->browidx);
  cudaFree(c->bcval);
  cudaFree(c->ws);
  cudaFree(c->ws_loss);
  cudaFree(c->sn_hd);
  cudaFree(c->sn_loss);
  cudaFree(c->sn_bar);
  cudaFree(c->tile_sync);
  cudaFree(c->d_loss);
  cudaFreeHost(c->h_loss);
  cudaFree(c->stage64);
  cudaFree(c->stage32);
  cudaFree(c->stage_all);
  cudaFree(c->grad_all);
  if (c->grad_host) cudaFreeHost(c->grad_host);
  cudaFree(c->flat);
  for (float* b : c->bias) cudaFree(b);
  for (auto e : c->mev) cudaEventDestroy(e);
  if (c->comm_st) cudaStreamDestroy(c->comm_st);
  if (c->local) {
    std::lock_guard<std::mutex> lk(c->local->mu);
    auto& lg = *c->local;
    for (auto* evs : {&lg.ev_pack, &lg.ev_red})
      if (c->peers.rank < static_cast<int>(evs->size()) && (*evs)[c->peers.rank]) {
        cudaEventDestroy((*evs)[c->peers.rank]);
        (*evs)[c->peers.rank] = nullptr;
      }
    lg.broken = true;  // a rank left: later merges of the others fail instead of waiting
    lg.cv.notify_all();
  }
  c->local.reset();
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  cudaFree(c->xbuf);
  if (c->pinned) cudaFreeHost(c->pinned);
  for (auto e : c->evpool) cudaEventDestroy(e);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (auto e : c->xfer_ev) cudaEventDestroy(e);
  if (c->snap_ev) cudaEventDestroy(c->snap_ev);
  if (c->merge_ev) cudaEventDestroy(c->merge_ev);
  if (c->xfer) cudaStreamDestroy(c->xfer);
  for (auto e : c->xsnap_ev) cudaEventDestroy(e);
  for (auto e : c->xgrad_ev) cudaEventDestroy(e);
  if (c->xseq_host) cudaFreeHost(c->xseq_host);
  for (auto e : c->xread_ev) cudaEventDestroy(e);
  if (c->xgrad_host) cudaFreeHost(c->xgrad_host);
  cudaFree(c->d_xseq);
  for (auto e : c->xchunk_ev) cudaEventDestroy(e);
  if (c->xstart_ev) cudaEventDestroy(c->xstart_ev);
  if (c->xdone_ev) cudaEventDestroy(c->xdone_ev);
  if (c->xh2d) cudaStreamDestroy(c->xh2d);
  if (c->xmrg) cudaStreamDestroy(c->xmrg);
  for (auto st_ : c->xmrg_l) cudaStreamDestroy(st_);
  for (auto e : c->xmdone_ev) cudaEventDestroy(e);
  for (auto e : c->bev) cudaEventDestroy(e);
  if (c->bev_loss) cudaEventDestroy(c->bev_loss);
  if (c->side) cudaStreamDestroy(c->side);
  cudaFree(c->ws_dw);
  cudaFree(c->ws_head);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return HB_OK;
}

int hb_set_weights_f64(hb_ctx* c, int layer, const double* w) {
  HB_TRY(ctx_check(c));
  HB_TRY(land_wait(c));  // (the staging buffer is reused)
  if (layer < 0 || layer >= c->L || !w) return fail(HB_EINVAL, "bad layer %d or null weights", layer);
  const int rows = c->d[layer + 1], cols = c->d[layer];
  const size_t n = static_cast<size_t>(rows) * cols;
  HB_CUDA(cudaMemcpyAsync(c->stage64, w, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 4096));
  if (layer == 0 && c->sparse)
    f64_to_f32_kernel<true><<<blocks, 256, 0, c->stream>>>(c->W[0], c->ldw[0], c->stage64, cols, rows, cols,
                                                           nullptr);
  else
    f64_to_f32_kernel<false><<<blocks, 256, 0, c->stream>>>(c->W[layer], c->ldw[layer], c->stage64, cols, rows, cols,
                                                            c->need_lo() ? c->W_lo[layer] : nullptr);
  HB_CUDA(cudaGetLastError());
  HB_CUDA(cudaStreamSynchronize(c->stream));
  return HB_OK;
}

int hb_get_weights_f64(hb_ctx* c, int layer, double* w) {
  HB_TRY(ctx_check(c));
  if (layer < 0 || layer >= c->L || !w) return fail(HB_EINVAL, "bad layer %d or null output", layer);
  const int rows = c->d[layer + 1], cols = c->d[layer];
  const size_t n = static_cast<size_t>(rows) * cols;
  const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 4096));
  if (layer == 0 && c->sparse)
    f32_to_f64_kernel<true><<<blocks, 256, 0, c->stream>>>(c->stage64, cols, c->W[0], c->ldw[0], rows, cols);
  else
    f32_to_f64_kernel<false><<<blocks, 256, 0, c->stream>>>(c->stage64, cols, c->W[layer], c->ldw[layer], rows, cols);
  HB_CUDA(cudaGetLastError());
  HB_CUDA(cudaMemcpyAsync(w, c->stage64, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  return HB_OK;
}

int hb_get_weights_f32(hb_ctx* c, int layer, float* w) {
  HB_TRY(ctx_check(c));
  if (layer < 0 || layer >= c->L || !w) return fail(HB_EINVAL, "bad layer %d or null output", layer);
  const int rows = c->d[layer + 1], cols = c->d[layer];
  if (layer == 0 && c->sparse) {
    std::vector<double> tmp(static_cast<size_t>(rows) * cols);
    HB_TRY(hb_get_weights_f64(c, layer, tmp.data()));
    for (size_t i = 0; i < tmp.size(); ++i) w[i] = static_cast<float>(tmp[i]);
    return HB_OK;
  }
  HB_CUDA(cudaMemcpy2DAsync(w, cols * sizeof(float), c->W[layer], c->ldw[layer] * sizeof(float), cols * sizeof(float),
                            rows, cudaMemcpyDeviceToHost, c->stream));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  return HB_OK;
}

int hb_get_grad_f32(hb_ctx* c, int layer, float* g) {
  HB_TRY(ctx_check(c));
  if (layer < 0 || layer >= c->L || !g) return fail(HB_EINVAL, "bad layer %d or null output", layer);
  if (!c->grads_valid) return fail(HB_ESTATE, "no gradient kept: run a step with HB_STEP_EMIT_GRAD first");
  const int rows = c->d[layer + 1], cols = c->d[layer];
  const size_t n = static_cast<size_t>(rows) * cols;
  if (layer == 0 && c->sparse) {
    // G[0] holds the transposed (d_in, d_out) gradient with row stride ldw[0]
    std::vector<float> t(static_cast<size_t>(cols) * c->ldw[0]);
    HB_CUDA(cudaMemcpyAsync(t.data(), c->G[0], t.size() * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    HB_CUDA(cudaStreamSynchronize(c->stream));
    for (int r = 0; r < rows; ++r)
      for (int k = 0; k < cols; ++k) g[static_cast<size_t>(r) * cols + k] = t[static_cast<size_t>(k) * c->ldw[0] + r];
    return HB_OK;
  }
  HB_CUDA(cudaMemcpyAsync(g, c->G[layer], n * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  return HB_OK;
}

// Registered (page-locked, device-mapped) host ranges: the snapshot kernel
// reads the shared float64 model straight over PCIe and the stale merge is a
// kernel doing W_host -= eta*g in place over PCIe (aligned 8-byte stores, so
// concurrent host readers never see a torn scalar, as linalg.py:3-7 requires).
int hb_host_register(const void* p, size_t bytes) {
  if (!p || bytes == 0) return fail(HB_EINVAL, "null pointer or zero size");
  std::lock_guard<std::mutex> lk(g_host_mu);
  if (g_host_ranges.count(reinterpret_cast<uintptr_t>(p))) {
    g_host_refs[reinterpret_cast<uintptr_t>(p)]++;
    return HB_OK;
  }
  cudaError_t e = cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    cudaGetLastError();
    return HB_OK;  // registered by someone else: used through the copy path
  }
  HB_CUDA(e);
  void* dptr = nullptr;
  HB_CUDA(cudaHostGetDevicePointer(&dptr, const_cast<void*>(p), 0));
  g_host_ranges[reinterpret_cast<uintptr_t>(p)] = {bytes, dptr};
  g_host_refs[reinterpret_cast<uintptr_t>(p)] = 1;
  return HB_OK;
}

int hb_host_unregister(const void* p) {
  if (!p) return fail(HB_EINVAL, "null pointer");
  std::lock_guard<std::mutex> lk(g_host_mu);
  auto it = g_host_ranges.find(reinterpret_cast<uintptr_t>(p));
  if (it == g_host_ranges.end()) return HB_OK;
  if (--g_host_refs[it->first] > 0) return HB_OK;  // still page-locked for another context
  g_host_refs.erase(it->first);
  g_host_ranges.erase(it);
  g_pin_epoch.fetch_add(1);  // contexts re-check their host model's page-lock
  cudaError_t e = cudaHostUnregister(const_cast<void*>(p));
  if (e == cudaErrorHostMemoryNotRegistered) {
    cudaGetLastError();
    return HB_OK;
  }
  HB_CUDA(e);
  return HB_OK;
}

// device alias of a registered host range covering [p, p+bytes), or null
static void* mapped_alias(const void* p, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_host_mu);
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  auto it = g_host_ranges.upper_bound(a);
  if (it == g_host_ranges.begin()) return nullptr;
  --it;
  if (a + bytes > it->first + it->second.first) return nullptr;
  return static_cast<char*>(it->second.second) + (a - it->first);
}

// page-locked host memory (registered or cudaMallocHost'd): DMA-able as is
static bool is_pinned(const void* p) {
  if (p == nullptr) return false;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Host->device copy that tolerates a source range straddling the end of a
// registered (page-locked) range -- e.g. a staged array whose head is a view
// that was pinned earlier: CUDA rejects such a copy as one transfer, so it is
// split at registered-range boundaries.  sync: wait for completion.
static cudaError_t h2d_copy(void* dst, const void* src, size_t bytes, cudaStream_t st, bool sync = false) {
  t_h2d_bytes += static_cast<long long>(bytes);
  const uintptr_t a = reinterpret_cast<uintptr_t>(src);
  size_t done = 0;
  while (done < bytes) {
    const uintptr_t p = a + done;
    size_t n = bytes - done;
    {
      std::lock_guard<std::mutex> lk(g_host_mu);
      auto it = g_host_ranges.upper_bound(p);
      if (it != g_host_ranges.begin()) {
        auto prev = std::prev(it);
        if (p < prev->first + prev->second.first) n = std::min<size_t>(n, prev->first + prev->second.first - p);
      }
      if (it != g_host_ranges.end() && it->first < p + n) n = it->first - p;  // stop at the next registered range
    }
    cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + done, reinterpret_cast<const void*>(p), n,
                                    cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    done += n;
  }
  return sync ? cudaStreamSynchronize(st) : cudaSuccess;
}

static int ensure_stage_all(hb_ctx* c) {
  if (c->stage_all) return HB_OK;
  HB_CUDA(cudaMalloc(&c->stage_all, c->n_params * sizeof(double)));
  HB_CUDA(cudaMalloc(&c->grad_all, c->n_params * sizeof(float)));
  HB_CUDA(cudaMallocHost(&c->grad_host, c->n_params * sizeof(float)));
  return HB_OK;
}

int hb_set_bias_f64(hb_ctx* c, int layer, const double* b) {
  HB_TRY(ctx_check(c));
  if (layer < 0 || layer >= c->L - 1)
    return fail(HB_EINVAL, "bias is supported on hidden layers 0..%d (the output layer has none)", c->L - 2);
  if (c->bias.empty()) c->bias.assign(c->L, nullptr);
  drop_graphs(c);  // the fused epilogues read the pointer at capture time
  if (b == nullptr) {
    cudaFree(c->bias[layer]);
    c->bias[layer] = nullptr;
    return HB_OK;
  }
  const int n = c->d[layer + 1];
  std::vector<float> h(round_up(n, 4), 0.f);
  for (int i = 0; i < n; ++i) h[i] = static_cast<float>(b[i]);
  if (!c->bias[layer]) HB_CUDA(cudaMalloc(&c->bias[layer], h.size() * sizeof(float)));
  HB_CUDA(cudaMemcpy(c->bias[layer], h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
  return HB_OK;
}

int hb_set_weights_all_f64(hb_ctx* c, const double* const* ws) {
  HB_TRY(ctx_check(c));
  HB_TRY(land_wait(c));  // (the staging buffer is reused)
  if (!ws) return fail(HB_EINVAL, "null weight array");
  HB_TRY(ensure_stage_all(c));
  c->mirror_valid = false;  // the staging buffer is reused below
  XferClock clk("snapshot");
  for (int l = 0; l < c->L; ++l)
    if (!ws[l]) return fail(HB_EINVAL, "null weights for layer %d", l);
  // DMA every layer into the f64 staging buffer (copy engine, full link rate
  // from page-locked memory), return once the bytes landed -- the snapshot is
  // taken -- and let the f64 -> f32 (+lo) conversions run behind the caller
  if (!c->snap_ev) HB_CUDA(cudaEventCreateWithFlags(&c->snap_ev, cudaEventDisableTiming));
  size_t off = 0;
  for (int l = 0; l < c->L; ++l) {
    const size_t n = static_cast<size_t>(c->d[l + 1]) * c->d[l];
    HB_CUDA(cudaMemcpyAsync(c->stage_all + off, ws[l], n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    off += n;
  }
  HB_CUDA(cudaEventRecord(c->snap_ev, c->stream));
  clk.mark("dma enqueued");
  off = 0;
  for (int l = 0; l < c->L; ++l) {
    const int rows = c->d[l + 1], cols = c->d[l];
    const size_t n = static_cast<size_t>(rows) * cols;
    const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 4096));
    if (l == 0 && c->sparse)
      f64_to_f32_kernel<true><<<blocks, 256, 0, c->stream>>>(c->W[0], c->ldw[0], c->stage_all + off, cols, rows, cols,
                                                             nullptr);
    else
      f64_to_f32_kernel<false><<<blocks, 256, 0, c->stream>>>(c->W[l], c->ldw[l], c->stage_all + off, cols, rows,
                                                              cols, c->need_lo() ? c->W_lo[l] : nullptr);
    HB_CUDA(cudaGetLastError());
    off += n;
  }
  clk.mark("kernels enqueued");
  HB_CUDA(cudaEventSynchronize(c->snap_ev));
  clk.mark("dma done");
  return HB_OK;
}

int hb_merge_grads_all_into_f64(hb_ctx* c, double* const* ws, double eta) {
  HB_TRY(ctx_check(c));
  HB_TRY(land_wait(c));  // (the staging buffer is reused)
  if (!ws) return fail(HB_EINVAL, "null weight array");
  if (!c->grads_valid) return fail(HB_ESTATE, "no gradient kept: run a step with HB_STEP_EMIT_GRAD first");
  HB_TRY(ensure_stage_all(c));
  c->mirror_valid = false;  // the staging buffer is reused below
  bool mapped = true;
  std::vector<double*> dws(c->L);
  for (int l = 0; l < c->L; ++l) {
    if (!ws[l]) return fail(HB_EINVAL, "null weights for layer %d", l);
    dws[l] = static_cast<double*>(mapped_alias(ws[l], static_cast<size_t>(c->d[l + 1]) * c->d[l] * sizeof(double)));
    mapped = mapped && dws[l] != nullptr;
  }
  if (mapped) {
    // page-locked host model: pipelined read-modify-write over the two copy
    // engines -- chunk k goes H2D on the xfer stream while chunk k-1 is
    // updated on the device (w += -eta*g in f64, linalg.py:79) and written
    // back D2H on the step stream
    XferClock clk("merge");
    if (!c->xfer) HB_CUDA(cudaStreamCreateWithFlags(&c->xfer, cudaStreamNonBlocking));
    static const size_t kChunk = getenv("HB_MERGE_CHUNK") ? static_cast<size_t>(atoll(getenv("HB_MERGE_CHUNK")))
                                                           : (size_t(1) << 17);  // doubles (1 MiB)
    if (!c->merge_ev) HB_CUDA(cudaEventCreateWithFlags(&c->merge_ev, cudaEventDisableTiming));
    HB_CUDA(cudaEventRecord(c->merge_ev, c->stream));
    HB_CUDA(cudaStreamWaitEvent(c->xfer, c->merge_ev, 0));  // the step (gradient) and any earlier use are done
    size_t off = 0;
    int k = 0;
    for (int l = 0; l < c->L; ++l) {
      const int rows = c->d[l + 1], cols = c->d[l];
      const size_t n = static_cast<size_t>(rows) * cols;
      const bool tr = (l == 0 && c->sparse);
      // chunks are whole rows of the (rows, cols) host layout
      const int rows_per = static_cast<int>(std::max<size_t>(1, kChunk / std::max(1, cols)));
      for (int r0 = 0; r0 < rows; r0 += rows_per, ++k) {
        const int nr = std::min(rows_per, rows - r0);
        const size_t e0 = static_cast<size_t>(r0) * cols, ne = static_cast<size_t>(nr) * cols;
        if (static_cast<int>(c->xfer_ev.size()) <= k) {
          cudaEvent_t e;
          HB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          c->xfer_ev.push_back(e);
        }
        double* dev = c->stage_all + off + e0;
        HB_CUDA(cudaMemcpyAsync(dev, ws[l] + e0, ne * sizeof(double), cudaMemcpyHostToDevice, c->xfer));
        HB_CUDA(cudaEventRecord(c->xfer_ev[k], c->xfer));
        HB_CUDA(cudaStreamWaitEvent(c->stream, c->xfer_ev[k], 0));
        const float* g = tr ? c->G[0] + r0 : c->G[l] + static_cast<size_t>(r0) * cols;
        merge_host_f64_kernel<<<static_cast<int>(std::min<size_t>((ne + 255) / 256, 148 * 8)), 256, 0, c->stream>>>(
            dev, g, tr ? c->ldw[0] : cols, nr, cols, tr ? 1 : 0, eta);
        HB_CUDA(cudaGetLastError());
        HB_CUDA(cudaMemcpyAsync(ws[l] + e0, dev, ne * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      }
      off += n;
    }
    clk.mark("enqueued");
    HB_CUDA(cudaStreamSynchronize(c->stream));
    clk.mark("done");
    return HB_OK;
  }
  // gather every layer's gradient in (d_{l+1}, d_l) order into one device
  // buffer (the sparse layer's transposed gradient is transposed back on the
  // device), one D2H, then the float64 axpy on the host
  size_t off = 0;
  std::vector<size_t> offs(c->L);
  for (int l = 0; l < c->L; ++l) {
    const int rows = c->d[l + 1], cols = c->d[l];
    const size_t n = static_cast<size_t>(rows) * cols;
    offs[l] = off;
    if (l == 0 && c->sparse) {
      const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 4096));
      transpose_f32_kernel<<<blocks, 256, 0, c->stream>>>(c->grad_all + off, c->G[0], c->ldw[0], rows, cols);
      HB_CUDA(cudaGetLastError());
    } else {
      HB_CUDA(cudaMemcpyAsync(c->grad_all + off, c->G[l], n * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
    }
    off += n;
  }
  HB_CUDA(cudaMemcpyAsync(c->grad_host, c->grad_all, off * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  XferClock clk2("merge-host");
  // linalg.py:79 np.add(target, scale*source, out=target), scale = -eta; elementwise,
  // so splitting the index range over threads changes nothing numerically
  const double scale = -eta;
  const int nthreads = static_cast<int>(std::max<size_t>(1, std::min<size_t>(8, off / (1 << 16))));
  auto work = [&](int t) {
    for (int l = 0; l < c->L; ++l) {
      const size_t n = static_cast<size_t>(c->d[l + 1]) * c->d[l];
      const size_t a = n * t / nthreads, b = n * (t + 1) / nthreads;
      double* w = ws[l];
      const float* g = c->grad_host + offs[l];
      for (size_t i = a; i < b; ++i) w[i] += scale * static_cast<double>(g[i]);
    }
  };
  if (nthreads == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int t = 1; t < nthreads; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
  }
  clk2.mark("axpy done");
  return HB_OK;
}

int hb_merge_grad_into_f64(hb_ctx* c, int layer, double* host_w, double eta) {
  HB_TRY(ctx_check(c));
  HB_TRY(land_wait(c));  // (the staging buffer is reused)
  if (layer < 0 || layer >= c->L || !host_w) return fail(HB_EINVAL, "bad layer %d or null weights", layer);
  const int rows = c->d[layer + 1], cols = c->d[layer];
  const size_t n = static_cast<size_t>(rows) * cols;
  HB_TRY(ensure_pinned(c, n * sizeof(float) + (layer == 0 && c->sparse ? n * sizeof(float) : 0)));
  float* g = static_cast<float*>(c->pinned);
  HB_TRY(hb_get_grad_f32(c, layer, g));
  // linalg.py:79 np.add(target, scale*source, out=target), scale = -eta
  const double scale = -eta;
  for (size_t i = 0; i < n; ++i) host_w[i] += scale * static_cast<double>(g[i]);
  return HB_OK;
}

// ------------------------------------------ fused replica step (drop-in call)
// Arms the overlapped exchange for exactly one step call.  The host model must
// be page-locked (hb_host_register) so its DMAs run at link speed and can be
// captured into the step graph.
// Which layers merge on the device lane.  Each layer's merge costs either
// host DRAM (host lane: read w, write w, read the fp32 gradient, 20 B per
// weight) plus 4 B of gradient D2H, or PCIe both ways (device lane: 8 B H2D
// merge read + 8 B D2H write-back per weight).  Layers are assigned greedily
// to keep max(H2D, D2H, host-DRAM time) of the merge phase lowest (measured
// B200 host: ~50 GB/s each PCIe direction, ~65 GB/s of host DRAM for this
// access mix; the snapshot's H2D precedes the merge phase and is not
// counted).  Only layers whose split-K reduce carries the merge and whose
// merge read can hide under the dW partial GEMM (large batches) qualify.
static void xchg_plan_lanes_impl(hb_ctx* c);
static void xchg_plan_mirror(hb_ctx* c);
static void xchg_plan_lanes(hb_ctx* c) {
  xchg_plan_lanes_impl(c);
  xchg_plan_mirror(c);
  if (xfer_debug())
    for (int l = 0; l < c->L; ++l)
      fprintf(stderr, "[xfer] layer %d merges on the %s lane\n", l, c->xdma[l] ? "device" : (c->xml[l] ? "mirror (sole writer)" : "host"));
}
// Mirror lane plan (sole-writer calls, §6): a mirror-lane layer moves 8 B per
// weight D2H (the merged float64 row) and no host work; a host-lane layer 4 B
// D2H (the fp32 gradient) plus ~20 B of host DRAM traffic for the float64
// read-modify-write.  Largest layers first, each goes where max(D2H time, host
// time) stays lowest.  Measured e2e with every layer on the mirror lane vs none:
// scaled 5.9e5 -> 6.2e5, w8a 1.65e7 -> 1.88e7, real-sim 1.3e6 -> 1.7e6 samples/s;
// the split this cost model picks (scaled: the two 4M-weight layers on the
// host) measured 5.9e5 vs 6.1e5 for all-mirror -- the B200 host's float64 merge
// is slower than PCIe -- so every layer takes the mirror lane by default.
// HB_MIRROR_LANE=0 / =plan: none / the cost-model split (HB_PCIE_GBS, HB_HOST_MERGE_GBS).
static void xchg_plan_mirror(hb_ctx* c) {
  c->xml.assign(c->L, 0);
  const char* e = getenv("HB_MIRROR_LANE");
  if (e && e[0] == '0') return;
  const bool all = !(e && strcmp(e, "plan") == 0);
  const double pcie = static_cast<double>(env_long("HB_PCIE_GBS", 50)), hostbw = static_cast<double>(env_long("HB_HOST_MERGE_GBS", 40));
  std::vector<int> order(c->L);
  for (int l = 0; l < c->L; ++l) order[l] = l;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    return static_cast<long long>(c->d[a + 1]) * c->d[a] > static_cast<long long>(c->d[b + 1]) * c->d[b];
  });
  double d2h = 0.0, host = 0.0;
  for (int l : order) {
    if (l < static_cast<int>(c->xdma.size()) && c->xdma[l]) continue;  // device lane
    const double n = static_cast<double>(c->d[l + 1]) * c->d[l];
    const double cm = std::max((d2h + 8 * n) / pcie, host / hostbw), ch = std::max((d2h + 4 * n) / pcie, (host + 20 * n) / hostbw);
    if (all || cm <= ch) {
      c->xml[l] = 1;
      d2h += 8 * n;
    } else {
      d2h += 4 * n;
      host += 20 * n;
    }
  }
}

static void xchg_plan_lanes_impl(hb_ctx* c) {
  c->xdma.assign(c->L, 0);
  if (c->xmode != 0 || !c->conc_bwd || c->cap < 4096 ||
      (getenv("HB_NO_XCHG_DEVICE_LANE") && getenv("HB_NO_XCHG_DEVICE_LANE")[0] == '1'))
    return;
  double h2d = 0.0, d2h = 0.0, host = 0.0;  // merge phase only: the snapshot's H2D is long done by then
  const int top = c->small_head ? c->L - 2 : c->L - 1;
  auto cost = [](double a, double b, double h) { return std::max(std::max(a / 50.0, b / 50.0), h / 65.0); };
  for (int l = c->L - 1; l >= 0; --l) {
    const double n = static_cast<double>(c->d[l + 1]) * c->d[l];
    bool capable = l >= 1 && l <= top && (layer_offset(c, l) % 2) == 0 && c->d[l] % 4 == 0 && c->ldw[l] % 4 == 0 &&
                   n / 4 >= 148 * 256;
    if (capable) {
      int splits, kb_per, kb_total;
      dw_plan(c, l, c->cap, &splits, &kb_per, &kb_total);
      capable = splits > 1;
    }
    if (capable && cost(h2d + 8 * n, d2h + 8 * n, host) < cost(h2d, d2h + 4 * n, host + 20 * n)) {
      c->xdma[l] = 1;
      h2d += 8 * n;
      d2h += 8 * n;
    } else {
      d2h += 4 * n;
      host += 20 * n;
    }
  }
}

// host-model fingerprint for the resident mirror: 64 evenly spaced values per layer
static void mirror_sample(const hb_ctx* c, double* const* ws, std::vector<double>& out) {
  constexpr int K = 64;
  out.clear();
  for (int l = 0; l < c->L; ++l) {
    const size_t n = static_cast<size_t>(c->d[l + 1]) * c->d[l];
    for (int k = 0; k < K; ++k) {
      const double v = reinterpret_cast<volatile const double*>(ws[l])[(n - 1) * k / (K - 1)];
      out.push_back(v);
    }
  }
}

// Wait until the write-backs of a deferred (HB_STEP_LAND_ASYNC) call are in
// the host model, then fingerprint it for the resident-mirror check.
static int land_wait(hb_ctx* c) {
  if (!c->land_pending) return HB_OK;
  c->land_pending = false;
  cudaError_t err = cudaSuccess;
  for (cudaStream_t st : c->xmrg_l) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (err == cudaSuccess) err = e;
  }
  if (err != cudaSuccess) {
    c->mirror_valid = false;
    return fail(HB_ECUDA, "deferred write-back failed: %s", cudaGetErrorString(err));
  }
  if (c->mirror_valid && c->land_ws.size() == static_cast<size_t>(c->L))
    mirror_sample(c, c->land_ws.data(), c->fp_vals);
  return HB_OK;
}

static int xchg_arm(hb_ctx* c, double* const* ws, uint32_t flags) {
  g_call_t0 = std::chrono::steady_clock::now();
  if (!ws) return fail(HB_EINVAL, "null weight array");
  const bool defer = (flags & HB_STEP_LAND_ASYNC) != 0;
  if (defer && !(flags & HB_STEP_SOLE_WRITER))
    return fail(HB_EINVAL, "HB_STEP_LAND_ASYNC needs HB_STEP_SOLE_WRITER (nobody else may write the host model)");
  // a deferred chain continues only on the same host arrays; anything else
  // (another model, a call that lands before returning) waits for the landing
  if (c->land_pending && !(defer && c->land_ws.size() == static_cast<size_t>(c->L) &&
                           std::equal(c->land_ws.begin(), c->land_ws.end(), ws)))
    HB_TRY(land_wait(c));
  // (the page-lock check costs a driver call per layer: once per pointer set)
  const long long epoch = g_pin_epoch.load();
  const bool same_set = c->xw_prev.size() == static_cast<size_t>(c->L) &&
                        std::equal(c->xw_prev.begin(), c->xw_prev.end(), ws) && c->pin_epoch == epoch;
  c->pin_epoch = epoch;
  for (int l = 0; l < c->L && !same_set; ++l) {
    if (!ws[l]) return fail(HB_EINVAL, "null weights for layer %d", l);
    if (!is_pinned(ws[l]))
      return fail(HB_EINVAL, "layer %d of the host model is not page-locked (hb_host_register it first)", l);
  }
  HB_TRY(ensure_stage_all(c));
  if (!c->xh2d) {
    int lo_prio = 0, hi_prio = 0;
    HB_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    HB_CUDA(cudaStreamCreateWithPriority(&c->xh2d, cudaStreamNonBlocking, hi_prio));
    HB_CUDA(cudaStreamCreateWithPriority(&c->xmrg, cudaStreamNonBlocking, hi_prio));
    c->xmrg_l.resize(c->L);
    c->xmdone_ev.resize(c->L);
    c->xmrg_used.assign(c->L, 0);
    c->xmerged_ev.resize(c->L);
    c->xmerged_rec.assign(c->L, 0);
    for (int l = 0; l < c->L; ++l) {
      HB_CUDA(cudaStreamCreateWithPriority(&c->xmrg_l[l], cudaStreamNonBlocking, hi_prio));
      HB_CUDA(cudaEventCreateWithFlags(&c->xmdone_ev[l], cudaEventDisableTiming));
      HB_CUDA(cudaEventCreateWithFlags(&c->xmerged_ev[l], cudaEventDisableTiming));
    }
    c->xd2h_ready_ev.resize(c->L);
    c->xd2h_done_ev.resize(c->L);
    c->xd2h_defer.assign(c->L, 0);
    for (int l = 0; l < c->L; ++l) {
      HB_CUDA(cudaEventCreateWithFlags(&c->xd2h_ready_ev[l], cudaEventDisableTiming));
      HB_CUDA(cudaEventCreateWithFlags(&c->xd2h_done_ev[l], cudaEventDisableTiming));
    }
    HB_CUDA(cudaEventCreateWithFlags(&c->xstart_ev, cudaEventDisableTiming));
    HB_CUDA(cudaEventCreateWithFlags(&c->xdone_ev, cudaEventDisableTiming));
    c->xsnap_ev.resize(c->L);
    c->xgrad_ev.resize(c->L);
    for (int l = 0; l < c->L; ++l) {
      HB_CUDA(cudaEventCreateWithFlags(&c->xsnap_ev[l], cudaEventDisableTiming));
      HB_CUDA(cudaEventCreateWithFlags(&c->xgrad_ev[l], cudaEventDisableTiming));
    }
    HB_CUDA(cudaMallocHost(&c->xseq_host, (c->L + 1) * sizeof(int32_t)));
    HB_CUDA(cudaHostAlloc(&c->xgrad_host, c->n_params * sizeof(float) + 64, cudaHostAllocDefault));
    std::memset(c->xseq_host, 0, (c->L + 1) * sizeof(int32_t));
    HB_CUDA(cudaMalloc(&c->d_xseq, sizeof(int32_t)));
    c->xread_ev.resize(c->L);
    for (auto& e : c->xread_ev) HB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    xchg_plan_lanes(c);
    if (const char* m = getenv("HB_XCHG_MERGE")) c->xmode_env = strcmp(m, "dma") == 0 ? 1 : 0;
  }
  std::vector<double*> cur(ws, ws + c->L);
  if (cur != c->xw_prev) {
    // graph key of this pointer set (a hash, so alternating between a few
    // host models reuses their captured graphs instead of re-capturing)
    unsigned long long h = 1469598103934665603ull;
    for (double* q : cur) h = (h ^ reinterpret_cast<uintptr_t>(q)) * 1099511628211ull;
    c->xw_prev = cur;
    c->xgen = static_cast<long long>(h >> 1) | 1;  // never 0 (0 = no exchange armed)
  }
  c->xw = cur;
  // resident mirror: a sole-writer call right after a sole-writer call on the
  // same arrays, and nobody touched the sampled host values in between
  c->xmode = (c->xmode_env == 1 && (flags & HB_STEP_SOLE_WRITER) != 0) ? 1 : 0;
  c->xsole = (flags & HB_STEP_SOLE_WRITER) != 0 && c->xmode == 0 &&
             !(getenv("HB_NO_MIRROR") && getenv("HB_NO_MIRROR")[0] == '1');
  c->xmirror = false;
  if (c->xsole && c->mirror_valid && c->mirror_gen == c->xgen) {
    if (c->land_pending) {
      // deferred chain: the host copy is still landing (it cannot be sampled);
      // the sole-writer declaration covers it until hb_replica_landed
      c->xmirror = true;
    } else {
      std::vector<double> now;
      mirror_sample(c, ws, now);
      c->xmirror = now.size() == c->fp_vals.size() &&
                   std::memcmp(now.data(), c->fp_vals.data(), now.size() * sizeof(double)) == 0;
    }
  }
  c->xland = defer && c->xsole;  // (the DMA merge mode lands before returning)
  c->mirror_valid = false;  // until this call completes
  c->xseq = c->xseq == 0x7fffffff ? 1 : c->xseq + 1;
  *reinterpret_cast<volatile int32_t*>(c->xseq_host) = c->xseq;
  return HB_OK;
}

struct XchgGuard {
  hb_ctx* c;
  ~XchgGuard() {
    c->xw.clear();
    xtl_dump();
  }
};

// Bytes the replica call moved over PCIe: the batch (counted as issued) plus
// the exchange copies captured in the step graph, per layer by lane.
static void xfer_account(hb_ctx* c, bool loss) {
  long long h2d = t_h2d_bytes, d2h = loss ? static_cast<long long>(sizeof(double)) : 0;
  if (c->xmode == 0) h2d += sizeof(int32_t);  // the sequence number the layer flags carry
  for (int l = 0; l < c->L; ++l) {
    const long long n = static_cast<long long>(c->d[l + 1]) * c->d[l];
    if (!c->xmirror) h2d += n * 8;  // snapshot (deep_copy, workers.py:132)
    const int lane = l < static_cast<int>(c->xdma_used.size()) ? c->xdma_used[l] : 0;
    const bool dev = c->xmode != 0 || lane != 0;
    if (dev) {
      if (!c->xmirror && lane != 2) h2d += n * 8;  // merge read of the host rows
      d2h += n * 8;  // merged rows written back
    } else {
      d2h += n * 4 + static_cast<long long>(sizeof(int32_t));  // fp32 gradient + the layer's flag
    }
  }
  c->last_h2d = h2d;
  c->last_d2h = d2h;
}

// Enqueue the step asynchronously (the exchange rides inside it), apply the
// host-mode merges as gradients land, then finish like do_step.
static int replica_finish(hb_ctx* c, int rc, int rows, double eta, uint32_t flags, double* out_loss,
                          bool ev1_recorded = false) {
  if (rc != HB_OK) {
    // nothing may still be reading or writing the host model when the call
    // returns: drain the step stream and the exchange's copy streams
    cudaStreamSynchronize(c->stream);
    if (c->xh2d) cudaStreamSynchronize(c->xh2d);
    if (c->xmrg) cudaStreamSynchronize(c->xmrg);
    for (auto st_ : c->xmrg_l) cudaStreamSynchronize(st_);
    if (c->side) cudaStreamSynchronize(c->side);
    c->land_pending = false;
    c->xland = false;
    c->mirror_valid = false;
    return rc;
  }
  const bool timed = (flags & HB_STEP_TIMED) != 0;
  if (timed && !ev1_recorded) HB_CUDA(cudaEventRecord(c->ev1, c->stream));
  HB_TRY(xchg_host_merges(c, eta));
  if (out_loss != nullptr) {
    double sum = 0.0;
    HB_TRY(read_loss(c, &sum));
    *out_loss = sum / rows;
  } else {
    HB_CUDA(cudaStreamSynchronize(c->stream));
  }
  if (timed) HB_CUDA(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
  xfer_account(c, out_loss != nullptr);
  if (c->xsole) {  // the staging buffer now equals the host model
    c->mirror_valid = true;
    c->mirror_gen = c->xgen;
    if (c->xland) {  // ... and will, once the write-backs land (fingerprinted then)
      c->land_pending = true;
      c->land_ws = c->xw;
    } else {
      mirror_sample(c, c->xw.data(), c->fp_vals);
    }
  }
  c->xland = false;
  xmark("done");
  return HB_OK;
}

static uint32_t replica_flags(hb_ctx* c, uint32_t flags) {
  t_h2d_bytes = 0;
  if (flags & HB_STEP_TIMED) cudaEventRecord(c->ev0, c->stream);
  return (flags | HB_STEP_EMIT_GRAD | HB_STEP_ASYNC) & ~HB_STEP_TIMED;
}

int hb_replica_step(hb_ctx* c, double* const* ws, int64_t start, int rows, double eta, uint32_t flags,
                    double* out_loss) {
  HB_TRY(ctx_check(c));
  HB_TRY(xchg_arm(c, ws, flags));
  XchgGuard g{c};
  const int rc = hb_train_step(c, start, rows, eta, replica_flags(c, flags), nullptr);
  return replica_finish(c, rc, rows, eta, flags, out_loss);
}

int hb_replica_begin(hb_ctx* c, double* const* ws, int64_t start, int rows, double eta, uint32_t flags) {
  HB_TRY(ctx_check(c));
  if (c->pend_active) return fail(HB_ESTATE, "a replica step is already in flight");
  HB_TRY(xchg_arm(c, ws, flags));
  const int rc = hb_train_step(c, start, rows, eta, replica_flags(c, flags), nullptr);
  if (rc != HB_OK) {
    XchgGuard g{c};
    replica_finish(c, rc, rows, eta, flags, nullptr);  // drains the streams
    return rc;
  }
  if (flags & HB_STEP_TIMED) HB_CUDA(cudaEventRecord(c->ev1, c->stream));  // the step's end, not end()'s call
  c->pend_active = true;
  c->pend_rows = rows;
  c->pend_eta = eta;
  c->pend_flags = flags;
  return HB_OK;
}

int hb_replica_end(hb_ctx* c, double* out_loss) {
  HB_TRY(ctx_check(c));
  if (!c->pend_active) return fail(HB_ESTATE, "no replica step in flight");
  c->pend_active = false;
  XchgGuard g{c};
  return replica_finish(c, HB_OK, c->pend_rows, c->pend_eta, c->pend_flags, out_loss, true);
}

int hb_replica_step_host_dense(hb_ctx* c, double* const* ws, const float* x, int64_t ld, const int64_t* labels,
                               int rows, double eta, uint32_t flags, double* out_loss) {
  HB_TRY(ctx_check(c));
  HB_TRY(xchg_arm(c, ws, flags));
  XchgGuard g{c};
  const int rc = hb_train_step_host_dense(c, x, ld, labels, rows, eta, replica_flags(c, flags), nullptr);
  return replica_finish(c, rc, rows, eta, flags, out_loss);
}

int hb_replica_step_host_csr(hb_ctx* c, double* const* ws, const int64_t* rowptr, const int32_t* col,
                             const float* val, const int64_t* labels, int rows, double eta, uint32_t flags,
                             double* out_loss) {
  HB_TRY(ctx_check(c));
  HB_TRY(xchg_arm(c, ws, flags));
  XchgGuard g{c};
  const int rc =
      hb_train_step_host_csr(c, rowptr, col, val, labels, rows, eta, replica_flags(c, flags), nullptr);
  return replica_finish(c, rc, rows, eta, flags, out_loss);
}

static int stage_dense_common(hb_ctx* c, int64_t n_rows, const int64_t* labels, bool gen_labels = false) {
  if (c->csr_in) return fail(HB_EINVAL, "context was created for sparse (CSR) input");
  if (n_rows < 1 || (!labels && !gen_labels)) return fail(HB_EINVAL, "need n_rows >= 1 and labels");
  HB_TRY(free_epoch(c));
  HB_CUDA(cudaMalloc(&c->ex, static_cast<size_t>(n_rows) * c->ld[0] * sizeof(float)));
  if (c->need_lo()) HB_CUDA(cudaMalloc(&c->ex_lo, static_cast<size_t>(n_rows) * c->ld[0] * sizeof(float)));
  if (c->ld[0] > c->d[0]) {
    // zero the pad columns once: no kernel reads them (the tensor maps stop at
    // d[0]), but row copies (hb_permute_epoch) move whole rows
    for (float* x : {c->ex, c->ex_lo}) {
      if (x == nullptr) continue;
      HB_CUDA(cudaMemset2DAsync(x + c->d[0], c->ld[0] * sizeof(float), 0, (c->ld[0] - c->d[0]) * sizeof(float),
                                n_rows, c->stream));
    }
  }
  HB_CUDA(cudaMalloc(&c->elabels, static_cast<size_t>(n_rows) * sizeof(int64_t)));
  if (labels) HB_CUDA(h2d_copy(c->elabels, labels, n_rows * sizeof(int64_t), c->stream));
  c->e_rows = n_rows;
  return HB_OK;
}

static int finish_dense_stage(hb_ctx* c) {
  c->epoch = DataView();
  c->epoch.x = c->ex;
  c->epoch.x_lo = c->ex_lo;
  if (c->ex_lo) {
    // every staged value exact in TF32 (lo twin all zero, e.g. binary inputs):
    // the layer-0 GEMMs then skip the lo tile and its MMA
    int* d_flag = nullptr;
    HB_CUDA(cudaMalloc(&d_flag, sizeof(int)));
    HB_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int), c->stream));
    const long long n = c->e_rows * c->d[0];
    any_nonzero_kernel<<<static_cast<int>(std::min<long long>(cdiv(n, 256), 148 * 8)), 256, 0, c->stream>>>(
        c->ex_lo, c->e_rows, c->d[0], c->ld[0], d_flag);
    int h = 1;
    const cudaError_t e1 = cudaGetLastError();
    const cudaError_t e2 = cudaMemcpyAsync(&h, d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
    const cudaError_t e3 = cudaStreamSynchronize(c->stream);
    cudaFree(d_flag);
    HB_CUDA(e1);
    HB_CUDA(e2);
    HB_CUDA(e3);
    c->epoch.x_lo_zero = (h == 0) && !(getenv("HB_NO_EXACT_X") && getenv("HB_NO_EXACT_X")[0] == '1');
  }
  c->epoch.ldx = c->ld[0];
  c->epoch.n_rows = c->e_rows;
  c->epoch.labels = c->elabels;
  HB_TRY(build_data_maps(c, c->epoch));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  c->staged = true;
  return HB_OK;
}

int hb_stage_dense_f64(hb_ctx* c, const double* x, int64_t n_rows, int64_t ld, const int64_t* labels) {
  HB_TRY(ctx_check(c));
  if (!x || ld < c->d[0]) return fail(HB_EINVAL, "null features or ld < %d", c->d[0]);
  HB_TRY(stage_dense_common(c, n_rows, labels));
  // chunked H2D of float64 rows through the f64 staging buffer, converted on device
  const long long chunk = std::max<long long>(1, static_cast<long long>(c->stage64_n) / ld);
  for (long long r0 = 0; r0 < n_rows; r0 += chunk) {
    const long long nr = std::min<long long>(chunk, n_rows - r0);
    HB_CUDA(h2d_copy(c->stage64, x + r0 * ld, nr * ld * sizeof(double), c->stream));
    const long long n = nr * c->d[0];
    f64_to_f32_kernel<false><<<static_cast<int>(std::min<long long>((n + 255) / 256, 4096)), 256, 0, c->stream>>>(
        c->ex + r0 * c->ld[0], c->ld[0], c->stage64, ld, static_cast<int>(nr), c->d[0],
        c->ex_lo ? c->ex_lo + r0 * c->ld[0] : nullptr);
    HB_CUDA(cudaGetLastError());
    HB_CUDA(cudaStreamSynchronize(c->stream));
  }
  return finish_dense_stage(c);
}

int hb_stage_dense_f32(hb_ctx* c, const float* x, int64_t n_rows, int64_t ld, const int64_t* labels) {
  HB_TRY(ctx_check(c));
  if (!x || ld < c->d[0]) return fail(HB_EINVAL, "null features or ld < %d", c->d[0]);
  HB_TRY(stage_dense_common(c, n_rows, labels));
  HB_CUDA(cudaMemcpy2DAsync(c->ex, c->ld[0] * sizeof(float), x, ld * sizeof(float), c->d[0] * sizeof(float), n_rows,
                            cudaMemcpyHostToDevice, c->stream));
  if (c->ex_lo) {
    split_lo_kernel<<<static_cast<int>(std::min<long long>(cdiv(n_rows * c->d[0], 256), 148 * 16)), 256, 0,
                      c->stream>>>(c->ex, c->ex_lo, c->ld[0], n_rows, c->d[0]);
    HB_CUDA(cudaGetLastError());
  }
  return finish_dense_stage(c);
}

int hb_stage_blobs(hb_ctx* c, int64_t n_rows, int64_t row0, int n_classes, const double* means, uint64_t seed) {
  HB_TRY(ctx_check(c));
  if (!means || n_classes < 2 || n_classes > c->d[c->L] || row0 < 0)
    return fail(HB_EINVAL, "need means, row0 >= 0 and 2 <= n_classes <= %d", c->d[c->L]);
  HB_TRY(stage_dense_common(c, n_rows, nullptr, true));
  const size_t nm = static_cast<size_t>(n_classes) * c->d[0];
  std::vector<float> m32(nm);
  for (size_t i = 0; i < nm; ++i) m32[i] = static_cast<float>(means[i]);
  float* d_means = nullptr;
  HB_CUDA(cudaMalloc(&d_means, nm * sizeof(float)));
  cudaError_t e = cudaMemcpyAsync(d_means, m32.data(), nm * sizeof(float), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) {
    blobs_kernel<<<static_cast<int>(std::min<long long>(n_rows, 148LL * 64)), 256, 0, c->stream>>>(
        c->ex, c->ex_lo, c->ld[0], row0, n_rows, c->d[0], d_means, n_classes, c->elabels, seed);
    e = cudaGetLastError();
  }
  const cudaError_t e2 = cudaStreamSynchronize(c->stream);
  cudaFree(d_means);
  HB_CUDA(e);
  HB_CUDA(e2);
  return finish_dense_stage(c);
}

int hb_read_staged(hb_ctx* c, int64_t start, int64_t rows, float* x, int64_t* labels) {
  HB_TRY(ctx_check(c));
  if (!c->staged || c->csr_in) return fail(HB_ESTATE, "no dense rows staged");
  if (start < 0 || rows < 0 || start + rows > c->e_rows)
    return fail(HB_EINVAL, "rows [%lld, %lld) outside the %lld staged rows", static_cast<long long>(start),
                static_cast<long long>(start + rows), c->e_rows);
  if (x)
    HB_CUDA(cudaMemcpy2DAsync(x, c->d[0] * sizeof(float), c->ex + start * c->ld[0], c->ld[0] * sizeof(float),
                              c->d[0] * sizeof(float), rows, cudaMemcpyDeviceToHost, c->stream));
  if (labels)
    HB_CUDA(cudaMemcpyAsync(labels, c->elabels + start, rows * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  return HB_OK;
}

// CSR rows -> dense rows (+ lo twin) for densified CSR contexts: a warp per
// row zeroes it, lane 0 adds the entries in CSR order (a repeated column sums,
// as the CSR kernels do), then the lanes write the lo twin of the touched
// entries.  rowptr may start at any offset (a batch of a staged epoch).
__global__ void densify_csr_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                   const float* __restrict__ val, long long rows, long long ld, float* __restrict__ x,
                                   float* __restrict__ x_lo) {
  const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (long long r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    float4* xr = reinterpret_cast<float4*>(x + r * ld);
    float4* lr = x_lo ? reinterpret_cast<float4*>(x_lo + r * ld) : nullptr;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (long long j = lane; j < ld / 4; j += 32) {
      xr[j] = z;
      if (lr) lr[j] = z;
    }
    __syncwarp();
    const long long e0 = rowptr[r], e1 = rowptr[r + 1];
    if (lane == 0)
      for (long long e = e0; e < e1; ++e) x[r * ld + col[e]] += val[e];
    __syncwarp();
    if (x_lo)
      for (long long e = e0 + lane; e < e1; e += 32) x_lo[r * ld + col[e]] = tf32_lo(x[r * ld + col[e]]);
  }
}

static int densify_launch(hb_ctx* c, const int64_t* rowptr, const int32_t* col, const float* val, long long rows,
                          float* x, float* x_lo) {
  const int grid = static_cast<int>(std::min<long long>(cdiv(rows, 8), 148 * 16));
  densify_csr_kernel<<<grid, 256, 0, c->stream>>>(rowptr, col, val, rows, c->ld[0], x, x_lo);
  HB_CUDA(cudaGetLastError());
  return HB_OK;
}

// Densified CSR staging: the CSR arrays go to the device once and are
// scattered into the dense epoch buffers the GEMM path reads.
static int stage_csr_densified(hb_ctx* c, const int64_t* rowptr, const int32_t* col, const float* val,
                               int64_t n_rows, const int64_t* labels) {
  const long long nnz = rowptr[n_rows];
  HB_TRY(free_epoch(c));
  HB_CUDA(cudaMalloc(&c->ex, static_cast<size_t>(n_rows) * c->ld[0] * sizeof(float)));
  if (c->need_lo()) HB_CUDA(cudaMalloc(&c->ex_lo, static_cast<size_t>(n_rows) * c->ld[0] * sizeof(float)));
  if (c->ld[0] > c->d[0]) {
    // zero the pad columns once: no kernel reads them (the tensor maps stop at
    // d[0]), but row copies (hb_permute_epoch) move whole rows
    for (float* x : {c->ex, c->ex_lo}) {
      if (x == nullptr) continue;
      HB_CUDA(cudaMemset2DAsync(x + c->d[0], c->ld[0] * sizeof(float), 0, (c->ld[0] - c->d[0]) * sizeof(float),
                                n_rows, c->stream));
    }
  }
  HB_CUDA(cudaMalloc(&c->elabels, static_cast<size_t>(n_rows) * sizeof(int64_t)));
  HB_CUDA(h2d_copy(c->elabels, labels, n_rows * sizeof(int64_t), c->stream));
  int64_t* d_rowptr = nullptr;
  int32_t* d_col = nullptr;
  float* d_val = nullptr;
  const size_t nz = std::max<long long>(nnz, 1);
  HB_CUDA(cudaMalloc(&d_rowptr, (n_rows + 1) * sizeof(int64_t)));
  HB_CUDA(cudaMalloc(&d_col, nz * sizeof(int32_t)));
  HB_CUDA(cudaMalloc(&d_val, nz * sizeof(float)));
  HB_CUDA(h2d_copy(d_rowptr, rowptr, (n_rows + 1) * sizeof(int64_t), c->stream));
  if (nnz > 0) {
    HB_CUDA(h2d_copy(d_col, col, nnz * sizeof(int32_t), c->stream));
    HB_CUDA(h2d_copy(d_val, val, nnz * sizeof(float), c->stream));
  }
  const int rc = densify_launch(c, d_rowptr, d_col, d_val, n_rows, c->ex, c->ex_lo);
  cudaStreamSynchronize(c->stream);
  cudaFree(d_rowptr);
  cudaFree(d_col);
  cudaFree(d_val);
  if (rc != HB_OK) return rc;
  c->e_rows = n_rows;
  c->e_nnz = nnz;
  c->nnz_per_row = static_cast<double>(nnz) / static_cast<double>(n_rows);
  return finish_dense_stage(c);
}

static int stage_csr_impl(hb_ctx* c, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n_rows,
                          const int64_t* labels);
int hb_stage_csr(hb_ctx* c, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n_rows,
                 const int64_t* labels) {
  HB_TRY(ctx_check(c));
  if (!c->csr_in) return fail(HB_EINVAL, "context was created for dense input");
  if (!rowptr || !labels || n_rows < 1) return fail(HB_EINVAL, "null CSR arrays or n_rows < 1");
  if (rowptr[0] != 0) return fail(HB_EINVAL, "rowptr[0] must be 0");
  const long long nnz = rowptr[n_rows];
  for (long long r = 0; r < n_rows; ++r)
    if (rowptr[r + 1] < rowptr[r]) return fail(HB_EINVAL, "rowptr not non-decreasing at row %lld", r);
  for (long long e = 0; e < nnz; ++e)
    if (col[e] < 0 || col[e] >= c->d[0])
      return fail(HB_EINVAL, "feature index %d outside [0, %d) at nnz %lld", col[e], c->d[0], e);
  return stage_csr_impl(c, rowptr, col, val, n_rows, labels);
}

// Stage a dense float64 (n_rows, d_0) dataset whose rows are mostly zeros --
// what the reference's LIBSVM loader hands a worker (data.py:128-140
// densifies, and BatchRef views that array) -- as CSR on a sparse-input
// context: the nonzeros are gathered on the host threads (values rounded to
// fp32, as every staging path does), so a 20958-wide real-sim epoch stages
// ~0.25% of its 12 GB and layer 0 runs on the CSR kernels.
int hb_stage_dense_as_csr_f64(hb_ctx* c, const double* x, int64_t n_rows, int64_t ld, const int64_t* labels) {
  HB_TRY(ctx_check(c));
  if (!c->csr_in) return fail(HB_EINVAL, "context was created for dense input");
  if (!x || !labels || n_rows < 1 || ld < c->d[0]) return fail(HB_EINVAL, "bad dense array (n_rows %lld, ld %lld)",
                                                               static_cast<long long>(n_rows), static_cast<long long>(ld));
  const int d0 = c->d[0];
  HostPool& pool = HostPool::get();
  const int parts = static_cast<int>(std::min<int64_t>(std::max(1, pool.size()) * 4, std::max<int64_t>(1, n_rows / 64)));
  std::vector<std::vector<int32_t>> pcol(parts);
  std::vector<std::vector<float>> pval(parts);
  std::vector<int64_t> rowlen(n_rows + 1, 0);
  pool.run(parts, [&](int t) {
    const int64_t r0 = n_rows * t / parts, r1 = n_rows * (t + 1) / parts;
    auto& cc = pcol[t];
    auto& vv = pval[t];
    for (int64_t r = r0; r < r1; ++r) {
      const double* row = x + r * ld;
      const size_t before = cc.size();
      for (int j = 0; j < d0; ++j)
        if (row[j] != 0.0) {
          cc.push_back(j);
          vv.push_back(static_cast<float>(row[j]));
        }
      rowlen[r + 1] = static_cast<int64_t>(cc.size() - before);
    }
  });
  for (int64_t r = 0; r < n_rows; ++r) rowlen[r + 1] += rowlen[r];
  std::vector<int32_t> col;
  std::vector<float> val;
  col.reserve(rowlen[n_rows]);
  val.reserve(rowlen[n_rows]);
  for (int t = 0; t < parts; ++t) {
    col.insert(col.end(), pcol[t].begin(), pcol[t].end());
    val.insert(val.end(), pval[t].begin(), pval[t].end());
  }
  return stage_csr_impl(c, rowlen.data(), col.data(), val.data(), n_rows, labels);
}

static int stage_csr_impl(hb_ctx* c, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n_rows,
                          const int64_t* labels) {
  const long long nnz = rowptr[n_rows];
  if (!c->sparse) return stage_csr_densified(c, rowptr, col, val, n_rows, labels);
  HB_TRY(free_epoch(c));
  std::vector<int64_t> colptr;
  std::vector<int32_t> rowidx;
  std::vector<float> cval;
  build_csc(rowptr, col, val, n_rows, c->d[0], colptr, rowidx, cval, 0);
  const size_t nz = std::max<long long>(nnz, 1);
  HB_CUDA(cudaMalloc(&c->erowptr, (n_rows + 1) * sizeof(int64_t)));
  HB_CUDA(cudaMalloc(&c->ecol, nz * sizeof(int32_t)));
  HB_CUDA(cudaMalloc(&c->eval_, nz * sizeof(float)));
  HB_CUDA(cudaMalloc(&c->ecolptr, (c->d[0] + 1) * sizeof(int64_t)));
  HB_CUDA(cudaMalloc(&c->erowidx, nz * sizeof(int32_t)));
  HB_CUDA(cudaMalloc(&c->ecval, nz * sizeof(float)));
  HB_CUDA(cudaMalloc(&c->elabels, n_rows * sizeof(int64_t)));
  HB_CUDA(h2d_copy(c->erowptr, rowptr, (n_rows + 1) * sizeof(int64_t), c->stream, true));
  if (nnz > 0) {
    HB_CUDA(h2d_copy(c->ecol, col, nnz * sizeof(int32_t), c->stream, true));
    HB_CUDA(h2d_copy(c->eval_, val, nnz * sizeof(float), c->stream, true));
    HB_CUDA(h2d_copy(c->erowidx, rowidx.data(), nnz * sizeof(int32_t), c->stream, true));
    HB_CUDA(h2d_copy(c->ecval, cval.data(), nnz * sizeof(float), c->stream, true));
  }
  HB_CUDA(h2d_copy(c->ecolptr, colptr.data(), (c->d[0] + 1) * sizeof(int64_t), c->stream, true));
  HB_CUDA(h2d_copy(c->elabels, labels, n_rows * sizeof(int64_t), c->stream, true));
  c->e_rows = n_rows;
  c->e_nnz = nnz;
  c->nnz_per_row = static_cast<double>(nnz) / static_cast<double>(n_rows);
  c->epoch = DataView();
  c->epoch.rowptr = c->erowptr;
  c->epoch.col = c->ecol;
  c->epoch.val = c->eval_;
  c->epoch.colptr = c->ecolptr;
  c->epoch.rowidx = c->erowidx;
  c->epoch.cval = c->ecval;
  c->epoch.labels = c->elabels;
  c->epoch.n_rows = n_rows;
  c->staged = true;
  return HB_OK;
}

int64_t hb_staged_rows(hb_ctx* c) { return c ? c->e_rows : 0; }

// ------------------------------------------------ on-device epoch reshuffle
// epoch[i] = base[perm[i]] (data.py:187-192 reorder), so a run stages its
// dataset once and every epoch's shuffled copy is a device gather instead of
// a host reorder + H2D.  Row data, labels and the CSC are bit-identical to
// staging the host-reordered copy.
__global__ void gather_rows_kernel(float* __restrict__ dst, const float* __restrict__ src,
                                   const int64_t* __restrict__ perm, long long n, long long ld) {
  const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (long long r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const float4* s4 = reinterpret_cast<const float4*>(src + perm[r] * ld);
    float4* d4 = reinterpret_cast<float4*>(dst + r * ld);
    for (long long j = lane; j < ld / 4; j += 32) d4[j] = s4[j];
  }
}
__global__ void gather_labels_kernel(int64_t* dst, const int64_t* src, const int64_t* perm, int64_t* inv,
                                     long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long p = perm[i];
    dst[i] = src[p];
    if (inv) inv[p] = i;
  }
}
__global__ void perm_rowlen_kernel(const int64_t* rowptr, const int64_t* perm, long long n, int64_t* len) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i <= n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    len[i] = i == 0 ? 0 : rowptr[perm[i - 1] + 1] - rowptr[perm[i - 1]];
}
__global__ void gather_csr_kernel(const int64_t* __restrict__ rowptr_src, const int32_t* __restrict__ col_src,
                                  const float* __restrict__ val_src, const int64_t* __restrict__ perm, long long n,
                                  const int64_t* __restrict__ rowptr_dst, int32_t* __restrict__ col_dst,
                                  float* __restrict__ val_dst) {
  const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (long long r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const long long s0 = rowptr_src[perm[r]], len = rowptr_src[perm[r] + 1] - s0, d0 = rowptr_dst[r];
    for (long long k = lane; k < len; k += 32) {
      col_dst[d0 + k] = col_src[s0 + k];
      val_dst[d0 + k] = val_src[s0 + k];
    }
  }
}
// key = feature * n + new_row over the base CSC; sorting the unique keys gives
// the permuted epoch's CSC in (feature, row) order -- what hb_stage_csr's
// stable counting sort produces for the host-reordered copy.
__global__ void perm_csc_keys_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                                     const int64_t* __restrict__ inv, int n_cols, long long n, uint64_t* keys,
                                     int32_t* idx) {
  const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (long long f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); f < n_cols; f += warps)
    for (long long k = colptr[f] + lane; k < colptr[f + 1]; k += 32) {
      keys[k] = static_cast<uint64_t>(f) * static_cast<uint64_t>(n) + static_cast<uint64_t>(inv[rowidx[k]]);
      idx[k] = static_cast<int32_t>(k);
    }
}
__global__ void perm_csc_gather_kernel(const uint64_t* keys, const int32_t* idx, const float* cval_src, long long nnz,
                                       long long n, int32_t* rowidx, float* cval) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    rowidx[k] = static_cast<int32_t>(keys[k] % static_cast<uint64_t>(n));
    cval[k] = cval_src[idx[k]];
  }
}

static int dup_device(void** dst, const void* src, size_t bytes, cudaStream_t st) {
  HB_CUDA(cudaMalloc(dst, std::max<size_t>(bytes, 1)));
  if (bytes) HB_CUDA(cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyDeviceToDevice, st));
  return HB_OK;
}

int hb_permute_epoch(hb_ctx* c, const int64_t* perm, int64_t n) {
  HB_TRY(ctx_check(c));
  if (!c->staged) return fail(HB_ESTATE, "no data staged");
  if (!perm || n != c->e_rows) return fail(HB_EINVAL, "permutation length %lld != staged rows %lld", (long long)n,
                                           c->e_rows);
  {  // a permutation of [0, n): numpy's fancy indexing would raise on anything else
    std::vector<uint8_t> seen(n, 0);
    for (long long i = 0; i < n; ++i) {
      if (perm[i] < 0 || perm[i] >= n) return fail(HB_EINVAL, "index %lld outside [0, %lld)", (long long)perm[i],
                                                   (long long)n);
      if (seen[perm[i]]++) return fail(HB_EINVAL, "index %lld repeated: not a permutation", (long long)perm[i]);
    }
  }
  cudaStream_t st = c->stream;
  const long long nnz = c->e_nnz;
  if (!c->has_base) {
    // the staged buffers become the base; fresh epoch buffers (same shapes)
    // receive base[perm] from now on -- one view_gen bump, then graphs reuse
    c->px = c->ex;
    c->px_lo = c->ex_lo;
    c->plabels = c->elabels;
    c->prowptr = c->erowptr;
    c->pcolptr = c->ecolptr;
    c->pcol = c->ecol;
    c->prowidx = c->erowidx;
    c->pval = c->eval_;
    c->pcval = c->ecval;
    HB_CUDA(cudaMalloc(&c->elabels, n * sizeof(int64_t)));
    HB_CUDA(cudaMalloc(&c->d_perm, n * sizeof(int64_t)));
    if (c->sparse) {
      const size_t nz = std::max<long long>(nnz, 1);
      HB_CUDA(cudaMalloc(&c->erowptr, (n + 1) * sizeof(int64_t)));
      HB_CUDA(cudaMalloc(&c->ecol, nz * sizeof(int32_t)));
      HB_CUDA(cudaMalloc(&c->eval_, nz * sizeof(float)));
      HB_CUDA(cudaMalloc(&c->erowidx, nz * sizeof(int32_t)));
      HB_CUDA(cudaMalloc(&c->ecval, nz * sizeof(float)));
      HB_TRY(dup_device(reinterpret_cast<void**>(&c->ecolptr), c->pcolptr, (c->d[0] + 1) * sizeof(int64_t), st));  // column counts do not move
      HB_CUDA(cudaMalloc(&c->d_inv, n * sizeof(int64_t)));
      HB_CUDA(cudaMalloc(&c->d_rowlen, (n + 1) * sizeof(int64_t)));
      HB_CUDA(cudaMalloc(&c->p_keys, 2 * nz * sizeof(uint64_t)));
      HB_CUDA(cudaMalloc(&c->p_idx, 2 * nz * sizeof(int32_t)));
      if (nnz >= (1ll << 31)) return fail(HB_EINVAL, "nnz %lld too large for the device CSC sort", nnz);
      size_t t1 = 0, t2 = 0;
      HB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, c->p_keys, c->p_keys + nz, c->p_idx, c->p_idx + nz,
                                              static_cast<int>(nz), 0, 64, st));
      HB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, t2, c->d_rowlen, c->erowptr, n + 1, st));
      c->p_temp_bytes = std::max(t1, t2);
      HB_CUDA(cudaMalloc(&c->p_temp, c->p_temp_bytes));
    } else {
      const size_t bytes = static_cast<size_t>(n) * c->ld[0] * sizeof(float);
      HB_CUDA(cudaMalloc(&c->ex, bytes));
      if (c->px_lo) HB_CUDA(cudaMalloc(&c->ex_lo, bytes));
    }
    c->has_base = true;
    c->view_gen++;
  }
  HB_CUDA(h2d_copy(c->d_perm, perm, n * sizeof(int64_t), st));
  const int g1 = static_cast<int>(std::min<long long>(cdiv(n, 256), 148 * 8));
  const int gw = static_cast<int>(std::min<long long>(cdiv(n, 8), 148 * 16));  // 8 warps per block
  gather_labels_kernel<<<g1, 256, 0, st>>>(c->elabels, c->plabels, c->d_perm, c->sparse ? c->d_inv : nullptr, n);
  HB_CUDA(cudaGetLastError());
  if (c->sparse) {
    perm_rowlen_kernel<<<static_cast<int>(std::min<long long>(cdiv(n + 1, 256), 148 * 8)), 256, 0, st>>>(
        c->prowptr, c->d_perm, n, c->d_rowlen);
    size_t tb = c->p_temp_bytes;
    HB_CUDA(cub::DeviceScan::InclusiveSum(c->p_temp, tb, c->d_rowlen, c->erowptr, n + 1, st));
    gather_csr_kernel<<<gw, 256, 0, st>>>(c->prowptr, c->pcol, c->pval, c->d_perm, n, c->erowptr, c->ecol, c->eval_);
    HB_CUDA(cudaGetLastError());
    if (nnz > 0) {
      const size_t nz = std::max<long long>(nnz, 1);
      perm_csc_keys_kernel<<<static_cast<int>(std::min<long long>(cdiv(c->d[0], 8), 148 * 16)), 256, 0, st>>>(
          c->pcolptr, c->prowidx, c->d_inv, c->d[0], n, c->p_keys, c->p_idx);
      HB_CUDA(cudaGetLastError());
      int end_bit = 1;
      while (end_bit < 64 && (static_cast<double>(1ull << end_bit) < static_cast<double>(c->d[0]) * n)) ++end_bit;
      tb = c->p_temp_bytes;
      HB_CUDA(cub::DeviceRadixSort::SortPairs(c->p_temp, tb, c->p_keys, c->p_keys + nz, c->p_idx, c->p_idx + nz,
                                              static_cast<int>(nnz), 0, end_bit, st));
      perm_csc_gather_kernel<<<static_cast<int>(std::min<long long>(cdiv(nnz, 256), 148 * 8)), 256, 0, st>>>(
          c->p_keys + nz, c->p_idx + nz, c->pcval, nnz, n, c->erowidx, c->ecval);
      HB_CUDA(cudaGetLastError());
    }
    c->epoch.rowptr = c->erowptr;
    c->epoch.col = c->ecol;
    c->epoch.val = c->eval_;
    c->epoch.colptr = c->ecolptr;
    c->epoch.rowidx = c->erowidx;
    c->epoch.cval = c->ecval;
    c->epoch.labels = c->elabels;
  } else {
    gather_rows_kernel<<<gw, 256, 0, st>>>(c->ex, c->px, c->d_perm, n, c->ld[0]);
    if (c->ex_lo) gather_rows_kernel<<<gw, 256, 0, st>>>(c->ex_lo, c->px_lo, c->d_perm, n, c->ld[0]);
    HB_CUDA(cudaGetLastError());
    if (c->epoch.x != c->ex) {
      c->epoch.x = c->ex;
      c->epoch.x_lo = c->ex_lo;
      c->epoch.labels = c->elabels;
      HB_TRY(build_data_maps(c, c->epoch));
    }
  }
  HB_CUDA(cudaStreamSynchronize(st));
  return HB_OK;
}

// range checks as branch-free min/max reductions (vectorised), then a scan
// for the offending value only on failure
// range checks as branch-free unsigned compares OR-reduced (no loop-carried
// min/max chain, so the compiler vectorises them); the slow scan only runs to
// name the offending entry
static int check_labels(const int64_t* y, long long n, int nc) {
  uint64_t bad = 0;
  for (long long i = 0; i < n; ++i) bad |= static_cast<uint64_t>(y[i]) >= static_cast<uint64_t>(nc);
  if (!bad) return HB_OK;
  for (long long i = 0; i < n; ++i)
    if (y[i] < 0 || y[i] >= nc) return fail(HB_EINVAL, "labels must lie in [0, %d), got %lld", nc, (long long)y[i]);
  return HB_OK;
}
static int check_cols(const int32_t* col, long long nnz, int d) {
  // (split over the merge pool: a batch's column ids come straight from DRAM)
  HostPool& pool = HostPool::get();
  const int parts = static_cast<int>(std::min<long long>(pool.size(), std::max<long long>(1, nnz / (1 << 14))));
  std::atomic<uint32_t> any{0};
  pool.run(parts, [&](int t) {
    const long long a = nnz * t / parts, b = nnz * (t + 1) / parts;
    uint32_t bad = 0;
    for (long long e = a; e < b; ++e) bad |= static_cast<uint32_t>(col[e]) >= static_cast<uint32_t>(d);
    if (bad) any.store(1, std::memory_order_relaxed);
  });
  if (!any.load()) return HB_OK;
  for (long long e = 0; e < nnz; ++e)
    if (col[e] < 0 || col[e] >= d) return fail(HB_EINVAL, "feature index %d outside [0, %d)", col[e], d);
  return HB_OK;
}

int hb_train_step(hb_ctx* c, int64_t start, int rows, double eta, uint32_t flags, double* out_loss) {
  HB_TRY(ctx_check(c));
  if (!c->staged) return fail(HB_ESTATE, "no data staged");
  if (start < 0 || rows < 1 || start + rows > c->e_rows)
    return fail(HB_EINVAL, "batch range [%lld, %lld) out of bounds for %lld rows", (long long)start,
                (long long)(start + rows), (long long)c->e_rows);
  return do_step(c, c->epoch, start, rows, eta, flags, out_loss);
}

int hb_train_step_host_dense(hb_ctx* c, const float* x, int64_t ld, const int64_t* labels, int rows, double eta,
                             uint32_t flags, double* out_loss) {
  HB_TRY(ctx_check(c));
  if (c->csr_in) return fail(HB_EINVAL, "context was created for sparse (CSR) input");
  if (!x || !labels || ld < c->d[0]) return fail(HB_EINVAL, "null batch or ld < %d", c->d[0]);
  if (rows < 1 || rows > c->max_batch) return fail(HB_EINVAL, "rows=%d outside [1, %d]", rows, c->max_batch);
  HB_TRY(check_labels(labels, rows, c->d[c->L]));
  const int d0 = c->d[0];
  const long long n = static_cast<long long>(rows) * d0;
  const int blocks = static_cast<int>(std::min<long long>(cdiv(n, 256), 148 * 16));
  // small batches in registered (mapped) host memory: read by the SMs directly
  static const long long zc_max = env_long("HB_ZC_BATCH_MAX", 4 << 20);
  const float* zx = n * 4 <= zc_max ? static_cast<const float*>(mapped_alias(x, ((rows - 1) * ld + d0) * sizeof(float)))
                                    : nullptr;
  const int64_t* zl = zx ? static_cast<const int64_t*>(mapped_alias(labels, rows * sizeof(int64_t))) : nullptr;
  if (zx && zl) {
    zc_batch_kernel<<<static_cast<int>(std::min<long long>(cdiv(n, 256), 148 * 8)), 256, 0, c->stream>>>(
        zx, ld, zl, c->bx, c->bx_lo, c->ld[0], c->blabels, rows, d0);
    HB_CUDA(cudaGetLastError());
    c->pre_launches++;
    t_h2d_bytes += n * static_cast<long long>(sizeof(float)) + rows * static_cast<long long>(sizeof(int64_t));
    return do_step(c, c->batch, 0, rows, eta, flags, out_loss);
  }
  if (ld == d0 && c->ld[0] == d0) {
    // contiguous on both sides: one linear DMA (a pitched 2D copy of
    // thousands of short rows runs far below link speed)
    HB_CUDA(h2d_copy(c->bx, x, n * sizeof(float), c->stream));
    if (c->bx_lo) {
      split_lo_kernel<<<blocks, 256, 0, c->stream>>>(c->bx, c->bx_lo, c->ld[0], rows, d0);
      HB_CUDA(cudaGetLastError());
    }
  } else if (ld == d0) {
    // contiguous host rows, padded device rows: linear DMA into a staging
    // slot, then one kernel re-pitches (and splits the lo twin)
    if (!c->bx_stage) HB_CUDA(cudaMalloc(&c->bx_stage, static_cast<size_t>(c->cap) * d0 * sizeof(float)));
    HB_CUDA(h2d_copy(c->bx_stage, x, n * sizeof(float), c->stream));
    repitch_split_kernel<<<blocks, 256, 0, c->stream>>>(c->bx_stage, c->bx, c->bx_lo, c->ld[0], rows, d0);
    HB_CUDA(cudaGetLastError());
  } else {
    HB_CUDA(cudaMemcpy2DAsync(c->bx, c->ld[0] * sizeof(float), x, ld * sizeof(float), d0 * sizeof(float), rows,
                              cudaMemcpyHostToDevice, c->stream));
    t_h2d_bytes += n * static_cast<long long>(sizeof(float));
    if (c->bx_lo) {
      split_lo_kernel<<<blocks, 256, 0, c->stream>>>(c->bx, c->bx_lo, c->ld[0], rows, d0);
      HB_CUDA(cudaGetLastError());
    }
  }
  HB_CUDA(h2d_copy(c->blabels, labels, rows * sizeof(int64_t), c->stream));
  return do_step(c, c->batch, 0, rows, eta, flags, out_loss);
}

int hb_train_step_host_csr(hb_ctx* c, const int64_t* rowptr, const int32_t* col, const float* val,
                           const int64_t* labels, int rows, double eta, uint32_t flags, double* out_loss) {
  HB_TRY(ctx_check(c));
  if (!c->csr_in) return fail(HB_EINVAL, "context was created for dense input");
  if (!rowptr || !labels) return fail(HB_EINVAL, "null batch");
  if (rows < 1 || rows > c->max_batch) return fail(HB_EINVAL, "rows=%d outside [1, %d]", rows, c->max_batch);
  if (rowptr[0] != 0) return fail(HB_EINVAL, "rowptr[0] must be 0");
  xmark("host csr: enter");
  HB_TRY(check_labels(labels, rows, c->d[c->L]));
  const long long nnz = rowptr[rows];
  HB_TRY(check_cols(col, nnz, c->d[0]));
  xmark("host csr: checked");
  if (nnz > c->b_nnz_cap) {
    cudaFree(c->bcol);
    cudaFree(c->bval);
    cudaFree(c->browidx);
    cudaFree(c->bcval);
    const long long cap = std::max<long long>(nnz, 1) * 3 / 2 + 64;
    HB_CUDA(cudaMalloc(&c->bcol, cap * sizeof(int32_t)));
    HB_CUDA(cudaMalloc(&c->bval, cap * sizeof(float)));
    HB_CUDA(cudaMalloc(&c->browidx, cap * sizeof(int32_t)));
    HB_CUDA(cudaMalloc(&c->bcval, cap * sizeof(float)));
    c->b_nnz_cap = cap;
    c->view_gen++;
  }
  c->nnz_per_row = static_cast<double>(nnz) / rows;
  // one pinned buffer carries the batch: [rowptr | labels | col | val] for the
  // forward, then [colptr | rowidx | cval] (the batch CSC for the sparse dW),
  // which is built on the host while the device runs the forward phase.
  const size_t b_rowptr = (rows + 1) * sizeof(int64_t), b_colptr = (c->d[0] + 1) * sizeof(int64_t),
               b_lab = rows * sizeof(int64_t), b_i32 = nnz * sizeof(int32_t), b_f32 = nnz * sizeof(float);
  HB_TRY(ensure_pinned(c, b_rowptr + b_colptr + b_lab + 2 * b_i32 + 2 * b_f32 + 64));
  char* p = static_cast<char*>(c->pinned);
  char* p_lab = p + b_rowptr;
  char* p_col = p_lab + b_lab;
  char* p_val = p_col + b_i32;
  char* p_colptr = p_val + b_f32;
  char* p_rowidx = p_colptr + b_colptr;
  char* p_cval = p_rowidx + b_i32;
  cudaStream_t st = c->stream;
  if (nnz > 0 && is_pinned(rowptr) && is_pinned(labels) && is_pinned(col) && is_pinned(val)) {
    // page-locked batch: DMA straight from the caller's arrays
    HB_CUDA(h2d_copy(c->browptr, rowptr, b_rowptr, st));
    HB_CUDA(h2d_copy(c->blabels, labels, b_lab, st));
    HB_CUDA(h2d_copy(c->bcol, col, b_i32, st));
    HB_CUDA(h2d_copy(c->bval, val, b_f32, st));
  } else {
    std::memcpy(p, rowptr, b_rowptr);
    std::memcpy(p_lab, labels, b_lab);
    std::memcpy(p_col, col, b_i32);
    std::memcpy(p_val, val, b_f32);
    HB_CUDA(h2d_copy(c->browptr, p, b_rowptr, st));
    HB_CUDA(h2d_copy(c->blabels, p_lab, b_lab, st));
    if (nnz > 0) {
      HB_CUDA(h2d_copy(c->bcol, p_col, b_i32, st));
      HB_CUDA(h2d_copy(c->bval, p_val, b_f32, st));
    }
  }
  if (!c->sparse) {
    // densified context: scatter the batch into the dense slot, then the GEMM path
    xmark("host csr: copies enqueued");
    HB_TRY(densify_launch(c, c->browptr, c->bcol, c->bval, rows, c->bx, c->bx_lo));
    xmark("host csr: densify enqueued");
    c->pre_launches = 1;
    return do_step(c, c->batch, 0, rows, eta, flags, out_loss);
  }
  const bool dev_csc = static_cast<double>(c->d[0]) * rows < 4294967295.0;
  if (dev_csc) {
    // batch CSC built on the device (stable by row, identical to the host sort)
    if (c->csc_cap < nnz + 1 || c->csc_temp == nullptr) {
      cudaFree(c->csc_keys);
      cudaFree(c->csc_idx);
      cudaFree(c->csc_temp);
      cudaFree(c->csc_counts);
      c->csc_cap = std::max<long long>(c->b_nnz_cap, nnz + 1);
      HB_CUDA(cudaMalloc(&c->csc_keys, 2 * c->csc_cap * sizeof(uint32_t)));
      HB_CUDA(cudaMalloc(&c->csc_idx, 2 * c->csc_cap * sizeof(int32_t)));
      HB_CUDA(cudaMalloc(&c->csc_counts, 2 * (c->d[0] + 2) * sizeof(int)));
      size_t t1 = 0, t2 = 0;
      HB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, c->csc_keys, c->csc_keys + c->csc_cap, c->csc_idx,
                                              c->csc_idx + c->csc_cap, static_cast<int>(c->csc_cap), 0, 32, st));
      HB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, t2, c->csc_counts, c->csc_counts + c->d[0] + 2, c->d[0] + 1, st));
      c->csc_temp_bytes = std::max(t1, t2);
      HB_CUDA(cudaMalloc(&c->csc_temp, c->csc_temp_bytes));
    }
    int* cnt = c->csc_counts;
    int* cnt_scan = c->csc_counts + c->d[0] + 2;
    HB_CUDA(cudaMemsetAsync(cnt, 0, (c->d[0] + 1) * sizeof(int), st));
    if (nnz > 0) {
      csc_keys_kernel<<<cdiv(rows, 8), 256, 0, st>>>(c->browptr, c->bcol, rows, c->csc_keys, c->csc_idx, cnt);
      HB_CUDA(cudaGetLastError());
    }
    size_t tb = c->csc_temp_bytes;
    HB_CUDA(cub::DeviceScan::InclusiveSum(c->csc_temp, tb, cnt, cnt_scan, c->d[0] + 1, st));
    counts_to_colptr_kernel<<<cdiv(c->d[0] + 1, 256), 256, 0, st>>>(cnt_scan, c->bcolptr, c->d[0]);
    HB_CUDA(cudaGetLastError());
    if (nnz > 0) {
      int end_bit = 1;
      while (end_bit < 32 && (static_cast<double>(1ull << end_bit) < static_cast<double>(c->d[0]) * rows)) ++end_bit;
      tb = c->csc_temp_bytes;
      HB_CUDA(cub::DeviceRadixSort::SortPairs(c->csc_temp, tb, c->csc_keys, c->csc_keys + c->csc_cap, c->csc_idx,
                                              c->csc_idx + c->csc_cap, static_cast<int>(nnz), 0, end_bit, st));
      csc_gather_kernel<<<static_cast<int>(std::min<long long>(cdiv(nnz, 256), 148 * 8)), 256, 0, st>>>(
          c->csc_keys + c->csc_cap, c->csc_idx + c->csc_cap, c->bval, nnz, rows, c->browidx, c->bcval);
      HB_CUDA(cudaGetLastError());
    }
    c->pre_launches = 3;  // keys, colptr, gather (the scan / radix sort are CUB)
  }
  auto csc_phase = [&]() -> int {
    if (dev_csc) return HB_OK;
    build_csc_into(rowptr, col, val, rows, c->d[0], reinterpret_cast<int64_t*>(p_colptr),
                   reinterpret_cast<int32_t*>(p_rowidx), reinterpret_cast<float*>(p_cval), c->h_colptr);
    HB_CUDA(h2d_copy(c->bcolptr, p_colptr, b_colptr, st));
    if (nnz > 0) {
      HB_CUDA(h2d_copy(c->browidx, p_rowidx, b_i32, st));
      HB_CUDA(h2d_copy(c->bcval, p_cval, b_f32, st));
    }
    return HB_OK;
  };
  DataView v;
  v.rowptr = c->browptr;
  v.col = c->bcol;
  v.val = c->bval;
  v.colptr = c->bcolptr;
  v.rowidx = c->browidx;
  v.cval = c->bcval;
  v.labels = c->blabels;
  v.n_rows = rows;
  if (dev_csc) return do_step(c, v, 0, rows, eta, flags, out_loss, true);
  return do_step(c, v, 0, rows, eta, flags, out_loss, true, csc_phase);
}

int hb_forward(hb_ctx* c, int64_t start, int rows) {
  HB_TRY(ctx_check(c));
  if (!c->staged) return fail(HB_ESTATE, "no data staged");
  if (start < 0 || rows < 1 || rows > c->max_batch || start + rows > c->e_rows)
    return fail(HB_EINVAL, "batch range out of bounds");
  c->last_launches = 0;
  HB_TRY(run_forward(c, c->epoch, start, rows, false, 0, 0.0, nullptr));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  return HB_OK;
}

int hb_get_activation_f32(hb_ctx* c, int layer, int rows, float* out) {
  HB_TRY(ctx_check(c));
  if (layer < 1 || layer >= c->L || !out || rows < 1 || rows > c->cap)
    return fail(HB_EINVAL, "activation layer must be in [1, %d)", c->L);
  HB_CUDA(cudaMemcpy2DAsync(out, c->d[layer] * sizeof(float), c->A[layer], c->ld[layer] * sizeof(float),
                            c->d[layer] * sizeof(float), rows, cudaMemcpyDeviceToHost, c->stream));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  return HB_OK;
}

int hb_eval_loss_sum(hb_ctx* c, int64_t start, int64_t rows, double* out_sum) {
  HB_TRY(ctx_check(c));
  if (!out_sum) return fail(HB_EINVAL, "null output");
  if (!c->staged) return fail(HB_ESTATE, "no data staged");
  if (start < 0 || rows < 1 || start + rows > c->e_rows) return fail(HB_EINVAL, "eval range out of bounds");
  double total = 0.0;
  for (long long s = start; s < start + rows; s += c->max_batch) {
    const int n = static_cast<int>(std::min<long long>(c->max_batch, start + rows - s));
    HB_TRY(run_forward(c, c->epoch, s, n, false, 0, 0.0, nullptr));
    double part = 0.0;
    HB_CUDA(cudaMemcpyAsync(&part, c->d_loss, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    HB_CUDA(cudaStreamSynchronize(c->stream));
    total += part;
  }
  *out_sum = total;
  return HB_OK;
}

int hb_last_step_ms(hb_ctx* c, float* ms) {
  if (!c || !ms) return fail(HB_EINVAL, "null argument");
  *ms = c->last_ms;
  return HB_OK;
}

int hb_last_step_launches(hb_ctx* c, int* n) {
  if (!c || !n) return fail(HB_EINVAL, "null argument");
  *n = c->last_launches;
  return HB_OK;
}

int hb_last_xfer_bytes(hb_ctx* c, int64_t* h2d, int64_t* d2h) {
  if (!c || !h2d || !d2h) return fail(HB_EINVAL, "null argument");
  *h2d = c->last_h2d;
  *d2h = c->last_d2h;
  return HB_OK;
}

int hb_profile_enable(hb_ctx* c, int on) {
  HB_TRY(ctx_check(c));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  c->prof_on = on != 0;
  c->ev_used = 0;
  c->step_marks.clear();
  c->prof_acc.clear();
  return HB_OK;
}

int hb_profile_filter(hb_ctx* c, const char* name) {
  HB_TRY(ctx_check(c));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  const std::string f = name ? name : "";
  if (f != c->prof_filter) {
    drop_graphs(c);  // captured graphs baked the old instrumentation
    c->prof_filter = f;
  }
  return HB_OK;
}

int hb_profile_read(hb_ctx* c, int max_entries, char* names, double* total_ms, int* counts, int* n_out) {
  HB_TRY(ctx_check(c));
  if (!n_out) return fail(HB_EINVAL, "null n_out");
  HB_CUDA(cudaStreamSynchronize(c->stream));
  int i = 0;
  for (auto& kv : c->prof_acc) {
    if (i >= max_entries) break;
    if (names) {
      std::memset(names + 64 * i, 0, 64);
      std::strncpy(names + 64 * i, kv.first.c_str(), 63);
    }
    if (total_ms) total_ms[i] = kv.second.first;
    if (counts) counts[i] = kv.second.second;
    ++i;
  }
  *n_out = i;
  c->prof_acc.clear();
  return HB_OK;
}

#ifdef HB_TRACE
// debug builds only: copy the pipeline timeline of the last traced GEMM
extern "C" int hb_trace_read(unsigned long long* out, int n) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, hb::hb_trace_buf, sizeof(unsigned long long) * std::min(n, 4096));
  cudaMemset(reinterpret_cast<void*>(0), 0, 0);
  unsigned long long zeros[4096] = {0};
  cudaMemcpyToSymbol(hb::hb_trace_buf, zeros, sizeof zeros);
  return HB_OK;
}
// per-CTA stamps of the last 8 GEMM launches ([slot][cta][4]); resets the launch counter
extern "C" int hb_trace_cta_read(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, hb::hb_trace_cta, sizeof(unsigned long long) * 8 * 1024 * 4);
  std::vector<unsigned long long> zeros(8 * 1024 * 4, 0);
  cudaMemcpyToSymbol(hb::hb_trace_cta, zeros.data(), zeros.size() * sizeof(unsigned long long));
  g_trace_launch_no = 0;
  return HB_OK;
}
#endif

int hb_synchronize(hb_ctx* c) {
  HB_TRY(ctx_check(c));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  return land_wait(c);
}

int hb_replica_landed(hb_ctx* c) {
  HB_TRY(ctx_check(c));
  if (c->pend_active) return fail(HB_ESTATE, "a replica step is in flight (hb_replica_end first)");
  return land_wait(c);
}

int hb_nccl_unique_id(void* out) {
  if (!out) return fail(HB_EINVAL, "null output");
  HB_TRY(load_nccl());
  nccl_uid_t id;
  int r = g_nccl.getUniqueId(&id);
  if (r != 0) return fail(HB_ENCCL, "ncclGetUniqueId: %s", g_nccl.errStr ? g_nccl.errStr(r) : "error");
  std::memcpy(out, &id, sizeof id);
  return HB_OK;
}

int hb_comm_init(hb_ctx* c, const void* id_bytes, int nranks, int rank) {
  HB_TRY(ctx_check(c));
  if (!id_bytes || nranks < 1 || rank < 0 || rank >= nranks) return fail(HB_EINVAL, "bad communicator arguments");
  HB_TRY(load_nccl());
  nccl_uid_t id;
  std::memcpy(&id, id_bytes, sizeof id);
  nccl_comm_t comm = nullptr;
  int r = g_nccl.commInitRank(&comm, nranks, id, rank);
  if (r != 0) return fail(HB_ENCCL, "ncclCommInitRank: %s", g_nccl.errStr ? g_nccl.errStr(r) : "error");
  c->comm = comm;
  c->nranks = nranks;
  ensure_flat_layout(c);
  if (!c->flat) HB_CUDA(cudaMalloc(&c->flat, c->flat_n * sizeof(float)));
  return HB_OK;
}

int hb_merge_allreduce(hb_ctx* c) {
  HB_TRY(ctx_check(c));
  HB_TRY(enqueue_merge(c));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  return peer_check(c);
}

int hb_host_pool_selftest(int jobs, int64_t* out_errors) {
  if (jobs < 1 || !out_errors) return fail(HB_EINVAL, "need jobs >= 1 and an output");
  HostPool& pool = HostPool::get();
  long long errors = 0;
  std::vector<std::atomic<int>> hits(64);
  for (int j = 0; j < jobs; ++j) {
    // part counts that grow and shrink from job to job: a stale ticket of the
    // previous job would run a part of this one twice (or with the wrong job)
    const int n = 1 + (j * 7919) % 61;
    for (auto& h : hits) h.store(0, std::memory_order_relaxed);
    const int tag = j;
    std::atomic<int> wrong{0};
    pool.run(n, [&, tag](int i) {
      if (tag != j) wrong.fetch_add(1);
      hits[i].fetch_add(1, std::memory_order_relaxed);
    });
    for (int i = 0; i < 64; ++i) errors += (hits[i].load() != (i < n ? 1 : 0)) ? 1 : 0;
    errors += wrong.load();
  }
  *out_errors = errors;
  return HB_OK;
}

int hb_host_merge_threads(int threads, int spin) {
  if (threads < 1 || spin < 0) return fail(HB_EINVAL, "need threads >= 1 and spin >= 0");
  HostPool::get().configure(threads, spin);
  return HB_OK;
}

int hb_probe_l2_gather(int device, int64_t rows, int cols, int per_warp, int unroll, double* out_gbps) {
  if (!out_gbps || rows < 1 || cols < 128 || cols > 1024 || cols % 128 != 0 || per_warp < 1)
    return fail(HB_EINVAL, "probe needs rows >= 1, cols a multiple of 128 up to 1024, per_warp >= 1");
  HB_CUDA(cudaSetDevice(device));
  float* m = nullptr;
  float* out = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = HB_OK;
  auto run = [&](int reps, float* ms) -> cudaError_t {
    const int sms = 148, warps = sms * 64;  // 8 blocks of 8 warps per SM
    const int grid = warps * 32 / 256;
    per_warp -= per_warp % std::max(1, unroll);
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; ++r) {
      if (unroll >= 4)
        l2_gather_probe_kernel<4><<<grid, 256, 0, st>>>(m, rows, cols, per_warp, out);
      else if (unroll == 2)
        l2_gather_probe_kernel<2><<<grid, 256, 0, st>>>(m, rows, cols, per_warp, out);
      else
        l2_gather_probe_kernel<1><<<grid, 256, 0, st>>>(m, rows, cols, per_warp, out);
    }
    cudaEventRecord(e1, st);
    cudaError_t e = cudaEventSynchronize(e1);
    if (e == cudaSuccess) e = cudaEventElapsedTime(ms, e0, e1);
    return e;
  };
  do {
    if (cudaMalloc(&m, static_cast<size_t>(rows) * cols * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&out, 148 * 64 * sizeof(float)) != cudaSuccess || cudaStreamCreate(&st) != cudaSuccess ||
        cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
      rc = fail(HB_ECUDA, "probe allocation failed");
      break;
    }
    cudaMemsetAsync(m, 0, static_cast<size_t>(rows) * cols * sizeof(float), st);
    float ms = 0.f;
    if (run(3, &ms) != cudaSuccess || run(10, &ms) != cudaSuccess) {  // warm (L2-resident), then timed
      rc = fail(HB_ECUDA, "probe kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
    const double bytes = 10.0 * 148 * 64 * static_cast<double>(per_warp) * cols * sizeof(float);
    *out_gbps = bytes / (ms * 1e-3) / 1e9;
  } while (false);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  cudaFree(m);
  cudaFree(out);
  return rc;
}

struct PeerHandle {  // HB_PEER_HANDLE_BYTES on the wire
  cudaIpcMemHandle_t ipc;
  int64_t pid;
  int64_t device;
  uint64_t ptr;
  int64_t n_params;
};
static_assert(sizeof(PeerHandle) <= HB_PEER_HANDLE_BYTES, "peer handle too large");

int hb_peer_handle(hb_ctx* c, void* out) {
  HB_TRY(ctx_check(c));
  if (!out) return fail(HB_EINVAL, "null handle buffer");
  if (!c->xbuf) {
    ensure_flat_layout(c);
    HB_CUDA(cudaMalloc(&c->xbuf, kPeerHeader + c->flat_n * sizeof(float)));
    HB_CUDA(cudaMemsetAsync(c->xbuf, 0, kPeerHeader, c->stream));
    HB_CUDA(cudaStreamSynchronize(c->stream));
  }
  PeerHandle h{};
  HB_CUDA(cudaIpcGetMemHandle(&h.ipc, c->xbuf));
  h.pid = static_cast<int64_t>(getpid());
  h.device = c->device;
  h.ptr = reinterpret_cast<uint64_t>(c->xbuf);
  h.n_params = static_cast<int64_t>(c->n_params);
  std::memset(out, 0, HB_PEER_HANDLE_BYTES);
  std::memcpy(out, &h, sizeof h);
  return HB_OK;
}

int hb_peer_attach(hb_ctx* c, int nranks, int rank, const void* handles) {
  HB_TRY(ctx_check(c));
  if (!handles || nranks < 1 || nranks > kMaxPeers || rank < 0 || rank >= nranks)
    return fail(HB_EINVAL, "bad peer group (nranks %d, rank %d; at most %d ranks)", nranks, rank, kMaxPeers);
  if (c->peers.n != 0) return fail(HB_ESTATE, "context already attached to a peer group");
  if (!c->xbuf) return fail(HB_ESTATE, "hb_peer_handle first");
  PeerTable t{};
  t.n = nranks;
  t.rank = rank;
  int local_peers = 0;
  const char* hs = static_cast<const char*>(handles);
  for (int q = 0; q < nranks; ++q) {
    PeerHandle h;
    std::memcpy(&h, hs + static_cast<size_t>(q) * HB_PEER_HANDLE_BYTES, sizeof h);
    if (h.n_params != static_cast<int64_t>(c->n_params))
      return fail(HB_EINVAL, "rank %d holds a model of %lld parameters, this one %zu", q,
                  static_cast<long long>(h.n_params), c->n_params);
    char* base = nullptr;
    if (q == rank) {
      if (h.ptr != reinterpret_cast<uint64_t>(c->xbuf)) return fail(HB_EINVAL, "handle %d is not this context's", q);
      base = c->xbuf;
    } else if (h.pid == static_cast<int64_t>(getpid())) {
      ++local_peers;
      if (h.device != c->device) {  // same process, another GPU: direct peer access over NVLink
        int ok = 0;
        HB_CUDA(cudaDeviceCanAccessPeer(&ok, c->device, static_cast<int>(h.device)));
        if (!ok) return fail(HB_ECUDA, "device %d cannot access device %lld", c->device, static_cast<long long>(h.device));
        cudaError_t e = cudaDeviceEnablePeerAccess(static_cast<int>(h.device), 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else HB_CUDA(e);
      }
      base = reinterpret_cast<char*>(h.ptr);
    } else {
      void* p = nullptr;
      HB_CUDA(cudaIpcOpenMemHandle(&p, h.ipc, cudaIpcMemLazyEnablePeerAccess));
      c->ipc_opened.push_back(p);
      base = static_cast<char*>(p);
    }
    t.flat[q] = reinterpret_cast<float*>(base + kPeerHeader);
    t.flag[q] = reinterpret_cast<unsigned long long*>(base);
  }
  if (local_peers == nranks - 1 && nranks > 1) {
    // every rank is in this process: join (or create) the group's ordering
    // state, keyed by rank 0's exchange buffer
    static std::mutex groups_mu;
    static std::map<uint64_t, std::weak_ptr<LocalGroup>> groups;
    PeerHandle h0;
    std::memcpy(&h0, hs, sizeof h0);
    std::lock_guard<std::mutex> lk(groups_mu);
    std::shared_ptr<LocalGroup> g = groups[h0.ptr].lock();
    if (!g) {
      g = std::make_shared<LocalGroup>();
      g->n = nranks;
      g->ev_pack.assign(nranks, nullptr);
      g->ev_red.assign(nranks, nullptr);
      groups[h0.ptr] = g;
    }
    HB_CUDA(cudaEventCreateWithFlags(&g->ev_pack[rank], cudaEventDisableTiming));
    HB_CUDA(cudaEventCreateWithFlags(&g->ev_red[rank], cudaEventDisableTiming));
    c->local = g;
  } else if (local_peers != 0) {
    return fail(HB_EINVAL, "a peer group is either all in this process or one rank per process");
  }
  c->peers = t;
  c->nranks = nranks;
  return HB_OK;
}

int hb_comm_destroy(hb_ctx* c) {
  if (!c || !c->comm) return HB_OK;
  if (g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
  c->comm = nullptr;
  return HB_OK;
}

}  // extern "C"
