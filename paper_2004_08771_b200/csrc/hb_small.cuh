// hb_small.cuh -- the whole replica step of a small net as ONE persistent kernel.
//
// Covtype-class steps (54-512-512-512-2 at b = 512, BASELINE configs[0]) are
// launch-latency bound on the per-layer tcgen05 path: ~13 dependent kernels of
// 10-18 us each for 1.7 GFLOP.  Here one cooperative launch (two CTAs per SM,
// all co-resident) walks the step's phases with a grid barrier between them:
//
//   F_h   A_{h+1} = sigmoid(A_h . W_h^T (+ b_h))           h = 0 .. L-2   (nn.py:108-121)
//   H     logits, softmax, CE, delta_out = (P - Y)/n         (nn.py:124-164)
//         delta_{L-2} = (delta_out . W_{L-1}) * A(1 - A)
//   B_h   delta_{h-1} = (delta_h . W_h) * A_h(1 - A_h)       (nn.py:170)
//         beside dW_{h+1} = delta_{h+1}^T A_{h+1}, W_{h+1} -= eta dW  (nn.py:168, 174-179)
//   last  dW_0 = delta_0^T X, W_0 -= eta dW_0; the batch loss sum
//
// W_{h+1} is updated in the phase after its last reader (dX of B_{h+1}, or
// the head), so every gradient is taken on the snapshot weights as the
// reference does.  The GEMM tiles run on the CUDA cores in fp32 FMA (round to
// nearest, each k-block of 32 products summed into a fresh register before it
// joins the running sum): at these sizes every phase is a one-wave problem fed
// from L2, and IEEE fp32 accumulation is more accurate than the 3xTF32 split.
// The head (logits, softmax, its dW) runs in float64 like head_small_kernel.
// Every sum has a fixed order: the step is deterministic.
#pragma once
#include "hb_kernels.cuh"
#include "hb_ptx.cuh"

namespace hb {

constexpr int kSnMaxL = 8;          // layers
constexpr int kSnMaxRows = 1024;    // batch rows a fused step takes
constexpr int kSnMaxWidth = 1024;   // layer width
constexpr int kSnThreads = 256;
constexpr int kSnBM = 64, kSnBN = 32, kSnBK = 32;
constexpr int kSnStages = 3;
constexpr int kSnLdA = kSnBM + 4;  // [k][m] row stride of an A stage (float4 rows stay aligned)
constexpr int kSnLdB = kSnBN + 2;  // [k][n] row stride of a B stage
constexpr int kSnAS = kSnBK * kSnLdA;
constexpr int kSnBS = kSnBK * kSnLdB;

struct SmallNetArgs {
  int L, rows, train;
  int d[kSnMaxL + 1];
  long long ld[kSnMaxL + 1];  // row stride of a width-d_l activation / error buffer
  const float* x;             // staged input rows (offset by start)
  long long ldx, start;
  const int64_t* labels;      // staged labels (offset by start)
  const DevStep* ds;
  float eta;
  float* W[kSnMaxL];
  float* W_lo[kSnMaxL];       // 3xTF32 lo twins kept current for the tensor-core paths (or null)
  long long ldw[kSnMaxL];
  const float* bias[kSnMaxL];
  float* A[kSnMaxL + 1];      // A[1 .. L-1]
  float* D[kSnMaxL];          // D[0 .. L-2]: error at the output of layer h, (rows, d_{h+1})
  float* G[kSnMaxL];          // raw gradients (EMIT_GRAD) or null
  float* hd;                  // (rows, 4) output error signal
  double* row_loss;           // (rows)
  double* loss_out;           // batch loss sum
  unsigned* bar;              // grid barrier counter, zero at launch
};

// All CTAs are co-resident (cooperative launch); a monotonically growing
// arrival counter, one generation per phase.
__device__ __forceinline__ void sn_grid_sync(unsigned* bar, unsigned& target) {
  target += gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (static_cast<unsigned>(ld_acquire_gpu(reinterpret_cast<const int*>(bar))) < target) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}

// C tile (kSnBM x kSnBN at m0, n0) of op(A) . op(B), M x N x K, in fp32 FMA.
//   A_MC: A(m, k) = A[k * lda + m] (m contiguous), else A[m * lda + k]
//   B_NC: B(k, n) = B[k * ldb + n] (n contiguous), else B[n * ldb + k]
// Thread (ty, tx) owns rows m0 + 4 ty + i (i < 4), cols n0 + 2 tx + j (j < 2).
// Operand k-blocks land in shared memory as [k][m] / [k][n] through 4-byte
// cp.async (zero-filled outside the matrix), kSnStages deep, so the L2
// latency of block kb + 2 hides under block kb's FMAs; each k row of a stage
// is one float4 (A) and one float2 (B) read per thread.
__device__ __forceinline__ void sn_cp4(float* smem, const float* gmem, const float* base, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(smem)), "l"(ok ? gmem : base),
               "r"(ok ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void sn_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N_>
__device__ __forceinline__ void sn_cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N_) : "memory"); }

template <bool A_MC, bool B_NC>
__device__ __forceinline__ void sn_tile(const float* __restrict__ A, long long lda, const float* __restrict__ B,
                                        long long ldb, int M, int N, int K, int m0, int n0, float (&acc)[4][2],
                                        float* As, float* Bs) {
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.f;
  auto issue = [&](int kb) {
    const int k0 = kb * kSnBK, s = kb % kSnStages;
    float* as = As + s * kSnAS;
    float* bs = Bs + s * kSnBS;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = t + kSnThreads * i;
      const int k = A_MC ? idx / kSnBM : idx % kSnBK;
      const int m = A_MC ? idx % kSnBM : idx / kSnBK;
      const int gm = m0 + m, gk = k0 + k;
      sn_cp4(as + k * kSnLdA + m,
             A_MC ? A + static_cast<long long>(gk) * lda + gm : A + static_cast<long long>(gm) * lda + gk, A,
             gm < M && gk < K);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = t + kSnThreads * i;
      const int k = B_NC ? idx / kSnBN : idx % kSnBK;
      const int n = B_NC ? idx % kSnBN : idx / kSnBK;
      const int gn = n0 + n, gk = k0 + k;
      sn_cp4(bs + k * kSnLdB + n,
             B_NC ? B + static_cast<long long>(gk) * ldb + gn : B + static_cast<long long>(gn) * ldb + gk, B,
             gn < N && gk < K);
    }
  };
  const int nkb = (K + kSnBK - 1) / kSnBK;
  __syncthreads();  // the previous tile's (or job's) readers are done with the stages
#pragma unroll
  for (int s = 0; s < kSnStages - 1; ++s) {
    if (s < nkb) issue(s);
    sn_cp_commit();
  }
  for (int kb = 0; kb < nkb; ++kb) {
    sn_cp_wait<kSnStages - 2>();  // block kb has landed (this thread's copies) ...
    __syncthreads();              // ... everyone's; and stage (kb - 1) % S is free again
    if (kb + kSnStages - 1 < nkb) issue(kb + kSnStages - 1);
    sn_cp_commit();
    const float* as = As + (kb % kSnStages) * kSnAS + 4 * ty;
    const float* bs = Bs + (kb % kSnStages) * kSnBS + 2 * tx;
    float blk[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) blk[i][0] = blk[i][1] = 0.f;
#pragma unroll
    for (int k = 0; k < kSnBK; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(as + k * kSnLdA);
      const float2 b = *reinterpret_cast<const float2*>(bs + k * kSnLdB);
      blk[0][0] = fmaf(a.x, b.x, blk[0][0]);
      blk[0][1] = fmaf(a.x, b.y, blk[0][1]);
      blk[1][0] = fmaf(a.y, b.x, blk[1][0]);
      blk[1][1] = fmaf(a.y, b.y, blk[1][1]);
      blk[2][0] = fmaf(a.z, b.x, blk[2][0]);
      blk[2][1] = fmaf(a.z, b.y, blk[2][1]);
      blk[3][0] = fmaf(a.w, b.x, blk[3][0]);
      blk[3][1] = fmaf(a.w, b.y, blk[3][1]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[i][0] += blk[i][0];
      acc[i][1] += blk[i][1];
    }
  }
  sn_cp_wait<0>();
}

// delta_{h-1} tile: (delta_h . W_h) * A_h (1 - A_h)
__device__ __forceinline__ void sn_dx_tile(const SmallNetArgs& p, int h, int tile, float* As, float* Bs) {
  const int M = p.rows, N = p.d[h], K = p.d[h + 1];
  const int tn = (N + kSnBN - 1) / kSnBN;
  const int m0 = (tile / tn) * kSnBM, n0 = (tile % tn) * kSnBN;
  float acc[4][2];
  sn_tile<false, true>(p.D[h], p.ld[h + 1], p.W[h], p.ldw[h], M, N, K, m0, n0, acc, As, Bs);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int m = m0 + 4 * ty + i, n = n0 + 2 * tx + j;
      if (m < M && n < N) {
        const float a = __ldcg(p.A[h] + m * p.ld[h] + n);
        p.D[h - 1][m * p.ld[h] + n] = acc[i][j] * (a * (1.f - a));
      }
    }
}

// dW_h = delta_h^T . A_h (A_0 = the batch), W_h -= eta dW_h (hidden layers)
__device__ __forceinline__ void sn_dw_tile(const SmallNetArgs& p, int h, int tile, const float* x, float eta,
                                           float* As, float* Bs) {
  const int M = p.d[h + 1], N = p.d[h], K = p.rows;
  const int tn = (N + kSnBN - 1) / kSnBN;
  const int m0 = (tile / tn) * kSnBM, n0 = (tile % tn) * kSnBN;
  const float* a = h == 0 ? x : p.A[h];
  const long long lda = h == 0 ? p.ldx : p.ld[h];
  float acc[4][2];
  sn_tile<true, true>(p.D[h], p.ld[h + 1], a, lda, M, N, K, m0, n0, acc, As, Bs);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int m = m0 + 4 * ty + i, n = n0 + 2 * tx + j;
      if (m < M && n < N) {
        const float g = acc[i][j];
        float* w = p.W[h] + m * p.ldw[h] + n;
        const float nw = *w - eta * g;
        *w = nw;
        if (p.W_lo[h] != nullptr) p.W_lo[h][m * p.ldw[h] + n] = tf32_lo(nw);
        if (p.G[h] != nullptr) p.G[h][static_cast<long long>(m) * N + n] = g;
      }
    }
}

// head dW for 32 columns j0..j0+31: G[c][j] = sum_r hd[r][c] A[r][j] in float64
// (8 row slices per column, summed in slice order), W -= eta G rounded once.
__device__ __forceinline__ void sn_head_dw(const SmallNetArgs& p, int job, float eta, double* red) {
  const int l = p.L - 1, d = p.d[l], nc = p.d[p.L];
  const int lane = threadIdx.x & 31, s = threadIdx.x >> 5;
  const int j = job * 32 + lane;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (j < d) {
    const float* a = p.A[l];
    // rows s, s + 8, ...: eight rows' loads in flight per round
    for (int r0 = s; r0 < p.rows; r0 += 64) {
      float av[8];
      float4 hv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int r = r0 + 8 * q;
        av[q] = r < p.rows ? __ldcg(a + r * p.ld[l] + j) : 0.f;
        hv[q] = r < p.rows ? __ldcg(reinterpret_cast<const float4*>(p.hd) + r) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double x = static_cast<double>(av[q]);
        acc[0] = fma(static_cast<double>(hv[q].x), x, acc[0]);
        acc[1] = fma(static_cast<double>(hv[q].y), x, acc[1]);
        acc[2] = fma(static_cast<double>(hv[q].z), x, acc[2]);
        acc[3] = fma(static_cast<double>(hv[q].w), x, acc[3]);
      }
    }
  }
  __syncthreads();  // (red is reused job after job)
#pragma unroll
  for (int c = 0; c < 4; ++c) red[(s * 4 + c) * 32 + lane] = acc[c];
  __syncthreads();
  if (s == 0 && j < d) {
    for (int c = 0; c < nc; ++c) {
      double g = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) g += red[(k * 4 + c) * 32 + lane];
      float* w = p.W[l] + c * p.ldw[l] + j;
      const float nw = static_cast<float>(static_cast<double>(*w) - static_cast<double>(eta) * g);
      *w = nw;
      if (p.W_lo[l] != nullptr) p.W_lo[l][c * p.ldw[l] + j] = tf32_lo(nw);
      if (p.G[l] != nullptr) p.G[l][c * d + j] = static_cast<float>(g);
    }
  }
}

// one warp per row: float64 logits / softmax / CE, the error signal, delta_{L-2}
__device__ __forceinline__ void sn_head_row(const SmallNetArgs& p, int r, const int64_t* labels) {
  const int l = p.L - 1, d = p.d[l], nc = p.d[p.L];
  const int lane = threadIdx.x & 31;
  const float* a = p.A[l] + r * p.ld[l];
  double z[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
  for (int j = lane; j < d; j += 32) {
    const double av = static_cast<double>(__ldcg(a + j));
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < nc) z[c] = fma(av, static_cast<double>(__ldcg(p.W[l] + c * p.ldw[l] + j)), z[c]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < 4; ++c) z[c] += __shfl_xor_sync(0xffffffffu, z[c], o);
  double zmax = -INFINITY;
  for (int c = 0; c < nc; ++c) zmax = fmax(zmax, z[c]);
  double e[4], esum = 0.0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    e[c] = c < nc ? exp(z[c] - zmax) : 0.0;
    esum += e[c];
  }
  const int y = static_cast<int>(labels[r]);
  double py = 0.0;
  for (int c = 0; c < nc; ++c)
    if (c == y) py = e[c] / esum;
  if (lane == 0) p.row_loss[r] = -log(fmax(py, 1e-12));
  if (!p.train) return;
  const double inv_n = static_cast<double>(1.0f / static_cast<float>(p.rows));
  float dl[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) dl[c] = c < nc ? static_cast<float>((e[c] / esum - (c == y ? 1.0 : 0.0)) * inv_n) : 0.f;
  if (lane == 0) reinterpret_cast<float4*>(p.hd)[r] = make_float4(dl[0], dl[1], dl[2], dl[3]);
  if (p.L < 2) return;
  float* dp = p.D[l - 1] + r * p.ld[l];
#pragma unroll 4
  for (int j = lane; j < d; j += 32) {
    float g = 0.f;
    for (int c = 0; c < nc; ++c) g = fmaf(dl[c], __ldcg(p.W[l] + c * p.ldw[l] + j), g);
    const float av = __ldcg(a + j);
    dp[j] = g * (av * (1.f - av));
  }
}

__global__ void __launch_bounds__(kSnThreads, 2) small_net_step_kernel(SmallNetArgs p) {
  __shared__ __align__(16) float As[kSnStages * kSnAS];
  __shared__ __align__(16) float Bs[kSnStages * kSnBS];
  const long long st = step_start(p.ds, p.start);
  const float eta = step_eta(p.ds, p.eta);
  const float* x = p.x + st * p.ldx;
  const int64_t* labels = p.labels + st;
  const int L = p.L;
  unsigned target = 0;
  const int tm_rows = (p.rows + kSnBM - 1) / kSnBM;
  // forward: hidden layers
  for (int h = 0; h < L - 1; ++h) {
    const float* in = h == 0 ? x : p.A[h];
    const long long ldin = h == 0 ? p.ldx : p.ld[h];
    const int N = p.d[h + 1], K = p.d[h];
    const int tn = (N + kSnBN - 1) / kSnBN;
    for (int tile = blockIdx.x; tile < tm_rows * tn; tile += gridDim.x) {
      const int m0 = (tile / tn) * kSnBM, n0 = (tile % tn) * kSnBN;
      float acc[4][2];
      sn_tile<false, false>(in, ldin, p.W[h], p.ldw[h], p.rows, N, K, m0, n0, acc, As, Bs);
      const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
      const float* b = p.bias[h];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int m = m0 + 4 * ty + i, n = n0 + 2 * tx + j;
          if (m < p.rows && n < N)
            p.A[h + 1][m * p.ld[h + 1] + n] = sigmoidf_stable(b != nullptr ? acc[i][j] + b[n] : acc[i][j]);
        }
    }
    sn_grid_sync(p.bar, target);
  }
  // head rows
  {
    const int warps = gridDim.x * (kSnThreads / 32);
    for (int r = blockIdx.x * (kSnThreads / 32) + (threadIdx.x >> 5); r < p.rows; r += warps) sn_head_row(p, r, labels);
  }
  if (p.train) {
    sn_grid_sync(p.bar, target);
    double* red = reinterpret_cast<double*>(As);  // 8 x 4 x 32 doubles = 8 KB (< the A stages)
    // backward: B_h = dX of layer h (h >= 1) beside dW of layer h + 1
    for (int h = L - 2; h >= 0; --h) {
      const int N = p.d[h], tn = (N + kSnBN - 1) / kSnBN;
      const int dx_tiles = h >= 1 ? tm_rows * tn : 0;
      const int u = h + 1;  // the layer whose update lands in this phase
      int dw_tiles;
      if (u == L - 1)
        dw_tiles = (p.d[u] + 31) / 32;
      else
        dw_tiles = ((p.d[u + 1] + kSnBM - 1) / kSnBM) * ((p.d[u] + kSnBN - 1) / kSnBN);
      for (int job = blockIdx.x; job < dx_tiles + dw_tiles; job += gridDim.x) {
        if (job < dx_tiles)
          sn_dx_tile(p, h, job, As, Bs);
        else if (u == L - 1)
          sn_head_dw(p, job - dx_tiles, eta, red);
        else
          sn_dw_tile(p, u, job - dx_tiles, x, eta, As, Bs);
      }
      sn_grid_sync(p.bar, target);
    }
    // layer 0's update
    {
      const int tiles = ((p.d[1] + kSnBM - 1) / kSnBM) * ((p.d[0] + kSnBN - 1) / kSnBN);
      for (int job = blockIdx.x; job < tiles; job += gridDim.x) sn_dw_tile(p, 0, job, x, eta, As, Bs);
    }
  } else {
    sn_grid_sync(p.bar, target);
  }
  // batch loss: CTA 0 sums the rows in a fixed order (row_loss is complete since the last barrier)
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    double s = 0.0;
    for (int r = threadIdx.x; r < p.rows; r += 32) s += p.row_loss[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *p.loss_out = s;
  }
}

}  // namespace hb
