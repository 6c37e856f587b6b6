// hb_kernels.cuh -- the non-GEMM kernels of the Hogbatch replica step:
// the fused small softmax/cross-entropy head, the wide-head softmax->delta
// pass, deterministic SGD reductions, the CSR-gather SpMM first layer and
// its sparse dW + update, precision conversion for the host exchange.
//
// Every reduction here runs in a fixed order (no float atomics), so a step is
// bit-reproducible run to run.
#pragma once
#include <cstdint>

#include "hb_ptx.cuh"

namespace hb {

constexpr float kProbFloor = 1e-12f;  // nn.py:26

// Per-step scalars read from device memory, so that one captured CUDA graph
// serves every batch of the same size: the batch's first row in the staged
// epoch and the learning rate (the coordinator's EXECUTE_WORK payload,
// messaging.py:91-96).  Kernels fall back to their by-value fields when the
// pointer is null (eager launches).
struct DevStep {
  long long start;
  float eta;
  int pad;
  double eta64;  // the merge's learning rate at the reference's float64 precision
  unsigned long long merge_gen;  // replica merges issued so far, this step's included (peer-merge flags)
};
__device__ __forceinline__ long long step_start(const DevStep* ds, long long s) { return ds ? ds->start : s; }
__device__ __forceinline__ float step_eta(const DevStep* ds, float e) { return ds ? ds->eta : e; }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ------------------------------------------------------------------------
// Fused small head (classes <= NCT, hidden width d <= 32*MAXT):
//   z = a . W^T, p = softmax(z)                               (nn.py:118-119)
//   loss_i = -log max(p_y, 1e-12)                              (nn.py:124-136)
//   delta = (p - onehot(y)) / n                                (nn.py:162-164)
//   delta_prev = (delta . W) * a (1 - a)                       (nn.py:170)
//   dW partial per block = sum_rows delta^T a                  (nn.py:168)
// One warp per row; lanes own columns j = lane + 32 t (coalesced).  A block
// owns HEAD_ROWS_PER_BLOCK consecutive rows and reduces its 8 warps' dW
// partials in warp order, so the result is deterministic.
constexpr int kHeadWarps = 8;
constexpr int kHeadRowsPerBlock = 16;


struct HeadArgs {
  const float* a;          // (rows, d) last hidden activation
  long long lda;
  const float* w;          // (nc, d) output weights
  long long ldw;
  const int64_t* labels;   // label array of the staged data (indexed from start)
  long long start;         // first batch row (ds->start when ds != null)
  int a_input;             // 1: `a` is the staged input itself (depth-1 nets), offset by start
  const DevStep* ds;
  int rows, d, nc;
  int zero_rows;           // delta_prev rows [rows, zero_rows) are zeroed
  int rows_per_block;      // vec kernel: rows walked by one block (multiple of kHeadRowsPerBlock)
  float inv_n;             // 1 / batch size
  int train;               // 0 = loss only (evaluation)
  float* delta_prev;       // (zero_rows, d) or null
  float* delta_prev_lo;    // its 3xTF32 lo twin (same layout) or null
  long long ld_dp;
  float* delta_out;        // (rows, nc) or null (tests)
  long long ld_do;
  double* ws_dw;           // [grid][nc][d] partials (float64: the block sums carry the cancellation of
                           // the softmax error signs, summed over hundreds of blocks)
  double* ws_loss;         // [grid] per-block loss sums
};

template <int NCT, int MAXT>
__global__ void __launch_bounds__(kHeadWarps * 32, (MAXT <= 16 && NCT <= 2) ? 2 : 1) head_small_kernel(HeadArgs p) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sW[NCT * 32 * MAXT];
  {
    const long long st = step_start(p.ds, p.start);
    p.labels += st;
    if (p.a_input) p.a += st * p.lda;
  }
  __shared__ double sLoss[kHeadWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = (p.d + 31) / 32;
  for (int i = threadIdx.x; i < NCT * 32 * MAXT; i += blockDim.x) {
    const int c = i / (32 * MAXT), j = i % (32 * MAXT);
    sW[i] = (c < p.nc && j < p.d) ? p.w[c * p.ldw + j] : 0.f;
  }
  __syncthreads();

  float acc[NCT][MAXT];
#pragma unroll
  for (int c = 0; c < NCT; ++c)
#pragma unroll
    for (int t = 0; t < MAXT; ++t) acc[c][t] = 0.f;
  double loss = 0.0;

  const int row0 = blockIdx.x * kHeadRowsPerBlock;
  for (int rr = warp; rr < kHeadRowsPerBlock; rr += kHeadWarps) {
    const int row = row0 + rr;
    if (row >= p.rows) {
      if (p.train && p.delta_prev != nullptr && row < p.zero_rows) {
        for (int t = 0; t < T; ++t) {
          const int j = lane + 32 * t;
          if (j < p.d) {
            p.delta_prev[row * p.ld_dp + j] = 0.f;
            if (p.delta_prev_lo != nullptr) p.delta_prev_lo[row * p.ld_dp + j] = 0.f;
          }
        }
      }
      continue;
    }
    float av[MAXT];
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      const int j = lane + 32 * t;
      av[t] = (t < T && j < p.d) ? p.a[row * p.lda + j] : 0.f;
    }
    // logits, softmax and the error signal in float64 (a handful of values per
    // row): p - 1 for a confident row loses its relative precision in fp32,
    // and the head's dW sum cancels those signals over the batch
    double z[NCT];
#pragma unroll
    for (int c = 0; c < NCT; ++c) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < MAXT; ++t) s = fma(static_cast<double>(av[t]), static_cast<double>(sW[c * 32 * MAXT + lane + 32 * t]), s);
      z[c] = warp_sum_f64(s);
    }
    double zmax = -INFINITY;
#pragma unroll
    for (int c = 0; c < NCT; ++c)
      if (c < p.nc) zmax = fmax(zmax, z[c]);
    double e[NCT], esum = 0.0;
#pragma unroll
    for (int c = 0; c < NCT; ++c) {
      e[c] = c < p.nc ? exp(z[c] - zmax) : 0.0;
      esum += e[c];
    }
    const int y = static_cast<int>(p.labels[row]);
    double py = 0.0;
#pragma unroll
    for (int c = 0; c < NCT; ++c)
      if (c == y) py = e[c] / esum;
    loss += -log(fmax(py, 1e-12));
    if (!p.train) continue;
    float dl[NCT];
#pragma unroll
    for (int c = 0; c < NCT; ++c)
      dl[c] = c < p.nc ? static_cast<float>((e[c] / esum - (c == y ? 1.0 : 0.0)) * static_cast<double>(p.inv_n)) : 0.f;
    if (p.delta_out != nullptr && lane < p.nc) {
#pragma unroll
      for (int c = 0; c < NCT; ++c)
        if (c == lane) p.delta_out[row * p.ld_do + c] = dl[c];
    }
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      const int j = lane + 32 * t;
      float g = 0.f;
#pragma unroll
      for (int c = 0; c < NCT; ++c) {
        g = fmaf(dl[c], sW[c * 32 * MAXT + j], g);
        acc[c][t] = fmaf(dl[c], av[t], acc[c][t]);
      }
      if (p.delta_prev != nullptr && t < T && j < p.d) {
        const float dv = g * (av[t] * (1.f - av[t]));
        p.delta_prev[row * p.ld_dp + j] = dv;
        if (p.delta_prev_lo != nullptr) p.delta_prev_lo[row * p.ld_dp + j] = tf32_lo(dv);
      }
    }
  }

  // deterministic block reduction of the loss
  if (lane == 0) sLoss[warp] = loss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kHeadWarps; ++w) s += sLoss[w];
    p.ws_loss[blockIdx.x] = s;
  }
  if (!p.train) return;
  // deterministic block reduction of the dW partials, one class at a time:
  // warps add into a shared row in warp order (sW is free after the row
  // loop); the block partial is stored as float64 for the long cross-block sum
  for (int c = 0; c < NCT && c < p.nc; ++c) {
    __syncthreads();
    for (int j = threadIdx.x; j < 32 * MAXT; j += blockDim.x) sW[j] = 0.f;
    __syncthreads();
    for (int w = 0; w < kHeadWarps; ++w) {
      if (warp == w) {
#pragma unroll
        for (int t = 0; t < MAXT; ++t) {
          const int j = lane + 32 * t;
          if (t < T && j < p.d) sW[j] += acc[c][t];
        }
      }
      __syncthreads();
    }
    for (int j = threadIdx.x; j < p.d; j += blockDim.x)
      p.ws_dw[(static_cast<long long>(blockIdx.x) * p.nc + c) * p.d + j] = static_cast<double>(sW[j]);
  }
}

// Vectorised variant for d % 4 == 0 (all padded row strides are multiples of
// 4 floats): lanes own float4 column groups 4*lane + 128*t, t < VPL, and each
// warp keeps its two rows' loads in flight together.  Same math and the same
// fixed reduction order (per-warp row order, then warps in order).
template <int NCT, int VPL>
__global__ void __launch_bounds__(kHeadWarps * 32) head_small_vec_kernel(HeadArgs p) {
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) float sW[NCT * 128 * VPL];
  {
    const long long st = step_start(p.ds, p.start);
    p.labels += st;
    if (p.a_input) p.a += st * p.lda;
  }
  __shared__ double sLoss[kHeadWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int D = 128 * VPL;
  for (int i = threadIdx.x; i < NCT * D; i += blockDim.x) {
    const int c = i / D, j = i % D;
    sW[i] = (c < p.nc && j < p.d) ? p.w[c * p.ldw + j] : 0.f;
  }
  __syncthreads();
  float4 acc[NCT][VPL];
#pragma unroll
  for (int c = 0; c < NCT; ++c)
#pragma unroll
    for (int t = 0; t < VPL; ++t) acc[c][t] = make_float4(0.f, 0.f, 0.f, 0.f);
  double loss = 0.0;
  constexpr int RPW = kHeadRowsPerBlock / kHeadWarps;  // rows per warp per pass (2)
  // a block owns rows [row_begin, row_end) and walks them kHeadRowsPerBlock at a time
  const int row_begin = blockIdx.x * p.rows_per_block;
  const int row_end = min(row_begin + p.rows_per_block, max(p.rows, p.zero_rows));
  for (int rb = row_begin; rb < row_end; rb += kHeadRowsPerBlock) {
  const int rbase = rb + warp * RPW;
  float4 av[RPW][VPL];
#pragma unroll
  for (int k = 0; k < RPW; ++k)
#pragma unroll
    for (int t = 0; t < VPL; ++t) {
      const int j = 4 * lane + 128 * t;
      const int row = rbase + k;
      av[k][t] = (row < p.rows && j < p.d) ? *reinterpret_cast<const float4*>(p.a + row * p.lda + j)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  double z[RPW][NCT];  // float64 logits / softmax / error signal (see head_small_kernel)
#pragma unroll
  for (int k = 0; k < RPW; ++k)
#pragma unroll
    for (int c = 0; c < NCT; ++c) {
      double sacc = 0.0;
#pragma unroll
      for (int t = 0; t < VPL; ++t) {
        const float4 w4 = *reinterpret_cast<const float4*>(&sW[c * D + 4 * lane + 128 * t]);
        sacc = fma(static_cast<double>(av[k][t].x), static_cast<double>(w4.x), sacc);
        sacc = fma(static_cast<double>(av[k][t].y), static_cast<double>(w4.y), sacc);
        sacc = fma(static_cast<double>(av[k][t].z), static_cast<double>(w4.z), sacc);
        sacc = fma(static_cast<double>(av[k][t].w), static_cast<double>(w4.w), sacc);
      }
      z[k][c] = sacc;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < RPW; ++k)
#pragma unroll
      for (int c = 0; c < NCT; ++c) z[k][c] += __shfl_xor_sync(0xffffffffu, z[k][c], o);
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int row = rbase + k;
    if (row >= p.rows) {
      if (p.train && p.delta_prev != nullptr && row < p.zero_rows) {
#pragma unroll
        for (int t = 0; t < VPL; ++t) {
          const int j = 4 * lane + 128 * t;
          if (j < p.d) {
            *reinterpret_cast<float4*>(p.delta_prev + row * p.ld_dp + j) = make_float4(0.f, 0.f, 0.f, 0.f);
            if (p.delta_prev_lo != nullptr)
              *reinterpret_cast<float4*>(p.delta_prev_lo + row * p.ld_dp + j) = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
      continue;
    }
    double zmax = -INFINITY;
#pragma unroll
    for (int c = 0; c < NCT; ++c)
      if (c < p.nc) zmax = fmax(zmax, z[k][c]);
    double e[NCT], esum = 0.0;
#pragma unroll
    for (int c = 0; c < NCT; ++c) {
      e[c] = c < p.nc ? exp(z[k][c] - zmax) : 0.0;
      esum += e[c];
    }
    const int y = static_cast<int>(p.labels[row]);
    double py = 0.0;
#pragma unroll
    for (int c = 0; c < NCT; ++c)
      if (c == y) py = e[c] / esum;
    loss += -log(fmax(py, 1e-12));
    if (!p.train) continue;
    float dl[NCT];
#pragma unroll
    for (int c = 0; c < NCT; ++c)
      dl[c] = c < p.nc ? static_cast<float>((e[c] / esum - (c == y ? 1.0 : 0.0)) * static_cast<double>(p.inv_n)) : 0.f;
#pragma unroll
    for (int t = 0; t < VPL; ++t) {
      const int j = 4 * lane + 128 * t;
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int c = 0; c < NCT; ++c) {
        const float4 w4 = *reinterpret_cast<const float4*>(&sW[c * D + j]);
        g.x = fmaf(dl[c], w4.x, g.x);
        g.y = fmaf(dl[c], w4.y, g.y);
        g.z = fmaf(dl[c], w4.z, g.z);
        g.w = fmaf(dl[c], w4.w, g.w);
        acc[c][t].x = fmaf(dl[c], av[k][t].x, acc[c][t].x);
        acc[c][t].y = fmaf(dl[c], av[k][t].y, acc[c][t].y);
        acc[c][t].z = fmaf(dl[c], av[k][t].z, acc[c][t].z);
        acc[c][t].w = fmaf(dl[c], av[k][t].w, acc[c][t].w);
      }
      if (p.delta_prev != nullptr && j < p.d) {
        const float4 a4 = av[k][t];
        const float4 dv = make_float4(g.x * (a4.x * (1.f - a4.x)), g.y * (a4.y * (1.f - a4.y)),
                                      g.z * (a4.z * (1.f - a4.z)), g.w * (a4.w * (1.f - a4.w)));
        *reinterpret_cast<float4*>(p.delta_prev + row * p.ld_dp + j) = dv;
        if (p.delta_prev_lo != nullptr) *reinterpret_cast<float4*>(p.delta_prev_lo + row * p.ld_dp + j) = lo4(dv);
      }
    }
  }
  }  // row passes
  if (lane == 0) sLoss[warp] = loss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kHeadWarps; ++w) t += sLoss[w];
    p.ws_loss[blockIdx.x] = t;
  }
  if (!p.train) return;
  // block partials: the warps' sums are added in warp order in fp32 (a few
  // rows each) -- every warp parks its row in shared memory, one barrier, then
  // each thread sums its columns over the warps in order -- and the partial is
  // stored as float64 for the long cross-block sum
  __shared__ __align__(16) float sRed[kHeadWarps * D];
  for (int c = 0; c < NCT && c < p.nc; ++c) {
    if (c > 0) __syncthreads();  // the previous class's sums have been read
#pragma unroll
    for (int t = 0; t < VPL; ++t)
      *reinterpret_cast<float4*>(&sRed[warp * D + 4 * lane + 128 * t]) = acc[c][t];
    __syncthreads();
    for (int j = threadIdx.x; j < p.d; j += blockDim.x) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < kHeadWarps; ++w) v += sRed[w * D + j];
      p.ws_dw[(static_cast<long long>(blockIdx.x) * p.nc + c) * p.d + j] = static_cast<double>(v);
    }
  }
}

// ------------------------------------------------------------------------
// Wide head second pass: logits (rows, nc) -> delta in place + per-row loss.
// One warp per row, row max shift as linalg.py:63-67.
struct SoftmaxArgs {
  float* z;  // (zero_rows, nc) logits in, delta out
  float* z_lo;  // lo twin of delta (or null)
  long long ldz;
  const int64_t* labels;  // staged label array, indexed from start
  long long start;
  const DevStep* ds;
  int rows, nc, zero_rows;
  float inv_n;
  int train;
  double* ws_loss;  // [grid]
};

__global__ void __launch_bounds__(256) softmax_delta_kernel(SoftmaxArgs p) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sLoss[8];
  p.labels += step_start(p.ds, p.start);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  double loss = 0.0;
  if (row < p.rows) {
    float* zr = p.z + row * p.ldz;
    float m = -INFINITY;
    for (int j = lane; j < p.nc; j += 32) m = fmaxf(m, zr[j]);
    m = warp_max(m);
    float s = 0.f;
    for (int j = lane; j < p.nc; j += 32) s += expf(zr[j] - m);
    s = warp_sum(s);
    const int y = static_cast<int>(p.labels[row]);
    if (lane == 0) {
      const float py = expf(zr[y] - m) / s;
      loss = -log(fmax(static_cast<double>(py), 1e-12));
    }
    if (p.train) {
      __syncwarp();
      for (int j = lane; j < p.nc; j += 32) {
        const float pj = expf(zr[j] - m) / s;
        const float dv = (pj - (j == y ? 1.f : 0.f)) * p.inv_n;
        zr[j] = dv;
        if (p.z_lo != nullptr) p.z_lo[row * p.ldz + j] = tf32_lo(dv);
      }
    }
  } else if (p.train && row < p.zero_rows) {
    for (int j = lane; j < p.nc; j += 32) {
      p.z[row * p.ldz + j] = 0.f;
      if (p.z_lo != nullptr) p.z_lo[row * p.ldz + j] = 0.f;
    }
  }
  if (lane == 0) sLoss[warp] = loss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += sLoss[w];
    p.ws_loss[blockIdx.x] = t;
  }
}

// Fixed-order sum of per-block loss partials: one warp, lane-strided partial
// sums then a fixed shuffle tree (deterministic).
__global__ void loss_reduce_kernel(const double* ws, int n, double* out, int accumulate) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s += ws[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) *out = accumulate ? *out + s : s;
}

// ------------------------------------------------------------------------
// W (rows, cols, ldw) -= eta * sum_{s<S} P[s] (rows, cols, dense), in place.
// The split-K / per-block partials are summed in slab order -> deterministic.
// Launch with one block of 256 threads per 32 consecutive elements: the 8
// warps split the slabs (warp w takes s = w, w+8, ...), then warp 0 adds the
// 8 warp sums in order -- a fixed summation order for every element.
__global__ void __launch_bounds__(256) reduce_sgd_kernel(float* w, long long ldw, const float* part, int S,
                                                           long long slab, int rows, int cols, float eta,
                                                           float* grad, long long ldg, const DevStep* ds,
                                                           float* w_lo) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[8][33];
  eta = step_eta(ds, eta);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long i = blockIdx.x * 32LL + lane;
  const long long total = static_cast<long long>(rows) * cols;
  // warp w sums slabs s = w, w+8, w+16, ... as four interleaved chains
  // (fixed order: chain k takes every fourth of the warp's slabs)
  // (8 independent loads in flight per thread per round)
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (i < total) {
    for (int s = warp; s < S; s += 64) {
      float t[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) t[k] = (s + 8 * k < S) ? __ldcs(part + (s + 8 * k) * slab + i) : 0.f;
      s0 += t[0] + t[4];
      s1 += t[1] + t[5];
      s2 += t[2] + t[6];
      s3 += t[3] + t[7];
    }
  }
  red[warp][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (warp == 0 && i < total) {
    float g = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) g += red[k][lane];
    const long long r = i / cols, c = i % cols;
    const float nw = w[r * ldw + c] - eta * g;
    w[r * ldw + c] = nw;
    if (w_lo != nullptr) w_lo[r * ldw + c] = tf32_lo(nw);
    if (grad != nullptr) grad[r * ldg + c] = g;
  }
}

// The small head's reduction: float64 block partials summed in float64 in a
// fixed order, the update applied in float64 and rounded once.
__global__ void __launch_bounds__(256) reduce_sgd_f64p_kernel(float* w, long long ldw, const double* part, int S,
                                                               long long slab, int rows, int cols, float eta,
                                                               float* grad, long long ldg, const DevStep* ds,
                                                               float* w_lo) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[8][33];
  eta = step_eta(ds, eta);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long i = blockIdx.x * 32LL + lane;
  const long long total = static_cast<long long>(rows) * cols;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (i < total) {
    for (int s = warp; s < S; s += 64) {
      double t[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) t[k] = (s + 8 * k < S) ? __ldcs(part + (s + 8 * k) * slab + i) : 0.0;
      s0 += t[0] + t[4];
      s1 += t[1] + t[5];
      s2 += t[2] + t[6];
      s3 += t[3] + t[7];
    }
  }
  red[warp][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (warp == 0 && i < total) {
    double g = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) g += red[k][lane];
    const long long r = i / cols, c = i % cols;
    const float nw = static_cast<float>(static_cast<double>(w[r * ldw + c]) - static_cast<double>(eta) * g);
    w[r * ldw + c] = nw;
    if (w_lo != nullptr) w_lo[r * ldw + c] = tf32_lo(nw);
    if (grad != nullptr) grad[r * ldg + c] = static_cast<float>(g);
  }
}

// Element-parallel variant for few slabs and many elements (split-K partials
// of large dW GEMMs): a grid-stride loop over float4 groups, every thread sums
// its 4 elements over the S slabs in slab order.  Needs cols % 4 == 0 and
// 16-byte-aligned rows of w / grad.
// host_w (optional): a float64 device copy of this layer's host model rows,
// read from the host just before this kernel; the stale merge
// host_w = host_w + (-eta) * g (linalg.py:79, NumPy rounding) is applied here
// too and the caller DMAs host_w back -- the device lane of the exchange.
__global__ void __launch_bounds__(256) reduce_sgd_vec_kernel(float* w, long long ldw, const float* part, int S,
                                                               long long slab, int rows, int cols, float eta,
                                                               float* grad, long long ldg, const DevStep* ds,
                                                               float* w_lo, double* host_w, double eta64) {
  pdl_wait();
  pdl_trigger();
  eta = step_eta(ds, eta);
  const long long quads = static_cast<long long>(rows) * cols / 4;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < quads;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = 4 * q;
    // issue the slab loads in batches of 8 independent loads, then sum in
    // slab order (the latency of one batch instead of S serial loads)
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < S; s0 += 8) {
      float4 t[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        t[k] = (s0 + k < S) ? __ldcs(reinterpret_cast<const float4*>(part + (s0 + k) * slab + i))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (s0 + k == 0) {
          g = t[0];
        } else if (s0 + k < S) {
          g.x += t[k].x;
          g.y += t[k].y;
          g.z += t[k].z;
          g.w += t[k].w;
        }
      }
    }
    const long long r = i / cols, c = i % cols;
    float4* wp = reinterpret_cast<float4*>(w + r * ldw + c);
    float4 wv = *wp;
    wv.x -= eta * g.x;
    wv.y -= eta * g.y;
    wv.z -= eta * g.z;
    wv.w -= eta * g.w;
    *wp = wv;
    if (w_lo != nullptr) *reinterpret_cast<float4*>(w_lo + r * ldw + c) = lo4(wv);
    if (grad != nullptr) *reinterpret_cast<float4*>(grad + r * ldg + c) = g;
    if (host_w != nullptr) {
      const double s = -(ds != nullptr ? ds->eta64 : eta64);
      double2* hp = reinterpret_cast<double2*>(host_w + i);
      double2 h0 = hp[0], h1 = hp[1];
      h0.x = __dadd_rn(h0.x, __dmul_rn(s, static_cast<double>(g.x)));
      h0.y = __dadd_rn(h0.y, __dmul_rn(s, static_cast<double>(g.y)));
      h1.x = __dadd_rn(h1.x, __dmul_rn(s, static_cast<double>(g.z)));
      h1.y = __dadd_rn(h1.y, __dmul_rn(s, static_cast<double>(g.w)));
      hp[0] = h0;
      hp[1] = h1;
    }
  }
}

// ------------------------------------------------------------------------
// CSR-gather SpMM first layer: A1[i, :] = sigmoid(sum_k val_k * W0T[col_k, :])
// for batch rows i in [0, rows) of the staged CSR starting at row `start`.
// W0 is held transposed, (d_in, d_out) row-major, so each nonzero gathers one
// contiguous d_out-long row.  One warp per example row; VEC = float4 columns.
struct SpmmArgs {
  const int64_t* rowptr;  // epoch CSR row pointer (n_rows + 1)
  const int32_t* col;
  const float* val;
  const DevStep* ds;
  long long start;
  int rows;
  const float* w0t;  // (d_in, d_out)
  long long ldw;
  int ldw_rows;      // d_in
  int d_out;
  float* out;  // (rows, d_out)
  long long ldo;
  float* out_lo;  // lo twin of out (or null)
  const float* bias;  // optional per-unit offset (d_out) added before the sigmoid (or null)
};

// CSR gather kernels: output columns per pass (HB_*_PASS float4 accumulators
// per lane = 128 * PASS columns) and blocks per SM (register cap).  Fewer
// accumulators let more warps -- more 4 KB row gathers -- be in flight per SM;
// measured on real-sim (b = 8192): SpMM 147 us at (8, 1) -> 118 us at (2, 8),
// sparse dW 213 us at (8, 1) -> 194 us at (4, 5).
#ifndef HB_SPMM_PASS
#define HB_SPMM_PASS 2
#endif
#ifndef HB_SPMM_MINB
#define HB_SPMM_MINB 8
#endif
#ifndef HB_SPDW_PASS
#define HB_SPDW_PASS 4
#endif
#ifndef HB_SPDW_MINB
#define HB_SPDW_MINB 5
#endif
#ifndef HB_SPMM_UNROLL
#define HB_SPMM_UNROLL 1  // nonzeros whose gathers a warp issues back to back
#endif
#ifndef HB_SPDW_UNROLL
#define HB_SPDW_UNROLL 2  // (sparse dW 194 -> 185 us at 2; the SpMM got slower)
#endif
#define HB_PRAGMA(x) _Pragma(#x)
#define HB_UNROLL_N(n) HB_PRAGMA(unroll n)

template <bool VEC>
__global__ void __launch_bounds__(256, HB_SPMM_MINB) spmm_sigmoid_kernel(SpmmArgs p) {
  pdl_wait();
  pdl_trigger();
  p.start = step_start(p.ds, p.start);
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= p.rows) return;
  const long long r = p.start + warp;
  const long long e0 = p.rowptr[r], e1 = p.rowptr[r + 1];
  float* o = p.out + warp * p.ldo;
  if (VEC) {
    // d_out % 128 == 0: lane owns float4 columns 4*lane + 128*t
    for (int base = 0; base < p.d_out; base += 128 * HB_SPMM_PASS) {
      float4 acc[HB_SPMM_PASS];
#pragma unroll
      for (int t = 0; t < HB_SPMM_PASS; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
      // the row's (col, val) pairs are fetched 32 at a time with one coalesced
      // load per lane and broadcast by shuffles, so the W0^T gathers of
      // consecutive nonzeros do not wait on index loads and overlap
      for (long long eb = e0; eb < e1; eb += 32) {
        const int cnt = static_cast<int>(min(32LL, e1 - eb));
        const int my_col = lane < cnt ? __ldg(p.col + eb + lane) : 0;
        const float my_val = lane < cnt ? __ldg(p.val + eb + lane) : 0.f;
        HB_UNROLL_N(HB_SPMM_UNROLL)
        for (int k = 0; k < cnt; ++k) {
          const float v = __shfl_sync(0xffffffffu, my_val, k);
          const float4* wr = reinterpret_cast<const float4*>(
              p.w0t + static_cast<long long>(__shfl_sync(0xffffffffu, my_col, k)) * p.ldw);
#pragma unroll
          for (int t = 0; t < HB_SPMM_PASS; ++t) {
            const int j = base + 4 * lane + 128 * t;
            if (j < p.d_out) {
              const float4 w = __ldg(wr + j / 4);
              acc[t].x = fmaf(v, w.x, acc[t].x);
              acc[t].y = fmaf(v, w.y, acc[t].y);
              acc[t].z = fmaf(v, w.z, acc[t].z);
              acc[t].w = fmaf(v, w.w, acc[t].w);
            }
          }
        }
      }
#pragma unroll
      for (int t = 0; t < HB_SPMM_PASS; ++t) {
        const int j = base + 4 * lane + 128 * t;
        if (j < p.d_out) {
          if (p.bias != nullptr) {
            const float4 b4 = *reinterpret_cast<const float4*>(p.bias + j);
            acc[t].x += b4.x;
            acc[t].y += b4.y;
            acc[t].z += b4.z;
            acc[t].w += b4.w;
          }
          const float4 sv = make_float4(sigmoidf_stable(acc[t].x), sigmoidf_stable(acc[t].y),
                                        sigmoidf_stable(acc[t].z), sigmoidf_stable(acc[t].w));
          reinterpret_cast<float4*>(o)[j / 4] = sv;
          if (p.out_lo != nullptr) reinterpret_cast<float4*>(p.out_lo + warp * p.ldo)[j / 4] = lo4(sv);
        }
      }
    }
  } else {
    for (int base = 0; base < p.d_out; base += 32 * 8) {
      float acc[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] = 0.f;
      for (long long e = e0; e < e1; ++e) {
        const float v = __ldg(p.val + e);
        const float* wr = p.w0t + static_cast<long long>(__ldg(p.col + e)) * p.ldw;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int j = base + lane + 32 * t;
          if (j < p.d_out) acc[t] = fmaf(v, __ldg(wr + j), acc[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int j = base + lane + 32 * t;
        if (j < p.d_out) {
          const float sv = sigmoidf_stable(p.bias != nullptr ? acc[t] + p.bias[j] : acc[t]);
          o[j] = sv;
          if (p.out_lo != nullptr) p.out_lo[warp * p.ldo + j] = tf32_lo(sv);
        }
      }
    }
  }
}


// Sparse dW0 + fused SGD update on the active feature rows only:
//   W0T[f, :] -= eta * sum_{i in batch, x_if != 0} x_if * delta0[i, :]
// using the epoch CSC (column pointer, ascending row index within a column).
// The batch [start, start+rows) is a contiguous row range of the epoch
// (engine.py:298-299), so its entries in column f are one contiguous slice
// found by binary search -- no per-batch transpose, fixed summation order.
struct SparseDwArgs {
  const int64_t* colptr;  // (d_in + 1)
  const int32_t* rowidx;  // ascending within each column (epoch row ids)
  const float* cval;
  const DevStep* ds;
  long long start;
  int rows;
  int d_in, d_out;
  const float* delta0;  // (rows, d_out)
  long long ldd;
  float* w0t;  // (d_in, d_out), updated in place
  long long ldw;
  float eta;
  float* grad;  // optional (d_in, d_out) raw gradient (transposed layout)
  long long ldg;
  const long long* lo_arr;  // per-feature batch slice of the CSC (csc_batch_ranges_kernel)
  const long long* hi_arr;
};

__device__ __forceinline__ long long lower_bound_i32(const int32_t* a, long long lo, long long hi, long long key) {
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (static_cast<long long>(a[mid]) < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// One block (8 warps) per (input feature f, 128-column chunk): the warps
// split the feature's batch entries round-robin (entry e -> warp (e-lo) % 8,
// four entries in flight per warp), each lane owns one float4 of the chunk;
// the 8 partial rows are added in warp order in shared memory and applied to
// W0T[f, chunk] in place (gradient optionally kept).  Fixed summation order.
template <bool VEC>
__global__ void __launch_bounds__(256) sparse_dw_kernel(SparseDwArgs p) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[8][128];
  p.start = step_start(p.ds, p.start);
  p.eta = step_eta(p.ds, p.eta);
  const int f = blockIdx.x;
  const int base = blockIdx.y * 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long lo = p.lo_arr[f], hi = p.hi_arr[f];
  const int width = min(128, p.d_out - base);
  float* wrow = p.w0t + static_cast<long long>(f) * p.ldw + base;
  float* grow = p.grad != nullptr ? p.grad + static_cast<long long>(f) * p.ldg + base : nullptr;
  if (lo == hi) {
    if (grow != nullptr && threadIdx.x < width) grow[threadIdx.x] = 0.f;
    return;
  }
  if (VEC) {
    const int j = 4 * lane;
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
    if (j < width) {
      // four entries in flight per warp (stride 8 warps), four fixed-order chains
      long long e = lo + warp;
      auto fma4 = [](float4& a, float v, const float4& d) {
        a.x = fmaf(v, d.x, a.x);
        a.y = fmaf(v, d.y, a.y);
        a.z = fmaf(v, d.z, a.z);
        a.w = fmaf(v, d.w, a.w);
      };
      auto drow = [&](long long ee) {
        return __ldg(reinterpret_cast<const float4*>(
            p.delta0 + (static_cast<long long>(__ldg(p.rowidx + ee)) - p.start) * p.ldd + base + j));
      };
      for (; e + 24 < hi; e += 32) {
        const float v0 = __ldg(p.cval + e), v1 = __ldg(p.cval + e + 8), v2 = __ldg(p.cval + e + 16),
                    v3 = __ldg(p.cval + e + 24);
        const float4 d0 = drow(e), d1 = drow(e + 8), d2 = drow(e + 16), d3 = drow(e + 24);
        fma4(a0, v0, d0);
        fma4(a1, v1, d1);
        fma4(a2, v2, d2);
        fma4(a3, v3, d3);
      }
      if (e < hi) fma4(a0, __ldg(p.cval + e), drow(e));
      if (e + 8 < hi) fma4(a1, __ldg(p.cval + e + 8), drow(e + 8));
      if (e + 16 < hi) fma4(a2, __ldg(p.cval + e + 16), drow(e + 16));
      a0 = make_float4(a0.x + a2.x, a0.y + a2.y, a0.z + a2.z, a0.w + a2.w);
      a1 = make_float4(a1.x + a3.x, a1.y + a3.y, a1.z + a3.z, a1.w + a3.w);
      *reinterpret_cast<float4*>(&red[warp][j]) =
          make_float4(a0.x + a1.x, a0.y + a1.y, a0.z + a1.z, a0.w + a1.w);
    }
  } else {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (long long e = lo + warp; e < hi; e += 8) {
      const float v = __ldg(p.cval + e);
      const float* dr = p.delta0 + (static_cast<long long>(__ldg(p.rowidx + e)) - p.start) * p.ldd + base;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int j = lane + 32 * t;
        if (j < width) acc[t] = fmaf(v, __ldg(dr + j), acc[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) red[warp][lane + 32 * t] = acc[t];
  }
  __syncthreads();
  if (threadIdx.x < width) {
    const int j = threadIdx.x;
    float g = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) g += (lo + k < hi) ? red[k][j] : 0.f;
    wrow[j] -= p.eta * g;
    if (grow != nullptr) grow[j] = g;
  }
}

// Per-feature slice [lo, hi) of the epoch CSC that falls in the batch rows
// [start, start+rows): one thread per feature, two binary searches.
// Same result with one warp per feature counting the column's entries below /
// inside the batch row range (ascending rows, so lo = c0 + #below): all loads
// independent instead of two chains of dependent binary-search probes --
// for epoch columns of up to a few hundred entries.
__global__ void __launch_bounds__(256) csc_batch_ranges_warp_kernel(const int64_t* colptr, const int32_t* rowidx,
                                                                    int d_in, long long start, int rows,
                                                                    const DevStep* ds, long long* lo_out,
                                                                    long long* hi_out) {
  pdl_wait();
  pdl_trigger();
  start = step_start(ds, start);
  const int lane = threadIdx.x & 31;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long f = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; f < d_in; f += nw) {
    const long long c0 = colptr[f], c1 = colptr[f + 1];
    int below = 0, inside = 0;
#pragma unroll 4
    for (long long e = c0 + lane; e < c1; e += 32) {
      const long long r = __ldg(rowidx + e);
      below += r < start;
      inside += (r >= start) & (r < start + rows);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      below += __shfl_xor_sync(0xffffffffu, below, o);
      inside += __shfl_xor_sync(0xffffffffu, inside, o);
    }
    if (lane == 0) {
      lo_out[f] = c0 + below;
      hi_out[f] = c0 + below + inside;
    }
  }
}
__global__ void csc_batch_ranges_kernel(const int64_t* colptr, const int32_t* rowidx, int d_in, long long start,
                                        int rows, const DevStep* ds, long long* lo_out, long long* hi_out) {
  pdl_wait();
  pdl_trigger();
  start = step_start(ds, start);
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < d_in; f += gridDim.x * blockDim.x) {
    const long long c0 = colptr[f], c1 = colptr[f + 1];
    const long long lo = lower_bound_i32(rowidx, c0, c1, start);
    lo_out[f] = lo;
    hi_out[f] = lower_bound_i32(rowidx, lo, c1, start + rows);
  }
}

// Sparse-feature regime (few batch entries per feature, e.g. real-sim's
// 20958 columns x ~20 entries): one warp per feature covering all d_out
// columns (float4 per lane, 1024-column chunks), entries in CSC order.
// Needs d_out % 4 == 0.
__global__ void __launch_bounds__(256, HB_SPDW_MINB) sparse_dw_warp_kernel(SparseDwArgs p) {
  pdl_wait();
  pdl_trigger();
  p.start = step_start(p.ds, p.start);
  p.eta = step_eta(p.ds, p.eta);
  const int f = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (f >= p.d_in) return;
  const long long lo = p.lo_arr[f], hi = p.hi_arr[f];
  float* wrow = p.w0t + static_cast<long long>(f) * p.ldw;
  float* grow = p.grad != nullptr ? p.grad + static_cast<long long>(f) * p.ldg : nullptr;
  if (lo == hi) {
    if (grow != nullptr)
      for (int j = lane * 4; j < p.d_out; j += 128) *reinterpret_cast<float4*>(grow + j) = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  for (int base = 0; base < p.d_out; base += 128 * HB_SPDW_PASS) {
    float4 acc[HB_SPDW_PASS];
#pragma unroll
    for (int t = 0; t < HB_SPDW_PASS; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    // the slice's (row, val) pairs are fetched 32 at a time with one
    // coalesced load per lane and broadcast by shuffles, so the delta0 row
    // gathers of consecutive entries do not wait on index loads
    for (long long eb = lo; eb < hi; eb += 32) {
      const int cnt = static_cast<int>(min(32LL, hi - eb));
      const long long my_row = lane < cnt ? static_cast<long long>(__ldg(p.rowidx + eb + lane)) - p.start : 0;
      const float my_val = lane < cnt ? __ldg(p.cval + eb + lane) : 0.f;
      HB_UNROLL_N(HB_SPDW_UNROLL)
      for (int k = 0; k < cnt; ++k) {
        const float v = __shfl_sync(0xffffffffu, my_val, k);
        const float* dr = p.delta0 + __shfl_sync(0xffffffffu, my_row, k) * p.ldd + base;
#pragma unroll
        for (int t = 0; t < HB_SPDW_PASS; ++t) {
          const int j = 4 * lane + 128 * t;
          if (base + j < p.d_out) {
            const float4 d = __ldg(reinterpret_cast<const float4*>(dr + j));
            acc[t].x = fmaf(v, d.x, acc[t].x);
            acc[t].y = fmaf(v, d.y, acc[t].y);
            acc[t].z = fmaf(v, d.z, acc[t].z);
            acc[t].w = fmaf(v, d.w, acc[t].w);
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < HB_SPDW_PASS; ++t) {
      const int j = base + 4 * lane + 128 * t;
      if (j < p.d_out) {
        float4 w = *reinterpret_cast<float4*>(wrow + j);
        w.x -= p.eta * acc[t].x;
        w.y -= p.eta * acc[t].y;
        w.z -= p.eta * acc[t].z;
        w.w -= p.eta * acc[t].w;
        *reinterpret_cast<float4*>(wrow + j) = w;
        if (grow != nullptr) *reinterpret_cast<float4*>(grow + j) = acc[t];
      }
    }
  }
}

// ------------------------------------------------------------------------
// Precision conversion / layout for the host <-> device model exchange.
// dst (rows, cols, ldd) fp32 <- src (rows, cols, lds) fp64; TRANSPOSE writes
// dst[c, r] (used for the transposed sparse first-layer weight).
template <bool TRANSPOSE>
__global__ void f64_to_f32_kernel(float* dst, long long ldd, const double* src, long long lds, int rows, int cols,
                                  float* dst_lo) {
  pdl_wait();
  pdl_trigger();
  const long long total = static_cast<long long>(rows) * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cols, c = i % cols;
    const float v = static_cast<float>(src[r * lds + c]);
    const long long o = TRANSPOSE ? c * ldd + r : r * ldd + c;
    dst[o] = v;
    if (dst_lo != nullptr) dst_lo[o] = tf32_lo(v);
  }
}
template <bool TRANSPOSE>
__global__ void f32_to_f64_kernel(double* dst, long long ldd, const float* src, long long lds, int rows, int cols) {
  const long long total = static_cast<long long>(rows) * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cols, c = i % cols;
    dst[r * ldd + c] = static_cast<double>(TRANSPOSE ? src[c * lds + r] : src[r * lds + c]);
  }
}

// Stale merge into the registered host model (workers.py:135 -> linalg.py:79):
// w_host[r, c] += -eta * g[r, c] (g transposed for the sparse first layer),
// float64, one aligned 8-byte store per element.
__global__ void merge_host_f64_kernel(double* w_host, const float* g, long long ldg, int rows, int cols,
                                      int transposed, double eta, const DevStep* ds = nullptr) {
  if (ds != nullptr) eta = ds->eta64;
  const long long total = static_cast<long long>(rows) * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cols, c = i % cols;
    const float gv = transposed ? g[c * ldg + r] : g[r * ldg + c];
    // np.add(target, scale*source, out=target): product and sum rounded
    // separately (no FMA contraction), exactly as NumPy evaluates it
    w_host[i] = __dadd_rn(w_host[i], __dmul_rn(-eta, static_cast<double>(gv)));
  }
}

// dst (rows, cols, dense) = src^T where src is (cols, rows) with row stride lds.
__global__ void transpose_f32_kernel(float* dst, const float* src, long long lds, int rows, int cols) {
  const long long total = static_cast<long long>(rows) * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cols, c = i % cols;
    dst[i] = src[c * lds + r];
  }
}

// lo (rows, cols, ld) = x - trunc_tf32(x): the 3xTF32 twin of a staged input.
// Split-K finish of a forward / dX GEMM whose output tile grid is too small
// to fill the SMs (small batches): out = op(sum_s part[s]) over S slabs in slab
// order (deterministic), op = sigmoid (forward, linalg.py:48-55), identity
// (logits) or x * a(1 - a) (dX, linalg.py:58-60); rows [M, zero_rows) of a dX
// output are written as 0; the lo twin is written when out_lo != null.
enum SplitEpi : int { SPLIT_SIGMOID = 0, SPLIT_STORE = 1, SPLIT_DSIG = 2 };
template <int MODE, bool VEC>
__global__ void __launch_bounds__(256) splitk_epi_kernel(float* __restrict__ out, float* __restrict__ out_lo,
                                                         long long ldo, const float* __restrict__ part, int S,
                                                         int M, int N, const float* __restrict__ aux, long long ld_aux,
                                                         int zero_rows, const float* __restrict__ bias = nullptr) {
  pdl_wait();
  pdl_trigger();
  const long long slab = static_cast<long long>(M) * N;
  const int rows_total = MODE == SPLIT_DSIG ? max(M, zero_rows) : M;
  constexpr int W = VEC ? 4 : 1;
  const long long items = static_cast<long long>(rows_total) * (N / W);
  for (long long it = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; it < items;
       it += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = it / (N / W);
    const int c = static_cast<int>(it % (N / W)) * W;
    float v[W];
    if (r >= M) {
#pragma unroll
      for (int k = 0; k < W; ++k) v[k] = 0.f;
    } else {
      const float* pp = part + r * N + c;
      if (VEC) {
        float4 g = __ldcs(reinterpret_cast<const float4*>(pp));
        for (int s0 = 1; s0 < S; s0 += 8) {
          float4 t[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            t[k] = s0 + k < S ? __ldcs(reinterpret_cast<const float4*>(pp + (s0 + k) * slab)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (s0 + k < S) {
              g.x += t[k].x;
              g.y += t[k].y;
              g.z += t[k].z;
              g.w += t[k].w;
            }
        }
        v[0] = g.x;
        v[W > 1 ? 1 : 0] = g.y;
        v[W > 2 ? 2 : 0] = g.z;
        v[W > 3 ? 3 : 0] = g.w;
      } else {
        float g = __ldcs(pp);
        for (int s = 1; s < S; ++s) g += __ldcs(pp + s * slab);
        v[0] = g;
      }
#pragma unroll
      for (int k = 0; k < W; ++k) {
        if (MODE != SPLIT_DSIG && bias != nullptr) v[k] += bias[c + k];
        if (MODE == SPLIT_SIGMOID) v[k] = sigmoidf_fast(v[k]);
        if (MODE == SPLIT_DSIG) {
          const float a = aux[r * ld_aux + c + k];
          v[k] = v[k] * (a * (1.f - a));
        }
      }
    }
    float* op = out + r * ldo + c;
    if (VEC) {
      const float4 o4 = make_float4(v[0], v[W > 1 ? 1 : 0], v[W > 2 ? 2 : 0], v[W > 3 ? 3 : 0]);
      *reinterpret_cast<float4*>(op) = o4;
      if (out_lo != nullptr) *reinterpret_cast<float4*>(out_lo + r * ldo + c) = lo4(o4);
    } else {
      op[0] = v[0];
      if (out_lo != nullptr) out_lo[r * ldo + c] = tf32_lo(v[0]);
    }
  }
}

// *flag = 1 if any x[r][c] (r < rows, c < cols, row stride ld) is nonzero;
// the pad columns [cols, ld) are never written by staging and never read
__global__ void any_nonzero_kernel(const float* x, long long rows, int cols, long long ld, int* flag) {
  int any = 0;
  const long long n = rows * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    any |= x[(i / cols) * ld + i % cols] != 0.f;
  if (__syncthreads_or(any) && threadIdx.x == 0) *flag = 1;
}

// dst (rows, cols) with row stride ld <- contiguous src (rows, cols); lo twin too
__global__ void repitch_split_kernel(const float* __restrict__ src, float* __restrict__ dst, float* __restrict__ lo,
                                     long long ld, long long rows, int cols) {
  const long long total = rows * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cols, c = i % cols;
    const float v = src[i];
    dst[r * ld + c] = v;
    if (lo != nullptr) lo[r * ld + c] = tf32_lo(v);
  }
}

__global__ void split_lo_kernel(const float* x, float* lo, long long ld, long long rows, int cols) {
  const long long total = rows * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cols, c = i % cols;
    lo[r * ld + c] = tf32_lo(x[r * ld + c]);
  }
}

// Zero-copy batch load: the SMs read a page-locked host batch through its
// mapped device alias (x rows of ldx floats, labels) and write the padded
// device rows, their lo twin and the labels.  Small batches take this path
// instead of a copy-engine DMA, which would queue behind the previous call's
// deferred float64 write-backs.
__global__ void zc_batch_kernel(const float* __restrict__ x, long long ldx, const int64_t* __restrict__ labels,
                                float* dst, float* dst_lo, long long ld, int64_t* dst_labels, long long rows,
                                int cols) {
  const long long total = rows * cols;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total; i += stride) {
    const long long r = i / cols, c = i % cols;
    const float v = x[r * ldx + c];
    dst[r * ld + c] = v;
    if (dst_lo != nullptr) dst_lo[r * ld + c] = tf32_lo(v);
  }
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < rows; i += stride)
    dst_labels[i] = labels[i];
}

// dst (rows, cols, ldd) = scale * src (rows, cols, dense): unpack of the
// allreduced flat model (replica averaging).
__global__ void unpack_scale_kernel(float* dst, long long ldd, const float* src, int rows, int cols, float scale,
                                    float* dst_lo) {
  const long long total = static_cast<long long>(rows) * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cols, c = i % cols;
    const float v = src[i] * scale;
    dst[r * ldd + c] = v;
    if (dst_lo != nullptr) dst_lo[r * ldd + c] = tf32_lo(v);
  }
}

// The whole model packed / unpacked in one launch each for the replica
// merge: layer l occupies [off[l], off[l+1]) of the flat buffer as a dense
// (rows, cols) block; its device layout has row stride ld[l] (+ lo twin).
constexpr int kMaxMergeLayers = 16;
struct ModelLayout {
  float* w[kMaxMergeLayers];
  float* w_lo[kMaxMergeLayers];
  long long ld[kMaxMergeLayers];
  int cols[kMaxMergeLayers];
  long long off[kMaxMergeLayers + 1];  // segment starts (multiples of 4; padding after each layer)
  long long size[kMaxMergeLayers];     // elements of each layer
  int n;
};
__device__ __forceinline__ int layout_layer(const ModelLayout& m, long long i) {
  int l = 0;
  while (l + 1 < m.n && i >= m.off[l + 1]) ++l;
  return l;
}
__global__ void pack_model_kernel(float* __restrict__ flat, const __grid_constant__ ModelLayout m) {
  pdl_wait();
  pdl_trigger();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m.off[m.n];
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int l = layout_layer(m, i);
    const long long k = i - m.off[l];
    flat[i] = k < m.size[l] ? m.w[l][(k / m.cols[l]) * m.ld[l] + k % m.cols[l]] : 0.f;
  }
}
__global__ void unpack_model_kernel(const float* __restrict__ flat, float scale, const __grid_constant__ ModelLayout m) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m.off[m.n];
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int l = layout_layer(m, i);
    const long long k = i - m.off[l];
    if (k >= m.size[l]) continue;  // segment padding
    const long long o = (k / m.cols[l]) * m.ld[l] + k % m.cols[l];
    const float v = flat[i] * scale;
    m.w[l][o] = v;
    if (m.w_lo[l] != nullptr) m.w_lo[l][o] = tf32_lo(v);
  }
}

// ------------------------------------------------------------------------
// Device-side synthetic Gaussian blobs (the shape of the reference's
// synthetic_blobs, data.py:226-252: unit-variance isotropic noise around a
// class mean; the means come from the host generator).  Used to stage the
// 10M-row scaled configuration without a host copy: row r's label and noise
// are a pure function of (seed, r), drawn from a counter-based Philox4x32-10
// stream, so any row range can be regenerated or read back (hb_read_staged).
__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint2 key) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const unsigned hi0 = __umulhi(0xD2511F53u, ctr.x), lo0 = 0xD2511F53u * ctr.x;
    const unsigned hi1 = __umulhi(0xCD9E8D57u, ctr.z), lo1 = 0xCD9E8D57u * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += 0x9E3779B9u;
    key.y += 0xBB67AE85u;
  }
  return ctr;
}
__device__ __forceinline__ float u01_open(unsigned v) {  // (0, 1]
  return (static_cast<float>(v >> 8) + 1.0f) * (1.0f / 16777216.0f);
}
// one block per row (grid-stride); threads own float4 column groups
__global__ void blobs_kernel(float* __restrict__ x, float* __restrict__ x_lo, long long ld, long long row0,
                             long long rows, int d, const float* __restrict__ means, int classes,
                             int64_t* __restrict__ labels, unsigned long long seed) {
  const uint2 key = make_uint2(static_cast<unsigned>(seed), static_cast<unsigned>(seed >> 32));
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    const long long g = row0 + r;  // global row id: the stream key
    const uint4 lh = philox4x32_10(make_uint4(0xFFFFFFFFu, static_cast<unsigned>(g), static_cast<unsigned>(g >> 32), 1u), key);
    const int y = static_cast<int>(((static_cast<unsigned long long>(lh.x) << 32 | lh.y) % static_cast<unsigned long long>(classes)));
    if (threadIdx.x == 0 && labels != nullptr) labels[r] = y;
    const float* mu = means + static_cast<long long>(y) * d;
    float* xr = x + r * ld;
    float* lr = x_lo ? x_lo + r * ld : nullptr;
    for (int k = threadIdx.x; 4 * k < d; k += blockDim.x) {
      const uint4 u = philox4x32_10(make_uint4(static_cast<unsigned>(k), static_cast<unsigned>(g),
                                               static_cast<unsigned>(g >> 32), 0u), key);
      // Box-Muller on two uniform pairs -> four standard normals
      float s0, c0, s1, c1;
      const float r0 = sqrtf(-2.0f * logf(u01_open(u.x))), r1 = sqrtf(-2.0f * logf(u01_open(u.z)));
      sincospif(2.0f * u01_open(u.y), &s0, &c0);
      sincospif(2.0f * u01_open(u.w), &s1, &c1);
      const float nz[4] = {r0 * c0, r0 * s0, r1 * c1, r1 * s1};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = 4 * k + q;
        if (j < d) {
          const float v = mu[j] + nz[q];
          xr[j] = v;
          if (lr) lr[j] = tf32_lo(v);
        }
      }
    }
  }
}

}  // namespace hb
