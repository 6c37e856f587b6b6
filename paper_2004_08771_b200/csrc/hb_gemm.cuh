// hb_gemm.cuh -- the fully-connected GEMMs of the Hogbatch replica step on
// sm_100a: TMA -> SMEM -> tcgen05.mma(kind::tf32) -> TMEM -> fused epilogue.
//
// One kernel template covers the three contractions of nn.py:108-171:
//   forward   Z = A_l . W_l^T        A K-major, B K-major  (nn.py:118)
//   dX        D = delta_l . W_l      A K-major, B MN-major (nn.py:170)
//   dW        G = delta_l^T . A_l    A MN-major, B MN-major (nn.py:168)
// and the epilogues that replace the reference's separate elementwise passes:
//   EPI_SIGMOID  A_{l+1} = sigmoid(Z)                      (linalg.py:48-55)
//   EPI_STORE    logits (wide softmax heads, finished by softmax_delta)
//   EPI_DSIG     delta_{l-1} = D * A_l (1 - A_l)            (linalg.py:58-60)
//   EPI_PARTIAL  split-K partial of G into a workspace slab
//   EPI_SGD      W_l -= eta * G in place (+ optional raw G) (nn.py:174-179)
//
// Precision: fp32 data; PASSES == 3 runs the 3xTF32 split
//   x = hi + lo, hi = x with the low 13 mantissa bits cleared,
//   A.B ~= A_lo.B_hi + A_hi.B_lo + A_hi.B_hi   (fp32 accumulate in TMEM)
// which meets the reference's per-step 1e-4 bar (SURVEY §7 hard part 1);
// PASSES == 1 is plain TF32.  The hi/lo split is done in shared memory by a
// dedicated warpgroup right after TMA lands each stage, so HBM/L2 traffic is
// the same as a plain fp32 GEMM.
//
// Warp roles (one CTA = one 128 x BN output tile, one split of K):
//   warp 0        TMA producer (one elected lane)
//   warp 1        MMA issuer   (one elected lane)
//   warp 2        TMEM allocator
//   warps 4..7    epilogue: tcgen05.ld TMEM -> registers -> fused op -> global
//   warps 8..11   (PASSES == 3) hi/lo splitter
#pragma once
#include "hb_ptx.cuh"

namespace hb {

enum Epi : int { EPI_SIGMOID = 0, EPI_STORE = 1, EPI_DSIG = 2, EPI_PARTIAL = 3, EPI_SGD = 4 };

struct GemmArgs {
  int M, N;               // valid output rows / cols
  int m_zero_rows;        // EPI_DSIG: rows in [M, m_zero_rows) are written as 0
  int a_off, b_off;       // row-coordinate offsets into A's / B's tensor maps
  int kb_total;           // ceil(K / 32)
  int kb_per_split;
  float* out;             // output / partial slab base / W (EPI_SGD, in place)
  long long ldo;
  long long split_stride; // EPI_PARTIAL: elements between split slabs
  const float* aux;       // EPI_DSIG: activation A_l (same indexing as out)
  long long ld_aux;
  float* grad;            // EPI_SGD: optional raw gradient output
  long long ld_grad;
  float eta;
};

constexpr int kBM = 128;
constexpr int kBK = 32;  // 32 fp32 = one 128-byte swizzle row

template <int BN, int PASSES>
struct GemmCfg {
  static constexpr int A_BYTES = kBM * kBK * 4;
  static constexpr int B_BYTES = BN * kBK * 4;
  static constexpr int OP_BYTES = A_BYTES + B_BYTES;  // raw (hi) operands of one stage
  static constexpr int STAGE_BYTES = OP_BYTES * (PASSES == 3 ? 2 : 1);
  static constexpr int BUDGET = 200 * 1024;
  static constexpr int STAGES_RAW = BUDGET / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  static constexpr int THREADS = PASSES == 3 ? 384 : 256;
  // TMEM accumulators: the tensor core's fp32 accumulation error grows with
  // the number of MMAs chained into one accumulator, so 3xTF32 keeps the two
  // small cross terms in their own accumulator and rotates the hi*hi term over
  // NBIG accumulators by k-block; the epilogue sums them in fp32 registers.
  static constexpr int NBIG_RAW = PASSES == 3 ? 512 / BN - 1 : 1;
  static constexpr int NBIG = NBIG_RAW > 15 ? 15 : (NBIG_RAW < 1 ? 1 : NBIG_RAW);
  static constexpr int NACC = PASSES == 3 ? NBIG + 1 : 1;
  static constexpr int TMEM_COLS_RAW = NACC * BN;
  static constexpr int TMEM_COLS = TMEM_COLS_RAW <= 32 ? 32 : TMEM_COLS_RAW <= 64 ? 64 : TMEM_COLS_RAW <= 128 ? 128
                                   : TMEM_COLS_RAW <= 256 ? 256 : 512;
  static_assert(TMEM_COLS_RAW <= 512, "TMEM holds 512 fp32 columns");
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align slack*/ + 256 /*barriers*/;
  static_assert(STAGES >= 2, "need at least double buffering");
};

__device__ __forceinline__ uint64_t op_desc(uint32_t tile, int kk, bool mn_major) {
  // K-major SW128: advance 32 B (8 tf32) along the 128-B row per MMA step.
  // MN-major SW128_BASE32B: advance 8 K-lines (1024 B) per MMA step; 32-wide
  // MN chunks are 4096 B apart (32 K-lines of 128 B each).
  return mn_major ? make_sdesc(tile + kk * 1024, 4096, 512, kLayoutSW128Base32B)
                  : make_sdesc(tile + kk * 32, 16, 1024, kLayoutSW128);
}

template <int BN, bool A_MN, bool B_MN, int EPI, int PASSES>
__global__ void __launch_bounds__(GemmCfg<BN, PASSES>::THREADS, 1)
    gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmArgs args) {
  using C = GemmCfg<BN, PASSES>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* ready = full + STAGES;
  uint64_t* empty = ready + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN;
  const int m0 = blockIdx.y * kBM;
  const int kb_begin = blockIdx.z * args.kb_per_split;
  const int kb_end = min(kb_begin + args.kb_per_split, args.kb_total);
  const int nkb = max(kb_end - kb_begin, 0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ready[s], 128);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sA = smem + s * C::STAGE_BYTES;
        uint8_t* sB = sA + C::A_BYTES;
        mbar_arrive_expect_tx(&full[s], C::OP_BYTES);
        const int k0 = (kb_begin + i) * kBK;
        if (!A_MN) {
          tma_load_2d(sA, &tmA, &full[s], k0, m0 + args.a_off);
        } else {
#pragma unroll
          for (int j = 0; j < kBM / 32; ++j) tma_load_2d(sA + j * 4096, &tmA, &full[s], m0 + 32 * j, k0 + args.a_off);
        }
        if (!B_MN) {
          tma_load_2d(sB, &tmB, &full[s], k0, n0 + args.b_off);
        } else {
#pragma unroll
          for (int j = 0; j < BN / 32; ++j) tma_load_2d(sB + j * 4096, &tmB, &full[s], n0 + 32 * j, k0 + args.b_off);
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_tf32(kBM, BN, A_MN, B_MN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(PASSES == 3 ? &ready[s] : &full[s], ph);
        tc_fence_after();
        const uint32_t aHi = smem_u32(smem + s * C::STAGE_BYTES);
        const uint32_t bHi = aHi + C::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < kBK / 8; ++kk) {
          const uint64_t ah = op_desc(aHi, kk, A_MN);
          const uint64_t bh = op_desc(bHi, kk, B_MN);
          if (PASSES == 3) {
            const uint64_t al = op_desc(aHi + C::OP_BYTES, kk, A_MN);
            const uint64_t bl = op_desc(bHi + C::OP_BYTES, kk, B_MN);
            const uint32_t t_small = tmem_base + C::NBIG * BN;
            const uint32_t t_big = tmem_base + (i % C::NBIG) * BN;
            mma_tf32(t_small, al, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u);
            mma_tf32(t_small, ah, bl, idesc, 1u);
            mma_tf32(t_big, ah, bh, idesc, (i >= C::NBIG || kk > 0) ? 1u : 0u);
          } else {
            mma_tf32(tmem_base, ah, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          }
        }
        mma_commit(&empty[s]);  // frees the smem stage once these MMAs retire
      }
      mma_commit(tmem_full);  // accumulator complete (immediate if nkb == 0)
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------------------------------------------------- epilogue
    const int q = warp - 4;  // TMEM lane quarter owned by this warp
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int row = m0 + q * 32 + lane;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + c;
      float v[32];
      {
        uint32_t r[32];
        // small-term accumulator first, then the hi*hi accumulators (only those
        // the k loop actually wrote)
        tmem_ld_32x32b_x32(lane_addr + (C::NACC - 1) * BN, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = nkb > 0 ? __uint_as_float(r[j]) : 0.f;
        if (C::NACC > 1) {
#pragma unroll 1
          for (int a = 0; a < C::NBIG; ++a) {
            tmem_ld_32x32b_x32(lane_addr + a * BN, r);
            tmem_ld_wait();
            if (a < nkb) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += __uint_as_float(r[j]);
            }
          }
        }
      }
      const int n = n0 + c;
      if (n >= args.N) continue;
      const int ncols = min(32, args.N - n);
      if (EPI == EPI_SIGMOID || EPI == EPI_STORE) {
        if (row < args.M) {
          float* o = args.out + static_cast<long long>(row) * args.ldo + n;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < ncols) o[j] = (EPI == EPI_SIGMOID) ? sigmoidf_stable(v[j]) : v[j];
        }
      } else if (EPI == EPI_DSIG) {
        if (row < args.M) {
          float* o = args.out + static_cast<long long>(row) * args.ldo + n;
          const float* a = args.aux + static_cast<long long>(row) * args.ld_aux + n;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < ncols) {
              const float s = a[j];
              o[j] = v[j] * (s * (1.f - s));
            }
        } else if (row < args.m_zero_rows) {
          float* o = args.out + static_cast<long long>(row) * args.ldo + n;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < ncols) o[j] = 0.f;
        }
      } else if (EPI == EPI_PARTIAL) {
        if (row < args.M) {
          float* o = args.out + blockIdx.z * args.split_stride + static_cast<long long>(row) * args.ldo + n;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < ncols) o[j] = v[j];
        }
      } else {  // EPI_SGD
        if (row < args.M) {
          float* w = args.out + static_cast<long long>(row) * args.ldo + n;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < ncols) w[j] = w[j] - args.eta * v[j];
          if (args.grad != nullptr) {
            float* g = args.grad + static_cast<long long>(row) * args.ld_grad + n;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncols) g[j] = v[j];
          }
        }
      }
    }
  } else if (PASSES == 3 && warp >= 8) {
    // ------------------------------------------------- hi/lo splitter
    const int t = threadIdx.x - 256;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      mbar_wait(&full[s], ph);
      uint4* hi = reinterpret_cast<uint4*>(smem + s * C::STAGE_BYTES);
      float4* lo = reinterpret_cast<float4*>(smem + s * C::STAGE_BYTES + C::OP_BYTES);
#pragma unroll 4
      for (int j = t; j < C::OP_BYTES / 16; j += 128) {
        uint4 x = hi[j];
        uint4 h = make_uint4(to_tf32_rna(x.x), to_tf32_rna(x.y), to_tf32_rna(x.z), to_tf32_rna(x.w));
        lo[j] = make_float4(__uint_as_float(x.x) - __uint_as_float(h.x), __uint_as_float(x.y) - __uint_as_float(h.y),
                            __uint_as_float(x.z) - __uint_as_float(h.z), __uint_as_float(x.w) - __uint_as_float(h.w));
        hi[j] = h;
      }
      fence_proxy_async_smem();
      mbar_arrive(&ready[s]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace hb
