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
//   EPI_SPLIT_SGD split-K partial into a slab, then the gridDim.z split CTAs of
//                an output tile meet (global arrive counter; all CTAs of the
//                launch are co-resident by construction, dw_plan) and each sums
//                a 1/S row share of the tile over the slabs in slab order and
//                applies W_l -= eta * G: the split-K reduction without a
//                second kernel
//
// Precision: fp32 data; PASSES == 3 runs the 3xTF32 split
//   x = hi + lo, hi = trunc_tf32(x) (what the tensor core reads from raw fp32),
//   lo = x - hi (exact in fp32), every operand tensor keeps its lo twin in HBM
//   (written by the kernel that produced it),
//   A.B ~= A_lo.B_hi + A_hi.B_lo + A_hi.B_hi   (fp32 accumulate in TMEM)
// which meets the reference's per-step 1e-4 bar (SURVEY §7 hard part 1);
// PASSES == 1 is plain TF32.  Pre-split twins cost one extra TMA load per
// operand but keep the in-CTA shared-memory traffic to TMA writes + MMA reads
// (an in-smem splitter made the kernel smem-bandwidth bound).
//
// Warp roles (one CTA = one 128 x BN output tile, one split of K):
//   warp 0        TMA producer (one elected lane)
//   warp 1        MMA issuer   (one elected lane)
//   warp 2        TMEM allocator
//   warps 4..11   epilogue: tcgen05.ld TMEM -> registers -> smem transpose -> fused op ->
//                 coalesced float4 global traffic (2 warps per TMEM lane quarter);
//                 operand-producing epilogues also write the lo twin
#pragma once
#include "hb_kernels.cuh"
#include "hb_ptx.cuh"

namespace hb {

enum Epi : int { EPI_SIGMOID = 0, EPI_STORE = 1, EPI_DSIG = 2, EPI_PARTIAL = 3, EPI_SGD = 4, EPI_SPLIT_SGD = 5 };

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
  float* out_lo;          // lo twin of the output (EPI_SIGMOID / EPI_DSIG: same indexing as out;
                          // EPI_SGD: lo twin of W), or null
  const DevStep* ds;      // graph launches: start / eta from device memory
  int a_start, b_start;   // add ds->start to a_off / b_off (staged-input operands)
  float* w;               // EPI_SPLIT_SGD: W_l (updated in place), its lo twin (or null), row stride
  float* w_lo;
  long long ldw;
  int* tile_sync;         // EPI_SPLIT_SGD: 2 zeroed counters per output tile (arrive, depart)
  int a_lo_zero, b_lo_zero;  // 3xTF32: that operand is exact in TF32 (lo twin all zero, e.g. binary
                             // w8a inputs) -- its lo tile is neither loaded nor multiplied
  int trace;              // HB_TRACE builds: record this launch's pipeline timeline
  int trace_slot;         // HB_TRACE builds: 1-based slot for the per-CTA stamps (0 = off)
  int drain_kb;           // > 0: accumulator drain every drain_kb k-blocks (GemmCfg), 0: rotating accumulators
  const float* bias;      // EPI_SIGMOID / EPI_STORE: optional per-column offset added before the op (or null)
};

// Optional pipeline timeline (debug builds, -DHB_TRACE): CTA (0,0,0) records
// globaltimer stamps per role and k-block into hb_trace_buf.
#ifdef HB_TRACE
__device__ unsigned long long hb_trace_buf[4096];
#define HB_STAMP(slot)                                                                   \
  do {                                                                                   \
    if (args.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (slot) < 4096) { \
      unsigned long long t_;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
      hb_trace_buf[(slot)] = t_;                                                         \
    }                                                                                    \
  } while (0)
// per-CTA stamps: [slot][cta][entry, setup done, epilogue start, end]
__device__ unsigned long long hb_trace_cta[8 * 1024 * 4];
#define HB_CTA_STAMP(k)                                                                          \
  do {                                                                                           \
    const int cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);             \
    if (args.trace_slot > 0 && cta_ < 1024) {                                                    \
      unsigned long long t_;                                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
      hb_trace_cta[((args.trace_slot - 1) * 1024 + cta_) * 4 + (k)] = t_;                        \
    }                                                                                            \
  } while (0)
#else
#define HB_CTA_STAMP(k) \
  do {                  \
  } while (0)
#define HB_STAMP(slot) \
  do {                 \
  } while (0)
#endif

#ifndef HB_GEMM_DRAIN
#define HB_GEMM_DRAIN 1
#endif

constexpr int kBM = 128;
constexpr int kBK = 32;  // 32 fp32 = one 128-byte swizzle row

// PAIR: 2-CTA tcgen05 (cta_group::2).  The two CTAs of a cluster pair compute a
// 256 x BN tile: each loads its own 128 rows of A and HALF of the B tile (so
// per-SM TMA ingest and shared-memory operand reads for B halve -- with fp32
// operands and 3xTF32 lo twins the single-CTA kernel was bound by per-SM TMA
// ingest, ~96 KB per k-block), the even CTA issues M=256 MMAs that read both
// CTAs' shared memory and write each CTA's own TMEM lanes.
template <int BN, int PASSES>
struct GemmCfg {
  static constexpr bool PAIR = (PASSES == 3) && (BN >= 64);
  static constexpr int BNL = PAIR ? BN / 2 : BN;  // B rows (K-major) / columns (MN-major) held per CTA
  static constexpr int A_BYTES = kBM * kBK * 4;
  static constexpr int B_BYTES = BNL * kBK * 4;
  static constexpr int OP_BYTES = A_BYTES + B_BYTES;  // raw (hi) operands of one stage
  static constexpr int STAGE_BYTES = OP_BYTES * (PASSES == 3 ? 2 : 1);
  static constexpr int BUDGET = 200 * 1024;
  static constexpr int STAGES_RAW = BUDGET / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int EPI_WARPS = 8;  // two per TMEM lane quarter, alternating 32-column chunks
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  // TMEM accumulators: the tensor core's fp32 accumulation error grows with
  // the number of MMAs chained into one accumulator, so 3xTF32 keeps the two
  // small cross terms in their own accumulator and rotates the hi*hi term over
  // NBIG accumulators by k-block; the epilogue sums them in fp32 registers.
  //
  // Drain mode (args.drain_kb = D > 0; 3xTF32, BN >= 64): instead, each run of
  // D k-blocks puts its three products into a fresh accumulator (two TMEM
  // slots, alternating), which the epilogue warps drain into fp32 registers
  // (round-to-nearest adds) while the tensor core fills the other slot: the
  // truncating accumulation covers 12 D MMAs, not the whole K.  TMEM reads run
  // at ~64 B/cycle per SM, so draining a 128 x BN tile costs ~2.7x the MMA time
  // of one k-block: D = 1 is for the few precision-critical GEMMs, D >= 3
  // hides the drain under the MMAs.
  static constexpr bool DRAIN_OK = (PASSES == 3) && (BN >= 64) && (HB_GEMM_DRAIN != 0);
  static constexpr int NBIG_RAW = PASSES == 3 ? 512 / BN - 1 : 1;
  static constexpr int NBIG = NBIG_RAW > 15 ? 15 : (NBIG_RAW < 1 ? 1 : NBIG_RAW);
  static constexpr int NACC = PASSES == 3 ? NBIG + 1 : 1;
  static constexpr int TMEM_COLS_RAW = (DRAIN_OK && 2 * BN > NACC * BN) ? 2 * BN : NACC * BN;
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
                     const __grid_constant__ CUtensorMap tmA_lo, const __grid_constant__ CUtensorMap tmB_lo,
                     const __grid_constant__ GemmArgs args) {
  using C = GemmCfg<BN, PASSES>;
  constexpr bool PAIR = C::PAIR;
  // args stays in the constant bank (a by-value copy that is modified spills
  // to the stack); the graph-mode per-step values live in registers
  int a_off = args.a_off, b_off = args.b_off;
  float eta = args.eta;
  if (args.ds != nullptr) {
    const int st = static_cast<int>(args.ds->start);
    if (args.a_start) a_off += st;
    if (args.b_start) b_off += st;
    eta = args.ds->eta;
  }
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint64_t* acc_full = tmem_full + 1;  // DRAIN: k-block slot s holds a finished partial
  uint64_t* acc_empty = acc_full + 2;  // DRAIN: slot s drained by every epilogue warp (of both CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) HB_STAMP(6 * 512 + 2);  // CTA start
  if (threadIdx.x == 0) HB_CTA_STAMP(0);
  const uint32_t crank = PAIR ? cluster_ctarank() : 0u;  // 0: MMA-issuing CTA of the pair
  const bool leader = crank == 0;
  // grid: x = M tiles (CTA pairs are x-adjacent: cluster (2,1,1)), y = N tiles, z = K splits
  const int n0 = blockIdx.y * BN;
  const int m0 = blockIdx.x * kBM;
  const int nl0 = n0 + static_cast<int>(crank) * C::BNL;  // this CTA's B slice
  const int kb_begin = blockIdx.z * args.kb_per_split;
  const int kb_end = min(kb_begin + args.kb_per_split, args.kb_total);
  const int nkb = max(kb_end - kb_begin, 0);
  const bool drain = C::DRAIN_OK && args.drain_kb > 0;
  const int dkb = drain ? args.drain_kb : 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (PASSES == 3) {
      tma_prefetch_desc(&tmA_lo);
      tma_prefetch_desc(&tmB_lo);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    // DRAIN: the drain warps publish the summed tile in TMEM (8 arrivals)
    mbar_init(tmem_full, (C::DRAIN_OK && args.drain_kb > 0) ? C::EPI_WARPS : 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], C::EPI_WARPS * (PAIR ? 2 : 1));
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if (PAIR) {
      tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
      tmem_relinquish_pair();
    } else {
      tmem_alloc(tmem_slot, C::TMEM_COLS);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if (PAIR)
    cluster_sync_all();  // the peer's barriers / TMEM must exist before any cross-CTA traffic
  else
    __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) HB_CTA_STAMP(1);
  const uint32_t tmem_base = *tmem_slot;
  // everything above is independent of the previous kernel's output (PDL)
  pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      // completion of both CTAs' loads is counted on the leader's full barrier
      const uint32_t full_leader0 = PAIR ? mapa_shared(smem_u32(&full[0]), 0) : smem_u32(&full[0]);
      const uint32_t stage_tx = C::STAGE_BYTES - (PASSES == 3 && args.a_lo_zero ? C::A_BYTES : 0) -
                                (PASSES == 3 && args.b_lo_zero ? C::B_BYTES : 0);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        HB_STAMP(0 * 512 + i);  // producer: stage free, issuing TMA
        uint8_t* sA = smem + s * C::STAGE_BYTES;
        uint8_t* sB = sA + C::A_BYTES;
        const uint32_t fb = full_leader0 + 8u * s;
        if (leader) mbar_arrive_expect_tx(&full[s], (PAIR ? 2 : 1) * stage_tx);
        const int k0 = (kb_begin + i) * kBK;
#pragma unroll
        for (int h = 0; h < (PASSES == 3 ? 2 : 1); ++h) {
          const CUtensorMap* ma = h ? &tmA_lo : &tmA;
          const CUtensorMap* mb = h ? &tmB_lo : &tmB;
          uint8_t* dA = sA + h * C::OP_BYTES;
          uint8_t* dB = sB + h * C::OP_BYTES;
          if (h && args.a_lo_zero) {
            // exact operand: no lo tile
          } else if (!A_MN) {
            tma_load_2d_to(dA, ma, fb, k0, m0 + a_off, PAIR);
          } else {
#pragma unroll
            for (int j = 0; j < kBM / 32; ++j) tma_load_2d_to(dA + j * 4096, ma, fb, m0 + 32 * j, k0 + a_off, PAIR);
          }
          // this CTA's half of B in 32-wide slices (4 KB: 32 K-major rows, or
          // 32 MN columns x 32 K-lines)
          if (h && args.b_lo_zero) continue;
#pragma unroll
          for (int j = 0; j < C::BNL / 32; ++j) {
            const int c0 = B_MN ? nl0 + 32 * j : k0;
            const int c1 = B_MN ? k0 + b_off : nl0 + 32 * j + b_off;
            tma_load_2d_to(dB + j * 4096, mb, fb, c0, c1, PAIR);
          }
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = make_idesc_tf32(PAIR ? 2 * kBM : kBM, BN, A_MN, B_MN);
      if (C::DRAIN_OK && drain) {
        uint32_t acc = 0u;
        for (int i = 0; i < nkb; ++i) {
          const int s = i % STAGES;
          const uint32_t ph = (i / STAGES) & 1;
          const int ci = i / dkb;  // chunk of dkb k-blocks -> one fresh accumulator
          const int slot = ci & 1;
          const bool first = (i % dkb) == 0;
          if (first && ci >= 2) mbar_wait(&acc_empty[slot], ((ci >> 1) - 1) & 1);  // drained (both CTAs)
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t aHi = smem_u32(smem + s * C::STAGE_BYTES);
          const uint32_t bHi = aHi + C::A_BYTES;
          const uint32_t t = tmem_base + slot * BN;
          // the two small cross terms first (into the fresh accumulator), then hi*hi
          if (first) acc = 0u;
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            if (!args.a_lo_zero) {
              mma_tf32_cg(t, op_desc(aHi + C::OP_BYTES, kk, A_MN), op_desc(bHi, kk, B_MN), idesc, acc, PAIR);
              acc = 1u;
            }
            if (!args.b_lo_zero) {
              mma_tf32_cg(t, op_desc(aHi, kk, A_MN), op_desc(bHi + C::OP_BYTES, kk, B_MN), idesc, acc, PAIR);
              acc = 1u;
            }
          }
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            mma_tf32_cg(t, op_desc(aHi, kk, A_MN), op_desc(bHi, kk, B_MN), idesc, acc, PAIR);
            acc = 1u;
          }
          mma_commit_cg(&empty[s], PAIR);
          if ((i % dkb) == dkb - 1 || i == nkb - 1) mma_commit_cg(&acc_full[slot], PAIR);
        }
      } else
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&full[s], ph);
        HB_STAMP(1 * 512 + i);  // MMA: operands ready, issuing
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
            // (at most one operand of a launch is exact, so t_small is always written)
            if (!args.a_lo_zero) mma_tf32_cg(t_small, al, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u, PAIR);
            if (!args.b_lo_zero)
              mma_tf32_cg(t_small, ah, bl, idesc, (args.a_lo_zero && i == 0 && kk == 0) ? 0u : 1u, PAIR);
            mma_tf32_cg(t_big, ah, bh, idesc, (i >= C::NBIG || kk > 0) ? 1u : 0u, PAIR);
          } else {
            mma_tf32_cg(tmem_base, ah, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u, PAIR);
          }
        }
        // frees the smem stage of both CTAs once these MMAs retire
        mma_commit_cg(&empty[s], PAIR);
        HB_STAMP(2 * 512 + i);  // MMA: issue done
      }
      if (!drain) mma_commit_cg(tmem_full, PAIR);  // accumulators complete (immediate if nkb == 0)
    }
  } else if (C::DRAIN_OK && drain && warp >= 4 && warp < 4 + C::EPI_WARPS) {
    // ------------------------------------- DRAIN: k-block partials -> registers
    // warp (q, h) owns TMEM lane quarter q and column half h of the tile
    constexpr int HC = BN / 2;  // columns per warp
    const int ew = warp - 4, q = ew & 3, h = ew >> 2;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + h * HC;
    const uint32_t leader_empty = PAIR ? mapa_shared(smem_u32(&acc_empty[0]), 0) : smem_u32(&acc_empty[0]);
    float sum[HC];
#pragma unroll
    for (int j = 0; j < HC; ++j) sum[j] = 0.f;
    const int nchunks = (nkb + dkb - 1) / dkb;
    for (int i = 0; i < nchunks; ++i) {
      const int slot = i & 1;
      mbar_wait(&acc_full[slot], (i >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < HC / 32; ++j) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(lane_base + slot * BN + 32 * j, r);
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 32; ++k) sum[32 * j + k] += __uint_as_float(r[k]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_empty + 8u * slot);
    }
    // publish the summed tile in slot 0 for the common epilogue below (every
    // MMA of this tile has retired: the last k-block's slot was just drained)
#pragma unroll
    for (int j = 0; j < HC / 32; ++j) {
      uint32_t r[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) r[k] = __float_as_uint(sum[32 * j + k]);
      tmem_st_32x32b_x32(lane_base + 32 * j, r);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(tmem_full);
  }
  // The producer / MMA / allocator warps (0-3) are idle once the accumulators
  // are complete, so they join the epilogue (12 warps, 3 per TMEM lane
  // quarter) -- the epilogue is the serialized tail of a CTA.  The fused
  // split-K rendezvous keeps its own 8-warp accounting.
  constexpr bool ALL_EPI = (EPI != EPI_SPLIT_SGD);
  if (ALL_EPI || (warp >= 4 && warp < 4 + C::EPI_WARPS)) {
    // ---------------------------------------------------------- epilogue
    // TMEM -> registers (thread = row) -> per-warp smem transpose -> coalesced
    // float4 global traffic (8 lanes per 128-byte row segment).  The mainloop
    // is finished once tmem_full fires, so stage 0 is reused as staging space.
    const int ew = ALL_EPI ? warp : warp - 4;
    const int q = ew & 3;          // TMEM lane quarter owned by this warp (warp % 4)
    const int half = ew >> 2;      // which interleaved 32-column chunks
    constexpr int NSLOT = ALL_EPI ? (4 + C::EPI_WARPS) / 4 : C::EPI_WARPS / 4;
    constexpr int CSTEP = 32 * NSLOT;
    // The epilogue's second operand (A_l for dX, W for the SGD update) does not
    // depend on the accumulator: it is loaded for a whole chunk at once (the
    // first chunk while the mainloop is still running) so its HBM latency is
    // paid once per chunk instead of once per 4-row group.
    constexpr bool HAS_PRE = (EPI == EPI_DSIG || EPI == EPI_SGD);
    float4 pre[8];
    auto load_pre = [&](int cc, float4(&dst)[8]) {
#pragma unroll
      for (int g = 0; g < 8; ++g) dst[g] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!HAS_PRE) return;
      const int gnn = n0 + cc + (lane & 7) * 4;
      const int left = args.N - gnn;
      if (cc >= BN || left <= 0) return;
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const long long gr = static_cast<long long>(m0) + q * 32 + 4 * g + (lane >> 3);
        if (gr >= args.M) continue;
        const float* ptr = (EPI == EPI_DSIG) ? args.aux + gr * args.ld_aux + gnn : args.out + gr * args.ldo + gnn;
        const bool vec = (EPI == EPI_DSIG) ? ((args.ld_aux & 3) == 0) : ((args.ldo & 3) == 0);
        if (vec && left >= 4) {
          dst[g] = *reinterpret_cast<const float4*>(ptr);
        } else {
          dst[g].x = ptr[0];
          if (left > 1) dst[g].y = ptr[1];
          if (left > 2) dst[g].z = ptr[2];
          if (left > 3) dst[g].w = ptr[3];
        }
      }
    };
    load_pre(32 * half, pre);
    mbar_wait(tmem_full, 0);
    __syncwarp();  // warps 0 / 1: lane 0 is back from its producer / MMA role
    if (threadIdx.x == 128) pdl_trigger();  // mainloop done: the next kernel may start its setup
    if (threadIdx.x == 128) HB_STAMP(6 * 512 + 0);  // epilogue start
    if (threadIdx.x == 128) HB_CTA_STAMP(2);
    tc_fence_after();
    constexpr int TP = 36;  // padded tile row (floats): conflict-free v4 in and out
    float* tile = reinterpret_cast<float*>(smem) + ew * 32 * TP;
    const bool vec_out = (args.ldo & 3) == 0;
    const bool vec_grad = (args.ld_grad & 3) == 0;
    const int sub_r = lane >> 3;       // row within a group of 4
    const int sub_c = (lane & 7) * 4;  // column quad within the 32-column chunk
#pragma unroll 1
    for (int c = 32 * half; c < BN; c += CSTEP) {
      if (c != 32 * half) load_pre(c, pre);  // one latency per chunk, overlapping the TMEM loads
      const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + c;
      float v[32];
      {
        uint32_t r[32];
        // small-term accumulator first, then the hi*hi accumulators (only those
        // the k loop actually wrote)
        tmem_ld_32x32b_x32(lane_addr + (drain ? 0 : (C::NACC - 1) * BN), r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (drain || nkb > 0) ? __uint_as_float(r[j]) : 0.f;
        if (C::NACC > 1 && !drain) {
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
      if (threadIdx.x == 128) HB_STAMP(7 * 512 + 4 * (c / CSTEP) + 0);  // epi: TMEM loaded
      const int n = n0 + c;
      if (n >= args.N) continue;  // warp-uniform (and then so are all later chunks)
#ifdef HB_DEBUG_NO_EPI_STORE
      if (v[0] == 12345.f) args.out[0] = v[1];  // timing experiment only: keep the TMEM loads alive
      continue;
#endif
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(tile + lane * TP + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      __syncwarp();
      if (threadIdx.x == 128) HB_STAMP(7 * 512 + 4 * (c / CSTEP) + 1);  // epi: transposed
      const int gn = n + sub_c;
      const int nleft = args.N - gn;  // columns of this quad still inside N
#pragma unroll
      for (int rr = 0; rr < 32; rr += 4) {
        const int tr = rr + sub_r;
        const long long grow = static_cast<long long>(m0) + q * 32 + tr;
        const float4 acc = *reinterpret_cast<const float4*>(tile + tr * TP + sub_c);
        if (nleft <= 0) continue;
        float o[4] = {acc.x, acc.y, acc.z, acc.w};
        bool write = grow < args.M;
        if ((EPI == EPI_SIGMOID || EPI == EPI_STORE) && args.bias != nullptr) {
#pragma unroll
          for (int k = 0; k < 4; ++k) o[k] += k < nleft ? args.bias[gn + k] : 0.f;
        }
        if (EPI == EPI_SIGMOID) {
#ifndef HB_DEBUG_EPI_NO_SIGMOID
#pragma unroll
          for (int k = 0; k < 4; ++k) o[k] = sigmoidf_fast(o[k]);
#endif
        } else if (EPI == EPI_DSIG) {
          if (write) {
            const float4 t4 = pre[rr / 4];
            const float av[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) o[k] = o[k] * (av[k] * (1.f - av[k]));
          } else if (grow < args.m_zero_rows) {
            write = true;
#pragma unroll
            for (int k = 0; k < 4; ++k) o[k] = 0.f;
          }
        }
        if (!write) continue;
#ifdef HB_DEBUG_EPI_NO_GLOBAL
        if (o[0] == 12345.f) args.out[0] = o[1];
        continue;
#endif
        if (EPI == EPI_SGD) {
          float* wp = args.out + grow * args.ldo + gn;
          float* lp = args.out_lo != nullptr ? args.out_lo + grow * args.ldo + gn : nullptr;
          if (vec_out && nleft >= 4) {
            float4 w4 = pre[rr / 4];
            w4.x -= eta * o[0];
            w4.y -= eta * o[1];
            w4.z -= eta * o[2];
            w4.w -= eta * o[3];
            *reinterpret_cast<float4*>(wp) = w4;
            if (lp != nullptr) *reinterpret_cast<float4*>(lp) = lo4(w4);
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (k < nleft) {
                const float prev = k == 0 ? pre[rr / 4].x : k == 1 ? pre[rr / 4].y : k == 2 ? pre[rr / 4].z : pre[rr / 4].w;
                const float nw = prev - eta * o[k];
                wp[k] = nw;
                if (lp != nullptr) lp[k] = tf32_lo(nw);
              }
          }
          if (args.grad != nullptr) {
            float* gp = args.grad + grow * args.ld_grad + gn;
            if (vec_grad && nleft >= 4) {
              *reinterpret_cast<float4*>(gp) = make_float4(o[0], o[1], o[2], o[3]);
            } else {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (k < nleft) gp[k] = o[k];
            }
          }
        } else {
          constexpr bool SLAB = (EPI == EPI_PARTIAL || EPI == EPI_SPLIT_SGD);
          float* op = args.out + (SLAB ? static_cast<long long>(blockIdx.z) * args.split_stride : 0LL) +
                      grow * args.ldo + gn;
          float* lp = (!SLAB && args.out_lo != nullptr) ? args.out_lo + grow * args.ldo + gn : nullptr;
          if (vec_out && nleft >= 4) {
            const float4 v4 = make_float4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<float4*>(op) = v4;
            if (lp != nullptr) *reinterpret_cast<float4*>(lp) = lo4(v4);
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (k < nleft) {
                op[k] = o[k];
                if (lp != nullptr) lp[k] = tf32_lo(o[k]);
              }
          }
        }
      }
    }
  }

  if (EPI == EPI_SPLIT_SGD && warp >= 4) {
    // ---- split-K rendezvous + distributed reduction (epilogue warps only)
    constexpr int ET = 32 * C::EPI_WARPS;
    const int S = gridDim.z;
    int* arrive = args.tile_sync + 2 * (blockIdx.x + gridDim.x * blockIdx.y);
    named_bar_sync(1, ET);  // this CTA's partial tile is fully stored
    if (threadIdx.x == 128) {
      __threadfence();
      atomicAdd(arrive, 1);
      long long spins = 0;
      while (ld_acquire_gpu(arrive) < S) {
        __nanosleep(64);
        if (++spins > (1ll << 25)) {  // seconds: the split CTAs were not co-resident
          printf("hogbatch_b200: split-K rendezvous timed out (tile %d,%d)\n", blockIdx.x, blockIdx.y);
          __trap();
        }
      }
      __threadfence();
    }
    named_bar_sync(1, ET);
    const int rows_per = (kBM + S - 1) / S;
    const int r0 = m0 + static_cast<int>(blockIdx.z) * rows_per;
    const int r1 = min(min(r0 + rows_per, m0 + kBM), args.M);
    const int ncols = min(BN, args.N - n0);
    const int quads = ncols / 4;  // host guarantees N % 4 == 0
    const int items = max(r1 - r0, 0) * quads;
    for (int it = threadIdx.x - 128; it < items; it += ET) {
      const int r = r0 + it / quads;
      const int cc = n0 + 4 * (it % quads);
      const float* part = args.out + static_cast<long long>(r) * args.ldo + cc;
      float4 g = __ldcg(reinterpret_cast<const float4*>(part));
      for (int sl = 1; sl < S; ++sl) {
        const float4 t = __ldcg(reinterpret_cast<const float4*>(part + sl * args.split_stride));
        g.x += t.x;
        g.y += t.y;
        g.z += t.z;
        g.w += t.w;
      }
      float4* wp = reinterpret_cast<float4*>(args.w + r * args.ldw + cc);
      float4 wv = *wp;
      wv.x -= eta * g.x;
      wv.y -= eta * g.y;
      wv.z -= eta * g.z;
      wv.w -= eta * g.w;
      *wp = wv;
      if (args.w_lo != nullptr) *reinterpret_cast<float4*>(args.w_lo + r * args.ldw + cc) = lo4(wv);
      if (args.grad != nullptr) *reinterpret_cast<float4*>(args.grad + r * args.ld_grad + cc) = g;
    }
    named_bar_sync(1, ET);
    // the partial slabs of this share are dead: drop their L2 lines without
    // the HBM write-back (they were written by this launch and read just above)
    if ((args.ldo & 31) == 0 && (ncols & 31) == 0) {
      const int lines_per_row = ncols / 32;
      const int nl = max(r1 - r0, 0) * lines_per_row * S;
      for (int it = threadIdx.x - 128; it < nl; it += ET) {
        const int sl = it % S;
        const int rl = it / S;
        const int r = r0 + rl / lines_per_row;
        const int cc = n0 + 32 * (rl % lines_per_row);
        discard_l2_line(args.out + sl * args.split_stride + static_cast<long long>(r) * args.ldo + cc);
      }
    }
    if (threadIdx.x == 128) {
      // the last CTA out re-arms the counters (every CTA has passed the wait)
      if (atomicAdd(arrive + 1, 1) == S - 1) {
        arrive[0] = 0;
        arrive[1] = 0;
        __threadfence();
      }
    }
  }

  tc_fence_before();
  if (PAIR)
    cluster_sync_all();  // no CTA may exit while its peer can still touch its smem / barriers
  else
    __syncthreads();
  if (threadIdx.x == 0) HB_STAMP(6 * 512 + 1);  // CTA end
  if (threadIdx.x == 0) HB_CTA_STAMP(3);
  if (warp == 2) {
    tc_fence_after();
    if (PAIR)
      tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
    else
      tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace hb
