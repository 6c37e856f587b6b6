// Replica averaging over peer memory (NVLink / NVSwitch P2P, or CUDA IPC
// between processes): the GPU-replica merge of SURVEY.md §8e without a
// collective library.  Every rank owns one exchange buffer
//
//   [0, 512)            flags (u64): whole-model pack @0, reduce @1; layer l pack @2+2l, reduce @3+2l;
//                       error word (u32) @ byte 448
//   [512, 512 + 4 n')   the packed fp32 model ("flat", layer-major, dense rows, each layer's segment
//                       padded to a multiple of 4 floats)
//
// and maps every peer's buffer (same process: the raw pointer with peer access
// enabled; another process: cudaIpcOpenMemHandle).  One merge is
//
//   pack own model -> flat; signal pack=g
//   wait until every rank signalled pack=g
//   reduce slice r of the flats: v = (flat_0 + flat_1 + ... + flat_{n-1}) * (1/n),
//      summed in rank order (identical bits on every rank), written into every
//      rank's flat (each rank owns a disjoint slice, so no two ranks touch the
//      same word); signal red=g
//   wait until every rank signalled red=g; unpack flat -> model (+ lo twins)
//
// i.e. a one-shot reduce-scatter + all-gather in a single kernel, reading and
// writing peers directly over NVLink: each rank moves 2(n-1)/n of the model in
// and out, like a ring allreduce, with one hop.  The waits are single-warp
// kernels polling the peers' flags with acquire loads (system scope), bounded
// by a timeout that raises the error word instead of hanging the GPU.
#pragma once

#include <cstdint>

#include "hb_kernels.cuh"

namespace hb {

constexpr int kMaxPeers = 8;
constexpr size_t kPeerHeader = 512;  // bytes before the flat model in an exchange buffer
constexpr int kPeerErrWord = 448 / 8;  // u64 index of the error word

struct PeerTable {
  float* flat[kMaxPeers];
  unsigned long long* flag[kMaxPeers];  // base of each rank's flag block
  int n;
  int rank;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The merge generation g: by value (eager steps) or from the step record in
// device memory (captured graphs replay with the current step's value).
__device__ __forceinline__ unsigned long long merge_gen(const DevStep* ds, unsigned long long g) {
  return ds != nullptr ? ds->merge_gen : g;
}

// flag word `which` (u64 index) of this rank := g, after everything this
// stream wrote before (kernel boundary + system fence)
__global__ void peer_signal_kernel(unsigned long long* flag_base, int which, unsigned long long g,
                                   const DevStep* ds = nullptr) {
  __threadfence_system();
  st_release_sys_u64(flag_base + which, merge_gen(ds, g));
}

// thread q waits for rank q's flag `which` to reach g (timeout: error word, no hang)
__global__ void peer_wait_kernel(const __grid_constant__ PeerTable t, int which, unsigned long long g,
                                 unsigned long long timeout_ns, const DevStep* ds = nullptr) {
  const int q = threadIdx.x;
  if (q >= t.n) return;
  g = merge_gen(ds, g);
  const unsigned long long* f = t.flag[q] + which;
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_sys_u64(f) < g) {
    if (globaltimer_ns() - t0 > timeout_ns) {
      atomicExch(reinterpret_cast<unsigned*>(t.flag[t.rank] + kPeerErrWord), 1u + static_cast<unsigned>(q));
      break;
    }
    __nanosleep(256);
  }
}

// slice `rank` of the n-way average of flat[base, base + n_elems) (base a
// multiple of 4), written back into every rank's flat
__global__ void __launch_bounds__(256) peer_reduce_kernel(PeerTable t, long long n_elems, float scale,
                                                          long long base = 0) {
  for (int q = 0; q < t.n; ++q) t.flat[q] += base;
  const long long n4 = n_elems / 4;
  const long long a = n4 * t.rank / t.n, b = n4 * (t.rank + 1) / t.n;
  for (long long i = a + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < b;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(t.flat[0])[i];
    for (int q = 1; q < t.n; ++q) {
      const float4 v = reinterpret_cast<const float4*>(t.flat[q])[i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    acc.x *= scale;
    acc.y *= scale;
    acc.z *= scale;
    acc.w *= scale;
    for (int q = 0; q < t.n; ++q) reinterpret_cast<float4*>(t.flat[q])[i] = acc;
  }
  if (t.rank == t.n - 1 && blockIdx.x == 0) {  // the < 4 tail elements
    for (long long i = 4 * n4 + threadIdx.x; i < n_elems; i += blockDim.x) {
      float acc = t.flat[0][i];
      for (int q = 1; q < t.n; ++q) acc += t.flat[q][i];
      acc *= scale;
      for (int q = 0; q < t.n; ++q) t.flat[q][i] = acc;
    }
  }
}

}  // namespace hb

namespace hb {
// L2 gather ceiling probe (bench.py's "l2" roofline for the CSR kernels): each
// warp gathers `per_warp` pseudo-random whole rows of a (rows x cols) fp32
// matrix -- the access pattern of the CSR SpMM (one W0^T row per nonzero) --
// with UNROLL rows in flight per lane, and reduces them into one float.
template <int UNROLL>
__global__ void __launch_bounds__(256) l2_gather_probe_kernel(const float* __restrict__ m, long long rows, int cols,
                                                              int per_warp, float* __restrict__ out) {
  const long long warp = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int k = 0; k < per_warp; k += UNROLL) {
    float4 v[UNROLL][8];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      unsigned h = static_cast<unsigned>(warp * 2654435761ull + (k + u) * 40503u);
      h ^= h >> 15;
      h *= 2246822519u;
      h ^= h >> 13;
      const float4* row = reinterpret_cast<const float4*>(m + (h % rows) * cols);
#pragma unroll
      for (int t = 0; t < 8; ++t) v[u][t] = (4 * lane + 128 * t < cols) ? __ldg(row + lane + 32 * t) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
#pragma unroll
      for (int t = 0; t < 8; ++t) acc += v[u][t].x + v[u][t].y + v[u][t].z + v[u][t].w;
  }
  if (acc == 1234.5f) out[warp] = acc;  // keep the loads alive
}
}  // namespace hb
