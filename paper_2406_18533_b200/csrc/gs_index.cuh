// gs_index.cuh -- the backward index shared by gs_project (writer) and gs_adam_step
// (reader): per-Gaussian bitmask over buckets k = d * n_views + v (destination-major), plus
// each CTA's exclusive base per bucket.  A record's send position is
//   base[k][cta] + (records of bucket k from lower warps of the CTA) + (lower lanes of the warp),
// recomputed identically by both kernels from the same masks with warp ballots.
#pragma once
#include <stdint.h>

#include "gs_device.cuh"

namespace gsd {

constexpr int kMaxBuckets = 256;  // n_views * world
constexpr int kMaxWords = kMaxBuckets / 32;
constexpr int kWarps = kBlock / 32;

struct gs_index_layout {
  int NW;
  int64_t ncta;
  size_t base_off, bytes;
};

inline gs_index_layout index_layout(int64_t n, int b, int G) {
  gs_index_layout L;
  int nb = b * G;
  L.NW = (nb + 31) / 32;
  L.ncta = (n + kBlock - 1) / kBlock;
  size_t mask_bytes = (size_t)L.NW * (size_t)n * 4;
  L.base_off = (mask_bytes + 255) & ~(size_t)255;
  L.bytes = L.base_off + ((size_t)nb * (size_t)L.ncta + 1) * 8;
  return L;
}

__device__ __forceinline__ void set_bit(uint32_t* m, int k) {
#pragma unroll
  for (int w = 0; w < kMaxWords; w++)
    if (w == (k >> 5)) m[w] |= 1u << (k & 31);
}
__device__ __forceinline__ bool get_bit(const uint32_t* m, int k) {
  uint32_t word = 0;
#pragma unroll
  for (int w = 0; w < kMaxWords; w++)
    if (w == (k >> 5)) word = m[w];
  return (word >> (k & 31)) & 1u;
}
__device__ __forceinline__ bool view_in_mask(const uint32_t* m, int v, int b, int G) {
  bool any = false;
  for (int d = 0; d < G; d++) any |= get_bit(m, d * b + v);
  return any;
}
__device__ __forceinline__ bool view_in_union(const uint32_t* u, int v, int b, int G) {
  return view_in_mask(u, v, b, G);
}

__device__ __forceinline__ void load_masks(const uint32_t* __restrict__ maskw, int64_t n, int64_t i,
                                           int NW, uint32_t* m) {
#pragma unroll
  for (int w = 0; w < kMaxWords; w++) m[w] = (w < NW && i < n) ? maskw[(int64_t)w * n + i] : 0u;
}

// Phase 1: zero the per-warp counters, form the warp's union masks u, count each bucket of
// the union per warp into s_cnt[wid * nb + k].  Ends with __syncthreads().
__device__ __forceinline__ void cta_rank_phase1(const uint32_t* m, uint32_t* u, int NW, int nb,
                                                int* s_cnt) {
  for (int k = threadIdx.x; k < kWarps * nb; k += kBlock) s_cnt[k] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int w = 0; w < kMaxWords; w++) {
    u[w] = w < NW ? __reduce_or_sync(0xffffffffu, m[w]) : 0u;
    uint32_t uu = u[w];
    while (uu) {
      int bit = __ffs(uu) - 1;
      uu &= uu - 1;
      unsigned bal = __ballot_sync(0xffffffffu, (m[w] >> bit) & 1u);
      if (lane == 0) s_cnt[wid * nb + w * 32 + bit] = __popc(bal);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ int warp_prefix(const int* s_cnt, int wid, int nb, int k) {
  int s = 0;
  for (int w = 0; w < wid; w++) s += s_cnt[w * nb + k];
  return s;
}

}  // namespace gsd
