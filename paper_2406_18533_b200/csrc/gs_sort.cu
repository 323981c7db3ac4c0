#include <chrono>
#include <cstdio>
// gs_sort.cu -- A3: Z-buffer build ("iterates over intersecting Gaussians in
// increasing depth"; App. A.2 "indices of intersecting gaussians for each pixel").
//
// B200 design (differs from the prior art's global (tile|depth) 64-bit radix sort):
//  1. per-block list lengths without per-pair atomics: every record adds +1/-1 at the four
//     corners of its tile rectangle in a 2D difference array of its view (4 atomics per
//     record), a row scan and a column scan give each block's count;
//  2. exclusive scan of the owned blocks' counts -> tile_range (host sync for capacity);
//  3. placement: each record appends key = depth_bits << 32 | recv_idx to every owned block
//     of its rectangle (one atomic cursor per pair);
//  4. per-block sort of the keys in shared memory (bitonic, <= 4096 keys) or, for the rare
//     longer lists, chunk sort + merge-path merges in global memory.
// (depth, recv_idx) is unique within a block and recv_idx is ascending in gid within a
// view (A1/A2 ordering), so the result is exactly the (depth, gid) order of O11 (R7)
// whatever the placement order: no stable sort is needed.
#include <algorithm>
#include <cstdlib>

#include "gs_device.cuh"
#include "gs_internal.h"

using namespace gsd;

namespace {

constexpr int kSortThreads = 256;
constexpr int kSmallCap = 4096;  // keys sorted in shared memory (32 KB)

__global__ void k_rect_diff(const gs_rec* __restrict__ rec, int64_t n_recv, gs_geom geo, int v_lo,
                            int v_hi, int* __restrict__ diff, int64_t* __restrict__ n_tiles) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j > n_recv) return;
  if (j == n_recv) { n_tiles[j] = 0; return; }
  n_tiles[j] = 0;
  float4 a = rec[j].a;
  int v = (int)(__float_as_uint(rec[j].d.w) & 31u);
  if (v < v_lo || v > v_hi) return;
  int tx0, tx1, ty0, ty1;
  if (!rect_of(a.x, a.y, a.w, geo.Wt, geo.Ht, tx0, tx1, ty0, ty1)) return;
  n_tiles[j] = (int64_t)(tx1 - tx0 + 1) * (ty1 - ty0 + 1);
  const int ld = geo.Wt + 1;
  int* D = diff + (int64_t)(v - v_lo) * (geo.Ht + 1) * ld;
  atomicAdd(&D[ty0 * ld + tx0], 1);
  atomicAdd(&D[ty0 * ld + tx1 + 1], -1);
  atomicAdd(&D[(ty1 + 1) * ld + tx0], -1);
  atomicAdd(&D[(ty1 + 1) * ld + tx1 + 1], 1);
}

__global__ void k_diff_rows(int* diff, int nrows, int ld) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int* p = diff + (int64_t)r * ld;
  int s = 0;
  for (int x = 0; x < ld; x++) p[x] = (s += p[x]);
}

__global__ void k_diff_cols(int* diff, int nviews, int rows, int ld) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nviews * ld) return;
  int v = t / ld, x = t % ld;
  int* p = diff + (int64_t)v * rows * ld + x;
  int s = 0;
  for (int y = 0; y < rows; y++) p[(int64_t)y * ld] = (s += p[(int64_t)y * ld]);
}

__global__ void k_owned_counts(const int* diff, gs_geom geo, int64_t B_lo, int64_t n_owned, int v_lo,
                               int64_t* counts) {
  int64_t lb = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (lb > n_owned) return;
  if (lb == n_owned) { counts[lb] = 0; return; }
  int64_t beta = B_lo + lb, v = beta / geo.per_view, loc = beta % geo.per_view;
  int tx = (int)(loc % geo.Wt), ty = (int)(loc / geo.Wt);
  counts[lb] = diff[((v - v_lo) * (geo.Ht + 1) + ty) * (int64_t)(geo.Wt + 1) + tx];
}

__global__ void k_to_range(const int64_t* off, int64_t n_owned, int32_t* range, int32_t* cursor) {
  int64_t lb = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (lb > n_owned) return;
  range[lb] = (int32_t)off[lb];
  if (lb < n_owned) cursor[lb] = (int32_t)off[lb];
}

// Pair-parallel placement: CTA c owns pairs [c*kPlacePairs, (c+1)*kPlacePairs) of the
// (record, tile-of-its-rectangle) enumeration (pair_start = exclusive scan of tile counts);
// every record has >= 1 tile, so at most kPlacePairs + 1 records overlap a CTA.  Their
// rectangles are staged in shared memory, each thread binary-searches the record of each of
// its pairs there and appends key = depth_bits << 32 | recv_idx to the block's list.
constexpr int kPlaceThreads = 256;
constexpr int kPlacePairs = 1024;

__global__ void __launch_bounds__(kPlaceThreads) k_place(
    const gs_rec* __restrict__ rec, int64_t n_recv, const int64_t* __restrict__ pair_start, int64_t n_full,
    gs_geom geo, int64_t B_lo, int64_t B_hi, int32_t* __restrict__ cursor, unsigned long long* __restrict__ keys) {
  __shared__ int64_t s_start[kPlacePairs + 2];
  __shared__ int s_tx0[kPlacePairs + 1], s_ty0[kPlacePairs + 1], s_w[kPlacePairs + 1], s_v[kPlacePairs + 1];
  __shared__ unsigned s_depth[kPlacePairs + 1];
  __shared__ int64_t s_jlo;
  __shared__ int s_nr;
  const int64_t P0 = (int64_t)blockIdx.x * kPlacePairs;
  const int64_t P1 = min(P0 + kPlacePairs, n_full);
  if (threadIdx.x == 0) {
    // first record whose range contains P0: last j with pair_start[j] <= P0
    int64_t lo = 0, hi = n_recv;  // pair_start[n_recv] = n_full > P0
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (pair_start[mid] <= P0) lo = mid; else hi = mid;
    }
    int64_t lo2 = lo, hi2 = n_recv;  // last j with pair_start[j] <= P1 - 1
    while (hi2 - lo2 > 1) {
      int64_t mid = (lo2 + hi2) >> 1;
      if (pair_start[mid] <= P1 - 1) lo2 = mid; else hi2 = mid;
    }
    s_jlo = lo;
    s_nr = (int)(lo2 - lo + 1);
  }
  __syncthreads();
  const int64_t jlo = s_jlo;
  const int nr = s_nr;
  for (int r = threadIdx.x; r < nr; r += kPlaceThreads) {
    const int64_t j = jlo + r;
    s_start[r] = pair_start[j];
    const float4 a = rec[j].a;
    int tx0, tx1, ty0, ty1;
    rect_of(a.x, a.y, a.w, geo.Wt, geo.Ht, tx0, tx1, ty0, ty1);
    s_tx0[r] = tx0;
    s_ty0[r] = ty0;
    s_w[r] = tx1 - tx0 + 1;
    s_v[r] = (int)(__float_as_uint(rec[j].d.w) & 31u);
    s_depth[r] = __float_as_uint(a.z);
  }
  if (threadIdx.x == 0) s_start[nr] = pair_start[jlo + nr];
  __syncthreads();
  for (int64_t pp = P0 + threadIdx.x; pp < P1; pp += kPlaceThreads) {
    int lo = 0, hi = nr;  // last r with s_start[r] <= pp
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (s_start[mid] <= pp) lo = mid; else hi = mid;
    }
    const int t = (int)(pp - s_start[lo]), w = s_w[lo];
    const int ty = s_ty0[lo] + t / w, tx = s_tx0[lo] + t % w;
    const int64_t beta = (int64_t)s_v[lo] * geo.per_view + (int64_t)ty * geo.Wt + tx;
    if (beta < B_lo || beta >= B_hi) continue;
    const int pos = atomicAdd(&cursor[beta - B_lo], 1);
    keys[pos] = ((unsigned long long)s_depth[lo] << 32) | (unsigned long long)(jlo + lo);
  }
}

// Bitonic network over P (power of two) keys in shared memory.  Compare-exchange t pairs
// i = 2t - (t & (j-1)) with i + j; for j <= 32 a warp's 32 consecutive t touch only its own
// 64 keys, so those stages synchronise with __syncwarp (when P/2 is a multiple of 32).
__device__ __forceinline__ void bitonic_smem(unsigned long long* s, int P) {
  const bool warp_local = (P / 2) % 32 == 0;
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < P / 2; t += kSortThreads) {
        const int i = 2 * t - (t & (j - 1)), l = i + j;
        const bool up = (i & k) == 0;
        const unsigned long long x = s[i], y = s[l];
        if ((x > y) == up) { s[i] = y; s[l] = x; }
      }
      if (j <= 32 && warp_local && (j > 1 || k < P)) {
        // next stage is warp-local too unless this was the last stage of a merge whose
        // successor has j' = k (k >= 64 crosses warps)
        const int jn = j > 1 ? j >> 1 : k;  // next stage's j
        if (jn <= 32) { __syncwarp(); continue; }
      }
      __syncthreads();
    }
  __syncthreads();
}

// Register bitonic sort of up to 32*E keys held by one warp, striped: key i = e*32 + lane.
// Stages with j >= 32 compare two registers of the same lane; j < 32 exchange with lane^j.
template <int E>
__device__ __forceinline__ void warp_bitonic(unsigned long long (&v)[E], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int je = j >> 5;
#pragma unroll
        for (int e = 0; e < E; e++) {
          if ((e & je) == 0) {
            const int i = e * 32 + lane;
            const bool up = (i & k) == 0;
            const unsigned long long a = v[e], b = v[e | je];
            if ((a > b) == up) { v[e] = b; v[e | je] = a; }
          }
        }
      } else {
        const bool lower = (lane & j) == 0;
#pragma unroll
        for (int e = 0; e < E; e++) {
          const int i = e * 32 + lane;
          const bool up = (i & k) == 0;
          const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[e], j);
          const unsigned long long mn = v[e] < o ? v[e] : o, mx = v[e] < o ? o : v[e];
          v[e] = (lower == up) ? mn : mx;
        }
      }
    }
  }
}

template <int E>
__device__ __forceinline__ void warp_sort_segment(const unsigned long long* __restrict__ keys,
                                                  uint32_t* __restrict__ out, int n, int lane) {
  unsigned long long v[E];
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int i = e * 32 + lane;
    v[e] = i < n ? keys[i] : ~0ull;
  }
  warp_bitonic<E>(v, lane);
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int i = e * 32 + lane;
    if (i < n) out[i] = (uint32_t)v[e];
  }
}

constexpr int kWarpCap = 256;  // lists up to this length are sorted by one warp in registers

// One warp per owned block: lists of <= 256 keys are sorted in registers; longer ones are
// queued for the shared-memory CTA sort (<= kSmallCap) or the merge sort (longer).
__global__ void __launch_bounds__(kSortThreads) k_sort_warp(const int32_t* __restrict__ range, int64_t n_owned,
                                                            const unsigned long long* __restrict__ keys,
                                                            uint32_t* __restrict__ sorted_idx, int32_t* mid_list,
                                                            int32_t* n_mid, int32_t* large_list, int32_t* n_large) {
  const int lane = threadIdx.x & 31;
  const int64_t lb = (int64_t)blockIdx.x * (kSortThreads / 32) + (threadIdx.x >> 5);
  if (lb >= n_owned) return;
  const int beg = range[lb], n = range[lb + 1] - beg;
  if (n <= 1) {
    if (n == 1 && lane == 0) sorted_idx[beg] = (uint32_t)keys[beg];
    return;
  }
  if (n > kWarpCap) {
    if (lane == 0) {
      if (n > kSmallCap) large_list[atomicAdd(n_large, 1)] = (int32_t)lb;
      else mid_list[atomicAdd(n_mid, 1)] = (int32_t)lb;
    }
    return;
  }
  if (n <= 32) warp_sort_segment<1>(keys + beg, sorted_idx + beg, n, lane);
  else if (n <= 64) warp_sort_segment<2>(keys + beg, sorted_idx + beg, n, lane);
  else if (n <= 128) warp_sort_segment<4>(keys + beg, sorted_idx + beg, n, lane);
  else warp_sort_segment<8>(keys + beg, sorted_idx + beg, n, lane);
}

// Shared-memory bitonic sort of the queued medium lists (kWarpCap < n <= kSmallCap);
// persistent CTAs take list after list.
__global__ void __launch_bounds__(kSortThreads) k_sort_small(const int32_t* __restrict__ range,
                                                             const unsigned long long* __restrict__ keys,
                                                             uint32_t* __restrict__ sorted_idx,
                                                             const int32_t* __restrict__ mid_list,
                                                             const int32_t* n_mid, int32_t* next) {
  __shared__ unsigned long long s[kSmallCap];
  __shared__ int s_item;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(next, 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= *n_mid) return;
    const int lb = mid_list[item];
    const int beg = range[lb], n = range[lb + 1] - beg;
    int P = 2;
    while (P < n) P <<= 1;
    for (int i = threadIdx.x; i < P; i += kSortThreads) s[i] = i < n ? keys[beg + i] : ~0ull;
    __syncthreads();
    bitonic_smem(s, P);
    for (int i = threadIdx.x; i < n; i += kSortThreads) sorted_idx[beg + i] = (uint32_t)s[i];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kSortThreads) k_sort_large(const int32_t* __restrict__ range,
                                                             unsigned long long* keys,
                                                             unsigned long long* tmp,
                                                             uint32_t* __restrict__ sorted_idx,
                                                             const int32_t* large_list,
                                                             const int32_t* n_large, int32_t* next) {
  __shared__ unsigned long long s[kSmallCap];
  __shared__ int s_item;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(next, 1);
    __syncthreads();
    int item = s_item;
    __syncthreads();
    if (item >= *n_large) return;
    int lb = large_list[item];
    int beg = range[lb], n = range[lb + 1] - beg;
    unsigned long long* src = keys + beg;
    unsigned long long* dst = tmp + beg;
    // 1. sort chunks of kSmallCap in shared memory
    for (int c0 = 0; c0 < n; c0 += kSmallCap) {
      int m = min(kSmallCap, n - c0);
      for (int i = threadIdx.x; i < kSmallCap; i += kSortThreads) s[i] = i < m ? src[c0 + i] : ~0ull;
      __syncthreads();
      bitonic_smem(s, kSmallCap);
      for (int i = threadIdx.x; i < m; i += kSortThreads) src[c0 + i] = s[i];
      __syncthreads();
    }
    // 2. merge-path merges of sorted runs, ping-pong src <-> dst
    for (int w = kSmallCap; w < n; w <<= 1) {
      for (int p0 = 0; p0 < n; p0 += 2 * w) {
        int na = min(w, n - p0), nbb = max(0, min(w, n - p0 - w));
        const unsigned long long* A = src + p0;
        const unsigned long long* Bv = src + p0 + na;
        int L = na + nbb, per = (L + kSortThreads - 1) / kSortThreads;
        int d0 = min(L, (int)threadIdx.x * per), d1 = min(L, d0 + per);
        // diagonal search: i = elements taken from A among the first d0 outputs
        int lo = max(0, d0 - nbb), hi = min(d0, na);
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (A[mid] < Bv[d0 - 1 - mid]) lo = mid + 1; else hi = mid;
        }
        int ia = lo, ib = d0 - lo;
        for (int d = d0; d < d1; d++) {
          bool takeA = ib >= nbb || (ia < na && A[ia] < Bv[ib]);
          dst[p0 + d] = takeA ? A[ia++] : Bv[ib++];
        }
      }
      __syncthreads();
      unsigned long long* t = src; src = dst; dst = t;
    }
    for (int i = threadIdx.x; i < n; i += kSortThreads) sorted_idx[beg + i] = (uint32_t)src[i];
    __syncthreads();
  }
}


// ---------------------------------------------------------------- radix path (default)
// Depth-presorted, stable block binning: sort the records by depth once (LSD radix over the
// 32 depth bits, stable, so equal depths stay in recv_idx order), emit the (block, record)
// pairs in that order -- each CTA writes a contiguous pair range, coalesced -- then stably
// radix-sort the pairs by owned-block index only (ceil(log2(n_owned + 1)) bits, 2-3 passes).
// Every block's list then comes out in (depth, recv_idx) order, whatever its length: no
// per-block comparison sort, no long-list special case, and traffic linear in the pairs.
// Pairs of non-owned blocks (G > 1, rectangles straddling the partition) get key n_owned and
// sort past the end (they are never written out).
constexpr int kRadixThreads = 256;
constexpr int kRadixItems = 16;
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 4096 elements per CTA
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixPerWarp = kRadixTile / kRadixWarps;   // 512 consecutive elements per warp

// Per-record tile count of the rectangle (0 outside the rank's views); no binning atomics.
__global__ void k_tile_counts(const gs_rec* __restrict__ rec, int64_t n_recv, gs_geom geo, int v_lo, int v_hi,
                              int64_t* __restrict__ n_tiles) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j > n_recv) return;
  int64_t t = 0;
  if (j < n_recv) {
    const float4 a = rec[j].a;
    const int v = (int)(__float_as_uint(rec[j].d.w) & 31u);
    int tx0, tx1, ty0, ty1;
    if (v >= v_lo && v <= v_hi && rect_of(a.x, a.y, a.w, geo.Wt, geo.Ht, tx0, tx1, ty0, ty1))
      t = (int64_t)(tx1 - tx0 + 1) * (ty1 - ty0 + 1);
  }
  n_tiles[j] = t;
}

// tile_range from the block-sorted keys: range[b] = first position with key >= b, for
// b in [0, n_owned] (position n_full stands for key n_owned; keys n_owned are other ranks').
__global__ void k_key_ranges(const uint32_t* __restrict__ keys, int64_t n_full, uint32_t n_owned,
                             int32_t* __restrict__ range) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n_full) return;
  const int64_t k = i < n_full ? (int64_t)keys[i] : (int64_t)n_owned;
  const int64_t prev = i > 0 ? (int64_t)keys[i - 1] : -1;
  for (int64_t b = prev + 1; b <= k && b <= (int64_t)n_owned; b++) range[b] = (int32_t)i;
}

// k_key_ranges over 4 consecutive keys per thread (one 16-byte load; keys 16-byte aligned):
// same output, a quarter of the threads and of the 64-bit index arithmetic.
__global__ void k_key_ranges4(const uint32_t* __restrict__ keys, int64_t n_full, uint32_t n_owned,
                              int32_t* __restrict__ range) {
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i0 > n_full) return;
  uint32_t k[4];
  if (i0 + 4 <= n_full) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(keys + i0));
    k[0] = v.x, k[1] = v.y, k[2] = v.z, k[3] = v.w;
  } else {
#pragma unroll
    for (int t = 0; t < 4; t++) k[t] = i0 + t < n_full ? __ldg(keys + i0 + t) : n_owned;
  }
  int64_t prev = i0 > 0 ? (int64_t)__ldg(keys + i0 - 1) : -1;
#pragma unroll
  for (int t = 0; t < 4; t++) {
    const int64_t i = i0 + t;
    if (i > n_full) break;
    const int64_t kk = (int64_t)k[t];
    for (int64_t b = prev + 1; b <= kk && b <= (int64_t)n_owned; b++) range[b] = (int32_t)i;
    prev = kk;
  }
}

// Per-tile digit histogram, digit-major: hist[d * ntiles + tile] (warp-aggregated smem adds).
__global__ void __launch_bounds__(kRadixThreads) k_radix_hist(const uint32_t* __restrict__ keys, int64_t n,
                                                              int shift, int bits, int64_t ntiles,
                                                              int64_t* __restrict__ hist) {
  __shared__ int h[kRadixWarps][256];  // one copy per warp: fewer same-address conflicts
  const int bins = 1 << bits;
  const int w = threadIdx.x >> 5;
  for (int i = threadIdx.x & 31; i < 256; i += 32) h[w][i] = 0;
  __syncwarp();
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
  const uint32_t mask = (uint32_t)(bins - 1);
#pragma unroll 4
  for (int r = 0; r < kRadixItems; r++) {
    const int64_t i = base + r * kRadixThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[w][(__ldg(keys + i) >> shift) & mask], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < bins; d += kRadixThreads) {
    int t = 0;
#pragma unroll
    for (int ww = 0; ww < kRadixWarps; ww++) t += h[ww][d];
    hist[(int64_t)d * ntiles + blockIdx.x] = t;
  }
}

// Stable scatter of one digit pass.  Warp w ranks its 512 consecutive elements in 16 rounds
// of 32 (match_any peers + a warp-private running count per digit), the CTA turns the
// per-warp counts into tile-local offsets, the tile is reordered by digit in shared memory and
// written out so that consecutive threads store consecutive positions of a digit's run.
// off = exclusive scan of hist (global start of each (digit, tile)).  Only positions < n_write
// are stored into vout (keys: all); kout == nullptr stores the values only.
#ifndef GS_SCATTER_MINB
#define GS_SCATTER_MINB 5
#endif
__global__ void __launch_bounds__(kRadixThreads, GS_SCATTER_MINB) k_radix_scatter(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, int64_t n, int64_t n_write, int shift, int bits, int64_t ntiles,
    const int64_t* __restrict__ off) {
  const int bins = 1 << bits;
  __shared__ int s_wh[kRadixWarps][257];
  __shared__ int s_toff[256];
  __shared__ int s_wsum[kRadixWarps];
  __shared__ long long s_gbase[256];
  __shared__ uint32_t s_k[kRadixTile], s_v[kRadixTile];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t mask = (uint32_t)(bins - 1);
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
  const int m = (int)min((int64_t)kRadixTile, n - base);
  for (int d = lane; d < 257; d += 32) s_wh[w][d] = 0;
  for (int d = tid; d < bins; d += kRadixThreads) s_gbase[d] = off[(int64_t)d * ntiles + blockIdx.x];
  __syncwarp();
  // values are loaded only when they are placed and the in-warp ranks (< 512) are packed two
  // per register: fewer live registers (5 CTAs per SM; 3 before)
  uint32_t kk[kRadixItems];
  uint32_t rk2[kRadixItems / 2];
#pragma unroll
  for (int r = 0; r < kRadixItems / 2; r++) rk2[r] = 0u;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < kRadixItems; r++) {
    const int li = w * kRadixPerWarp + r * 32 + lane;
    const bool valid = li < m;
    kk[r] = valid ? __ldg(kin + base + li) : 0u;
    const int d = valid ? (int)((kk[r] >> shift) & mask) : 256;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int cur = s_wh[w][d];
    rk2[r / 2] |= (uint32_t)(cur + __popc(peers & lt)) << (16 * (r & 1));
    __syncwarp();
    if ((peers & lt) == 0) s_wh[w][d] = cur + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive over warps, tile total
  int tot = 0;
  if (tid < bins) {
#pragma unroll
    for (int ww = 0; ww < kRadixWarps; ww++) {
      const int t = s_wh[ww][tid];
      s_wh[ww][tid] = tot;
      tot += t;
    }
  }
  // exclusive scan of the tile totals over digits (tid = digit)
  int incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[w] = incl;
  __syncthreads();
  int wpre = 0;
  for (int ww = 0; ww < w; ww++) wpre += s_wsum[ww];
  s_toff[tid] = wpre + incl - tot;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRadixItems; r++) {
    const int li = w * kRadixPerWarp + r * 32 + lane;
    if (li < m) {
      const int d = (int)((kk[r] >> shift) & mask);
      const int pos = s_toff[d] + s_wh[w][d] + (int)((rk2[r / 2] >> (16 * (r & 1))) & 0xffffu);
      s_k[pos] = kk[r];
      s_v[pos] = __ldg(vin + base + li);
    }
  }
  __syncthreads();
  for (int i = tid; i < m; i += kRadixThreads) {
    const uint32_t k = s_k[i];
    const int d = (int)((k >> shift) & mask);
    const int64_t pos = s_gbase[d] + (i - s_toff[d]);
    if (kout) kout[pos] = k;
    if (pos < n_write) vout[pos] = s_v[i];
  }
}

__global__ void k_depth_keys(const gs_rec* __restrict__ rec, int64_t n, uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ vals) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  keys[j] = __float_as_uint(rec[j].a.z);  // depth > 0: the bit pattern orders like the value
  vals[j] = (uint32_t)j;
}

__global__ void k_gather_tiles(const uint32_t* __restrict__ order, const int64_t* __restrict__ ntiles, int64_t n,
                               int64_t* __restrict__ ps) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > n) return;
  ps[s] = s < n ? ntiles[order[s]] : 0;
}

// First record (in depth order) of every emission CTA: record s covers pairs
// [ps[s], ps[s+1]); it is the first record of CTA c iff its range contains c * kPlacePairs.
__global__ void k_cta_first(const int64_t* __restrict__ ps, int64_t n, int64_t* __restrict__ first) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t a = ps[s], b = ps[s + 1];
  for (int64_t c = (a + kPlacePairs - 1) / kPlacePairs; c * kPlacePairs < b; c++) first[c] = s;
}

// Emit the pairs of the depth-ordered records: CTA c writes pairs [c*kPlacePairs, ...) of
// the enumeration pair_start (= scan of the tile counts in depth order); key = owned-block
// index (n_owned for a block of another rank), value = recv_idx.  Every received record has
// >= 1 tile (A1 emits a record only for a non-empty rectangle with an owned block), so at most
// kPlacePairs + 1 records overlap a CTA.
__global__ void __launch_bounds__(kPlaceThreads) k_emit(
    const gs_rec* __restrict__ rec, const uint32_t* __restrict__ order, int64_t n_recv,
    const int64_t* __restrict__ pair_start, const int64_t* __restrict__ first, int64_t n_full, gs_geom geo,
    int64_t B_lo, int64_t B_hi, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  __shared__ int64_t s_start[kPlacePairs + 2];
  __shared__ int s_tx0[kPlacePairs + 1], s_ty0[kPlacePairs + 1], s_w[kPlacePairs + 1], s_v[kPlacePairs + 1];
  __shared__ uint32_t s_j[kPlacePairs + 1];
  __shared__ int64_t s_slo;
  __shared__ int s_nr;
  const int64_t P0 = (int64_t)blockIdx.x * kPlacePairs;
  const int64_t P1 = min(P0 + kPlacePairs, n_full);
  if (threadIdx.x == 0) {
    const int64_t lo = first[blockIdx.x];
    int64_t hi = n_recv - 1;  // record holding pair P1 - 1
    if (P1 < n_full) {
      const int64_t t = first[blockIdx.x + 1];
      hi = pair_start[t] == P1 ? t - 1 : t;
    }
    s_slo = lo;
    s_nr = (int)(hi - lo + 1);
  }
  __syncthreads();
  const int64_t slo = s_slo;
  const int nr = s_nr;
  for (int r = threadIdx.x; r < nr; r += kPlaceThreads) {
    const int64_t sidx = slo + r;
    s_start[r] = pair_start[sidx];
    const uint32_t j = order[sidx];
    const float4 a = rec[j].a;
    int tx0, tx1, ty0, ty1;
    rect_of(a.x, a.y, a.w, geo.Wt, geo.Ht, tx0, tx1, ty0, ty1);
    s_tx0[r] = tx0;
    s_ty0[r] = ty0;
    s_w[r] = tx1 - tx0 + 1;
    s_v[r] = (int)(__float_as_uint(rec[j].d.w) & 31u);
    s_j[r] = j;
  }
  if (threadIdx.x == 0) s_start[nr] = pair_start[slo + nr];
  // record of each of the CTA's pairs without a per-pair binary search: mark each record at its
  // first pair in the CTA, then an inclusive max-scan over the kPlacePairs positions
  __shared__ int s_own[kPlacePairs];
  __shared__ int s_wmax[kPlaceThreads / 32];
  for (int i = threadIdx.x; i < kPlacePairs; i += kPlaceThreads) s_own[i] = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < nr; r += kPlaceThreads) {
    const int64_t off = s_start[r] - P0;
    if (off > 0 && off < kPlacePairs) s_own[off] = r;  // record 0 owns position 0 (it starts at or before P0)
  }
  __syncthreads();
  {
    constexpr int kPer = kPlacePairs / kPlaceThreads;  // consecutive positions per thread
    int m = 0;
#pragma unroll
    for (int k = 0; k < kPer; k++) m = max(m, s_own[threadIdx.x * kPer + k]);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int inc = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc = max(inc, y);
    }
    if (lane == 31) s_wmax[wid] = inc;
    __syncthreads();
    int run = 0;
    for (int w2 = 0; w2 < wid; w2++) run = max(run, s_wmax[w2]);
    int ex = __shfl_up_sync(0xffffffffu, inc, 1);
    ex = max(run, lane > 0 ? ex : 0);
#pragma unroll
    for (int k = 0; k < kPer; k++) {
      ex = max(ex, s_own[threadIdx.x * kPer + k]);
      s_own[threadIdx.x * kPer + k] = ex;
    }
  }
  __syncthreads();
  const uint32_t n_owned = (uint32_t)(B_hi - B_lo);
  for (int64_t pp = P0 + threadIdx.x; pp < P1; pp += kPlaceThreads) {
    const int lo = s_own[pp - P0];
    const int t = (int)(pp - s_start[lo]), w = s_w[lo];
    // t / w through a float reciprocal and one correction step (t < 2^24, w >= 1: exact)
    int q = (int)((float)t * __frcp_rn((float)w));
    int rm = t - q * w;
    if (rm < 0) q--, rm += w;
    else if (rm >= w) q++, rm -= w;
    const int ty = s_ty0[lo] + q, tx = s_tx0[lo] + rm;
    const int64_t beta = (int64_t)s_v[lo] * geo.per_view + (int64_t)ty * geo.Wt + tx;
    keys[pp] = (beta < B_lo || beta >= B_hi) ? n_owned : (uint32_t)(beta - B_lo);
    vals[pp] = s_j[lo];
  }
}

}  // namespace

// Binning algorithm: radix (default) or the per-block comparison sorts (GS_BIN_SORT=bitonic).
static bool bin_mode_radix() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("GS_BIN_SORT");
    mode = (e && e[0] == 'b') ? 0 : 1;
  }
  return mode == 1;
}

// One stable LSD pass over n (key, value) elements (keys/values in kin/vin) on `bits` digit
// bits at `shift`; kout may be null (values only).  Scratch: SLOT_RADIX_HIST.
static gs_status radix_pass(gs_ctx* c, const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                            int64_t n, int64_t n_write, int shift, int bits, cudaStream_t st) {
  if (n == 0) return GS_OK;
  const int bins = 1 << bits;
  const int64_t ntiles = (n + kRadixTile - 1) / kRadixTile;
  int64_t* hist = (int64_t*)gs_slot_get(c, SLOT_RADIX_HIST, (size_t)bins * ntiles * sizeof(int64_t), st);
  if (!hist) return gs_fail(c, GS_ECUDA, "radix histogram scratch");
  ++c->launches;
  k_radix_hist<<<(unsigned)ntiles, kRadixThreads, 0, st>>>(kin, n, shift, bits, ntiles, hist);
  gs_status s = gs_scan_i64(c, hist, hist, (int64_t)bins * ntiles, 0, st);
  if (s != GS_OK) return s;
  ++c->launches;
  k_radix_scatter<<<(unsigned)ntiles, kRadixThreads, 0, st>>>(kin, vin, kout, vout, n, n_write, shift, bits, ntiles,
                                                              hist);
  GS_LAUNCH_CHECK(c, "radix pass");
  return GS_OK;
}

namespace {
}  // namespace

// Radix binning (see the comment above k_radix_hist).  Two host syncs: the pair total (scratch
// sizing) and the owned pair count K (capacity, *n_pairs_h).
static gs_status bin_sort_radix(gs_ctx* c, const gs_rec* rec, int64_t n_recv, gs_geom geo, int64_t B_lo,
                                int64_t B_hi, uint32_t* sorted_idx, int64_t pair_cap, int32_t* tile_range,
                                int64_t* n_pairs_h, cudaStream_t st) {
  const int64_t n_owned = B_hi - B_lo;
  const int v_lo = (int)(B_lo / geo.per_view), v_hi = (int)((B_hi - 1) / geo.per_view);
  if (n_recv == 0) {
    GS_CUDA(c, cudaMemsetAsync(tile_range, 0, (n_owned + 1) * sizeof(int32_t), st));
    return GS_OK;
  }
  GS_REQUIRE(c, rec != nullptr, "null recv_rec");
  int64_t* ntiles = (int64_t*)gs_slot_get(c, SLOT_RECTILES, (n_recv + 1) * sizeof(int64_t), st);
  int64_t* ps = (int64_t*)gs_slot_get(c, SLOT_PSTART, (n_recv + 1) * sizeof(int64_t), st);
  if (!ntiles || !ps) return gs_fail(c, GS_ECUDA, "scratch");
  ++c->launches;
  k_tile_counts<<<(unsigned)((n_recv + 256) / 256), 256, 0, st>>>(rec, n_recv, geo, v_lo, v_hi, ntiles);
  gs_status s = gs_scan_i64(c, ntiles, ps, n_recv + 1, 0, st);  // only for the total
  if (s != GS_OK) return s;
  static const bool dbg = getenv("GS_DEBUG_SORT") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t0 = now();
  GS_CUDA(c, cudaMemcpyAsync(c->pinned, ps + n_recv, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  auto t1 = now();
  const int64_t n_full = c->pinned[0];
  // tile_range holds int32 positions: bound the pair total (a superset of the owned pairs)
  if (n_full >= (1ll << 31))
    return gs_fail(c, GS_ENOTSUP, "pair total %lld exceeds int32 positions", (long long)n_full);
  const int64_t cap = max(n_full, n_recv);
  uint32_t* A = (uint32_t*)gs_slot_get(c, SLOT_KEYS, 2 * cap * sizeof(uint32_t), st);
  uint32_t* Bf = (uint32_t*)gs_slot_get(c, SLOT_KEYS_TMP, 2 * cap * sizeof(uint32_t), st);
  if (!A || !Bf) return gs_fail(c, GS_ECUDA, "radix scratch (%lld pairs)", (long long)cap);
  uint32_t *ka = A, *va = A + cap, *kb = Bf, *vb = Bf + cap;
  // 1. records by depth (4 stable 8-bit passes: A -> B -> A -> B -> A)
  ++c->launches;
  k_depth_keys<<<(unsigned)((n_recv + 255) / 256), 256, 0, st>>>(rec, n_recv, ka, va);
  for (int p = 0; p < 4; p++) {
    s = (p & 1) ? radix_pass(c, kb, vb, ka, va, n_recv, n_recv, 8 * p, 8, st)
                : radix_pass(c, ka, va, kb, vb, n_recv, n_recv, 8 * p, 8, st);
    if (s != GS_OK) return s;
  }
  // 2. pair starts in depth order; 3. pairs (block, recv_idx) in depth order -> B
  ++c->launches;
  k_gather_tiles<<<(unsigned)((n_recv + 256) / 256), 256, 0, st>>>(va, ntiles, n_recv, ps);
  s = gs_scan_i64(c, ps, ps, n_recv + 1, 0, st);
  if (s != GS_OK) return s;
  if (n_full > 0) {
    const int64_t nct = (n_full + kPlacePairs - 1) / kPlacePairs;
    int64_t* first = (int64_t*)gs_slot_get(c, SLOT_LARGE, (nct + 1) * sizeof(int64_t), st);
    if (!first) return gs_fail(c, GS_ECUDA, "scratch");
    ++c->launches;
    k_cta_first<<<(unsigned)((n_recv + 255) / 256), 256, 0, st>>>(ps, n_recv, first);
    ++c->launches;
    k_emit<<<(unsigned)nct, kPlaceThreads, 0, st>>>(rec, va, n_recv, ps, first, n_full, geo, B_lo, B_hi, kb, vb);
    GS_LAUNCH_CHECK(c, "bin_sort emit");
  }
  // 4. stable sort by owned-block index (other ranks' blocks: key n_owned, sorted last); the
  //    last pass writes the values into sorted_idx (up to its capacity) and the keys into scratch
  const int nbits = 32 - __builtin_clz((unsigned)n_owned);
  const int passes = (nbits + 7) / 8, width = (nbits + passes - 1) / passes;
  uint32_t *kin = kb, *vin = vb, *kout = ka, *vout = va;
  for (int p = 0; p < passes; p++) {
    const int shift = p * width, bits = min(width, nbits - shift);
    const bool last = p == passes - 1;
    s = radix_pass(c, kin, vin, kout, last ? sorted_idx : vout, n_full, last ? min(n_full, pair_cap) : n_full,
                   shift, bits, st);
    if (s != GS_OK) return s;
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  // 5. ranges from the sorted keys (now in kin)
  ++c->launches;
  k_key_ranges4<<<(unsigned)((n_full / 4 + 256) / 256), 256, 0, st>>>(kin, n_full, (uint32_t)n_owned, tile_range);
  GS_LAUNCH_CHECK(c, "bin_sort ranges");
  int32_t* kp = (int32_t*)(c->pinned + 1);
  auto t2 = now();
  GS_CUDA(c, cudaMemcpyAsync(kp, tile_range + n_owned, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  auto t3 = now();
  if (dbg) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr, "libgs bin_sort: n_full %lld  sync1 %.2f ms  enqueue %.2f ms  sync2 %.2f ms\n",
            (long long)n_full, ms(t0, t1), ms(t1, t2), ms(t2, t3));
  }
  const int64_t K = *kp;
  *n_pairs_h = K;
  if (K > pair_cap) return gs_fail(c, GS_ECAPACITY, "pair capacity %lld < %lld", (long long)pair_cap, (long long)K);
  return GS_OK;
}

extern "C" gs_status gs_bin_sort(gs_ctx* c, const void* recv_rec, int64_t n_recv, const gs_camera* cams_h,
                                 int n_views, const int64_t* dp_h, uint32_t* sorted_idx, int64_t pair_cap,
                                 int32_t* tile_range, int64_t* n_pairs_h, void* stream) {
  if (!c) return GS_EINVAL;
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, tile_range && n_pairs_h, "null argument");
  GS_REQUIRE(c, n_recv >= 0 && n_recv < (1ll << 32), "n_recv out of range");
  cudaStream_t st = (cudaStream_t)stream;
  gs_geom geo = gs_make_geom(&cams_h[0]);
  const int64_t B_lo = dp_h[c->rank], B_hi = dp_h[c->rank + 1], n_owned = B_hi - B_lo;
  *n_pairs_h = 0;
  if (n_owned == 0) {
    GS_CUDA(c, cudaMemsetAsync(tile_range, 0, sizeof(int32_t), st));
    return GS_OK;
  }
  if (bin_mode_radix()) {
    GS_REQUIRE(c, n_owned < (1ll << 31) - 1, "too many owned blocks");
    return bin_sort_radix(c, (const gs_rec*)recv_rec, n_recv, geo, B_lo, B_hi, sorted_idx, pair_cap, tile_range,
                          n_pairs_h, st);
  }
  const int v_lo = (int)(B_lo / geo.per_view), v_hi = (int)((B_hi - 1) / geo.per_view);
  const int nvl = v_hi - v_lo + 1;
  const int64_t diff_n = (int64_t)nvl * (geo.Ht + 1) * (geo.Wt + 1);
  int* diff = (int*)gs_slot_get(c, SLOT_DIFF, diff_n * sizeof(int), st);
  int64_t* counts = (int64_t*)gs_slot_get(c, SLOT_COUNTS, (n_owned + 1) * sizeof(int64_t), st);
  int32_t* cursor = (int32_t*)gs_slot_get(c, SLOT_CURSOR, (n_owned + 1) * sizeof(int32_t), st);
  int32_t* large = (int32_t*)gs_slot_get(c, SLOT_LARGE, (2 * n_owned + 8) * sizeof(int32_t), st);
  int64_t* ntiles = (int64_t*)gs_slot_get(c, SLOT_RECTILES, (n_recv + 1) * sizeof(int64_t), st);
  if (!diff || !counts || !cursor || !large || !ntiles) return gs_fail(c, GS_ECUDA, "scratch");
  GS_CUDA(c, cudaMemsetAsync(diff, 0, diff_n * sizeof(int), st));
  if (n_recv > 0) {
    GS_REQUIRE(c, recv_rec != nullptr, "null recv_rec");
    ++c->launches;
    k_rect_diff<<<(unsigned)((n_recv + 256) / 256), 256, 0, st>>>((const gs_rec*)recv_rec, n_recv, geo,
                                                                  v_lo, v_hi, diff, ntiles);
    s = gs_scan_i64(c, ntiles, ntiles, n_recv + 1, 0, st);  // pair_start
    if (s != GS_OK) return s;
  }
  const int ld = geo.Wt + 1, rows = geo.Ht + 1;
  ++c->launches;
  k_diff_rows<<<(nvl * rows + 127) / 128, 128, 0, st>>>(diff, nvl * rows, ld);
  ++c->launches;
  k_diff_cols<<<(nvl * ld + 127) / 128, 128, 0, st>>>(diff, nvl, rows, ld);
  ++c->launches;
  k_owned_counts<<<(unsigned)((n_owned + 256) / 256), 256, 0, st>>>(diff, geo, B_lo, n_owned, v_lo, counts);
  GS_LAUNCH_CHECK(c, "bin_sort counts");
  s = gs_scan_i64(c, counts, counts, n_owned + 1, 0, st);
  if (s != GS_OK) return s;
  GS_CUDA(c, cudaMemcpyAsync(c->pinned, counts + n_owned, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  if (n_recv > 0)
    GS_CUDA(c, cudaMemcpyAsync(c->pinned + 1, ntiles + n_recv, sizeof(int64_t),
                               cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  const int64_t K = c->pinned[0], n_full = n_recv > 0 ? c->pinned[1] : 0;
  *n_pairs_h = K;
  if (K > pair_cap || K >= (1ll << 31))
    return gs_fail(c, GS_ECAPACITY, "pair capacity %lld < %lld", (long long)pair_cap, (long long)K);
  ++c->launches;
  k_to_range<<<(unsigned)((n_owned + 256) / 256), 256, 0, st>>>(counts, n_owned, tile_range, cursor);
  GS_LAUNCH_CHECK(c, "bin_sort range");
  if (K == 0) return GS_OK;
  GS_REQUIRE(c, sorted_idx != nullptr, "null sorted_idx");
  unsigned long long* keys = (unsigned long long*)gs_slot_get(c, SLOT_KEYS, K * sizeof(unsigned long long), st);
  if (!keys) return gs_fail(c, GS_ECUDA, "key scratch (%lld pairs)", (long long)K);
  ++c->launches;
  k_place<<<(unsigned)((n_full + kPlacePairs - 1) / kPlacePairs), kPlaceThreads, 0, st>>>(
      (const gs_rec*)recv_rec, n_recv, ntiles, n_full, geo, B_lo, B_hi, cursor, keys);
  // lists: mid (n_owned) then large (n_owned), then 4 counters
  int32_t* mid = large;
  int32_t* lrg = large + n_owned;
  int32_t* ctr = large + 2 * n_owned;  // n_mid, next_mid, n_large, next_large
  GS_CUDA(c, cudaMemsetAsync(ctr, 0, 4 * sizeof(int32_t), st));
  ++c->launches;
  k_sort_warp<<<(unsigned)((n_owned + kSortThreads / 32 - 1) / (kSortThreads / 32)), kSortThreads, 0, st>>>(
      tile_range, n_owned, keys, sorted_idx, mid, ctr, lrg, ctr + 2);
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->device);
  ++c->launches;
  k_sort_small<<<dev_sms * 4, kSortThreads, 0, st>>>(tile_range, keys, sorted_idx, mid, ctr, ctr + 1);
  GS_LAUNCH_CHECK(c, "bin_sort small");
  unsigned long long* tmp = (unsigned long long*)gs_slot_get(c, SLOT_KEYS_TMP, K * sizeof(unsigned long long), st);
  if (!tmp) return gs_fail(c, GS_ECUDA, "merge scratch");
  ++c->launches;
  k_sort_large<<<dev_sms * 4, kSortThreads, 0, st>>>(tile_range, keys, tmp, sorted_idx, lrg, ctr + 2, ctr + 3);
  GS_LAUNCH_CHECK(c, "bin_sort large");
  return GS_OK;
}
