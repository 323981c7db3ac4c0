// gs_sort.cu -- A3: Z-buffer build ("iterates over intersecting Gaussians in
// increasing depth"; App. A.2 "indices of intersecting gaussians for each pixel").
//
// B200 design (differs from the prior art's global 64-bit (tile | depth) radix sort of the
// pairs): the RECORDS are sorted by (view, depth) -- stable LSD radix over the 32 depth bits,
// then the view -- so equal depths stay in receive order (= gid order within a view, R7); the
// (block, record) pairs are emitted in that order, each view's pairs into its own segment of
// the pair array, padded to whole radix tiles; then the pairs of every segment are stably
// radix-sorted by their VIEW-LOCAL block index (16 bits for a 4591x3436 view: 2 passes of 8;
// 13 bits at 1080p: 7 + 6) with one digit histogram laid out [view][digit][tile], so one
// exclusive scan keeps every segment in place.  Each block's list then comes out in exact
// (depth, gid) order (O11) with no per-block sort and traffic linear in the pairs; tile_range
// is read off the sorted keys.  Pairs of blocks the rank does not own (G > 1: rectangles
// straddling the partition) and the padding carry the sentinel key 2^nbits - 1, sort to the
// end of their segment and are never written.  One host sync per call: the per-view pair
// counts (scratch sizing, segment layout, the capacity check and *n_pairs_h).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "gs_device.cuh"
#include "gs_internal.h"

using namespace gsd;

namespace {

#ifndef GS_RADIX_THREADS
#define GS_RADIX_THREADS 256
#endif
constexpr int kRadixThreads = GS_RADIX_THREADS;  // 256 (4096-element tiles): 512 (8192) measured slower
#ifndef GS_RADIX_ITEMS
#define GS_RADIX_ITEMS 16
#endif
constexpr int kRadixItems = GS_RADIX_ITEMS;  // elements per thread (A/B builds may vary it)
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // elements per CTA
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixPerWarp = kRadixTile / kRadixWarps;   // 512 consecutive elements per warp
constexpr int kEmitThreads = 256;
constexpr int kEmitPairs = 1024;  // pairs per emission CTA

// The segment layout of the rank's views v_lo .. v_lo + nv - 1 (host-computed after the sync):
// view k's pairs occupy padded positions [seg[k], seg[k+1]) (tile-aligned), its owned pairs
// come first after sorting and land in sorted_idx at [kcum[k], kcum[k+1]).
struct seg_arg {
  int nv, v_lo;
  long long seg[GS_MAX_VIEWS + 1];    // padded element offsets (multiples of kRadixTile)
  long long kcum[GS_MAX_VIEWS + 1];   // owned-pair offsets in sorted_idx
  long long shift[GS_MAX_VIEWS];      // emission: padded = unpadded position + shift[k]
  int lo[GS_MAX_VIEWS], hi[GS_MAX_VIEWS];  // owned view-local blocks [lo, hi) of view k
  long long B_lo;                     // first owned block (global index)
  unsigned sentinel;                  // 2^nbits - 1
};

__device__ __forceinline__ int seg_of_tile(const seg_arg& g, long long t) {
  int k = 0;
  while (k + 1 < g.nv && t * kRadixTile >= g.seg[k + 1]) k++;
  return k;
}
// histogram index of (segment k, digit d, tile t): layout [segment][digit][tile in segment]
__device__ __forceinline__ long long seg_hidx(const seg_arg& g, int k, int d, long long t, int bins) {
  const long long t0 = g.seg[k] / kRadixTile, nt = (g.seg[k + 1] - g.seg[k]) / kRadixTile;
  return t0 * bins + (long long)d * nt + (t - t0);
}

// Per-record tile count of its rectangle in its view (all blocks: the emission enumerates the
// rectangle), and per view the pair total and the owned-pair total (owned = view-local block in
// [lo, hi): per rectangle row an interval intersection).  cnt[k] / own[k] over the rank's views.
__global__ void k_tile_counts(const gs_rec* __restrict__ rec, int64_t n_recv, gs_geom geo, seg_arg g,
                              int64_t* __restrict__ n_tiles, unsigned long long* __restrict__ cnt,
                              unsigned long long* __restrict__ own) {
  __shared__ unsigned long long s_c[GS_MAX_VIEWS], s_o[GS_MAX_VIEWS];
  if (threadIdx.x < GS_MAX_VIEWS) s_c[threadIdx.x] = s_o[threadIdx.x] = 0;
  __syncthreads();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned t = 0, o = 0;
  int k = -1;
  if (j < n_recv) {
    const float4 a = rec[j].a;
    k = (int)(__float_as_uint(rec[j].d.w) & 31u) - g.v_lo;
    int tx0, tx1, ty0, ty1;
    if (k >= 0 && k < g.nv && rect_of(a.x, a.y, a.w, geo.Wt, geo.Ht, tx0, tx1, ty0, ty1)) {
      t = (unsigned)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
      for (int ty = ty0; ty <= ty1; ty++) {
        const long long r0 = (long long)ty * geo.Wt + tx0, r1 = (long long)ty * geo.Wt + tx1 + 1;
        o += (unsigned)max(0ll, min(r1, (long long)g.hi[k]) - max(r0, (long long)g.lo[k]));
      }
    } else {
      k = -1;
    }
  }
  if (j <= n_recv) n_tiles[j] = t;
  // per view: the lanes of a view add their counts once (a warp's records mostly share a view)
  const unsigned peers = __match_any_sync(0xffffffffu, k);
  const int leader = __ffs(peers) - 1;
  const unsigned ts = __reduce_add_sync(peers, t), os = __reduce_add_sync(peers, o);
  if (k >= 0 && (int)(threadIdx.x & 31) == leader) {
    atomicAdd(&s_c[k], (unsigned long long)ts);
    if (os) atomicAdd(&s_o[k], (unsigned long long)os);
  }
  __syncthreads();
  if (threadIdx.x < GS_MAX_VIEWS && s_c[threadIdx.x]) {
    atomicAdd(&cnt[threadIdx.x], s_c[threadIdx.x]);
    if (s_o[threadIdx.x]) atomicAdd(&own[threadIdx.x], s_o[threadIdx.x]);
  }
}

__global__ void k_depth_keys(const gs_rec* __restrict__ rec, int64_t n, uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ vals) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  keys[j] = __float_as_uint(rec[j].a.z);  // depth > 0: the bit pattern orders like the value
  vals[j] = (uint32_t)j;
}

// view keys of the depth-ordered records (the last, stable, record pass groups them by view)
__global__ void k_view_keys(const gs_rec* __restrict__ rec, const uint32_t* __restrict__ order, int64_t n,
                            int v_lo, uint32_t* __restrict__ keys) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  keys[s] = (__float_as_uint(rec[order[s]].d.w) & 31u) - (uint32_t)v_lo;
}

__global__ void k_gather_tiles(const uint32_t* __restrict__ order, const int64_t* __restrict__ ntiles, int64_t n,
                               int64_t* __restrict__ ps) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > n) return;
  ps[s] = s < n ? ntiles[order[s]] : 0;
}

// First record (in (view, depth) order) of every emission CTA: record s covers unpadded pairs
// [ps[s], ps[s+1]); it is the first record of CTA c iff its range contains c * kEmitPairs.
__global__ void k_cta_first(const int64_t* __restrict__ ps, int64_t n, int64_t* __restrict__ first) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t a = ps[s], b = ps[s + 1];
  for (int64_t c = (a + kEmitPairs - 1) / kEmitPairs; c * kEmitPairs < b; c++) first[c] = s;
}

// Emit the pairs of the ordered records: CTA c enumerates unpadded pairs [c*kEmitPairs, ...)
// of pair_start (= scan of the tile counts in (view, depth) order) and stores each at its
// padded position (+ shift of its view's segment): key = view-local block index if the rank
// owns the block, else the sentinel; value = recv_idx.  The histogram of the first digit
// pass (bits [0, bits0)) is accumulated on the way ([segment][digit][tile] layout).  Every
// received record has >= 1 tile (A1 emits a record only for a rectangle with an owned block),
// so at most kEmitPairs + 1 records overlap a CTA.
__global__ void __launch_bounds__(kEmitThreads) k_emit(
    const gs_rec* __restrict__ rec, const uint32_t* __restrict__ order, int64_t n_recv,
    const int64_t* __restrict__ pair_start, const int64_t* __restrict__ first, int64_t n_full, gs_geom geo,
    seg_arg g, int bits0, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
    unsigned long long* __restrict__ hist) {
  __shared__ int64_t s_start[kEmitPairs + 2];
  __shared__ int s_tx0[kEmitPairs + 1], s_ty0[kEmitPairs + 1], s_w[kEmitPairs + 1], s_k[kEmitPairs + 1];
  __shared__ uint32_t s_j[kEmitPairs + 1];
  __shared__ int64_t s_slo;
  __shared__ int s_nr;
  __shared__ int s_own[kEmitPairs];
  __shared__ int s_wmax[kEmitThreads / 32];
  __shared__ unsigned s_h[2][256];  // first-pass histogram of the (at most 2) padded tiles hit
  const int64_t P0 = (int64_t)blockIdx.x * kEmitPairs;
  const int64_t P1 = min(P0 + kEmitPairs, n_full);
  for (int i = threadIdx.x; i < 512; i += kEmitThreads) (&s_h[0][0])[i] = 0;
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
  for (int r = threadIdx.x; r < nr; r += kEmitThreads) {
    const int64_t sidx = slo + r;
    s_start[r] = pair_start[sidx];
    const uint32_t j = order[sidx];
    const float4 a = rec[j].a;
    int tx0, tx1, ty0, ty1;
    rect_of(a.x, a.y, a.w, geo.Wt, geo.Ht, tx0, tx1, ty0, ty1);
    s_tx0[r] = tx0;
    s_ty0[r] = ty0;
    s_w[r] = tx1 - tx0 + 1;
    s_k[r] = (int)(__float_as_uint(rec[j].d.w) & 31u) - g.v_lo;
    s_j[r] = j;
  }
  if (threadIdx.x == 0) s_start[nr] = pair_start[slo + nr];
  // record of each of the CTA's pairs without a per-pair binary search: mark each record at its
  // first pair in the CTA, then an inclusive max-scan over the kEmitPairs positions
  for (int i = threadIdx.x; i < kEmitPairs; i += kEmitThreads) s_own[i] = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < nr; r += kEmitThreads) {
    const int64_t off = s_start[r] - P0;
    if (off > 0 && off < kEmitPairs) s_own[off] = r;  // record 0 owns position 0 (it starts at or before P0)
  }
  __syncthreads();
  {
    constexpr int kPer = kEmitPairs / kEmitThreads;  // consecutive positions per thread
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
  // the padded tiles this CTA's pairs land in: the first pair's tile and possibly the next
  // (a CTA's 1024 pairs span at most one view boundary only at padding, which moves them to a
  // later tile: track up to two tiles, else fall back to global atomics)
  const int64_t tbase = (P0 + g.shift[s_k[0]]) / kRadixTile;
  __shared__ long long s_hb[2], s_hn[2];  // histogram base and digit stride of the two tiles
  if (threadIdx.x < 2) {
    const int64_t tile = tbase + threadIdx.x;
    const int k = seg_of_tile(g, tile);
    const long long t0 = g.seg[k] / kRadixTile;
    s_hn[threadIdx.x] = (g.seg[k + 1] - g.seg[k]) / kRadixTile;
    s_hb[threadIdx.x] = t0 * (1 << bits0) + (tile - t0);
  }
  const unsigned dmask = (1u << bits0) - 1u;
  for (int64_t pp = P0 + threadIdx.x; pp < P1; pp += kEmitThreads) {
    const int lo = s_own[pp - P0];
    const int t = (int)(pp - s_start[lo]), w = s_w[lo], k = s_k[lo];
    // t / w through a float reciprocal and one correction step (t < 2^24, w >= 1: exact)
    int q = (int)((float)t * __frcp_rn((float)w));
    int rm = t - q * w;
    if (rm < 0) q--, rm += w;
    else if (rm >= w) q++, rm -= w;
    const int local = (s_ty0[lo] + q) * geo.Wt + s_tx0[lo] + rm;
    const uint32_t key = (local >= g.lo[k] && local < g.hi[k]) ? (uint32_t)local : g.sentinel;
    const int64_t pos = pp + g.shift[k];
    keys[pos] = key;
    vals[pos] = s_j[lo];
    const int64_t tile = pos / kRadixTile;
    const int d = (int)(key & dmask);
    if (tile - tbase < 2)
      atomicAdd(&s_h[tile - tbase][d], 1u);
    else
      atomicAdd(&hist[seg_hidx(g, k, d, tile, 1 << bits0)], 1ull);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += kEmitThreads) {
    const int tt = i >> 8, d = i & 255;
    const unsigned c = s_h[tt][d];
    if (c) atomicAdd(&hist[s_hb[tt] + (long long)d * s_hn[tt]], (unsigned long long)c);
  }
}

// Padding of every segment: the sentinel key (value unused), counted in the first-pass histogram.
__global__ void k_pad(seg_arg g, const unsigned long long* __restrict__ cnt, int bits0, uint32_t* __restrict__ keys,
                      unsigned long long* __restrict__ hist) {
  const int k = blockIdx.y;
  const int64_t a = g.seg[k] + (int64_t)cnt[k], b = g.seg[k + 1];
  const int d = (int)(g.sentinel & ((1u << bits0) - 1u));
  for (int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = g.sentinel;
    atomicAdd(&hist[seg_hidx(g, k, d, i / kRadixTile, 1 << bits0)], 1ull);
  }
}

// Per-tile digit histogram (passes after the first), [segment][digit][tile] layout
// (kSeg), or digit-major [digit][tile] over n elements (the record passes).
template <bool kSeg>
__global__ void __launch_bounds__(kRadixThreads) k_radix_hist(const uint32_t* __restrict__ keys, int64_t n,
                                                              int shift, int bits, int64_t ntiles, seg_arg g,
                                                              unsigned long long* __restrict__ hist) {
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
  const int k = kSeg ? seg_of_tile(g, blockIdx.x) : 0;
  for (int d = threadIdx.x; d < bins; d += kRadixThreads) {
    int t = 0;
#pragma unroll
    for (int ww = 0; ww < kRadixWarps; ww++) t += h[ww][d];
    hist[kSeg ? seg_hidx(g, k, d, blockIdx.x, bins) : (long long)d * ntiles + blockIdx.x] = t;
  }
}

// Stable scatter of one digit pass.  Warp w ranks its 512 consecutive elements in 16 rounds
// of 32 (match_any peers + a warp-private running count per digit), the CTA turns the
// per-warp counts into tile-local offsets, the tile is reordered by digit in shared memory and
// written out so that consecutive threads store consecutive positions of a digit's run.
// off = exclusive scan of the histogram (global start of each (digit, tile)).  kSeg: the
// segmented layout; kLast (kSeg only): values go to sorted_idx at their compact position
// (kcum of the segment + position in it), the sentinel's are dropped; keys to kout (all).
template <bool kSeg, bool kLast>
__global__ void __launch_bounds__(kRadixThreads, 5 * 256 / kRadixThreads) k_radix_scatter(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, int64_t n, int shift, int bits, int64_t ntiles, seg_arg g,
    const unsigned long long* __restrict__ off, int64_t vcap) {
  const int bins = 1 << bits;
  __shared__ int s_wh[kRadixWarps][257];
  __shared__ int s_toff[kRadixThreads];
  __shared__ int s_wsum[kRadixWarps];
  __shared__ long long s_gbase[256];
  extern __shared__ uint32_t s_kv[];  // dynamic: the tile's keys, then its values
  uint32_t* const s_k = s_kv;
  uint32_t* const s_v = s_kv + kRadixTile;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t mask = (uint32_t)(bins - 1);
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
  const int m = (int)min((int64_t)kRadixTile, n - base);
  const int sk = kSeg ? seg_of_tile(g, blockIdx.x) : 0;
  for (int d = lane; d < 257; d += 32) s_wh[w][d] = 0;
  for (int d = tid; d < bins; d += kRadixThreads)
    s_gbase[d] = (long long)off[kSeg ? seg_hidx(g, sk, d, blockIdx.x, bins) : (long long)d * ntiles + blockIdx.x];
  __syncwarp();
  // values are loaded only when they are placed and the in-warp ranks (< 512) are packed two
  // per register: fewer live registers (5 CTAs per SM)
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
  const long long vshift = kLast ? g.kcum[sk] - g.seg[sk] : 0;  // padded -> compact (owned pairs first)
  for (int i = tid; i < m; i += kRadixThreads) {
    const uint32_t k = s_k[i];
    const int d = (int)((k >> shift) & mask);
    const int64_t pos = s_gbase[d] + (i - s_toff[d]);
    kout[pos] = k;
    if (kLast) {
      if (k != g.sentinel && pos + vshift < vcap) vout[pos + vshift] = s_v[i];
    } else {
      vout[pos] = s_v[i];
    }
  }
}

// tile_range from the sorted segments: range[b] = first compact position of owned block b.
// Position i of segment k holds the view-local key keys[i] (the sentinel stands for hi[k]); the
// owned blocks with local index in (previous key, key] start at i's compact position.  Every
// segment ends in >= 1 sentinel, so its last owned blocks and range[n_owned] are written too.
// Four consecutive positions per thread (one 16-byte load); a CTA's 1024 positions lie in one
// radix tile, hence in one segment.
__global__ void k_seg_ranges(const uint32_t* __restrict__ keys, seg_arg g, int64_t per_view, int32_t* __restrict__ range) {
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  __shared__ int s_seg;
  if (threadIdx.x == 0) s_seg = seg_of_tile(g, ((int64_t)blockIdx.x * blockDim.x * 4) / kRadixTile);
  __syncthreads();
  if (i0 >= g.seg[g.nv]) return;
  const int k = s_seg;
  const int lo = g.lo[k], hi = g.hi[k];
  const uint4 v = __ldg(reinterpret_cast<const uint4*>(keys + i0));
  const uint32_t kk[4] = {v.x, v.y, v.z, v.w};
  int prev = lo - 1;
  if (i0 > g.seg[k]) {
    const uint32_t kp = __ldg(keys + i0 - 1);
    prev = kp == g.sentinel ? hi : (int)kp;
  }
  int32_t* rb = range + ((long long)(g.v_lo + k) * per_view - g.B_lo);  // owned index of local block 0
  const int32_t c0 = (int32_t)(g.kcum[k] + (i0 - g.seg[k]));
#pragma unroll
  for (int t = 0; t < 4; t++) {
    const int cur = kk[t] == g.sentinel ? hi : (int)kk[t];
    for (int bb = max(prev + 1, lo); bb <= cur && bb <= hi; bb++) rb[bb] = c0 + t;
    prev = cur;
  }
}

constexpr int kScatterSmem = 2 * kRadixTile * (int)sizeof(uint32_t);
// the scatter kernels' dynamic shared memory above the 48 KB default (once per process)
bool scatter_smem_ready() {
  static const bool ok = [] {
    bool r = true;
    r &= cudaFuncSetAttribute(k_radix_scatter<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kScatterSmem) == cudaSuccess;
    r &= cudaFuncSetAttribute(k_radix_scatter<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kScatterSmem) == cudaSuccess;
    r &= cudaFuncSetAttribute(k_radix_scatter<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kScatterSmem) == cudaSuccess;
    return r;
  }();
  return ok;
}

// One stable LSD pass over n (key, value) elements on `bits` digit bits at `shift` (record
// passes: digit-major histogram over tiles).  Scratch: SLOT_RADIX_HIST.
gs_status radix_pass(gs_ctx* c, const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout, int64_t n,
                     int shift, int bits, const seg_arg& g, cudaStream_t st) {
  if (n == 0) return GS_OK;
  const int bins = 1 << bits;
  const int64_t ntiles = (n + kRadixTile - 1) / kRadixTile;
  unsigned long long* hist =
      (unsigned long long*)gs_slot_get(c, SLOT_RADIX_HIST, (size_t)bins * ntiles * sizeof(int64_t), st);
  if (!hist) return gs_fail(c, GS_ECUDA, "radix histogram scratch");
  ++c->launches;
  k_radix_hist<false><<<(unsigned)ntiles, kRadixThreads, 0, st>>>(kin, n, shift, bits, ntiles, g, hist);
  gs_status s = gs_scan_i64(c, (const int64_t*)hist, (int64_t*)hist, (int64_t)bins * ntiles, 0, st);
  if (s != GS_OK) return s;
  ++c->launches;
  k_radix_scatter<false, false><<<(unsigned)ntiles, kRadixThreads, kScatterSmem, st>>>(kin, vin, kout, vout, n, shift, bits,
                                                                            ntiles, g, hist, 0);
  GS_LAUNCH_CHECK(c, "radix pass");
  return GS_OK;
}

}  // namespace

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
  GS_REQUIRE(c, n_owned < (1ll << 31) - 1, "too many owned blocks");
  if (n_recv == 0) {
    GS_CUDA(c, cudaMemsetAsync(tile_range, 0, (n_owned + 1) * sizeof(int32_t), st));
    return GS_OK;
  }
  GS_REQUIRE(c, recv_rec != nullptr, "null recv_rec");
  if (!scatter_smem_ready()) return gs_fail(c, GS_ECUDA, "radix scatter shared-memory attribute");
  const gs_rec* rec = (const gs_rec*)recv_rec;
  const int64_t pv = geo.per_view;
  seg_arg g;
  memset(&g, 0, sizeof(g));
  g.v_lo = (int)(B_lo / pv);
  g.nv = (int)((B_hi - 1) / pv) - g.v_lo + 1;
  g.B_lo = B_lo;
  for (int k = 0; k < g.nv; k++) {
    const int64_t v = g.v_lo + k;
    g.lo[k] = (int)std::max<int64_t>(B_lo - v * pv, 0);
    g.hi[k] = (int)std::min<int64_t>(B_hi - v * pv, pv);
  }
  const int nbits = 32 - __builtin_clz((unsigned)pv);  // 2^nbits > pv: the sentinel exceeds every key
  g.sentinel = (nbits >= 32) ? 0xffffffffu : ((1u << nbits) - 1u);
  const int passes = (nbits + 7) / 8, width = (nbits + passes - 1) / passes;
  // 1. per-record tile counts, per-view pair and owned-pair totals (one host sync)
  int64_t* ntiles = (int64_t*)gs_slot_get(c, SLOT_RECTILES, (n_recv + 1) * sizeof(int64_t), st);
  int64_t* ps = (int64_t*)gs_slot_get(c, SLOT_PSTART, (n_recv + 1) * sizeof(int64_t), st);
  unsigned long long* vc = (unsigned long long*)gs_slot_get(c, SLOT_COUNTS, 2 * GS_MAX_VIEWS * sizeof(int64_t), st);
  if (!ntiles || !ps || !vc) return gs_fail(c, GS_ECUDA, "scratch");
  GS_CUDA(c, cudaMemsetAsync(vc, 0, 2 * GS_MAX_VIEWS * sizeof(int64_t), st));
  ++c->launches;
  k_tile_counts<<<(unsigned)((n_recv + 256) / 256), 256, 0, st>>>(rec, n_recv, geo, g, ntiles, vc,
                                                                  vc + GS_MAX_VIEWS);
  GS_LAUNCH_CHECK(c, "tile counts");
  GS_CUDA(c, cudaMemcpyAsync(c->pinned, vc, 2 * GS_MAX_VIEWS * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  int64_t n_full = 0, K = 0;
  g.seg[0] = 0;
  g.kcum[0] = 0;
  for (int k = 0; k < g.nv; k++) {
    const int64_t cnt = c->pinned[k], own = c->pinned[GS_MAX_VIEWS + k];
    // >= 1 padding sentinel per segment (k_seg_ranges reads the segment's end off it)
    g.seg[k + 1] = g.seg[k] + (cnt + 1 + kRadixTile - 1) / kRadixTile * kRadixTile;
    g.shift[k] = g.seg[k] - n_full;
    g.kcum[k + 1] = g.kcum[k] + own;
    n_full += cnt;
    K += own;
  }
  const int64_t n_pad = g.seg[g.nv];
  *n_pairs_h = K;
  if (n_pad >= (1ll << 31))
    return gs_fail(c, GS_ENOTSUP, "pair total %lld exceeds int32 positions", (long long)n_pad);
  if (K > pair_cap) return gs_fail(c, GS_ECAPACITY, "pair capacity %lld < %lld", (long long)pair_cap, (long long)K);
  GS_REQUIRE(c, K == 0 || sorted_idx != nullptr, "null sorted_idx");
  const int64_t cap = std::max(n_pad, n_recv);
  uint32_t* A = (uint32_t*)gs_slot_get(c, SLOT_KEYS, 2 * cap * sizeof(uint32_t), st);
  uint32_t* Bf = (uint32_t*)gs_slot_get(c, SLOT_KEYS_TMP, 2 * cap * sizeof(uint32_t), st);
  if (!A || !Bf) return gs_fail(c, GS_ECUDA, "radix scratch (%lld pairs)", (long long)cap);
  uint32_t *ka = A, *va = A + cap, *kb = Bf, *vb = Bf + cap;
  // 2. records by (view, depth): 4 stable 8-bit depth passes (A -> B -> A -> B -> A), then the
  //    view (-> B -> A, values only kept)
  ++c->launches;
  k_depth_keys<<<(unsigned)((n_recv + 255) / 256), 256, 0, st>>>(rec, n_recv, ka, va);
  for (int p = 0; p < 4; p++) {
    s = (p & 1) ? radix_pass(c, kb, vb, ka, va, n_recv, 8 * p, 8, g, st)
                : radix_pass(c, ka, va, kb, vb, n_recv, 8 * p, 8, g, st);
    if (s != GS_OK) return s;
  }
  if (g.nv > 1) {
    ++c->launches;
    k_view_keys<<<(unsigned)((n_recv + 255) / 256), 256, 0, st>>>(rec, va, n_recv, g.v_lo, ka);
    s = radix_pass(c, ka, va, kb, vb, n_recv, 0, 32 - __builtin_clz((unsigned)(g.nv - 1)), g, st);
    if (s != GS_OK) return s;
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  // 3. pair starts in (view, depth) order; pairs (local block or sentinel, recv_idx) -> B, with
  //    the first pass's histogram
  ++c->launches;
  k_gather_tiles<<<(unsigned)((n_recv + 256) / 256), 256, 0, st>>>(va, ntiles, n_recv, ps);
  s = gs_scan_i64(c, ps, ps, n_recv + 1, 0, st);
  if (s != GS_OK) return s;
  const int64_t ntl = n_pad / kRadixTile;
  const int bins0 = 1 << std::min(width, nbits);
  unsigned long long* hist =
      (unsigned long long*)gs_slot_get(c, SLOT_RADIX_HIST, (size_t)(1 << width) * ntl * sizeof(int64_t), st);
  if (!hist) return gs_fail(c, GS_ECUDA, "radix histogram scratch");
  GS_CUDA(c, cudaMemsetAsync(hist, 0, (size_t)bins0 * ntl * sizeof(int64_t), st));
  if (n_full > 0) {
    const int64_t nct = (n_full + kEmitPairs - 1) / kEmitPairs;
    int64_t* first = (int64_t*)gs_slot_get(c, SLOT_LARGE, (nct + 1) * sizeof(int64_t), st);
    if (!first) return gs_fail(c, GS_ECUDA, "scratch");
    ++c->launches;
    k_cta_first<<<(unsigned)((n_recv + 255) / 256), 256, 0, st>>>(ps, n_recv, first);
    ++c->launches;
    k_emit<<<(unsigned)nct, kEmitThreads, 0, st>>>(rec, va, n_recv, ps, first, n_full, geo, g, std::min(width, nbits),
                                                   kb, vb, hist);
  }
  ++c->launches;
  k_pad<<<dim3(4, g.nv), 256, 0, st>>>(g, vc, std::min(width, nbits), kb, hist);
  GS_LAUNCH_CHECK(c, "bin_sort emit");
  // 4. stable segmented sort by view-local block index; the last pass writes the owned values
  //    compactly into sorted_idx and the keys into scratch
  uint32_t *kin = kb, *vin = vb, *kout = ka, *vout = va;
  for (int p = 0; p < passes; p++) {
    const int shift = p * width, bits = std::min(width, nbits - shift), bins = 1 << bits;
    if (p > 0) {
      ++c->launches;
      k_radix_hist<true><<<(unsigned)ntl, kRadixThreads, 0, st>>>(kin, n_pad, shift, bits, ntl, g, hist);
    }
    s = gs_scan_i64(c, (const int64_t*)hist, (int64_t*)hist, (int64_t)bins * ntl, 0, st);
    if (s != GS_OK) return s;
    ++c->launches;
    if (p == passes - 1)
      k_radix_scatter<true, true><<<(unsigned)ntl, kRadixThreads, kScatterSmem, st>>>(kin, vin, kout, sorted_idx, n_pad, shift,
                                                                          bits, ntl, g, hist, pair_cap);
    else
      k_radix_scatter<true, false><<<(unsigned)ntl, kRadixThreads, kScatterSmem, st>>>(kin, vin, kout, vout, n_pad, shift, bits,
                                                                           ntl, g, hist, 0);
    GS_LAUNCH_CHECK(c, "bin_sort pass");
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  // 5. ranges from the sorted keys (now in kin)
  ++c->launches;
  k_seg_ranges<<<(unsigned)(n_pad / 1024), 256, 0, st>>>(kin, g, pv, tile_range);
  GS_LAUNCH_CHECK(c, "bin_sort ranges");
  return GS_OK;
}
