// gs_sort.cu -- A3: Z-buffer build ("iterates over intersecting Gaussians in
// increasing depth"; App. A.2 "indices of intersecting gaussians for each pixel").
//
// B200 design (differs from the prior art's global 64-bit (tile | depth) radix sort of every
// (tile, Gaussian) pair): two levels.
//  1. The RECORDS are sorted by (view, depth) -- stable LSD radix over the 32 depth bits, then
//     the view -- so equal depths stay in receive order (= gid order within a view, R7).
//  2. Coarse binning: each record is paired with the SUPER-TILES (8 x 8 blocks, 128 x 128 px)
//     its tile rectangle touches (~2 per record instead of ~17 blocks), emitted in (view,
//     depth) order into per-view segments padded to radix tiles and stably radix-sorted by the
//     view-local super-tile index (10 bits at 4591x3436: 2 passes of 5; 8 bits at 1080p: one
//     pass) with one digit histogram laid out [view][digit][tile].  Each super-tile's coarse
//     list is then in (depth, gid) order.
//  3. Block offsets without storing any pair: each super-tile's coarse list is cut into
//     segments of kFineSeg records; per segment the hits of each of its 64 blocks are counted
//     (ballot popcounts of the records' block masks), a running sum over the super-tile's
//     segments gives every segment its blocks' starting ranks and every block its pair count,
//     and an exclusive scan over the owned blocks gives tile_range.  (A per-view 2D difference
//     array of the rectangles needs 4 atomics per record, which serialise when many records
//     share a rectangle corner -- the screen-clamped Gaussians of street views: 44 ms of C4.)
//  4. Fine emission: one CTA per super-tile walks its coarse list in order, 128 records at a
//     time; each record's blocks inside the super-tile are a 64-bit mask, the in-order rank of
//     a record among those hitting a block is a ballot popcount (plus the earlier warps'
//     counts), and the record index is stored at tile_range[block] + rank.  Block lists come
//     out in exact (depth, gid) order (O11) with no per-block sort, no pair keys and no pass
//     over the pairs besides the one store of each.
// Blocks the rank does not own (G > 1: rectangles straddling the partition) are masked out in
// step 4 and never counted in step 3.  One host sync per call: the per-view coarse and owned
// pair counts (scratch sizing, segment layout, the capacity check and *n_pairs_h).
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
constexpr int kSTShift = 3;        // super-tile side: 2^3 = 8 blocks (64 blocks: one 64-bit mask)
constexpr int kST = 1 << kSTShift;
constexpr int kFineThreads = 128;  // fine emission: records per chunk (4 warps)
constexpr int kFineSeg = 2048;     // fine emission: coarse-list records per CTA (16 chunks)

// The coarse grid: super-tile (sx, sy) = blocks [8 sx, 8 sx + 7] x [8 sy, 8 sy + 7] of the
// view, view-local index sy * Cw + sx.
struct cgrid {
  int Cw, Ch;
};
// A record's tile rectangle and view packed into 8 bytes (k_tile_counts, read by the emission
// kernels instead of the 64-byte record): x = tx0 | tx1 << 16, y = ty0 | ty1 << 13 | view << 26
// (Wt < 2^16, Ht < 2^13); an empty rectangle has tx0 > tx1.
__device__ __forceinline__ uint2 pack_rect(int tx0, int tx1, int ty0, int ty1, int v) {
  return make_uint2((unsigned)tx0 | (unsigned)tx1 << 16, (unsigned)ty0 | (unsigned)ty1 << 13 | (unsigned)v << 26);
}
__device__ __forceinline__ void unpack_rect(uint2 r, int& tx0, int& tx1, int& ty0, int& ty1, int& v) {
  tx0 = (int)(r.x & 0xffffu);
  tx1 = (int)(r.x >> 16);
  ty0 = (int)(r.y & 0x1fffu);
  ty1 = (int)((r.y >> 13) & 0x1fffu);
  v = (int)(r.y >> 26);
}
__device__ __forceinline__ void coarse_rect(int tx0, int tx1, int ty0, int ty1, int& sx0, int& sx1, int& sy0,
                                            int& sy1) {
  sx0 = tx0 >> kSTShift;
  sx1 = tx1 >> kSTShift;
  sy0 = ty0 >> kSTShift;
  sy1 = ty1 >> kSTShift;
}

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

// Per record: its coarse-pair count (super-tiles its tile rectangle touches), its packed
// rectangle, and per view the coarse-pair total and the owned-pair total (owned = view-local
// block in [lo, hi): per rectangle row an interval intersection).  cnt[k] / own[k] over the
// rank's views; g.lo / g.hi are the FINE ownership bounds here.
// nrec[k]: records of view k; unord: set when a record's view is below its predecessor's
// (the receive buffer is then not view-contiguous and the records take the general sort).
__global__ void k_tile_counts(const gs_rec* __restrict__ rec, int64_t n_recv, gs_geom geo, seg_arg g,
                              int64_t* __restrict__ n_coarse, unsigned long long* __restrict__ cnt,
                              unsigned long long* __restrict__ own, uint2* __restrict__ rect8,
                              unsigned long long* __restrict__ nrec, unsigned long long* __restrict__ unord,
                              uint32_t* __restrict__ dbits) {
  __shared__ unsigned long long s_c[GS_MAX_VIEWS], s_o[GS_MAX_VIEWS];
  __shared__ unsigned s_r[GS_MAX_VIEWS];
  if (threadIdx.x < GS_MAX_VIEWS) s_c[threadIdx.x] = s_o[threadIdx.x] = 0, s_r[threadIdx.x] = 0;
  __syncthreads();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned t = 0, o = 0;
  int k = -1;
  if (j < n_recv) {
    const float4 a = rec[j].a;
    dbits[j] = __float_as_uint(a.z);  // depth > 0: the bit pattern orders like the value
    const int v = (int)(__float_as_uint(rec[j].d.w) & 31u);
    if (j > 0 && (int)(__float_as_uint(rec[j - 1].d.w) & 31u) > v) atomicOr(unord, 1ull);
    if (v - g.v_lo >= 0 && v - g.v_lo < g.nv) atomicAdd(&s_r[v - g.v_lo], 1u);
    k = v - g.v_lo;
    int tx0, tx1, ty0, ty1;
    const bool ok = k >= 0 && k < g.nv && rect_of(a.x, a.y, a.w, geo.Wt, geo.Ht, tx0, tx1, ty0, ty1);
    rect8[j] = ok ? pack_rect(tx0, tx1, ty0, ty1, v) : pack_rect(1, 0, 0, 0, v);
    if (ok) {
      int sx0, sx1, sy0, sy1;
      coarse_rect(tx0, tx1, ty0, ty1, sx0, sx1, sy0, sy1);
      t = (unsigned)((sx1 - sx0 + 1) * (sy1 - sy0 + 1));
      for (int ty = ty0; ty <= ty1; ty++) {
        const long long r0 = (long long)ty * geo.Wt + tx0, r1 = (long long)ty * geo.Wt + tx1 + 1;
        o += (unsigned)max(0ll, min(r1, (long long)g.hi[k]) - max(r0, (long long)g.lo[k]));
      }
    } else {
      k = -1;
    }
  }
  if (j <= n_recv) n_coarse[j] = t;
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
  if (threadIdx.x < GS_MAX_VIEWS && s_r[threadIdx.x]) atomicAdd(&nrec[threadIdx.x], (unsigned long long)s_r[threadIdx.x]);
}

__global__ void k_depth_keys(const uint32_t* __restrict__ dbits, int64_t n, uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ vals) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  keys[j] = dbits[j];
  vals[j] = (uint32_t)j;
}

// View-contiguous records (the receive buffer of one rank's own views): depth keys laid out
// in per-view segments padded to radix tiles (padded position p of segment k holds record
// kcum[k] + p - seg[k], or the sentinel 0xffffffff -- above every depth's bits -- past the
// view's records), so four segmented stable passes sort each view by depth with no view pass.
__global__ void k_depth_keys_seg(const uint32_t* __restrict__ dbits, seg_arg r, uint32_t* __restrict__ keys,
                                 uint32_t* __restrict__ vals) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= r.seg[r.nv]) return;
  const int k = seg_of_tile(r, p / kRadixTile);
  const int64_t o = p - r.seg[k], nk = r.kcum[k + 1] - r.kcum[k];
  const int64_t j = r.kcum[k] + o;
  keys[p] = o < nk ? dbits[j] : 0xffffffffu;
  vals[p] = o < nk ? (uint32_t)j : 0u;
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

// Emit the coarse pairs of the ordered records: CTA c enumerates unpadded pairs
// [c*kEmitPairs, ...) of pair_start (= scan of the coarse counts in (view, depth) order) and
// stores each at its padded position (+ shift of its view's segment): key = view-local
// super-tile index; value = recv_idx.  The histogram of the first digit
// pass (bits [0, bits0)) is accumulated on the way ([segment][digit][tile] layout).  Every
// received record has >= 1 tile (A1 emits a record only for a rectangle with an owned block),
// so at most kEmitPairs + 1 records overlap a CTA.
__global__ void __launch_bounds__(kEmitThreads) k_emit(
    const uint2* __restrict__ rect8, const uint32_t* __restrict__ order, int64_t n_recv,
    const int64_t* __restrict__ pair_start, const int64_t* __restrict__ first, int64_t n_full, gs_geom geo,
    cgrid cg, seg_arg g, int bits0, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
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
    int tx0, tx1, ty0, ty1, v, sx0, sx1, sy0, sy1;
    unpack_rect(rect8[j], tx0, tx1, ty0, ty1, v);
    coarse_rect(tx0, tx1, ty0, ty1, sx0, sx1, sy0, sy1);
    s_tx0[r] = sx0;
    s_ty0[r] = sy0;
    s_w[r] = sx1 - sx0 + 1;
    s_k[r] = v - g.v_lo;
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
    const int local = (s_ty0[lo] + q) * cg.Cw + s_tx0[lo] + rm;
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

__global__ void k_to_i32(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int32_t)in[i];
}

// 32 x 32 bit-matrix transpose across a warp: lane i holds row i (bit k = column k); lane k
// gets column k (bit i = row i's bit k).  Five stages; stage j swaps the off-diagonal j x j
// blocks between lanes i and i ^ j.
__device__ __forceinline__ unsigned warp_transpose32(unsigned v, int lane) {
  const unsigned masks[5] = {0x0000ffffu, 0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int s = 0; s < 5; s++) {
    const int j = 16 >> s;
    const unsigned m = masks[s];
    const unsigned o = __shfl_xor_sync(0xffffffffu, v, j);
    v = (lane & j) ? ((v & ~m) | ((o >> j) & m)) : ((v & m) | ((o << j) & ~m));
  }
  return v;
}

// Fine emission, one CTA per segment of kFineSeg records of a (view k, super-tile)'s coarse
// list (crange, in (depth, gid) order; fseg[t] = the first segment of super-tile t), in chunks
// of 128 records, one per thread.  Each segment's block cursors start at tile_range + the
// hits of the super-tile's earlier segments (fcnt, k_fine_count + k_fine_prefix), so the
// segments of a long list (the horizon rows of street views reach ~10^5 records per
// super-tile) run in parallel and each block list still comes out in order.  A record's owned blocks
// inside the super-tile form a 64-bit mask (bit 8 j + i = block (8 sx + i, 8 sy + j)).  Each
// warp transposes its 32 masks, so lane l holds the 32-bit sets of its lanes (= records, in
// order) hitting block l and block l + 32; their popcounts are the warp's counts (phase 1).
// Phase 2 (warp 0) turns them into offsets: per block the earlier warps' counts, and the
// block's place in the chunk's staging array (blocks back to back, an exclusive scan of the
// chunk's per-block totals).  In phase 3 lane l places the record indices of its two blocks,
// in lane order, into the staging array (and the block of every staged entry); in phase 4 the
// CTA walks the staged entries linearly and stores each at its block's cursor (started at
// tile_range) + its place in the block's run: consecutive threads store mostly consecutive
// addresses.  Every block list keeps the coarse (depth, gid) order.
struct fine_arg {
  int nv, v_lo, nST;
  int lo[GS_MAX_VIEWS], hi[GS_MAX_VIEWS];  // owned view-local blocks [lo, hi) of view k
  long long B_lo;
};
// The segment of CTA `bid`: its super-tile t (fseg[t] <= bid < fseg[t + 1], binary search)
// and coarse-list range [cs, ce); false past the last segment.  Also the super-tile's owned
// blocks (bit b of own_lo / own_hi: block b / b + 32, every lane computes the same mask).
struct fine_seg {
  int t, k, bx0, by0, cs, ce, seg;
  unsigned own_lo, own_hi;
};
__device__ __forceinline__ bool find_fine_seg(int64_t bid, const int64_t* __restrict__ fseg, int nt,
                                              const int32_t* __restrict__ crange, const gs_geom& geo,
                                              const cgrid& cg, const fine_arg& f, fine_seg& q) {
  if (bid >= fseg[nt]) return false;
  int lo = 0, hi = nt;  // largest t with fseg[t] <= bid (empty super-tiles have fseg[t] == fseg[t+1])
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (fseg[mid] <= bid) lo = mid; else hi = mid;
  }
  q.t = lo;
  q.seg = (int)(bid - fseg[lo]);
  const int cs0 = crange[lo], ce0 = crange[lo + 1];
  q.cs = cs0 + q.seg * kFineSeg;
  q.ce = min(ce0, q.cs + kFineSeg);
  q.k = lo / f.nST;
  const int sidx = lo - q.k * f.nST;
  q.bx0 = (sidx % cg.Cw) * kST;
  q.by0 = (sidx / cg.Cw) * kST;
  const int lane = threadIdx.x & 31;
  bool ob[2];
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int b = lane + 32 * h, bx = q.bx0 + (b & (kST - 1)), by = q.by0 + (b >> kSTShift);
    const int loc = by * geo.Wt + bx;
    ob[h] = bx < geo.Wt && by < geo.Ht && loc >= f.lo[q.k] && loc < f.hi[q.k];
  }
  q.own_lo = __ballot_sync(0xffffffffu, ob[0]);
  q.own_hi = __ballot_sync(0xffffffffu, ob[1]);
  return true;
}

// The owned blocks of the super-tile that coarse-list record i hits, as a 64-bit mask.
__device__ __forceinline__ void fine_mask(const uint2* __restrict__ rect8, uint32_t j, const fine_seg& q,
                                          unsigned& mlo, unsigned& mhi) {
  int tx0, tx1, ty0, ty1, v;
  unpack_rect(__ldg(&rect8[j]), tx0, tx1, ty0, ty1, v);
  const int ix0 = max(tx0 - q.bx0, 0), ix1 = min(tx1 - q.bx0, kST - 1);
  const int iy0 = max(ty0 - q.by0, 0), iy1 = min(ty1 - q.by0, kST - 1);
  mlo = mhi = 0;
  if (ix0 <= ix1 && iy0 <= iy1) {
    const unsigned long long cols =
        (unsigned long long)((0xffu << ix0) & (0xffu >> (kST - 1 - ix1))) * 0x0101010101010101ull;
    const unsigned long long rows = (~0ull << (8 * iy0)) & (~0ull >> (8 * (kST - 1 - iy1)));
    const unsigned long long m = cols & rows;
    mlo = (unsigned)m & q.own_lo;
    mhi = (unsigned)(m >> 32) & q.own_hi;
  }
}

// Segments per super-tile: fseg[t] = ceil(len_t / kFineSeg) (then exclusively scanned).
__global__ void k_fine_nseg(const int32_t* __restrict__ crange, int nt, int64_t* __restrict__ fseg) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nt) fseg[t] = (crange[t + 1] - crange[t] + kFineSeg - 1) / kFineSeg;
}

// Per-block hit counts of every segment: fcnt[seg][64].
__global__ void __launch_bounds__(kFineThreads) k_fine_count(const uint2* __restrict__ rect8,
                                                             const uint32_t* __restrict__ clist,
                                                             const int32_t* __restrict__ crange,
                                                             const int64_t* __restrict__ fseg, int nt, gs_geom geo,
                                                             cgrid cg, fine_arg f, int* __restrict__ fcnt) {
  constexpr int kB = kST * kST;
  __shared__ int s_c[kB];
  fine_seg q;
  if (!find_fine_seg(blockIdx.x, fseg, nt, crange, geo, cg, f, q)) return;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < kB) s_c[tid] = 0;
  __syncthreads();
  int a = 0, b = 0;  // this lane's counts of blocks lane, lane + 32 (over its warp's chunks)
  for (int c0 = q.cs; c0 < q.ce; c0 += kFineThreads) {
    const int i = c0 + tid;
    unsigned mlo = 0, mhi = 0;
    if (i < q.ce) fine_mask(rect8, clist[i], q, mlo, mhi);
    a += __popc(warp_transpose32(mlo, lane));
    b += __popc(warp_transpose32(mhi, lane));
  }
  atomicAdd(&s_c[lane], a);
  atomicAdd(&s_c[lane + 32], b);
  __syncthreads();
  if (tid < kB) fcnt[(int64_t)blockIdx.x * kB + tid] = s_c[tid];
}

// fcnt[seg][b] -> the hits of block b in the super-tile's earlier segments, and the block's
// pair count (all its segments) to bcnt at its owned index (one thread per (super-tile,
// block), sequential over the super-tile's segments; every owned block is written once).
__global__ void k_fine_prefix(const int64_t* __restrict__ fseg, int nt, int* __restrict__ fcnt, gs_geom geo,
                              cgrid cg, fine_arg f, int64_t* __restrict__ bcnt) {
  constexpr int kB = kST * kST;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int64_t)nt * kB) return;
  const int t = (int)(g / kB), b = (int)(g % kB);
  const int k = t / f.nST, sidx = t - k * f.nST;
  const int bx = (sidx % cg.Cw) * kST + (b & (kST - 1)), by = (sidx / cg.Cw) * kST + (b >> kSTShift);
  const int loc = by * geo.Wt + bx;
  const bool own = bx < geo.Wt && by < geo.Ht && loc >= f.lo[k] && loc < f.hi[k];
  const int64_t s0 = fseg[t], s1 = fseg[t + 1];
  int run = 0;
  for (int64_t s = s0; s < s1; s++) {
    const int x = fcnt[s * kB + b];
    fcnt[s * kB + b] = run;
    run += x;
  }
  if (own) bcnt[(int64_t)(f.v_lo + k) * geo.per_view + loc - f.B_lo] = run;
}

__global__ void __launch_bounds__(kFineThreads) k_fine(const uint2* __restrict__ rect8,
                                                       const uint32_t* __restrict__ clist,
                                                       const int32_t* __restrict__ crange,
                                                       const int64_t* __restrict__ fseg, int nt,
                                                       const int* __restrict__ fcnt, gs_geom geo, cgrid cg,
                                                       fine_arg f, const int32_t* __restrict__ range,
                                                       uint32_t* __restrict__ out) {
  constexpr int kW = kFineThreads / 32, kB = kST * kST;
  constexpr int kStage = kB / 2 * kFineThreads;  // staged entries per pass (one half of the blocks)
  __shared__ int s_cur[kB];   // block cursor (next free position of its list)
  __shared__ int s_dst[kB];   // this chunk: cursor - staging start of the block
  __shared__ int s_wc[kW][kB];
  __shared__ int s_tot, s_tot_a;
  __shared__ uint32_t s_flat[kStage + 1];
  __shared__ uint8_t s_blk[kStage + 1];
  fine_seg q;
  if (!find_fine_seg(blockIdx.x, fseg, nt, crange, geo, cg, f, q)) return;
  const int cs = q.cs, ce = q.ce, k = q.k, bx0 = q.bx0, by0 = q.by0;
  const unsigned own_lo = q.own_lo, own_hi = q.own_hi;
  if (cs >= ce || (own_lo | own_hi) == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid < kB) {
    const int loc = (by0 + (tid >> kSTShift)) * geo.Wt + bx0 + (tid & (kST - 1));
    s_cur[tid] = ((tid >> 5 ? own_hi : own_lo) >> (tid & 31) & 1u)
                     ? range[(int64_t)(f.v_lo + k) * geo.per_view + loc - f.B_lo] + fcnt[(int64_t)blockIdx.x * kB + tid]
                     : 0;
  }
  for (int c0 = cs; c0 < ce; c0 += kFineThreads) {
    __syncthreads();  // s_cur initialised / the previous chunk's staging written out
    const int i = c0 + tid;
    uint32_t j = 0;
    unsigned mlo = 0, mhi = 0;
    if (i < ce) {
      j = clist[i];
      fine_mask(rect8, j, q, mlo, mhi);
    }
    // lane l: which of the warp's records hit block l (tlo) and block l + 32 (thi)
    unsigned tlo = warp_transpose32(mlo, lane), thi = warp_transpose32(mhi, lane);
    s_wc[w][lane] = __popc(tlo);  // phase 1
    s_wc[w][lane + 32] = __popc(thi);
    __syncthreads();
    if (w == 0) {  // phase 2: blocks lane and lane + 32
      int ra = 0, rb = 0;
#pragma unroll
      for (int ww = 0; ww < kW; ww++) {
        const int ta = s_wc[ww][lane], tb = s_wc[ww][lane + 32];
        s_wc[ww][lane] = ra;
        s_wc[ww][lane + 32] = rb;
        ra += ta;
        rb += tb;
      }
      // staging starts: exclusive scan of the 64 block totals (blocks 0..31, then 32..63)
      int ia = ra, ib = rb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ya = __shfl_up_sync(0xffffffffu, ia, o), yb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) ia += ya, ib += yb;
      }
      const int tot_a = __shfl_sync(0xffffffffu, ia, 31);
      const int sa = ia - ra, sb = tot_a + ib - rb;
      // the warp offsets become staging positions; s_dst maps them to list positions
      for (int ww = 0; ww < kW; ww++) s_wc[ww][lane] += sa, s_wc[ww][lane + 32] += sb;
      const int ca = s_cur[lane], cb = s_cur[lane + 32];
      s_dst[lane] = ca - sa;
      s_dst[lane + 32] = cb - sb;
      s_cur[lane] = ca + ra;
      s_cur[lane + 32] = cb + rb;
      if (lane == 31) s_tot = tot_a + ib, s_tot_a = tot_a;
    }
    __syncthreads();
    // phases 3 + 4 over the staging array; a chunk with more than kStage entries is staged in
    // two halves (blocks 0..31, then 32..63: at most 32 x 128 entries each)
    const int tot = s_tot, tot_a = s_tot_a;
    const bool split = tot > kStage;
    for (int half = 0; half < (split ? 2 : 1); half++) {
      unsigned xa = (split && half == 1) ? 0u : tlo, xb = (split && half == 0) ? 0u : thi;
      const int sh = (split && half == 1) ? tot_a : 0;  // staging position of the pass's first entry
      int plo = s_wc[w][lane] - sh, phi = s_wc[w][lane + 32] - sh;
      while (__any_sync(0xffffffffu, (xa | xb) != 0)) {  // phase 3: lane order = record order
        const int ra = __ffs(xa) - 1, rb = __ffs(xb) - 1;  // -1 (unused) when empty
        const uint32_t ja = __shfl_sync(0xffffffffu, j, ra & 31), jb = __shfl_sync(0xffffffffu, j, rb & 31);
        const int da = xa ? plo : kStage, db = xb ? phi : kStage;  // kStage: a dummy slot
        s_flat[da] = ja;
        s_blk[da] = (uint8_t)lane;
        s_flat[db] = jb;
        s_blk[db] = (uint8_t)(lane + 32);
        plo += xa != 0u;
        phi += xb != 0u;
        xa &= xa - 1;
        xb &= xb - 1;
      }
      __syncthreads();
      const int n = split ? (half ? tot - tot_a : tot_a) : tot;
      for (int e = tid; e < n; e += kFineThreads) out[s_dst[s_blk[e]] + sh + e] = s_flat[e];  // phase 4
      if (split && half == 0) __syncthreads();  // the staging is reused by the second half
    }
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

// One stable segmented 8-bit pass over n_pad padded elements (layout of g); last: values
// to vout at their compact positions (sentinels dropped).  Scratch: SLOT_RADIX_HIST.
gs_status seg_radix_pass(gs_ctx* c, const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                         int64_t n_pad, int shift, const seg_arg& g, bool last, int64_t vcap, cudaStream_t st) {
  if (n_pad == 0) return GS_OK;
  const int bins = 256;
  const int64_t ntl = n_pad / kRadixTile;
  unsigned long long* hist =
      (unsigned long long*)gs_slot_get(c, SLOT_RADIX_HIST, (size_t)bins * ntl * sizeof(int64_t), st);
  if (!hist) return gs_fail(c, GS_ECUDA, "radix histogram scratch");
  ++c->launches;
  k_radix_hist<true><<<(unsigned)ntl, kRadixThreads, 0, st>>>(kin, n_pad, shift, 8, ntl, g, hist);
  gs_status s = gs_scan_i64(c, (const int64_t*)hist, (int64_t*)hist, (int64_t)bins * ntl, 0, st);
  if (s != GS_OK) return s;
  ++c->launches;
  if (last)
    k_radix_scatter<true, true><<<(unsigned)ntl, kRadixThreads, kScatterSmem, st>>>(kin, vin, kout, vout, n_pad, shift,
                                                                                    8, ntl, g, hist, vcap);
  else
    k_radix_scatter<true, false><<<(unsigned)ntl, kRadixThreads, kScatterSmem, st>>>(kin, vin, kout, vout, n_pad,
                                                                                     shift, 8, ntl, g, hist, 0);
  GS_LAUNCH_CHECK(c, "segmented radix pass");
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
  // the coarse grid (super-tiles of 8 x 8 blocks) and its segment layout arguments
  cgrid cg;
  cg.Cw = (geo.Wt + kST - 1) / kST;
  cg.Ch = (geo.Ht + kST - 1) / kST;
  const int nST = cg.Cw * cg.Ch;
  fine_arg fa;
  memset(&fa, 0, sizeof(fa));
  fa.nv = g.nv;
  fa.v_lo = g.v_lo;
  fa.nST = nST;
  fa.B_lo = B_lo;
  for (int k = 0; k < g.nv; k++) fa.lo[k] = g.lo[k], fa.hi[k] = g.hi[k];
  GS_REQUIRE(c, (int64_t)g.nv * nST < (1ll << 31) - 1, "too many super-tiles");
  GS_REQUIRE(c, geo.Wt < (1 << 16) && geo.Ht < (1 << 13), "image of %d x %d blocks exceeds the packed rectangle",
             geo.Wt, geo.Ht);
  // 1. per-record coarse counts, per-view coarse and owned-pair totals (one host sync)
  int64_t* ncoarse = (int64_t*)gs_slot_get(c, SLOT_RECTILES, (n_recv + 1) * sizeof(int64_t), st);
  // ps: the depth bits of the records (k_tile_counts -> the depth keys), later the coarse pair
  // starts in (view, depth) order (k_gather_tiles)
  int64_t* ps = (int64_t*)gs_slot_get(c, SLOT_PSTART, (n_recv + 1) * sizeof(int64_t), st);
  // per view: coarse pairs, owned pairs, records; then the view-order flag
  unsigned long long* vc = (unsigned long long*)gs_slot_get(c, SLOT_COUNTS, (3 * GS_MAX_VIEWS + 1) * sizeof(int64_t), st);
  uint2* rect8 = (uint2*)gs_slot_get(c, SLOT_RECT8, n_recv * sizeof(uint2), st);
  if (!ncoarse || !ps || !vc || !rect8) return gs_fail(c, GS_ECUDA, "scratch");
  GS_CUDA(c, cudaMemsetAsync(vc, 0, (3 * GS_MAX_VIEWS + 1) * sizeof(int64_t), st));
  ++c->launches;
  k_tile_counts<<<(unsigned)((n_recv + 256) / 256), 256, 0, st>>>(rec, n_recv, geo, g, ncoarse, vc,
                                                                  vc + GS_MAX_VIEWS, rect8, vc + 2 * GS_MAX_VIEWS,
                                                                  vc + 3 * GS_MAX_VIEWS, (uint32_t*)ps);
  GS_LAUNCH_CHECK(c, "tile counts");
  GS_CUDA(c, cudaMemcpyAsync(c->pinned, vc, (3 * GS_MAX_VIEWS + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  // coarse segments: every super-tile key is "owned" ([0, nST)); the sentinel pads
  seg_arg cgs = g;
  const int nbits = 32 - __builtin_clz((unsigned)nST);  // 2^nbits > nST: the sentinel exceeds every key
  cgs.sentinel = (1u << nbits) - 1u;
  cgs.B_lo = (long long)g.v_lo * nST;
  const int passes = (nbits + 7) / 8, width = (nbits + passes - 1) / passes;
  int64_t n_full = 0, K = 0;
  cgs.seg[0] = 0;
  cgs.kcum[0] = 0;
  for (int k = 0; k < g.nv; k++) {
    const int64_t cnt = c->pinned[k], own = c->pinned[GS_MAX_VIEWS + k];
    cgs.lo[k] = 0;
    cgs.hi[k] = nST;
    // >= 1 padding sentinel per segment (k_seg_ranges reads the segment's end off it)
    cgs.seg[k + 1] = cgs.seg[k] + (cnt + 1 + kRadixTile - 1) / kRadixTile * kRadixTile;
    cgs.shift[k] = cgs.seg[k] - n_full;
    cgs.kcum[k + 1] = cgs.kcum[k] + cnt;
    n_full += cnt;
    K += own;
  }
  const int64_t n_pad = cgs.seg[g.nv];
  *n_pairs_h = K;
  if (n_pad >= (1ll << 31) || K >= (1ll << 31))
    return gs_fail(c, GS_ENOTSUP, "pair total %lld exceeds int32 positions", (long long)std::max(n_pad, K));
  if (K > pair_cap) return gs_fail(c, GS_ECAPACITY, "pair capacity %lld < %lld", (long long)pair_cap, (long long)K);
  GS_REQUIRE(c, K == 0 || sorted_idx != nullptr, "null sorted_idx");
  if (K == 0) {  // no owned pair: empty lists
    GS_CUDA(c, cudaMemsetAsync(tile_range, 0, (n_owned + 1) * sizeof(int32_t), st));
    return GS_OK;
  }

  // 3. records by (view, depth): view-contiguous records in 4 segmented stable 8-bit depth
  //    passes; otherwise 4 stable depth passes (A -> B -> A -> B -> A), then the view (-> B -> A,
  //    values only kept)
  // view-contiguous records (one rank's own receive buffer at G = 1 is bucketed by view): the
  // records' own per-view segments, sorted by depth in 4 segmented passes
  seg_arg rs = g;
  bool vseg = c->pinned[3 * GS_MAX_VIEWS] == 0;
  {
    int64_t tot = 0;
    rs.seg[0] = 0;
    rs.kcum[0] = 0;
    for (int k = 0; k < g.nv; k++) {
      const int64_t nk = c->pinned[2 * GS_MAX_VIEWS + k];
      rs.seg[k + 1] = rs.seg[k] + (nk + kRadixTile - 1) / kRadixTile * kRadixTile;
      rs.kcum[k + 1] = rs.kcum[k] + nk;
      tot += nk;
    }
    rs.sentinel = 0xffffffffu;
    vseg = vseg && tot == n_recv && g.nv > 1;  // every record in an owned view (else: general path)
  }
  const int64_t cap = std::max(std::max(n_pad, n_recv), vseg ? (int64_t)rs.seg[g.nv] : 0);
  uint32_t* A = (uint32_t*)gs_slot_get(c, SLOT_KEYS, 2 * cap * sizeof(uint32_t), st);
  uint32_t* Bf = (uint32_t*)gs_slot_get(c, SLOT_KEYS_TMP, 2 * cap * sizeof(uint32_t), st);
  uint32_t* clist = (uint32_t*)gs_slot_get(c, SLOT_CLIST, std::max<int64_t>(n_full, 1) * sizeof(uint32_t), st);
  int32_t* crange = (int32_t*)gs_slot_get(c, SLOT_CRANGE, ((int64_t)g.nv * nST + 1) * sizeof(int32_t), st);
  if (!A || !Bf || !clist || !crange) return gs_fail(c, GS_ECUDA, "radix scratch (%lld pairs)", (long long)cap);
  uint32_t *ka = A, *va = A + cap, *kb = Bf, *vb = Bf + cap;
  if (vseg) {
    const int64_t np_ = rs.seg[g.nv];
    ++c->launches;
    k_depth_keys_seg<<<(unsigned)((np_ + 255) / 256), 256, 0, st>>>((const uint32_t*)ps, rs, ka, va);
    // A -> B -> A -> B, the last pass writing the values compact into va (sentinels dropped)
    for (int p = 0; p < 4; p++) {
      s = (p & 1) ? seg_radix_pass(c, kb, vb, ka, va, np_, 8 * p, rs, p == 3, n_recv, st)
                  : seg_radix_pass(c, ka, va, kb, vb, np_, 8 * p, rs, false, 0, st);
      if (s != GS_OK) return s;
    }
  } else {
    ++c->launches;
    k_depth_keys<<<(unsigned)((n_recv + 255) / 256), 256, 0, st>>>((const uint32_t*)ps, n_recv, ka, va);
    for (int p = 0; p < 4; p++) {
      s = (p & 1) ? radix_pass(c, kb, vb, ka, va, n_recv, 8 * p, 8, g, st)
                  : radix_pass(c, ka, va, kb, vb, n_recv, 8 * p, 8, g, st);
      if (s != GS_OK) return s;
    }
  }
  if (!vseg && g.nv > 1) {
    ++c->launches;
    k_view_keys<<<(unsigned)((n_recv + 255) / 256), 256, 0, st>>>(rec, va, n_recv, g.v_lo, ka);
    s = radix_pass(c, ka, va, kb, vb, n_recv, 0, 32 - __builtin_clz((unsigned)(g.nv - 1)), g, st);
    if (s != GS_OK) return s;
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  // 4. coarse pair starts in (view, depth) order; coarse pairs (super-tile, recv_idx) -> B,
  //    with the first pass's histogram
  ++c->launches;
  k_gather_tiles<<<(unsigned)((n_recv + 256) / 256), 256, 0, st>>>(va, ncoarse, n_recv, ps);
  s = gs_scan_i64(c, ps, ps, n_recv + 1, 0, st);
  if (s != GS_OK) return s;
  const int64_t ntl = n_pad / kRadixTile;
  const int bins0 = 1 << std::min(width, nbits);
  unsigned long long* hist =
      (unsigned long long*)gs_slot_get(c, SLOT_RADIX_HIST, (size_t)(1 << width) * ntl * sizeof(int64_t), st);
  if (!hist) return gs_fail(c, GS_ECUDA, "radix histogram scratch");
  GS_CUDA(c, cudaMemsetAsync(hist, 0, (size_t)bins0 * ntl * sizeof(int64_t), st));
  {
    const int64_t nct = (n_full + kEmitPairs - 1) / kEmitPairs;
    int64_t* first = (int64_t*)gs_slot_get(c, SLOT_LARGE, (nct + 1) * sizeof(int64_t), st);
    if (!first) return gs_fail(c, GS_ECUDA, "scratch");
    ++c->launches;
    k_cta_first<<<(unsigned)((n_recv + 255) / 256), 256, 0, st>>>(ps, n_recv, first);
    ++c->launches;
    k_emit<<<(unsigned)nct, kEmitThreads, 0, st>>>(rect8, va, n_recv, ps, first, n_full, geo, cg, cgs,
                                                   std::min(width, nbits), kb, vb, hist);
  }
  ++c->launches;
  k_pad<<<dim3(4, g.nv), 256, 0, st>>>(cgs, vc, std::min(width, nbits), kb, hist);
  GS_LAUNCH_CHECK(c, "bin_sort emit");
  // 5. stable segmented sort by view-local super-tile; the last pass writes the record indices
  //    compactly into clist and the keys into scratch
  uint32_t *kin = kb, *vin = vb, *kout = ka, *vout = va;
  for (int p = 0; p < passes; p++) {
    const int shift = p * width, bits = std::min(width, nbits - shift), bins = 1 << bits;
    if (p > 0) {
      ++c->launches;
      k_radix_hist<true><<<(unsigned)ntl, kRadixThreads, 0, st>>>(kin, n_pad, shift, bits, ntl, cgs, hist);
    }
    s = gs_scan_i64(c, (const int64_t*)hist, (int64_t*)hist, (int64_t)bins * ntl, 0, st);
    if (s != GS_OK) return s;
    ++c->launches;
    if (p == passes - 1)
      k_radix_scatter<true, true><<<(unsigned)ntl, kRadixThreads, kScatterSmem, st>>>(kin, vin, kout, clist, n_pad,
                                                                                      shift, bits, ntl, cgs, hist,
                                                                                      n_full);
    else
      k_radix_scatter<true, false><<<(unsigned)ntl, kRadixThreads, kScatterSmem, st>>>(kin, vin, kout, vout, n_pad,
                                                                                       shift, bits, ntl, cgs, hist, 0);
    GS_LAUNCH_CHECK(c, "bin_sort pass");
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  // 6. super-tile ranges of the coarse lists (sorted keys now in kin), then the fine emission
  ++c->launches;
  k_seg_ranges<<<(unsigned)(n_pad / 1024), 256, 0, st>>>(kin, cgs, nST, crange);
  // fine emission over segments of kFineSeg coarse records (long lists split across CTAs)
  const int nt = g.nv * nST;
  const int64_t nseg_max = nt + n_full / kFineSeg + 1;  // >= sum over t of ceil(len_t / kFineSeg)
  int64_t* fseg = (int64_t*)gs_slot_get(c, SLOT_CURSOR, ((int64_t)nt + 1) * sizeof(int64_t), st);
  int* fcnt = (int*)gs_slot_get(c, SLOT_FSEG_CNT, nseg_max * kST * kST * sizeof(int), st);
  if (!fseg || !fcnt) return gs_fail(c, GS_ECUDA, "fine emission scratch");
  ++c->launches;
  k_fine_nseg<<<(unsigned)((nt + 256) / 256), 256, 0, st>>>(crange, nt, fseg);
  GS_CUDA(c, cudaMemsetAsync(fseg + nt, 0, sizeof(int64_t), st));
  s = gs_scan_i64(c, fseg, fseg, (int64_t)nt + 1, 0, st);
  if (s != GS_OK) return s;
  // block pair counts -> tile_range (exclusive scan over the owned blocks)
  int64_t* bcnt = (int64_t*)gs_slot_get(c, SLOT_BCOUNT, (n_owned + 1) * sizeof(int64_t), st);
  if (!bcnt) return gs_fail(c, GS_ECUDA, "scratch");
  GS_CUDA(c, cudaMemsetAsync(bcnt + n_owned, 0, sizeof(int64_t), st));
  ++c->launches;
  k_fine_count<<<(unsigned)nseg_max, kFineThreads, 0, st>>>(rect8, clist, crange, fseg, nt, geo, cg, fa, fcnt);
  ++c->launches;
  k_fine_prefix<<<(unsigned)(((int64_t)nt * kST * kST + 255) / 256), 256, 0, st>>>(fseg, nt, fcnt, geo, cg, fa,
                                                                                   bcnt);
  GS_LAUNCH_CHECK(c, "block counts");
  s = gs_scan_i64(c, bcnt, bcnt, n_owned + 1, 0, st);
  if (s != GS_OK) return s;
  ++c->launches;
  k_to_i32<<<(unsigned)((n_owned + 256) / 256), 256, 0, st>>>(bcnt, n_owned + 1, tile_range);
  ++c->launches;
  k_fine<<<(unsigned)nseg_max, kFineThreads, 0, st>>>(rect8, clist, crange, fseg, nt, fcnt, geo, cg, fa,
                                                     tile_range, sorted_idx);
  GS_LAUNCH_CHECK(c, "bin_sort fine");
  return GS_OK;
}
