// gs_render.cu -- A4/A5: front-to-back alpha compositing and its backward over the rank's
// owned 16x16 blocks.
//
// One CTA per owned block; each thread owns PPT pixels of one column, 16/PPT rows apart
// (PPT = 4: 64 threads per block, measured fastest on C2; 2 and 8 kept for A/B runs), laid out
// so that the 32 pixels of a warp sharing a j form an 8x4 patch (strip_layout).  The block's
// depth-sorted list is staged through shared memory in batches (coalesced gathers: the sorted
// index, then the 48-byte record); records that no pixel of the block can composite are culled
// at staging (block_may_hit) and the rest are stored compacted, padded with opacity-0 entries.
// The conic is carried as its Cholesky factor L, prescaled by sqrt(0.5 log2 e), so the
// Gaussian weight is one MUFU.EX2 of a sum of two squares (no cancellation for thin Gaussians):
//   u = l11 dx + l21 dy, w = l22 dy, G = 2^-(u^2 + w^2) = exp(-0.5 d^T conic d),
// and between a thread's pixels dy drops by 16/PPT, so u and w of the next pixel are one FADD
// each (q_strip).  A pixel skips an entry (alpha < 1/255) iff q > log2(255 o), precomputed per
// staged record, so skipped evaluations need no exponential.
// Early termination: a thread stops evaluating a pixel once its T would drop below 1e-4, and
// the CTA stops staging once every pixel has stopped (__syncthreads_count).
// The forward fuses the L1 loss epilogue and the per-block cost counters.
// The backward walks each pixel's list back to front from n_last, reconstructs
// T_k = T_{k+1} / (1 - alpha_k), accumulates per entry three moments of the thread's pixels
// from which the 6 geometric gradients follow in closed form (strip_grads) plus the 3 colour
// gradients, then reduces the 9 values across the warp with a transpose (recursive-halving)
// reduction (12 shuffles, only when some lane contributes) into per-warp shared-memory slots.
#include <cstdlib>
#include <type_traits>

#include "gs_device.cuh"
#include "gs_internal.h"

using namespace gsd;

namespace {

constexpr int kFB = 128;    // forward: records staged per round
#ifndef GS_FWD_KFW
#define GS_FWD_KFW 64
#endif
constexpr int kFW = GS_FWD_KFW;  // warp-independent forward: records staged per warp round
constexpr int kUnroll = 4;  // forward entries per unrolled group (batch padded to a multiple; 4 measured
                            // faster than 8 and 16 on C2)

// Could any pixel centre of the 16x16 block at (bx0, by0) see the staged record with
// alpha >= 1/255?  Minimum of q(d) = |L'^T d|^2 over the continuous box of offsets
// d = m - p (a convex quadratic: 0 if the box contains d = 0, else on one of its edges)
// against qmax with a wide margin (5% of 1 + qmax in the exponent), so an entry is dropped only
// when every pixel would skip it: a conservative, semantics-free cull (dropped entries are
// no-ops for every pixel of the block).
// box_may_hit: the same test over the pixel centres [bx0, bx0 + ex] x [by0, by0 + ey] (the
// warp-independent kernels test each warp's 8x16 half of the block).
__device__ __forceinline__ bool box_may_hit(const float4& A, const float4& Bq, float qmax, float bx0, float by0,
                                            float ex, float ey) {
  if (!(qmax >= 0.f)) return false;  // opacity < 1/255: never composited
  const float l11 = A.z, l21 = A.w, l22 = Bq.x;
  const float dxh = A.x - bx0, dxl = dxh - ex, dyh = A.y - by0, dyl = dyh - ey;
  if (dxl <= 0.f && dxh >= 0.f && dyl <= 0.f && dyh >= 0.f) return true;
  const float a = l11 * l11, b = l11 * l21, c = l21 * l21 + l22 * l22;
  auto Q = [&](float dx, float dy) {
    const float u = fmaf(l11, dx, l21 * dy), w = l22 * dy;
    return fmaf(u, u, w * w);
  };
  // edge minimisers -b dx / c and -b dy / a through one approximate reciprocal each (no IEEE
  // division sequences): an error e in the minimiser raises q by O(e^2), far inside the margin
  float rc, ra;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(c));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(a));
  const float bc = -b * rc, ba = -b * ra;
  float qmin = Q(dxl, fminf(fmaxf(bc * dxl, dyl), dyh));
  qmin = fminf(qmin, Q(dxh, fminf(fmaxf(bc * dxh, dyl), dyh)));
  qmin = fminf(qmin, Q(fminf(fmaxf(ba * dyl, dxl), dxh), dyl));
  qmin = fminf(qmin, Q(fminf(fmaxf(ba * dyh, dxl), dxh), dyh));
  return !(qmin > qmax + 0.05f * (1.0f + qmax));
}
__device__ __forceinline__ bool block_may_hit(const float4& A, const float4& Bq, float qmax, float bx0, float by0) {
  return box_may_hit(A, Bq, qmax, bx0, by0, 15.f, 15.f);
}

// Stage the batch's records [0, cnt) *compacted*: the records that may be hit
// (block_may_hit; all of them when !cull) are written, in list order, to slots [0, kept) as
// (mx, my, l11', l21'), (l22', o, r, g), (b, qmax, list position, receive index) with
// L' = L sqrt(0.5 log2 e) and qmax = log2(255 o): alpha = o 2^-q >= 1/255 <=> q <= qmax, so the
// skip test needs no exponential (both passes decide skips with exactly this comparison);
// followed by
// opacity-0 padding entries (qmax < 0 <= q: never composited) up to a multiple of `pad`.  The
// render loops then read consecutive slots (no index indirection).  Returns kept; the caller
// syncs before reading and must have synced before calling (slots are overwritten).
template <int NT, int BATCH>
__device__ __forceinline__ int stage_records(const gs_rec* __restrict__ rec, const uint32_t* __restrict__ sidx,
                                             int cnt, int pos0, float4* s_a, float4* s_b, float4* s_c, int* s_wc,
                                             float bx0, float by0, bool cull, int pad) {
  constexpr int kW = NT / 32, kI = BATCH / NT;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t jr[kI];
  unsigned bal[kI];
  // pass 1: the cull test (only the index survives the barrier; pass 2 re-reads the record
  // from L1, keeping the register footprint of the staging small)
#pragma unroll
  for (int i = 0; i < kI; i++) {
    const int t = tid + NT * i;
    bool keep = false;
    jr[i] = 0;
    if (t < cnt) {
      jr[i] = sidx[t];
      keep = true;
      if (cull) {
        const float4* p = reinterpret_cast<const float4*>(rec + jr[i]);
        const float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
        (void)c;
        keep = block_may_hit(make_float4(a.x, a.y, b.x * kLScale, b.y * kLScale),
                             make_float4(b.z * kLScale, b.w, 0.f, 0.f),
                             b.w > 0.f ? __log2f(255.0f * b.w) : -1.0f, bx0, by0);
      }
    }
    bal[i] = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_wc[i * kW + wid] = __popc(bal[i]);
  }
  __syncthreads();
  int total = 0;
#pragma unroll
  for (int x = 0; x < kI * kW; x++) total += s_wc[x];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kI; i++) {
    if ((bal[i] >> lane) & 1u) {
      int off = __popc(bal[i] & lt);
      for (int x = 0; x < i * kW + wid; x++) off += s_wc[x];
      const float4* p = reinterpret_cast<const float4*>(rec + jr[i]);
      const float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
      s_a[off] = make_float4(a.x, a.y, b.x * kLScale, b.y * kLScale);
      s_b[off] = make_float4(b.z * kLScale, b.w, c.x, c.y);
      s_c[off] = make_float4(c.z, b.w > 0.f ? __log2f(255.0f * b.w) : -1.0f, __int_as_float(pos0 + tid + NT * i),
                             __uint_as_float(jr[i]));
    }
  }
  const int padded = (total + pad - 1) / pad * pad;
  for (int t = total + tid; t < padded; t += NT) {
    s_a[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    s_b[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    s_c[t] = make_float4(0.f, -1.0f, 0.f, 0.f);
  }
  return total;
}

// Warp-private form of stage_records for the warp-independent kernels (kWarp): the calling
// warp stages records [0, cnt) of its own walk (KW / 32 per lane), culled against the pixel
// centres of *its* 8x16 half of the block [hx0, hx0 + 7] x [hy0, hy0 + 15], compacted by
// ballot into its private slots and padded to a multiple of `pad`.  No CTA barrier; the caller
// must have __syncwarp'ed since its last read of the slots.
template <int KW, int ST = 1>
__device__ __forceinline__ int stage_warp(const gs_rec* __restrict__ rec, const uint32_t* __restrict__ sidx, int cnt,
                                          int pos0, float4* s_a, float4* s_b, float4* s_c, float hx0, float hy0,
                                          bool cull, int pad) {
  constexpr int kI = KW / 32;
  const int lane = threadIdx.x & 31;
  uint32_t jr[kI];
  unsigned bal[kI];
#pragma unroll
  for (int i = 0; i < kI; i++) {
    const int t = lane + 32 * i;
    bool keep = false;
    jr[i] = 0;
    if (t < cnt) {
      jr[i] = sidx[t];
      keep = true;
      if (cull) {
        const float4* p = reinterpret_cast<const float4*>(rec + jr[i]);
        const float4 a = __ldg(p), b = __ldg(p + 1);
        keep = box_may_hit(make_float4(a.x, a.y, b.x * kLScale, b.y * kLScale),
                           make_float4(b.z * kLScale, b.w, 0.f, 0.f),
                           b.w > 0.f ? __log2f(255.0f * b.w) : -1.0f, hx0, hy0, 7.f, 15.f);
      }
    }
    bal[i] = __ballot_sync(0xffffffffu, keep);
  }
  const unsigned lt = (1u << lane) - 1u;
  int base = 0;
#pragma unroll
  for (int i = 0; i < kI; i++) {
    if ((bal[i] >> lane) & 1u) {
      const int off = base + __popc(bal[i] & lt);
      const float4* p = reinterpret_cast<const float4*>(rec + jr[i]);
      const float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
      s_a[ST * off] = make_float4(a.x, a.y, b.x * kLScale, b.y * kLScale);
      s_b[ST * off] = make_float4(b.z * kLScale, b.w, c.x, c.y);
      s_c[ST * off] = make_float4(c.z, b.w > 0.f ? __log2f(255.0f * b.w) : -1.0f, __int_as_float(pos0 + lane + 32 * i),
                             __uint_as_float(jr[i]));
    }
    base += __popc(bal[i]);
  }
  const int padded = (base + pad - 1) / pad * pad;
  for (int t = base + lane; t < padded; t += 32) {
    s_a[ST * t] = make_float4(0.f, 0.f, 0.f, 0.f);
    s_b[ST * t] = make_float4(0.f, 0.f, 0.f, 0.f);
    s_c[ST * t] = make_float4(0.f, -1.0f, 0.f, 0.f);
  }
  __syncwarp();
  return base;
}

template <int NT, typename T>
__device__ __forceinline__ T block_sum(T v, T* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (NT == 32) return v;  // valid in every lane
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  T s = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; w++) s += sm[w];
  return s;  // valid in thread 0
}

// Pixel layout: thread t of a block's CTA owns PPT pixels of one column, RS = 16 / PPT rows
// apart: (x, r + RS j), j < PPT.  A warp covers 8 columns x 4 values of r (RS >= 4), so the
// 32 pixels sharing a j -- the lanes that take one compositing branch together -- form a
// compact 8x4 patch (a small Gaussian's footprint fills more of it than of a 16x2 or strided
// patch).
template <int PPT>
struct strip_layout {
  static constexpr int RS = 16 / PPT;
  __device__ static void of(int tid, int& x, int& r) {
    const int w = tid >> 5, l = tid & 31;
    if (RS >= 4) {
      x = 8 * (w & 1) + (l & 7);
      r = 4 * (w >> 1) + (l >> 3);
    } else {
      x = l & 15;
      r = l >> 4;
    }
  }
};

// Exponents of a staged record at the thread's pixels (px, py0 + RS j), j < PPT:
// q_j = u_j^2 + w_j^2 with G_j = 2^-q_j.  dx is shared; dy_j = dy0 - RS j, so
// u_j = u_{j-1} - RS l21 and w_j = w_{j-1} - RS l22 (RS a power of two: exact products).
// Both render passes call exactly this, so their skip/stop decisions agree bit for bit.
template <int PPT>
struct gs_strip {
  float dx, dy0, u[PPT], w[PPT], q[PPT];
};
// pen (forward): per-pixel penalty added inside the FMA that forms w^2 -- 0 for a live pixel
// (w * w + 0 rounds exactly like w * w, so q is unchanged) and +inf for a finished one (q = inf
// fails every skip test): the done flags cost no instruction per entry.  nullptr: no penalty.
template <int PPT>
__device__ __forceinline__ void q_strip(const float4& A, const float4& Bq, float px, float py0, gs_strip<PPT>& e,
                                        const float2* pen = nullptr) {
  constexpr float RS = (float)strip_layout<PPT>::RS;
  const float l11 = A.z, l21 = A.w, l22 = Bq.x;

  // (dx, dy0) and the exponents of pixel pairs with packed fp32x2 operations (FADD2 / FFMA2 /
  // FMUL2: one issue slot for two lanes' worth of work; per element identical to the scalar
  // __fsub_rn / __fmaf_rn(u, u, w * w))
  const float2 d = __fadd2_rn(make_float2(A.x, A.y), make_float2(-px, -py0));
  e.dx = d.x;
  e.dy0 = d.y;
  e.u[0] = __fmaf_rn(l11, e.dx, __fmul_rn(l21, e.dy0));
  e.w[0] = __fmul_rn(l22, e.dy0);
#pragma unroll
  for (int j = 1; j < PPT; j++) {
    // u - RS l21 with RS a power of two: the product is exact, so the FMA equals the
    // subtraction of the product (one instruction instead of two)
    e.u[j] = __fmaf_rn(-RS, l21, e.u[j - 1]);
    e.w[j] = __fmaf_rn(-RS, l22, e.w[j - 1]);
  }
#pragma unroll
  for (int j = 0; j < PPT; j += 2) {
    const float2 u = make_float2(e.u[j], e.u[j + 1]), w = make_float2(e.w[j], e.w[j + 1]);
    const float2 q = __ffma2_rn(u, u, pen ? __ffma2_rn(w, w, pen[j / 2]) : __fmul2_rn(w, w));
    e.q[j] = q.x;
    e.q[j + 1] = q.y;
  }
}

// kCap = false: the entry's opacity is at most kCapFree, so raw = o G <= o (G = ex2(-q) <= 1,
// q >= 0) never reaches the cap and the clamp and its zero-gradient select are skipped
// (identical results).  kCapFree sits 1e-4 below the cap: raw would need G > 1.0001.
constexpr float kCapFree = 0.9899f;
// Composite one staged entry into one pixel (O12) given its capped alpha >= 1/255.  A pixel
// that stops gets the +inf penalty (pen) and counts towards ndone; kTrack keeps its stop
// position (evaluation counts: statistics and the WORK cost mode).
template <bool kStats, bool kTrack>
__device__ __forceinline__ void fwd_comp(float alpha, float cr, float cg, float cb, int pos, float& T, float& C0,
                                         float& C1, float& C2, float& pen, int& ndone, int& nlast, int& stop_pos,
                                         int& efc) {
  const float Tn = T * (1.0f - alpha);
  if (Tn < kTStop) {  // R3: stop before compositing this entry
    pen = __int_as_float(0x7f800000);
    ndone++;
    if (kTrack) stop_pos = pos;
    return;
  }
  const float wgt = alpha * T;
  C0 = fmaf(wgt, cr, C0);
  C1 = fmaf(wgt, cg, C1);
  C2 = fmaf(wgt, cb, C2);
  T = Tn;
  nlast = pos + 1;
  if (kStats) efc++;
}

// kWarp (PPT = 4 only): the two warps walk the list independently, each over its own 8x16
// half (stage_warp), with no CTA barrier until the epilogue.
template <int PPT, bool kStats, int MINB = 1, bool kWarp = false, bool kTrack = true>
__global__ void __launch_bounds__(256 / PPT, MINB) k_render_fwd(
    const gs_rec* __restrict__ rec, const uint32_t* __restrict__ sorted_idx,
    const int32_t* __restrict__ range, gs_geom geo, int64_t B_lo, float bg0, float bg1, float bg2,
    const uint8_t* __restrict__ gt, float norm, float* __restrict__ out_rgb,
    float* __restrict__ T_final, int32_t* __restrict__ n_last, float* __restrict__ dL_dpix,
    double* __restrict__ loss_sum, int64_t* __restrict__ tile_cost, int cost_mode,
    long long* __restrict__ stats, int cull) {
  constexpr int NT = 256 / PPT;
  static_assert(!kWarp || PPT == 4, "warp-independent render needs PPT = 4 (one 8x16 half per warp)");
  constexpr int kSlots = kWarp ? 2 * (kFW + kUnroll) : kFB + kUnroll;
  __shared__ float4 s_a[kSlots], s_b[kSlots], s_c[kSlots];
  __shared__ int s_wc[kFB / 32];
  __shared__ long long s_red[NT / 32];
  __shared__ double s_redd[NT / 32];
  const long long t0 = clock64();
  const int tid = threadIdx.x;
  const int64_t lb = blockIdx.x, beta = B_lo + lb;
  const int64_t v = beta / geo.per_view, loc = beta % geo.per_view;
  const int tx = (int)(loc % geo.Wt), ty = (int)(loc / geo.Wt);
  constexpr int RS = strip_layout<PPT>::RS;
  int x, y0;
  strip_layout<PPT>::of(tid, x, y0);
  const int px = tx * 16 + x, py0 = ty * 16 + y0;
  const float fpx = (float)px, fpy0 = (float)py0;
  const int beg = range[lb], end = range[lb + 1];
  float T[PPT], C0[PPT], C1[PPT], C2[PPT];
  static_assert(kTrack || !kStats, "statistics need the stop positions");
  int nl[PPT], sp[PPT];
  float2 pen[PPT / 2];  // pixel pairs; 0: live pixel, +inf: stopped or outside the image (q_strip)
  int ndone = 0;
  unsigned inside = 0;
#pragma unroll
  for (int j = 0; j < PPT; j++) {
    T[j] = 1.f;
    C0[j] = C1[j] = C2[j] = 0.f;
    nl[j] = 0;
    sp[j] = -1;
    const bool in = px < geo.W && py0 + RS * j < geo.H;
    inside |= (unsigned)in << j;
    (j & 1 ? pen[j / 2].y : pen[j / 2].x) = in ? 0.f : __int_as_float(0x7f800000);
    ndone += !in;
  }
  int efc = 0;
  auto all_done = [&]() { return ndone == PPT; };
  const float bx0 = (float)(tx * 16), by0 = (float)(ty * 16);
  constexpr int kStep = kWarp ? kFW : kFB;
  const int wofs = kWarp ? (tid >> 5) * (kFW + kUnroll) : 0;  // this warp's slots (kWarp)
  for (int b0 = beg; b0 < end; b0 += kStep) {
    const int cnt = min(kStep, end - b0);
    int kept;
    if constexpr (kWarp) {
      if (__all_sync(0xffffffffu, all_done())) break;
      kept = stage_warp<kFW>(rec, sorted_idx + b0, cnt, b0 - beg, s_a + wofs, s_b + wofs, s_c + wofs,
                             bx0 + (float)(8 * (tid >> 5)), by0, cull != 0, kUnroll);
    } else {
      if (__syncthreads_count(all_done()) == NT) break;
      kept = stage_records<NT, kFB>(rec, sorted_idx + b0, cnt, b0 - beg, s_a, s_b, s_c, s_wc, bx0, by0,
                                    cull != 0, kUnroll);
      __syncthreads();
    }
    const int kept8 = (kept + kUnroll - 1) & ~(kUnroll - 1);
    for (int k0 = 0; k0 < kept8; k0 += kUnroll) {
      if (all_done()) break;
#pragma unroll
      for (int kk = 0; kk < kUnroll; kk++) {
        const float4 A = s_a[wofs + k0 + kk], Bq = s_b[wofs + k0 + kk], cq = s_c[wofs + k0 + kk];
        gs_strip<PPT> e;
        q_strip<PPT>(A, Bq, fpx, fpy0, e, pen);
        bool cj[PPT], any = false;
#pragma unroll
        for (int j = 0; j < PPT; j++) {
          cj[j] = e.q[j] <= cq.y;  // finished pixels have q = +inf
          any = any || cj[j];
        }
        if (any) {  // the common case (every pixel skips the entry) takes one branch
#pragma unroll
          for (int j = 0; j < PPT; j++)
            if (cj[j]) {
              const float al = fminf(kAlphaCap, __fmul_rn(Bq.y, ex2_approx(-e.q[j])));
              fwd_comp<kStats, kTrack>(al, Bq.z, Bq.w, cq.x, __float_as_int(cq.z), T[j], C0[j], C1[j], C2[j],
                                       j & 1 ? pen[j / 2].y : pen[j / 2].x, ndone, nl[j], sp[j], efc);
            }
        }
      }
    }
    if constexpr (kWarp) __syncwarp();  // every lane is done with the slots before restaging
  }
  // evaluations: an in-image pixel evaluates every entry up to its stopping entry (or all)
  const int n = end - beg;
  int ef = 0, nstop = 0, nlsum = 0;
  double lsum = 0.0;
#pragma unroll
  for (int j = 0; j < PPT; j++) {
    const bool in = inside >> j & 1;
    const int p = (y0 + RS * j) * 16 + x;
    const int64_t o = lb * 256 + p;
    if (in) {
      ef += sp[j] >= 0 ? sp[j] + 1 : n;
      nstop += sp[j] >= 0;
    }
    nlsum += nl[j];
    const float col[3] = {fmaf(T[j], bg0, C0[j]), fmaf(T[j], bg1, C1[j]), fmaf(T[j], bg2, C2[j])};
    T_final[o] = in ? T[j] : 1.f;
    n_last[o] = nl[j];
    if (out_rgb) {
#pragma unroll
      for (int ch = 0; ch < 3; ch++) out_rgb[lb * 768 + ch * 256 + p] = in ? col[ch] : 0.f;
    }
    if (gt) {
      const uint8_t* g = gt + ((v * geo.H + py0 + RS * j) * (int64_t)geo.W + px) * 3;
#pragma unroll
      for (int ch = 0; ch < 3; ch++) {
        float e = 0.f;
        if (in) e = col[ch] - (float)g[ch] * (1.0f / 255.0f);
        if (dL_dpix) dL_dpix[lb * 768 + ch * 256 + p] = (e > 0.f ? 1.f : (e < 0.f ? -1.f : 0.f)) * norm;
        lsum += (double)fabsf(e);
      }
    }
  }
  if (gt && loss_sum) {
    double s = block_sum<NT, double>(lsum, s_redd);
    if (tid == 0 && s != 0.0) atomicAdd(loss_sum, s * (double)norm);
  }
  if (kStats) {
    long long a = block_sum<NT, long long>(ef, s_red);
    long long b2 = block_sum<NT, long long>(efc, s_red);
    long long d2 = block_sum<NT, long long>(nstop, s_red);
    if (tid == 0) {
      atomicAdd((unsigned long long*)&stats[0], (unsigned long long)a);
      atomicAdd((unsigned long long*)&stats[1], (unsigned long long)b2);
      atomicAdd((unsigned long long*)&stats[2], (unsigned long long)(a - b2 - d2));
      atomicAdd((unsigned long long*)&stats[3], (unsigned long long)d2);
    }
  }
  (void)nlsum;
  if (tile_cost) {
    if (cost_mode == GS_COST_WORK) {
      long long w = block_sum<NT, long long>(ef, s_red);
      if (tid == 0) tile_cost[lb] += w;
    } else {
      __syncthreads();
      if (tid == 0) tile_cost[lb] += clock64() - t0;
    }
  }
}

// 1 / x for x in [1/255, 1] (1 - alpha >= 0.01, or an opacity of a compositing entry): one
// MUFU.RCP, no range fix-up (normal inputs only).
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Strip form of bwd_comp for the thread's pixel D rows below its first.  The six geometric
// gradients are linear in q = o G dA with coefficients polynomial in D (u = u_0 - D l21,
// w = w_0 - D l22, dy = dy_0 - D), so per pixel only the moments
// acc = (sum q, sum D q, sum D^2 q) are accumulated (q = o G dA = alpha dA, zero through the
// cap, R6; with a black background q = wgt . dot, one product); strip_grads turns them into
// the 6 gradients once per entry.  (O14; R6: zero gradient through the 0.99 cap.)
template <int D, bool kBg = true, bool kCap = true>
__device__ __forceinline__ void bwd_comp_strip(float raw, float G, const float4& Bq, float cb, float& T, float& P,
                                               float2 g01, float g2, float Tf, float bgdot, float acc[3],
                                               float2& gc01, float& gc2) {
  const float alpha = kCap ? fminf(kAlphaCap, raw) : raw;
  const float rom = rcp_approx(1.0f - alpha);
  T *= rom;  // transmittance in front of this entry
  const float wgt = alpha * T;
  gc01 = __ffma2_rn(make_float2(wgt, wgt), g01, gc01);
  gc2 = fmaf(wgt, g2, gc2);
  // the behind-colour S enters only through (c - S) . dL/dC, so the pixel keeps P = S . dL/dC
  // (S <- S + alpha (c - S)  =>  P <- P + alpha (c . dL/dC - P)): one scalar instead of S
  const float dot = fmaf(cb, g2, fmaf(Bq.w, g01.y, fmaf(Bq.z, g01.x, -P)));  // (c - S) . dL/dC
  // kBg = false: black background (bg = 0), the T_final term vanishes (not left to the
  // compiler: x * 0 does not fold in IEEE arithmetic)
  // q = alpha dA, dA = T dot (- T_final rom bgdot): alpha T dot = wgt dot
  const float qa = kBg ? alpha * (T * dot - Tf * rom * bgdot) : wgt * dot;
  P = fmaf(alpha, dot, P);
  const float gG = (!kCap || raw <= kAlphaCap) ? qa : 0.f;
  (void)G;
  acc[0] += gG;
  if (D == 1) acc[1] += gG, acc[2] += gG;
  if (D >= 2) acc[1] = fmaf((float)D, gG, acc[1]), acc[2] = fmaf((float)(D * D), gG, acc[2]);
}

// gr[0..5] of one entry from the strip moments of q = o G dA (2 ln 2 = 1 / kLScale^2):
//   dL/dl11' = -2ln2 l11 sum q_j u_j,  dL/dl21' = -2ln2 sum q_j (l21 u_j + l22 w_j),
//   dL/dconic-like (gr2..4) = -1/2 sum q dx^2, -sum q dx dy_j, -1/2 sum q dy_j^2,
//   dL/do = sum G dA = sum q / o (o > 1/255 for any entry that composites).
__device__ __forceinline__ void strip_grads(const float4& A, const float4& Bq, float dx, float dy0, float u0,
                                            float w0, const float acc[3], float gr[9]) {
  const float l11 = A.z, l21 = A.w, l22 = Bq.x, o = Bq.y;
  const float Q0 = acc[0], Q1 = acc[1], Q2 = acc[2];
  const float k = -1.3862943611198906f;
  gr[5] = Q0 * rcp_approx(o);
  gr[0] = k * l11 * fmaf(u0, Q0, -l21 * Q1);
  gr[1] = k * fmaf(fmaf(l21, u0, l22 * w0), Q0, -fmaf(l21, l21, l22 * l22) * Q1);
  gr[2] = -0.5f * dx * dx * Q0;
  gr[3] = -dx * fmaf(dy0, Q0, -Q1);
  gr[4] = -0.5f * fmaf(dy0, fmaf(dy0, Q0, -2.0f * Q1), Q2);
}

// Transpose (recursive-halving) warp reduction of 9 values: afterwards lane l holds the warp
// sum of value red_index(l) (valid lanes: 0,2,4,8,10,16,18,20,24).
__device__ __forceinline__ float warp_reduce9(const float v[9], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
  float w[5], x[3], y[2];
#pragma unroll
  for (int i = 0; i < 5; i++) {
    const float hi = i < 4 ? v[5 + i] : 0.f;
    const float send = b4 ? v[i] : hi;
    const float r = __shfl_xor_sync(0xffffffffu, send, 16);
    w[i] = (b4 ? hi : v[i]) + r;
  }
#pragma unroll
  for (int i = 0; i < 3; i++) {
    const float hi = i < 2 ? w[3 + i] : 0.f;
    const float send = b3 ? w[i] : hi;
    const float r = __shfl_xor_sync(0xffffffffu, send, 8);
    x[i] = (b3 ? hi : w[i]) + r;
  }
#pragma unroll
  for (int i = 0; i < 2; i++) {
    const float hi = i < 1 ? x[2] : 0.f;
    const float send = b2 ? x[i] : hi;
    const float r = __shfl_xor_sync(0xffffffffu, send, 4);
    y[i] = (b2 ? hi : x[i]) + r;
  }
  float z = (b1 ? y[1] : y[0]) + __shfl_xor_sync(0xffffffffu, b1 ? y[0] : y[1], 2);
  z += __shfl_xor_sync(0xffffffffu, z, 1);
  return z;
}

__device__ __forceinline__ int red_index(int lane, bool& valid) {
  const int b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1, b1 = (lane >> 1) & 1;
  const int sA = b4 ? 4 : 5, a = b4 ? 5 : 0;
  const int b = b3 ? 3 : 0, sB = b3 ? max(0, min(2, sA - 3)) : min(3, sA);
  const int c = b2 ? 2 : 0, sC = b2 ? max(0, min(1, sB - 2)) : min(2, sB);
  const int d = b1, sD = b1 ? max(0, min(1, sC - 1)) : min(1, sC);
  valid = sD > 0 && !(lane & 1);
  return a + b + c + d;
}

// kWarp (PPT = 4 only): each warp walks its own 8x16 half back to front from its own
// largest n_last (stage_warp), and adds its per-entry warp sums straight to dL/d(record)
// (no per-warp slots, no CTA barrier).
// Buffered warp reduction (kWarp backward): the per-lane gradients of kF contributing
// entries are stored as rows of 32 floats, row (slot, value) = the 32 lanes' values, then each
// row is summed by one lane (8 float4 loads at XOR-swizzled chunks: conflict-free; the sum's
// order does not matter) and added to dL/d(record).  9 kF rows: with kF = 3 (default) lanes
// 0..26 take one row each; with kF = 4 lanes 0..31 take rows 0..31 and the 4 remaining rows
// are split over 8 lanes each and finished by shuffles.  ~9 stores + ~17 instructions per
// entry instead of the 12-shuffle transpose reduction with its selects (~47).
#ifndef GS_BWD_KF
#define GS_BWD_KF 3
#endif
constexpr int kF = GS_BWD_KF;  // entries per flush (4: 36 rows = 32 + 4 x 8 lanes; 3: 27 rows, one lane each)

// Where the gradient of received record j goes: row base[s] + 9 j for the source s with
// seg[s] <= j < seg[s+1].  Own buffer: nseg = 1, base[0] = dL/d(record).  NEXT-3
// (gs_render_bwd_put): base[s] = source s's dL/dsend + 9 (owner_off[s] - seg[s]), so the
// reduction lands in the owner's buffer over NVLink (the reverse exchange, fused).
struct gs_gdst {
  float* base[GS_MAX_WORLD];
  long long seg[GS_MAX_WORLD + 1];
  int nseg;
};
__device__ __forceinline__ float* gdst_row(const gs_gdst& g, uint32_t j) {
  if (g.nseg == 1) return g.base[0] + (int64_t)j * 9;  // own buffer (uniform branch)
  int s = 0;
  while (s + 1 < g.nseg && (long long)j >= g.seg[s + 1]) s++;
  return g.base[s] + (int64_t)j * 9;
}
__device__ __forceinline__ void flush_rows(const float* __restrict__ rows_all, int wbytes, uint32_t ridreg, int nslot,
                                           const gs_gdst& dst, int lane) {
  // rows_all: the CTA's row buffer (128-byte aligned); wbytes: this warp's byte offset (a
  // multiple of 128, so it commutes with the chunk XOR below)
  const float* rows = rows_all + wbytes / 4;
  // lane s of ridreg holds the record of buffered entry s
  constexpr int NP = 9 * kF, R = NP > 32 ? NP - 32 : 1, LPP = 32 / R;
  static_assert(NP <= 32 || (32 % R == 0 && LPP <= 8 && 8 % LPP == 0), "flush layout");
  static_assert((kF * 9 * 32 * 4) % 128 == 0, "warp row buffers 128-byte aligned");
  const int np = 9 * nslot;
  const uint32_t rid0 = __shfl_sync(0xffffffffu, ridreg, lane / 9);
  if (lane < np) {
    // chunk c of row `lane` read at chunk (c ^ lane) & 7: the 8 lanes of a phase hit 8
    // different bank groups (conflict-free), one LOP3 per chunk (rows 128-byte aligned)
    const char* rb = reinterpret_cast<const char*>(rows_all);
    const int ob = wbytes + (lane * 8 + (lane & 7)) * 16;
    float4 a = *reinterpret_cast<const float4*>(rb + ob);
#pragma unroll
    for (int c = 1; c < 8; c++) {
      const float4 x = *reinterpret_cast<const float4*>(rb + (ob ^ (c * 16)));
      const float2 lo = __fadd2_rn(make_float2(a.x, a.y), make_float2(x.x, x.y));
      const float2 hi = __fadd2_rn(make_float2(a.z, a.w), make_float2(x.z, x.w));
      a = make_float4(lo.x, lo.y, hi.x, hi.y);
    }
    const float z = (a.x + a.y) + (a.z + a.w);
    if (z != 0.f) atomicAdd(gdst_row(dst, rid0) + lane % 9, z);
  }
  if constexpr (NP > 32) {  // rows 32.. : LPP lanes per row
    const int p = 32 + lane / LPP, part = lane % LPP;
    float z = 0.f;
    if (p < np) {
      const float4* r = reinterpret_cast<const float4*>(rows + p * 32);
#pragma unroll
      for (int c = 0; c < 8 / LPP; c++) {
        const float4 x = r[part * (8 / LPP) + c];
        z += (x.x + x.y) + (x.z + x.w);
      }
    }
#pragma unroll
    for (int o = LPP / 2; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    const uint32_t rid1 = __shfl_sync(0xffffffffu, ridreg, min(p, np - 1) / 9);
    if (part == 0 && p < np && z != 0.f) atomicAdd(gdst_row(dst, rid1) + p % 9, z);
  }
}

template <int PPT, bool kStats, int MINB = 1, bool kWarp = false, bool kBg = true>
__global__ void __launch_bounds__(256 / PPT, MINB) k_render_bwd(
    const gs_rec* __restrict__ rec, const uint32_t* __restrict__ sorted_idx,
    const int32_t* __restrict__ range, gs_geom geo, int64_t B_lo, float bg0, float bg1, float bg2,
    const float* __restrict__ dL_dpix, const float* __restrict__ T_final,
    const int32_t* __restrict__ n_last, float* __restrict__ dL_drec, int64_t* __restrict__ tile_cost,
    int cost_mode, long long* __restrict__ stats, int cull, gs_gdst gdst) {
  constexpr int NT = 256 / PPT;
  constexpr bool kOneWarp = NT == 32;
  constexpr int kNW = NT / 32;   // warps per block
  constexpr int kBB = 128;        // records staged per round
#ifndef GS_BWD_KBW16
#define GS_BWD_KBW16 64
#endif
  // kWarp: records staged per warp round (64 fits 16 CTAs/SM with 3-entry flushes: 14.2 KB per CTA)
  constexpr int kBW = MINB >= 18 ? 32 : (MINB >= 14 ? GS_BWD_KBW16 : 64);
  static_assert(!kWarp || PPT == 4, "warp-independent render needs PPT = 4 (one 8x16 half per warp)");
  constexpr bool kDirect = kOneWarp || kWarp;  // warp sums go straight to global memory
  __shared__ float4 s_a[kWarp ? 1 : kBB], s_b[kWarp ? 1 : kBB], s_c[kWarp ? 1 : kBB];
  // kWarp: the staged entries as (A, Bq, cq) triples, so one pointer walks them (the three
  // planes' base addresses were rematerialised per entry under the register cap)
  __shared__ float4 s_e[kWarp ? 3 * 2 * kBW : 1];
  __shared__ int s_wc[kBB / 32];
  // per-warp gradient slots: each (warp, entry, value) is written by exactly one lane, so no
  // shared-memory atomics (a float atomicAdd on shared memory is a CAS loop on sm_100)
  __shared__ float s_g[kDirect ? 1 : kNW * kBB * 9];
  // kWarp: per-warp buffered reduction rows (flush_rows) and the buffered entries' records
  __shared__ __align__(128) float s_rows[kWarp ? 2 * kF * 9 * 32 : 4];
  int nslot = 0;  // kWarp: buffered entries (warp-uniform)
  uint32_t ridreg = 0;  // kWarp: lane s holds the record of buffered entry s
  float* rowp = s_rows + (threadIdx.x >> 5) * kF * 9 * 32 + (threadIdx.x & 31);  // kWarp: this lane's next row slot
  __shared__ int s_max[NT / 32];
  __shared__ long long s_red[NT / 32];
  const long long t0 = clock64();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t lb = blockIdx.x, beta = B_lo + lb;
  const int64_t loc = beta % geo.per_view;
  const int tx = (int)(loc % geo.Wt), ty = (int)(loc / geo.Wt);
  constexpr int RS = strip_layout<PPT>::RS;
  int x, y0;
  strip_layout<PPT>::of(tid, x, y0);
  const int px = tx * 16 + x, py0 = ty * 16 + y0;
  const float fpx = (float)px, fpy0 = (float)py0;
  int nl[PPT];
  float Tf[PPT], T[PPT], P[PPT], g2[PPT], bgd[PPT];
  float2 g01[PPT];  // (r, g) pairs for packed fp32x2 updates
  int mymax = 0, nlsum = 0;
#pragma unroll
  for (int j = 0; j < PPT; j++) {
    const bool in = px < geo.W && py0 + RS * j < geo.H;
    const int64_t o = lb * 256 + (y0 + RS * j) * 16 + x;
    nl[j] = in ? n_last[o] : 0;
    Tf[j] = in ? T_final[o] : 1.f;
    T[j] = Tf[j];
    P[j] = 0.f;
    g01[j] = make_float2(in ? dL_dpix[lb * 768 + (o - lb * 256)] : 0.f, in ? dL_dpix[lb * 768 + 256 + (o - lb * 256)] : 0.f);
    g2[j] = in ? dL_dpix[lb * 768 + 512 + (o - lb * 256)] : 0.f;
    bgd[j] = bg0 * g01[j].x + bg1 * g01[j].y + bg2 * g2[j];
    mymax = max(mymax, nl[j]);
    nlsum += nl[j];
  }
  const int wmax = __reduce_max_sync(0xffffffffu, mymax);
  int maxn = wmax;
  if (!kOneWarp && !kWarp) {
    if (lane == 0) s_max[wid] = wmax;
    __syncthreads();
    maxn = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; w++) maxn = max(maxn, s_max[w]);
  }
  // this lane's gradient slot offset within an entry (value index, or -1), read back from
  // shared memory when the register cap evicts it (cheaper than recomputing red_index)
  // (kWarp uses the buffered rows instead: no slot table, its shared memory goes to staging)
  __shared__ int s_ridx[kWarp ? 1 : NT];
  int ridx_s = -1;
  if constexpr (!kWarp) {
    bool v;
    const int r = red_index(lane, v);
    s_ridx[tid] = v ? r : -1;
    __syncwarp();
    ridx_s = s_ridx[tid];
  }
  const bool rvalid = ridx_s >= 0;
  const int ridx = rvalid ? ridx_s : 0;
  const int beg = range[lb];
  int ebc = 0;
  float acc[3] = {0.f, 0.f, 0.f};  // per-entry strip moments and colour gradients
  float2 gc01 = make_float2(0.f, 0.f);
  float gc2 = 0.f;
  constexpr int kStep = kWarp ? kBW : kBB;
  const int wofs = kWarp ? wid * kBW : 0;  // this warp's slots (kWarp)
  for (int bi = (maxn + kStep - 1) / kStep - 1; bi >= 0; bi--) {
    const int p0 = bi * kStep;  // list position of the batch start
    const int cnt = min(kStep, maxn - p0);
    int kept;
    if constexpr (kWarp) {
      __syncwarp();
      kept = stage_warp<kBW, 3>(rec, sorted_idx + beg + p0, cnt, p0, s_e + 3 * wofs, s_e + 3 * wofs + 1,
                                s_e + 3 * wofs + 2, (float)(tx * 16 + 8 * wid), (float)(ty * 16), cull != 0, 1);
    } else {
      __syncthreads();
      kept = stage_records<NT, kBB>(rec, sorted_idx + beg + p0, cnt, p0, s_a, s_b, s_c, s_wc,
                                    (float)(tx * 16), (float)(ty * 16), cull != 0, 1);
      if (!kOneWarp)
        for (int t = tid; t < kNW * kBB * 9; t += NT) s_g[t] = 0.f;
      __syncthreads();
    }
    const float4* ep = s_e + 3 * (wofs + kept - 1);  // kWarp: entry k's triple
    for (int k = kept - 1; k >= 0; k--, ep -= 3) {
      const float4 cq = kWarp ? ep[2] : s_c[k];
      const int pos = __float_as_int(cq.z);
      if (!kWarp && pos >= wmax) continue;  // warp-uniform (kWarp stages only positions < wmax)
      const float4 A = kWarp ? ep[0] : s_a[k], Bq = kWarp ? ep[1] : s_b[k];
      gs_strip<PPT> e;
      q_strip<PPT>(A, Bq, fpx, fpy0, e);
      bool cj[PPT], any = false;
#pragma unroll
      for (int j = 0; j < PPT; j++) {
        cj[j] = pos < nl[j] && e.q[j] <= cq.y;
        any = any || cj[j];
      }
      // lanes without a contributing pixel keep zero moments, so their strip_grads are zeros
      // (the accumulators live across entries and are re-zeroed after each warp sum: no
      // per-entry zero moves)
      if (any) {
        // warp-uniform: entries with o <= kCapFree skip the alpha clamp (bwd_comp_strip)
        auto pixels = [&](auto capc) {
          constexpr bool kCap = decltype(capc)::value;
#pragma unroll
          for (int j = 0; j < PPT; j++)
            if (cj[j]) {
              const float G = ex2_approx(-e.q[j]);
              const float raw = __fmul_rn(Bq.y, G);
              switch (j) {
                case 0: bwd_comp_strip<0 * RS, kBg, kCap>(raw, G, Bq, cq.x, T[j], P[j], g01[j], g2[j], Tf[j], bgd[j], acc, gc01, gc2); break;
                case 1: bwd_comp_strip<1 * RS, kBg, kCap>(raw, G, Bq, cq.x, T[j], P[j], g01[j], g2[j], Tf[j], bgd[j], acc, gc01, gc2); break;
                case 2: bwd_comp_strip<2 * RS, kBg, kCap>(raw, G, Bq, cq.x, T[j], P[j], g01[j], g2[j], Tf[j], bgd[j], acc, gc01, gc2); break;
                case 3: bwd_comp_strip<3 * RS, kBg, kCap>(raw, G, Bq, cq.x, T[j], P[j], g01[j], g2[j], Tf[j], bgd[j], acc, gc01, gc2); break;
                case 4: bwd_comp_strip<4 * RS, kBg, kCap>(raw, G, Bq, cq.x, T[j], P[j], g01[j], g2[j], Tf[j], bgd[j], acc, gc01, gc2); break;
                case 5: bwd_comp_strip<5 * RS, kBg, kCap>(raw, G, Bq, cq.x, T[j], P[j], g01[j], g2[j], Tf[j], bgd[j], acc, gc01, gc2); break;
                case 6: bwd_comp_strip<6 * RS, kBg, kCap>(raw, G, Bq, cq.x, T[j], P[j], g01[j], g2[j], Tf[j], bgd[j], acc, gc01, gc2); break;
                default: bwd_comp_strip<7 * RS, kBg, kCap>(raw, G, Bq, cq.x, T[j], P[j], g01[j], g2[j], Tf[j], bgd[j], acc, gc01, gc2); break;
              }
            }
        };
        if (Bq.y > kCapFree)
          pixels(std::true_type{});
        else
          pixels(std::false_type{});
        if (kStats) {
#pragma unroll
          for (int j = 0; j < PPT; j++) ebc += cj[j];
        }
      }
      if (__any_sync(0xffffffffu, any)) {
        float gr[9];
        strip_grads(A, Bq, e.dx, e.dy0, e.u[0], e.w[0], acc, gr);
        gr[6] = gc01.x;
        gr[7] = gc01.y;
        gr[8] = gc2;
        acc[0] = acc[1] = acc[2] = 0.f;
        gc01 = make_float2(0.f, 0.f);
        gc2 = 0.f;
        if constexpr (kWarp) {
#pragma unroll
          for (int q = 0; q < 9; q++) rowp[q * 32] = gr[q];
          rowp += 9 * 32;
          if (lane == nslot) ridreg = __float_as_uint(cq.w);
          if (++nslot == kF) {
            __syncwarp();
            flush_rows(s_rows, wid * kF * 9 * 32 * 4, ridreg, kF, gdst, lane);
            __syncwarp();
            nslot = 0;
            rowp -= kF * 9 * 32;
          }
        } else {
          const float z = warp_reduce9(gr, lane);
          if (rvalid) {
            if (kDirect) {
              if (z != 0.f) atomicAdd(dL_drec + (int64_t)__float_as_uint(cq.w) * 9 + ridx, z);
            } else {
              s_g[(wid * kBB + k) * 9 + ridx] = z;
            }
          }
        }
      }
    }
    if (!kDirect) {
      __syncthreads();
      for (int t = tid; t < kept; t += NT) {
        float* dst = dL_drec + (int64_t)__float_as_uint(s_c[t].w) * 9;
#pragma unroll
        for (int q = 0; q < 9; q++) {
          float xv = 0.f;
#pragma unroll
          for (int w = 0; w < kNW; w++) xv += s_g[(w * kBB + t) * 9 + q];
          if (xv != 0.f) atomicAdd(dst + q, xv);
        }
      }
    }
  }
  if constexpr (kWarp) {
    if (nslot > 0) {
      __syncwarp();
      flush_rows(s_rows, wid * kF * 9 * 32 * 4, ridreg, nslot, gdst, lane);
    }
  }
  if (kStats) {
    long long a = block_sum<NT, long long>(nlsum, s_red);
    long long b2 = block_sum<NT, long long>(ebc, s_red);
    if (tid == 0) {
      atomicAdd((unsigned long long*)&stats[4], (unsigned long long)a);
      atomicAdd((unsigned long long*)&stats[5], (unsigned long long)b2);
    }
  }
  if (tile_cost) {
    if (cost_mode == GS_COST_WORK) {
      long long w = block_sum<NT, long long>(nlsum, s_red);
      if (tid == 0) tile_cost[lb] += w;
    } else {
      __syncthreads();
      if (tid == 0) tile_cost[lb] += clock64() - t0;
    }
  }
}

// per-block ellipse cull of staged entries (A/B knob: GS_RENDER_CULL bit 0 forward, bit 1
// backward; default both)
static int render_cull() {
  static int cull = -1;
  if (cull < 0) {
    const char* e = getenv("GS_RENDER_CULL");
    cull = e ? atoi(e) & 3 : 3;
  }
  return cull;
}

// resident-CTA floor of the PPT = 4 kernels, i.e. their register cap (A/B knobs:
// GS_RENDER_FWD_MINB: 12 or 16 for the block-staged forward, 16 / 18 / 20 for the
// warp-independent one; default 18 = 56 registers (C2 18.6 -> 18.0 ms against 16);
// GS_RENDER_BWD_MINB: 8 / 10 / 12 for the block-staged backward (else 12), 12 / 14 / 16 / 18
// for the warp-independent black-background one; default 16 = 64 registers (C2 34.3 -> 33.8
// ms against 14)).
static int render_minb(int bwd) {
  static int mb[2] = {-1, -1};
  if (mb[bwd] < 0) {
    const char* e = getenv(bwd ? "GS_RENDER_BWD_MINB" : "GS_RENDER_FWD_MINB");
    mb[bwd] = e ? atoi(e) : (bwd ? 16 : 18);
  }
  return mb[bwd];
}

// pixels per thread (A/B knob: GS_RENDER_PPT = 2, 4 or 8; default 4, measured best on C2)
static int render_ppt() {
  static int ppt = -1;
  if (ppt < 0) {
    const char* e = getenv("GS_RENDER_PPT");
    ppt = e ? atoi(e) : 4;
    if (ppt != 2 && ppt != 4 && ppt != 8) ppt = 4;
  }
  return ppt;
}

// warp-independent 8x16 halves (A/B knob: GS_RENDER_WARP bit 0 forward, bit 1 backward;
// PPT = 4 only; default both: C2 forward 22.65 -> 22.47 ms, backward 45.65 -> 44.27 ms)
static int render_warp() {
  static int w = -1;
  if (w < 0) {
    const char* e = getenv("GS_RENDER_WARP");
    w = e ? atoi(e) & 3 : 3;
  }
  return w;
}

}  // namespace

extern "C" gs_status gs_render_fwd(gs_ctx* c, const void* recv_rec, const uint32_t* sorted_idx,
                                   const int32_t* tile_range, const gs_camera* cams_h, int n_views,
                                   const int64_t* dp_h, const float* bg_h, const uint8_t* gt, int b_loss,
                                   float* out_rgb, float* T_final, int32_t* n_last, float* dL_dpix,
                                   double* loss_sum, int64_t* tile_cost, int cost_mode, int64_t* stats,
                                   void* stream) {
  if (!c) return GS_EINVAL;
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, !gt || b_loss >= 1, "b_loss must be >= 1 with gt");
  const int64_t B_lo = dp_h[c->rank], n_owned = dp_h[c->rank + 1] - B_lo;
  if (n_owned == 0) return GS_OK;
  GS_REQUIRE(c, tile_range && T_final && n_last, "null argument");
  GS_REQUIRE(c, n_owned < (1ll << 31), "too many owned blocks");
  gs_geom geo = gs_make_geom(&cams_h[0]);
  float bg[3] = {0.f, 0.f, 0.f};
  if (bg_h) for (int k = 0; k < 3; k++) bg[k] = bg_h[k];
  const float norm = gt ? (float)(1.0 / (3.0 * (double)geo.W * (double)geo.H * (double)b_loss)) : 0.f;
  ++c->launches;
  const int ppt = render_ppt();
  const int mb = render_minb(0);
  auto kf = ppt == 2 ? (stats ? k_render_fwd<2, true> : k_render_fwd<2, false>)
          : ppt == 8 ? (stats ? k_render_fwd<8, true> : k_render_fwd<8, false>)
          : (render_warp() & 1) ? (stats ? k_render_fwd<4, true, 16, true>
                                   : cost_mode == GS_COST_WORK ? k_render_fwd<4, false, 16, true>
                                   : mb == 16 ? k_render_fwd<4, false, 16, true, false>
                                   : mb == 20 ? k_render_fwd<4, false, 20, true, false>
                                              : k_render_fwd<4, false, 18, true, false>)
          : mb == 12 ? (stats ? k_render_fwd<4, true, 12> : k_render_fwd<4, false, 12>)
                     : (stats ? k_render_fwd<4, true, 16> : k_render_fwd<4, false, 16>);
  kf<<<(unsigned)n_owned, 256 / ppt, 0, (cudaStream_t)stream>>>(
      (const gs_rec*)recv_rec, sorted_idx, tile_range, geo, B_lo, bg[0], bg[1], bg[2], gt, norm, out_rgb,
      T_final, n_last, dL_dpix, loss_sum, tile_cost, cost_mode, (long long*)stats, render_cull() & 1);
  GS_LAUNCH_CHECK(c, "render_fwd");
  return GS_OK;
}

// Shared launcher of gs_render_bwd and gs_render_bwd_put (gradient rows through gdst).
static gs_status render_bwd_launch(gs_ctx* c, const void* recv_rec, const uint32_t* sorted_idx,
                                   const int32_t* tile_range, const gs_camera* cams_h, const int64_t* dp_h,
                                   const float* bg_h, const float* dL_dpix, const float* T_final,
                                   const int32_t* n_last, float* dL_drec, const gs_gdst& gdst, bool put,
                                   int64_t* tile_cost, int cost_mode, int64_t* stats, cudaStream_t st) {
  const int64_t B_lo = dp_h[c->rank], n_owned = dp_h[c->rank + 1] - B_lo;
  if (n_owned == 0) return GS_OK;
  GS_REQUIRE(c, tile_range && T_final && n_last && dL_dpix, "null argument");
  gs_geom geo = gs_make_geom(&cams_h[0]);
  float bg[3] = {0.f, 0.f, 0.f};
  if (bg_h) for (int k = 0; k < 3; k++) bg[k] = bg_h[k];
  const int ppt = render_ppt();
  const int mb = render_minb(1);
  const bool black = bg[0] == 0.f && bg[1] == 0.f && bg[2] == 0.f;
  if (put && !(ppt == 4 && (render_warp() & 2) && black))
    return gs_fail(c, GS_ENOTSUP, "gs_render_bwd_put needs the warp-independent PPT=4 backward and bg = 0");
  ++c->launches;
  auto kb = ppt == 2 ? (stats ? k_render_bwd<2, true> : k_render_bwd<2, false>)
          : ppt == 8 ? (stats ? k_render_bwd<8, true> : k_render_bwd<8, false>)
          : (render_warp() & 2) ? (black
                                       ? (mb == 12 ? (stats ? k_render_bwd<4, true, 12, true, false> : k_render_bwd<4, false, 12, true, false>)
                                                   : mb == 14 ? (stats ? k_render_bwd<4, true, 14, true, false> : k_render_bwd<4, false, 14, true, false>)
                                                   : mb == 18 ? (stats ? k_render_bwd<4, true, 18, true, false> : k_render_bwd<4, false, 18, true, false>)
                                                   : (stats ? k_render_bwd<4, true, 16, true, false> : k_render_bwd<4, false, 16, true, false>))
                                       : (stats ? k_render_bwd<4, true, 12, true> : k_render_bwd<4, false, 12, true>))
          : mb == 8 ? (stats ? k_render_bwd<4, true, 8> : k_render_bwd<4, false, 8>)
          : mb == 10 ? (stats ? k_render_bwd<4, true, 10> : k_render_bwd<4, false, 10>)
                     : (stats ? k_render_bwd<4, true, 12> : k_render_bwd<4, false, 12>);
  const int threads = 256 / ppt;
  kb<<<(unsigned)n_owned, threads, 0, st>>>(
      (const gs_rec*)recv_rec, sorted_idx, tile_range, geo, B_lo, bg[0], bg[1], bg[2], dL_dpix, T_final, n_last,
      dL_drec, tile_cost, cost_mode, (long long*)stats, (render_cull() >> 1) & 1, gdst);
  GS_LAUNCH_CHECK(c, "render_bwd");
  return GS_OK;
}

extern "C" gs_status gs_render_bwd(gs_ctx* c, const void* recv_rec, int64_t n_recv,
                                   const uint32_t* sorted_idx, const int32_t* tile_range,
                                   const gs_camera* cams_h, int n_views, const int64_t* dp_h,
                                   const float* bg_h, const float* dL_dpix, const float* T_final,
                                   const int32_t* n_last, float* dL_drec, int64_t* tile_cost, int cost_mode,
                                   int64_t* stats, void* stream) {
  if (!c) return GS_EINVAL;
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_recv > 0) {
    GS_REQUIRE(c, dL_drec != nullptr, "null dL_drec");
    GS_CUDA(c, cudaMemsetAsync(dL_drec, 0, (size_t)n_recv * 9 * sizeof(float), st));
  }
  gs_gdst g;
  for (int k = 0; k < GS_MAX_WORLD; k++) g.base[k] = nullptr;
  for (int k = 0; k <= GS_MAX_WORLD; k++) g.seg[k] = 0;
  g.base[0] = dL_drec;
  g.seg[1] = n_recv;
  g.nseg = 1;
  return render_bwd_launch(c, recv_rec, sorted_idx, tile_range, cams_h, dp_h, bg_h, dL_dpix, T_final, n_last,
                           dL_drec, g, false, tile_cost, cost_mode, stats, st);
}

extern "C" gs_status gs_render_bwd_put(gs_ctx* c, const void* recv_rec, int64_t n_recv, const uint32_t* sorted_idx,
                                       const int32_t* tile_range, const gs_camera* cams_h, int n_views,
                                       const int64_t* dp_h, const float* dL_dpix, const float* T_final,
                                       const int32_t* n_last, int64_t* tile_cost, int cost_mode, int64_t* stats,
                                       void* stream) {
  if (!c) return GS_EINVAL;
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, c->p2p.attached && c->p2p.planned, "gs_render_bwd_put needs gs_p2p_attach and gs_p2p_plan");
  const int G = c->world;
  int64_t seg[GS_MAX_WORLD + 1], put[GS_MAX_WORLD], soff[GS_MAX_WORLD + 1], own[GS_MAX_WORLD];
  s = gs_p2p_offsets(c->p2p.counts.data(), G, c->rank, seg, put, soff, own);
  if (s != GS_OK) return gs_fail(c, s, "bad plan");
  GS_REQUIRE(c, n_recv == seg[G], "n_recv %lld does not match the plan (%lld)", (long long)n_recv,
             (long long)seg[G]);
  gs_gdst g;
  for (int k = 0; k < GS_MAX_WORLD; k++) g.base[k] = nullptr;
  for (int k = 0; k <= GS_MAX_WORLD; k++) g.seg[k] = k <= G ? seg[k] : seg[G];
  for (int k = 0; k < G; k++)
    if (seg[k + 1] > seg[k]) {
      GS_REQUIRE(c, c->p2p.dsend[k] != nullptr, "rank %d has no dL/dsend buffer", k);
      g.base[k] = c->p2p.dsend[k] + 9 * (own[k] - seg[k]);
    }
  g.nseg = G;
  return render_bwd_launch(c, recv_rec, sorted_idx, tile_range, cams_h, dp_h, nullptr, dL_dpix, T_final, n_last,
                           nullptr, g, true, tile_cost, cost_mode, stats, (cudaStream_t)stream);
}
