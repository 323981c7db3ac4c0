// gs_render.cu -- A4/A5: front-to-back alpha compositing and its backward over the rank's
// owned 16x16 blocks.
//
// One CTA of 64 threads per owned block.  Each of its two warps owns one 8x16 half of the
// block and walks the block's depth-sorted list on its own (no CTA barrier until the
// epilogue): it stages 64 records per round into warp-private shared memory, drops the ones no
// pixel centre of its half can composite (box_may_hit) and stores the rest compacted.  Each
// thread owns 4 pixels of one column, 4 rows apart, so the 32 pixels of a warp that share a
// row index j form a compact 8x4 patch.
//
// Evaluation (R16).  The record carries the conic as its Cholesky factor L' prescaled by
// sqrt(0.5 log2 e) (G = 2^-q, q = u^2 + w^2, u = l11 dx + l21 dy, w = l22 dy), in double-float
// form.  At staging the warp evaluates u and w at its half's centre r = (hx0 + 3.5, hy0 + 7.5)
// in fp64 (u_ref, w_ref, rounded to fp32); a pixel then needs only its offset from r, which
// is at most (3.5, 7.5) px, a per-lane constant:  u = u_ref + l11 (rx - px) + l21 (ry - py).
// For a thin Gaussian far from its mean, u is a small difference of large terms; evaluated
// from the mean, its fp32 error grows with the distance, evaluated from r it does not.
// A pixel skips an entry (alpha < 1/255) iff q > qmax = log2(255 o) (per record, rounded to
// nearest), so skipped evaluations need no exponential; both passes take every decision
// through the same instructions, so they agree bit for bit.
// Early termination: a pixel stops once its T would drop below 1e-4 (R3), a warp once all its
// pixels have.  The forward fuses the L1 loss epilogue and the per-block cost counters
// (P:210).  The backward walks each pixel's list back to front from n_last, reconstructs
// T_k = T_{k+1} / (1 - alpha_k), accumulates per entry three moments of the thread's pixels
// from which the 6 geometric gradients follow in closed form (strip_grads) plus the 3 colour
// gradients, and reduces them over the warp through buffered shared-memory rows (flush_rows).
#include <cstdlib>
#include <type_traits>

#include "gs_device.cuh"
#include "gs_internal.h"

using namespace gsd;

namespace {

constexpr int kPPT = 4;     // pixels per thread (one column, kRS rows apart)
constexpr int kRS = 4;      // row stride between a thread's pixels
constexpr int kNT = 64;     // threads per block CTA (two warps, one 8x16 half each)
constexpr int kFW = 64;     // forward: records staged per warp round
constexpr int kBW = 64;     // backward: records staged per warp round
constexpr int kUnroll = 4;  // forward entries per unrolled group (4 measured faster than 8 and 16 on C2)
// resident-CTA floors (register caps) of the default kernels; compile-time so A/B builds can
// vary them (python -m paper_2406_18533_b200.build extra defines), never selected at run time
#ifndef GS_FWD_MINB
#define GS_FWD_MINB 18
#endif
#ifndef GS_BWD_MINB
#define GS_BWD_MINB 14
#endif
// 0: the backward ignores the forward's cull bits and repeats the test (A/B builds only)
#ifndef GS_CULL_REUSE
#define GS_CULL_REUSE 1
#endif

// Could any pixel centre of the box [bx0, bx0 + ex] x [by0, by0 + ey] see the record (mean
// (mx, my), prescaled factor l11, l21, l22) with alpha >= 1/255?  Minimum of q(d) = |L'^T d|^2
// over the continuous box of offsets d = m - p (a convex quadratic: 0 if the box contains
// d = 0, else on one of its edges) against qmax with a wide margin (5% of 1 + qmax in the
// exponent), so an entry is dropped only when every pixel would skip it: a conservative,
// semantics-free cull (dropped entries are no-ops for every pixel of the box).
__device__ __forceinline__ bool box_may_hit(float mx, float my, float l11, float l21, float l22, float qmax,
                                            float bx0, float by0, float ex, float ey) {
  if (!(qmax >= 0.f)) return false;  // opacity < 1/255: never composited
  const float dxh = mx - bx0, dxl = dxh - ex, dyh = my - by0, dyl = dyh - ey;
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

// Receive indices [0, cnt) of a staging round: lane + 32 i (0 past cnt).
template <int KW>
__device__ __forceinline__ void load_idx(const uint32_t* __restrict__ sidx, int cnt, uint32_t (&jr)[KW / 32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < KW / 32; i++) jr[i] = lane + 32 * i < cnt ? __ldg(sidx + lane + 32 * i) : 0u;
}

// u and w of the prescaled factor at the reference point (rx, ry), in fp64 from the
// double-float factor (hi + lo), rounded to nearest (R16).  Explicit fp64 intrinsics: every
// kernel that stages a record gets the same bits for the same reference point.
__device__ __forceinline__ float ref_u(const float4& a, const float4& b, const float4& d, double rx, double ry) {
  const double dmx = __dsub_rn((double)a.x, rx), dmy = __dsub_rn((double)a.y, ry);
  return __double2float_rn(__fma_rn(__dadd_rn((double)b.x, (double)d.x), dmx,
                                    __dmul_rn(__dadd_rn((double)b.y, (double)d.y), dmy)));
}
__device__ __forceinline__ float ref_w(const float4& a, const float4& b, const float4& d, double ry) {
  return __double2float_rn(__dmul_rn(__dadd_rn((double)b.z, (double)d.z), __dsub_rn((double)a.y, ry)));
}

// Stage records [0, cnt) of the calling warp's walk (jr: their receive indices in list
// order, list positions pos0 + t), culled against the pixel centres of its 8x16 half
// [hx0, hx0 + 7] x [hy0, hy0 + 15], compacted by ballot into the warp's slots and padded to a
// multiple of `pad` with entries no pixel composites.  Slot k is the triple s[3k .. 3k+2]:
//   A  = (u_ref, w_ref, l11', l21')      u, w at the half's centre r = (hx0 + 3.5, hy0 + 7.5),
//                                        in fp64 from the double-float factor, rounded
//   Bq = (l22', o, r, g)
//   cq = (b, qmax, list position, receive index)
// No CTA barrier; the caller must have __syncwarp'ed since its last read of the slots.
// S = 4 (backward): a fourth float4 per slot carries entry constants of the gradient formation,
//   E = (m_x - r_x, m_y - r_y, 1 / o, l21'^2 + l22'^2)   (mean relative to the half's centre).
// jr: the round's receive indices (load_idx); the backward loads them one round ahead, so its
// staging waits on one level of dependent loads (the records), not two.
// Cull bits (gs_render_fwd's cull_bits): word k of the round holds the keep ballot of entries
// 32k .. 32k + 31; bal (out) returns them to the forward, which stores them; bits_in
// (backward, nullable: the round's first word of this half, consecutive words 2 apart as the
// halves interleave) replaces the test -- the same decisions, so the same staged entries.
template <int KW, int S = 3>
__device__ __forceinline__ int stage_warp(const gs_rec* __restrict__ rec, const uint32_t (&jr)[KW / 32], int cnt,
                                          int pos0, float4* s, float hx0, float hy0, int pad,
                                          unsigned (&bal)[KW / 32], const uint32_t* __restrict__ bits_in = nullptr) {
  constexpr int kI = KW / 32;
  const int lane = threadIdx.x & 31;
  if (bits_in) {
#pragma unroll
    for (int i = 0; i < kI; i++) {
      const int c = cnt - 32 * i;
      bal[i] = c <= 0 ? 0u : (__ldg(bits_in + 2 * i) & (c >= 32 ? 0xffffffffu : (1u << c) - 1u));
    }
  } else {
#pragma unroll
    for (int i = 0; i < kI; i++) {
      const int t = lane + 32 * i;
      bool keep = false;
      if (t < cnt) {
        const gs_rec* r = rec + jr[i];
        const float4 a = __ldg(&r->a), b = __ldg(&r->b);
        const float qmax = __ldg(&r->c.w);
        keep = box_may_hit(a.x, a.y, b.x, b.y, b.z, qmax, hx0, hy0, 7.f, 15.f);
      }
      bal[i] = __ballot_sync(0xffffffffu, keep);
    }
  }
  const double rx = (double)hx0 + 3.5, ry = (double)hy0 + 7.5;
  const unsigned lt = (1u << lane) - 1u;
  int base = 0;
#pragma unroll
  for (int i = 0; i < kI; i++) {
    if ((bal[i] >> lane) & 1u) {
      const int off = base + __popc(bal[i] & lt);
      const gs_rec* r = rec + jr[i];
      const float4 a = __ldg(&r->a), b = __ldg(&r->b), c = __ldg(&r->c), d = __ldg(&r->d);
      const float uref = ref_u(a, b, d, rx, ry), wref = ref_w(a, b, d, ry);
      s[S * off] = make_float4(uref, wref, b.x, b.y);
      s[S * off + 1] = make_float4(b.z, b.w, c.x, c.y);
      s[S * off + 2] = make_float4(c.z, c.w, __int_as_float(pos0 + lane + 32 * i), __uint_as_float(jr[i]));
      if (S == 4)
        s[S * off + 3] = make_float4(a.x - (hx0 + 3.5f), a.y - (hy0 + 7.5f), __frcp_rn(b.w), fmaf(b.y, b.y, b.z * b.z));
    }
    base += __popc(bal[i]);
  }
  const int padded = (base + pad - 1) / pad * pad;
  for (int t = base + lane; t < padded; t += 32) {
    s[S * t] = make_float4(0.f, 0.f, 0.f, 0.f);
    s[S * t + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
    s[S * t + 2] = make_float4(0.f, -1.0f, 0.f, 0.f);  // qmax < 0 <= q: never composited
  }
  __syncwarp();
  return base;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  T s = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kNT / 32; w++) s += sm[w];
  return s;  // valid in thread 0
}

// Pixel layout: thread t owns pixels (x, r + 4 j), j < 4, with x = 8 (t / 32) + (t & 7),
// r = (t & 31) / 8: warp w covers columns 8w .. 8w + 7, and the 32 pixels sharing a j form an
// 8x4 patch.
__device__ __forceinline__ void pixel_of(int tid, int& x, int& r) {
  const int w = tid >> 5, l = tid & 31;
  x = 8 * w + (l & 7);
  r = l >> 3;
}

// Exponents of a staged entry at the thread's pixels: q_j = u_j^2 + w_j^2 with G_j = 2^-q_j,
// from the half's centre r: u_0 = u_ref + l11 ex + l21 ey0, w_0 = w_ref + l22 ey0 (ex = rx - px,
// ey0 = ry - py0: exact, per-lane constants), then u_j = u_{j-1} - 4 l21, w_j = w_{j-1} - 4 l22
// (exact products).  Both render passes call exactly this.
struct gs_strip {
  float u[kPPT], w[kPPT], q[kPPT];
};
// pen (forward): per-pixel penalty added inside the FMA that forms w^2 -- 0 for a live pixel
// (w * w + 0 rounds exactly like w * w, so q is unchanged) and +inf for a finished one (q = inf
// fails every skip test): the done flags cost no instruction per entry.  nullptr: no penalty.
__device__ __forceinline__ void q_strip(const float4& A, const float4& Bq, float ex, float ey0, gs_strip& e,
                                        const float2* pen = nullptr) {
  const float l11 = A.z, l21 = A.w, l22 = Bq.x;
  e.u[0] = __fmaf_rn(l11, ex, __fmaf_rn(l21, ey0, A.x));
  e.w[0] = __fmaf_rn(l22, ey0, A.y);
#pragma unroll
  for (int j = 1; j < kPPT; j++) {
    e.u[j] = __fmaf_rn(-(float)kRS, l21, e.u[j - 1]);
    e.w[j] = __fmaf_rn(-(float)kRS, l22, e.w[j - 1]);
  }
  // the exponents of pixel pairs with packed fp32x2 operations (FFMA2 / FMUL2: one issue slot
  // for two lanes' worth of work; per element identical to __fmaf_rn(u, u, w * w))
#pragma unroll
  for (int j = 0; j < kPPT; j += 2) {
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

template <bool kStats, int MINB, bool kTrack = true>
__global__ void __launch_bounds__(kNT, MINB) k_render_fwd(
    const gs_rec* __restrict__ rec, const uint32_t* __restrict__ sorted_idx,
    const int32_t* __restrict__ range, gs_geom geo, int64_t B_lo, float bg0, float bg1, float bg2,
    const uint8_t* __restrict__ gt, float norm, float* __restrict__ out_rgb,
    float* __restrict__ T_final, int32_t* __restrict__ n_last, float* __restrict__ dL_dpix,
    double* __restrict__ loss_sum, int64_t* __restrict__ tile_cost, int cost_mode,
    long long* __restrict__ stats, uint32_t* __restrict__ cull) {
  static_assert(kTrack || !kStats, "statistics need the stop positions");
  constexpr int kSlots = kFW + kUnroll;
  __shared__ float4 s_e[2 * 3 * kSlots];
  __shared__ long long s_red[kNT / 32];
  __shared__ double s_redd[kNT / 32];
  const long long t0 = clock64();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t lb = blockIdx.x, beta = B_lo + lb;
  const int64_t v = beta / geo.per_view, loc = beta % geo.per_view;
  const int tx = (int)(loc % geo.Wt), ty = (int)(loc / geo.Wt);
  int x, y0;
  pixel_of(tid, x, y0);
  const int px = tx * 16 + x, py0 = ty * 16 + y0;
  const float hx0 = (float)(tx * 16 + 8 * wid), hy0 = (float)(ty * 16);
  // offsets from the half's centre (exact); formed from px, py0 (which depend on the block index)
  // so that the register allocator keeps them rather than recomputing them per entry
  const float ex = (hx0 + 3.5f) - (float)px, ey0 = (hy0 + 7.5f) - (float)py0;
  const int beg = range[lb], end = range[lb + 1];
  float T[kPPT], C0[kPPT], C1[kPPT], C2[kPPT];
  int nl[kPPT], sp[kPPT];
  float2 pen[kPPT / 2];  // pixel pairs; 0: live pixel, +inf: stopped or outside the image (q_strip)
  int ndone = 0;
  unsigned inside = 0;
#pragma unroll
  for (int j = 0; j < kPPT; j++) {
    T[j] = 1.f;
    C0[j] = C1[j] = C2[j] = 0.f;
    nl[j] = 0;
    sp[j] = -1;
    const bool in = px < geo.W && py0 + kRS * j < geo.H;
    inside |= (unsigned)in << j;
    (j & 1 ? pen[j / 2].y : pen[j / 2].x) = in ? 0.f : __int_as_float(0x7f800000);
    ndone += !in;
  }
  int efc = 0;
  auto all_done = [&]() { return ndone == kPPT; };
  float4* const s = s_e + wid * 3 * kSlots;  // this warp's slots
  for (int b0 = beg; b0 < end; b0 += kFW) {
    if (__all_sync(0xffffffffu, all_done())) break;
    const int cnt = min(kFW, end - b0);
    // (loading the next round's indices here as the backward does spills at the forward's
    // 56-register cap: 18.41 -> 18.55 ms)
    uint32_t jc[kFW / 32];
    load_idx<kFW>(sorted_idx + b0, cnt, jc);
    unsigned bal[kFW / 32];
    const int kept = stage_warp<kFW>(rec, jc, cnt, b0 - beg, s, hx0, hy0, kUnroll, bal);
    if (cull && lane == 0) {
      // this half's cull words of the round: word (beg / 32 + lb + position / 32), halves interleaved
      uint32_t* const bo = cull + 2 * ((int64_t)(beg >> 5) + lb + ((b0 - beg) >> 5)) + wid;
#pragma unroll
      for (int i = 0; i < kFW / 32; i++)
        if (32 * i < cnt) bo[2 * i] = bal[i];
    }
    const int kept8 = (kept + kUnroll - 1) & ~(kUnroll - 1);
    for (int k0 = 0; k0 < kept8; k0 += kUnroll) {
      if (all_done()) break;
#pragma unroll
      for (int kk = 0; kk < kUnroll; kk++) {
        const float4 A = s[3 * (k0 + kk)], Bq = s[3 * (k0 + kk) + 1], cq = s[3 * (k0 + kk) + 2];
        gs_strip e;
        q_strip(A, Bq, ex, ey0, e, pen);
        bool cj[kPPT], any = false;
#pragma unroll
        for (int j = 0; j < kPPT; j++) {
          cj[j] = e.q[j] <= cq.y;  // finished pixels have q = +inf
          any = any || cj[j];
        }
        if (any) {  // the common case (every pixel skips the entry) takes one branch
#pragma unroll
          for (int j = 0; j < kPPT; j++)
            if (cj[j]) {
              const float al = fminf(kAlphaCap, __fmul_rn(Bq.y, ex2_approx(-e.q[j])));
              fwd_comp<kStats, kTrack>(al, Bq.z, Bq.w, cq.x, __float_as_int(cq.z), T[j], C0[j], C1[j], C2[j],
                                       j & 1 ? pen[j / 2].y : pen[j / 2].x, ndone, nl[j], sp[j], efc);
            }
        }
      }
    }
    __syncwarp();  // every lane is done with the slots before restaging
  }
  // evaluations: an in-image pixel evaluates every entry up to its stopping entry (or all)
  const int n = end - beg;
  int ef = 0, efmax = 0, nstop = 0;
  double lsum = 0.0;
#pragma unroll
  for (int j = 0; j < kPPT; j++) {
    const bool in = inside >> j & 1;
    const int p = (y0 + kRS * j) * 16 + x;
    const int64_t o = lb * 256 + p;
    if (in) {
      const int e = sp[j] >= 0 ? sp[j] + 1 : n;
      ef += e;
      efmax = max(efmax, e);
      nstop += sp[j] >= 0;
    }
    const float col[3] = {fmaf(T[j], bg0, C0[j]), fmaf(T[j], bg1, C1[j]), fmaf(T[j], bg2, C2[j])};
    T_final[o] = in ? T[j] : 1.f;
    n_last[o] = nl[j];
    if (out_rgb) {
#pragma unroll
      for (int ch = 0; ch < 3; ch++) out_rgb[lb * 768 + ch * 256 + p] = in ? col[ch] : 0.f;
    }
    if (gt) {
      const uint8_t* g = gt + ((v * geo.H + py0 + kRS * j) * (int64_t)geo.W + px) * 3;
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
    double sm = block_sum<double>(lsum, s_redd);
    if (tid == 0 && sm != 0.0) atomicAdd(loss_sum, sm * (double)norm);
  }
  if (kStats) {
    long long a = block_sum<long long>(ef, s_red);
    long long b2 = block_sum<long long>(efc, s_red);
    long long d2 = block_sum<long long>(nstop, s_red);
    if (tid == 0) {
      atomicAdd((unsigned long long*)&stats[0], (unsigned long long)a);
      atomicAdd((unsigned long long*)&stats[1], (unsigned long long)b2);
      atomicAdd((unsigned long long*)&stats[2], (unsigned long long)(a - b2 - d2));
      atomicAdd((unsigned long long*)&stats[3], (unsigned long long)d2);
    }
  }
  if (tile_cost) {
    if (cost_mode == GS_COST_WORK) {
      // R17: the entries each warp walks (its half's largest E_f), summed over the two warps
      const int wmax = __reduce_max_sync(0xffffffffu, efmax);
      const long long w = block_sum<long long>(lane == 0 ? wmax : 0, s_red);
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

// Strip form of the backward of one composited entry for the thread's pixel D rows below its
// first.  The six geometric gradients are linear in q = o G dA with coefficients polynomial in
// D (u = u_0 - D l21, w = w_0 - D l22, dy = dy_0 - D), so per pixel only the moments
// acc = (sum q, sum D q, sum D^2 q) are accumulated (q = o G dA = alpha dA, zero through the
// cap, R6; with a black background q = wgt . dot, one product); strip_grads turns them into
// the 6 gradients once per entry.  (O14; R6: zero gradient through the 0.99 cap.)
template <int D, bool kBg = true, bool kCap = true>
__device__ __forceinline__ void bwd_comp_strip(float raw, const float4& Bq, float cb, float& T, float& P,
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
  acc[0] += gG;
  if (D == 1) acc[1] += gG, acc[2] += gG;
  if (D >= 2) acc[1] = fmaf((float)D, gG, acc[1]), acc[2] = fmaf((float)(D * D), gG, acc[2]);
}

// gr[0..5] of one entry from the strip moments of q = o G dA (2 ln 2 = 1 / kLScale^2), with
// (dx, dy0) = m - p of the thread's first pixel and (u0, w0) its exponent terms:
//   dL/dl11' = -2ln2 l11 sum q_j u_j,  dL/dl21' = -2ln2 sum q_j (l21 u_j + l22 w_j),
//   dL/dconic-like (gr2..4) = -1/2 sum q dx^2, -sum q dx dy_j, -1/2 sum q dy_j^2,
//   dL/do = sum G dA = sum q / o (o > 1/255 for any entry that composites).
// E: the staged entry constants (stage_warp<., 4>): E.z = 1 / o, E.w = l21'^2 + l22'^2.
__device__ __forceinline__ void strip_grads(const float4& A, const float4& Bq, const float4& E, float dx, float dy0,
                                            float u0, float w0, const float acc[3], float gr[9]) {
  const float l11 = A.z, l21 = A.w, l22 = Bq.x;
  const float Q0 = acc[0], Q1 = acc[1], Q2 = acc[2];
  const float k = -1.3862943611198906f;
  gr[5] = Q0 * E.z;
  gr[0] = k * l11 * fmaf(u0, Q0, -l21 * Q1);
  gr[1] = k * fmaf(fmaf(l21, u0, l22 * w0), Q0, -E.w * Q1);
  gr[2] = -0.5f * dx * dx * Q0;
  gr[3] = -dx * fmaf(dy0, Q0, -Q1);
  gr[4] = -0.5f * fmaf(dy0, fmaf(dy0, Q0, -2.0f * Q1), Q2);
}

// Buffered warp reduction: the per-lane gradients of kF contributing entries are stored as
// rows of 32 floats, row (slot, value) = the 32 lanes' values, then each row is summed by one
// lane (8 float4 loads at XOR-swizzled chunks: conflict-free; the sum's order does not
// matter) and added to dL/d(record).  kF = 3: 27 rows, one lane each.  ~9 stores + ~17
// instructions per entry instead of a 12-shuffle transpose reduction with its selects (~47).
constexpr int kF = 3;

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
  static_assert((kF * 9 * 32 * 4) % 128 == 0, "warp row buffers 128-byte aligned");
  static_assert(9 * kF <= 32, "one lane per row");
  const int np = 9 * nslot;
  // lane s of ridreg holds the record of buffered entry s
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
}

// Each warp walks its own 8x16 half back to front from its own largest n_last and adds its
// per-entry warp sums to the gradient rows (no CTA barrier).  kBg: background term (bg != 0).
template <bool kStats, int MINB, bool kBg>
__global__ void __launch_bounds__(kNT, MINB) k_render_bwd(
    const gs_rec* __restrict__ rec, const uint32_t* __restrict__ sorted_idx,
    const int32_t* __restrict__ range, gs_geom geo, int64_t B_lo, float bg0, float bg1, float bg2,
    const float* __restrict__ dL_dpix, const float* __restrict__ T_final,
    const int32_t* __restrict__ n_last, int64_t* __restrict__ tile_cost, int cost_mode,
    long long* __restrict__ stats, gs_gdst gdst, const uint32_t* __restrict__ cull) {
  // the staged entries as (A, Bq, cq, E) quadruples, so one pointer walks them
  __shared__ float4 s_e[4 * 2 * kBW];
  // per-warp buffered reduction rows (flush_rows)
  __shared__ __align__(128) float s_rows[2 * kF * 9 * 32];
  __shared__ long long s_red[kNT / 32];
  int nslot = 0;        // buffered entries (warp-uniform)
  uint32_t ridreg = 0;  // lane s holds the record of buffered entry s
  float* rowp = s_rows + (threadIdx.x >> 5) * kF * 9 * 32 + (threadIdx.x & 31);  // this lane's next row slot
  const long long t0 = clock64();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t lb = blockIdx.x, beta = B_lo + lb;
  const int64_t loc = beta % geo.per_view;
  const int tx = (int)(loc % geo.Wt), ty = (int)(loc / geo.Wt);
  int x, y0;
  pixel_of(tid, x, y0);
  const int px = tx * 16 + x, py0 = ty * 16 + y0;
  const float hx0 = (float)(tx * 16 + 8 * wid), hy0 = (float)(ty * 16);
  const float ex = (hx0 + 3.5f) - (float)px, ey0 = (hy0 + 7.5f) - (float)py0;  // (see k_render_fwd)
  int nl[kPPT];
  float Tf[kPPT], T[kPPT], P[kPPT], g2[kPPT], bgd[kPPT];
  float2 g01[kPPT];  // (r, g) pairs for packed fp32x2 updates
  int mymax = 0, nlsum = 0;
#pragma unroll
  for (int j = 0; j < kPPT; j++) {
    const bool in = px < geo.W && py0 + kRS * j < geo.H;
    const int64_t o = lb * 256 + (y0 + kRS * j) * 16 + x;
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
  const int maxn = __reduce_max_sync(0xffffffffu, mymax);
  const int beg = range[lb];
  int ebc = 0;
  float acc[3] = {0.f, 0.f, 0.f};  // per-entry strip moments and colour gradients
  float2 gc01 = make_float2(0.f, 0.f);
  float gc2 = 0.f;
  float4* const s = s_e + wid * 4 * kBW;  // this warp's slots
  uint32_t jn[kBW / 32];
  const int bi0 = (maxn + kBW - 1) / kBW - 1;
  if (bi0 >= 0) load_idx<kBW>(sorted_idx + beg + bi0 * kBW, maxn - bi0 * kBW, jn);
  for (int bi = bi0; bi >= 0; bi--) {
    const int p0 = bi * kBW;  // list position of the batch start
    const int cnt = min(kBW, maxn - p0);
    uint32_t jc[kBW / 32];
#pragma unroll
    for (int i = 0; i < kBW / 32; i++) jc[i] = jn[i];
    if (bi > 0) load_idx<kBW>(sorted_idx + beg + p0 - kBW, kBW, jn);
    __syncwarp();
    const uint32_t* const bi_ =
        GS_CULL_REUSE && cull ? cull + 2 * ((int64_t)(beg >> 5) + lb + (p0 >> 5)) + wid : nullptr;
    unsigned bal[kBW / 32];
    const int kept = stage_warp<kBW, 4>(rec, jc, cnt, p0, s, hx0, hy0, 1, bal, bi_);
    const float4* ep = s + 4 * (kept - 1);  // entry k's quadruple
    for (int k = kept - 1; k >= 0; k--, ep -= 4) {
      const float4 cq = ep[2];
      const int pos = __float_as_int(cq.z);
      const float4 A = ep[0], Bq = ep[1];
      gs_strip e;
      q_strip(A, Bq, ex, ey0, e);
      bool cj[kPPT], any = false;
#pragma unroll
      for (int j = 0; j < kPPT; j++) {
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
          for (int j = 0; j < kPPT; j++)
            if (cj[j]) {
              const float raw = __fmul_rn(Bq.y, ex2_approx(-e.q[j]));
              switch (j) {
                case 0: bwd_comp_strip<0 * kRS, kBg, kCap>(raw, Bq, cq.x, T[j], P[j], g01[j], g2[j], Tf[j], bgd[j], acc, gc01, gc2); break;
                case 1: bwd_comp_strip<1 * kRS, kBg, kCap>(raw, Bq, cq.x, T[j], P[j], g01[j], g2[j], Tf[j], bgd[j], acc, gc01, gc2); break;
                case 2: bwd_comp_strip<2 * kRS, kBg, kCap>(raw, Bq, cq.x, T[j], P[j], g01[j], g2[j], Tf[j], bgd[j], acc, gc01, gc2); break;
                default: bwd_comp_strip<3 * kRS, kBg, kCap>(raw, Bq, cq.x, T[j], P[j], g01[j], g2[j], Tf[j], bgd[j], acc, gc01, gc2); break;
              }
            }
        };
        if (Bq.y > kCapFree)
          pixels(std::true_type{});
        else
          pixels(std::false_type{});
        if (kStats) {
#pragma unroll
          for (int j = 0; j < kPPT; j++) ebc += cj[j];
        }
      }
      if (__any_sync(0xffffffffu, any)) {
        // the mean-to-pixel offset of the thread's first pixel: (m - r) + (r - p)
        const float4 E = ep[3];
        float gr[9];
        strip_grads(A, Bq, E, E.x + ex, E.y + ey0, e.u[0], e.w[0], acc, gr);
        gr[6] = gc01.x;
        gr[7] = gc01.y;
        gr[8] = gc2;
        acc[0] = acc[1] = acc[2] = 0.f;
        gc01 = make_float2(0.f, 0.f);
        gc2 = 0.f;
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
      }
    }
  }
  if (nslot > 0) {
    __syncwarp();
    flush_rows(s_rows, wid * kF * 9 * 32 * 4, ridreg, nslot, gdst, lane);
  }
  if (kStats) {
    long long a = block_sum<long long>(nlsum, s_red);
    long long b2 = block_sum<long long>(ebc, s_red);
    if (tid == 0) {
      atomicAdd((unsigned long long*)&stats[4], (unsigned long long)a);
      atomicAdd((unsigned long long*)&stats[5], (unsigned long long)b2);
    }
  }
  if (tile_cost) {
    if (cost_mode == GS_COST_WORK) {
      // R17: the entries each warp walks back (its half's largest n_last), over the two warps
      const long long w = block_sum<long long>(lane == 0 ? maxn : 0, s_red);
      if (tid == 0) tile_cost[lb] += w;
    } else {
      __syncthreads();
      if (tid == 0) tile_cost[lb] += clock64() - t0;
    }
  }
}

// ex2.approx self-check: max relative error over every fp32 x in [lo, hi] (grid-stride), as
// an ordered uint64 of the double value (non-negative doubles order like their bits).
__global__ void k_selftest_ex2(uint32_t b_lo, uint32_t n, unsigned long long* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float x = __uint_as_float(b_lo + i);
    const double ref = exp2((double)x);
    const double err = fabs((double)ex2_approx(x) - ref) / ref;
    atomicMax(out, (unsigned long long)__double_as_longlong(err));
  }
}

}  // namespace

extern "C" int64_t gs_cull_words(int64_t n_pairs, int64_t n_owned) {
  return n_pairs < 0 || n_owned < 0 ? 0 : 2 * (n_pairs / 32 + n_owned + 1);
}

extern "C" gs_status gs_render_fwd(gs_ctx* c, const void* recv_rec, const uint32_t* sorted_idx,
                                   const int32_t* tile_range, const gs_camera* cams_h, int n_views,
                                   const int64_t* dp_h, const float* bg_h, const uint8_t* gt, int b_loss,
                                   float* out_rgb, float* T_final, int32_t* n_last, float* dL_dpix,
                                   double* loss_sum, int64_t* tile_cost, int cost_mode, int64_t* stats,
                                   uint32_t* cull_bits, void* stream) {
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
  // register caps (resident CTAs per SM): 16 with the stop positions tracked (statistics and
  // the WORK cost mode), 18 = 56 registers otherwise (C2 18.6 -> 18.0 ms against 16)
  auto kf = stats ? k_render_fwd<true, 16> : cost_mode == GS_COST_WORK ? k_render_fwd<false, 16>
                                                                        : k_render_fwd<false, GS_FWD_MINB, false>;
  kf<<<(unsigned)n_owned, kNT, 0, (cudaStream_t)stream>>>(
      (const gs_rec*)recv_rec, sorted_idx, tile_range, geo, B_lo, bg[0], bg[1], bg[2], gt, norm, out_rgb,
      T_final, n_last, dL_dpix, loss_sum, tile_cost, cost_mode, (long long*)stats, cull_bits);
  GS_LAUNCH_CHECK(c, "render_fwd");
  return GS_OK;
}

// Shared launcher of gs_render_bwd and gs_render_bwd_put (gradient rows through gdst).
static gs_status render_bwd_launch(gs_ctx* c, const void* recv_rec, const uint32_t* sorted_idx,
                                   const int32_t* tile_range, const gs_camera* cams_h, const int64_t* dp_h,
                                   const float* bg_h, const float* dL_dpix, const float* T_final,
                                   const int32_t* n_last, const gs_gdst& gdst, int64_t* tile_cost, int cost_mode,
                                   int64_t* stats, const uint32_t* cull_bits, cudaStream_t st) {
  const int64_t B_lo = dp_h[c->rank], n_owned = dp_h[c->rank + 1] - B_lo;
  if (n_owned == 0) return GS_OK;
  GS_REQUIRE(c, tile_range && T_final && n_last && dL_dpix, "null argument");
  gs_geom geo = gs_make_geom(&cams_h[0]);
  float bg[3] = {0.f, 0.f, 0.f};
  if (bg_h) for (int k = 0; k < 3; k++) bg[k] = bg_h[k];
  const bool black = bg[0] == 0.f && bg[1] == 0.f && bg[2] == 0.f;
  ++c->launches;
  // register caps: GS_BWD_MINB = 14 resident CTAs (72 registers) for the black-background kernel
  // (C2 33.17 -> 32.55 ms against 16 with the fp64 reference staging; 12: 33.96 ms), 12 with the
  // background term
  auto kb = black ? (stats ? k_render_bwd<true, 16, false> : k_render_bwd<false, GS_BWD_MINB, false>)
                  : (stats ? k_render_bwd<true, 12, true> : k_render_bwd<false, 12, true>);
  kb<<<(unsigned)n_owned, kNT, 0, st>>>((const gs_rec*)recv_rec, sorted_idx, tile_range, geo, B_lo, bg[0], bg[1],
                                        bg[2], dL_dpix, T_final, n_last, tile_cost, cost_mode, (long long*)stats,
                                        gdst, cull_bits);
  GS_LAUNCH_CHECK(c, "render_bwd");
  return GS_OK;
}

extern "C" gs_status gs_render_bwd(gs_ctx* c, const void* recv_rec, int64_t n_recv,
                                   const uint32_t* sorted_idx, const int32_t* tile_range,
                                   const gs_camera* cams_h, int n_views, const int64_t* dp_h,
                                   const float* bg_h, const float* dL_dpix, const float* T_final,
                                   const int32_t* n_last, float* dL_drec, int64_t* tile_cost, int cost_mode,
                                   int64_t* stats, const uint32_t* cull_bits, void* stream) {
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
  return render_bwd_launch(c, recv_rec, sorted_idx, tile_range, cams_h, dp_h, bg_h, dL_dpix, T_final, n_last, g,
                           tile_cost, cost_mode, stats, cull_bits, st);
}

extern "C" gs_status gs_render_bwd_put(gs_ctx* c, const void* recv_rec, int64_t n_recv, const uint32_t* sorted_idx,
                                       const int32_t* tile_range, const gs_camera* cams_h, int n_views,
                                       const int64_t* dp_h, const float* dL_dpix, const float* T_final,
                                       const int32_t* n_last, int64_t* tile_cost, int cost_mode, int64_t* stats,
                                       const uint32_t* cull_bits, void* stream) {
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
  return render_bwd_launch(c, recv_rec, sorted_idx, tile_range, cams_h, dp_h, nullptr, dL_dpix, T_final, n_last, g,
                           tile_cost, cost_mode, stats, cull_bits, (cudaStream_t)stream);
}

extern "C" gs_status gs_selftest_ex2(gs_ctx* c, float lo, float hi, double* max_rel_err_h, void* stream) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, max_rel_err_h && lo <= hi && lo < 0.f && hi <= 0.f,
             "need lo <= hi <= 0 (negative arguments; the bit range is walked downward from -0)");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* d = (unsigned long long*)gs_slot_get(c, SLOT_MISC, 64, st);
  if (!d) return gs_fail(c, GS_ECUDA, "scratch");
  GS_CUDA(c, cudaMemsetAsync(d, 0, 8, st));
  // negative floats: bits grow as the value falls, so [lo, hi] is bits [bits(hi), bits(lo)]
  const uint32_t b0 = hi == 0.f ? 0x80000000u : *reinterpret_cast<const uint32_t*>(&hi);
  const uint32_t b1 = *reinterpret_cast<const uint32_t*>(&lo);
  ++c->launches;
  k_selftest_ex2<<<148 * 8, 256, 0, st>>>(b0, b1 - b0 + 1, d);
  GS_LAUNCH_CHECK(c, "selftest_ex2");
  unsigned long long r = 0;
  GS_CUDA(c, cudaMemcpyAsync(&r, d, 8, cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  *max_rel_err_h = *reinterpret_cast<const double*>(&r);
  return GS_OK;
}
