// gs_render.cu -- A4/A5: front-to-back alpha compositing and its backward over the rank's
// owned 16x16 blocks.
//
// One CTA of 128 threads per owned block, two vertically adjacent pixels per thread (a warp
// covers a compact 16x4 pixel region).  The block's depth-sorted list is staged through
// shared memory in batches of 256 records (coalesced gathers: the sorted index, then the
// 48-byte record); every thread then walks the batch for its two pixels, so each shared-memory
// record read and each loop iteration is amortised over two evaluations.  The conic is
// carried as its Cholesky factor L, prescaled by sqrt(0.5 log2 e), so the Gaussian weight is
// one MUFU.EX2 of a sum of two squares (no cancellation for thin Gaussians):
//   u = l11 dx + l21 dy, w = l22 dy, G = 2^-(u^2 + w^2) = exp(-0.5 d^T conic d).
// Early termination: a CTA stops staging once every pixel has stopped
// (__syncthreads_count), a thread stops evaluating once its T would drop below 1e-4.
// The forward fuses the L1 loss epilogue and the per-block cost counters.
// The backward walks each pixel's list back to front from n_last, reconstructs
// T_k = T_{k+1} / (1 - alpha_k), sums the 9 record gradients of an entry over the thread's two
// pixels, then reduces them across the warp with a transpose (recursive-halving) reduction
// (12 shuffles instead of 45; only when some lane contributes) that leaves value c in one lane,
// so the 9 values are added to the batch entry's shared-memory accumulator by one warp-wide
// atomic instruction; each batch flushes one global atomic per (record, block, value).
#include "gs_device.cuh"
#include "gs_internal.h"

using namespace gsd;

namespace {

constexpr int kThreads = 128;  // 2 pixels per thread
constexpr int kBatch = 256;    // records staged per round

__device__ __forceinline__ void stage(const gs_rec* __restrict__ rec, uint32_t j, float4* s_a, float4* s_b,
                                      float* s_c, int t) {
  const float4* p = reinterpret_cast<const float4*>(rec + j);
  float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
  s_a[t] = make_float4(a.x, a.y, b.x * kLScale, b.y * kLScale);
  s_b[t] = make_float4(b.z * kLScale, b.w, c.x, c.y);
  s_c[t] = c.z;
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
    for (int w = 0; w < kThreads / 32; w++) s += sm[w];
  return s;  // valid in thread 0
}

// pixel pair of this thread inside the 16x16 block: (x, y) and (x, y + 1)
struct px_pair {
  int x, y, p0;  // p0 = y*16 + x, second pixel p0 + 16
};
__device__ __forceinline__ px_pair pair_of(int tid) {
  const int lane = tid & 31, wid = tid >> 5;
  px_pair q;
  q.x = lane & 15;
  q.y = wid * 4 + (lane >> 4) * 2;
  q.p0 = q.y * 16 + q.x;
  return q;
}

// One forward evaluation (O12) of staged entry (A, Bq, cb) at list position pos.
template <bool kStats>
__device__ __forceinline__ void fwd_px(const float4& A, const float4& Bq, float cb, float px, float py, int pos,
                                       float& T, float& C0, float& C1, float& C2, bool& done, int& nlast,
                                       int& stop_pos, int& efc) {
  float G, dx, dy, u, w;
  const float alpha = fminf(kAlphaCap, alpha_at(A.x, A.y, A.z, A.w, Bq.x, Bq.y, px, py, G, dx, dy, u, w));
  if (alpha < kAlphaMin) return;
  const float Tn = T * (1.0f - alpha);
  if (Tn < kTStop) {  // R3: stop before compositing this entry
    done = true;
    stop_pos = pos;
    return;
  }
  const float wgt = alpha * T;
  C0 = fmaf(wgt, Bq.z, C0);
  C1 = fmaf(wgt, Bq.w, C1);
  C2 = fmaf(wgt, cb, C2);
  T = Tn;
  nlast = pos + 1;
  if (kStats) efc++;
}

template <bool kStats>
__global__ void __launch_bounds__(kThreads) k_render_fwd(
    const gs_rec* __restrict__ rec, const uint32_t* __restrict__ sorted_idx,
    const int32_t* __restrict__ range, gs_geom geo, int64_t B_lo, float bg0, float bg1, float bg2,
    const uint8_t* __restrict__ gt, float norm, float* __restrict__ out_rgb,
    float* __restrict__ T_final, int32_t* __restrict__ n_last, float* __restrict__ dL_dpix,
    double* __restrict__ loss_sum, int64_t* __restrict__ tile_cost, int cost_mode,
    long long* __restrict__ stats) {
  __shared__ float4 s_a[kBatch], s_b[kBatch];
  __shared__ float s_c[kBatch];
  __shared__ long long s_red[kThreads / 32];
  __shared__ double s_redd[kThreads / 32];
  const long long t0 = clock64();
  const int tid = threadIdx.x;
  const int64_t lb = blockIdx.x, beta = B_lo + lb;
  const int64_t v = beta / geo.per_view, loc = beta % geo.per_view;
  const int tx = (int)(loc % geo.Wt), ty = (int)(loc / geo.Wt);
  const px_pair q = pair_of(tid);
  const int px = tx * 16 + q.x, py0 = ty * 16 + q.y, py1 = py0 + 1;
  const bool in0 = px < geo.W && py0 < geo.H, in1 = px < geo.W && py1 < geo.H;
  const float fpx = (float)px, fpy0 = (float)py0, fpy1 = (float)py1;
  const int beg = range[lb], end = range[lb + 1];
  float T0 = 1.f, T1 = 1.f, a0 = 0.f, a1 = 0.f, a2 = 0.f, b0c = 0.f, b1c = 0.f, b2c = 0.f;
  bool d0 = !in0, d1 = !in1;
  int nl0 = 0, nl1 = 0, sp0 = -1, sp1 = -1, efc0 = 0, efc1 = 0;
  for (int b0 = beg; b0 < end; b0 += kBatch) {
    if (__syncthreads_count(d0 && d1) == kThreads) break;
    if (b0 + tid < end) stage(rec, sorted_idx[b0 + tid], s_a, s_b, s_c, tid);
    if (b0 + tid + kThreads < end) stage(rec, sorted_idx[b0 + tid + kThreads], s_a, s_b, s_c, tid + kThreads);
    __syncthreads();
    const int cnt = min(kBatch, end - b0);
    const int pbase = b0 - beg;
    for (int k = 0; k < cnt; k++) {
      if (d0 && d1) break;
      const float4 A = s_a[k], Bq = s_b[k];
      const float cb = s_c[k];
      if (!d0) fwd_px<kStats>(A, Bq, cb, fpx, fpy0, pbase + k, T0, a0, a1, a2, d0, nl0, sp0, efc0);
      if (!d1) fwd_px<kStats>(A, Bq, cb, fpx, fpy1, pbase + k, T1, b0c, b1c, b2c, d1, nl1, sp1, efc1);
    }
  }
  // evaluations: an in-image pixel evaluates every entry up to its stopping entry (or all)
  const int n = end - beg;
  const int ef0 = in0 ? (sp0 >= 0 ? sp0 + 1 : n) : 0, ef1 = in1 ? (sp1 >= 0 ? sp1 + 1 : n) : 0;
  double lsum = 0.0;
  const int64_t o0 = lb * 256 + q.p0, o1 = o0 + 16;
  const float col0[3] = {fmaf(T0, bg0, a0), fmaf(T0, bg1, a1), fmaf(T0, bg2, a2)};
  const float col1[3] = {fmaf(T1, bg0, b0c), fmaf(T1, bg1, b1c), fmaf(T1, bg2, b2c)};
  T_final[o0] = in0 ? T0 : 1.f;
  T_final[o1] = in1 ? T1 : 1.f;
  n_last[o0] = nl0;
  n_last[o1] = nl1;
  if (out_rgb)
    for (int ch = 0; ch < 3; ch++) {
      out_rgb[lb * 768 + ch * 256 + q.p0] = in0 ? col0[ch] : 0.f;
      out_rgb[lb * 768 + ch * 256 + q.p0 + 16] = in1 ? col1[ch] : 0.f;
    }
  if (gt) {
    const uint8_t* g0 = gt + ((v * geo.H + py0) * (int64_t)geo.W + px) * 3;
    const uint8_t* g1 = g0 + (int64_t)geo.W * 3;
    for (int ch = 0; ch < 3; ch++) {
      float e0 = 0.f, e1 = 0.f;
      if (in0) e0 = col0[ch] - (float)g0[ch] * (1.0f / 255.0f);
      if (in1) e1 = col1[ch] - (float)g1[ch] * (1.0f / 255.0f);
      if (dL_dpix) {
        dL_dpix[lb * 768 + ch * 256 + q.p0] = (e0 > 0.f ? 1.f : (e0 < 0.f ? -1.f : 0.f)) * norm;
        dL_dpix[lb * 768 + ch * 256 + q.p0 + 16] = (e1 > 0.f ? 1.f : (e1 < 0.f ? -1.f : 0.f)) * norm;
      }
      lsum += (double)fabsf(e0) + (double)fabsf(e1);
    }
    if (loss_sum) {
      double s = block_sum<double>(lsum, s_redd);
      if (tid == 0 && s != 0.0) atomicAdd(loss_sum, s * (double)norm);
    }
  }
  if (kStats) {
    const int st0 = sp0 >= 0, st1 = sp1 >= 0;
    long long a = block_sum<long long>(ef0 + ef1, s_red);
    long long b2 = block_sum<long long>(efc0 + efc1, s_red);
    long long c2 = block_sum<long long>(ef0 - efc0 - (in0 && st0) + ef1 - efc1 - (in1 && st1), s_red);
    long long d2 = block_sum<long long>((in0 && st0) + (in1 && st1), s_red);
    if (tid == 0) {
      atomicAdd((unsigned long long*)&stats[0], (unsigned long long)a);
      atomicAdd((unsigned long long*)&stats[1], (unsigned long long)b2);
      atomicAdd((unsigned long long*)&stats[2], (unsigned long long)c2);
      atomicAdd((unsigned long long*)&stats[3], (unsigned long long)d2);
    }
  }
  if (tile_cost) {
    if (cost_mode == GS_COST_WORK) {
      long long w = block_sum<long long>(ef0 + ef1, s_red);
      if (tid == 0) tile_cost[lb] += w;
    } else {
      __syncthreads();
      if (tid == 0) tile_cost[lb] += clock64() - t0;
    }
  }
}

// Backward of one composited-or-skipped entry for one pixel (O14); accumulates into gr.
__device__ __forceinline__ bool bwd_px(const float4& A, const float4& Bq, float cb, float px, float py, float& T,
                                       float& S0, float& S1, float& S2, float g0, float g1, float g2, float Tf,
                                       float bgdot, float gr[9]) {
  float G, dx, dy, u, w;
  const float raw = alpha_at(A.x, A.y, A.z, A.w, Bq.x, Bq.y, px, py, G, dx, dy, u, w);
  const float alpha = fminf(kAlphaCap, raw);
  if (alpha < kAlphaMin) return false;
  const float om = 1.0f - alpha;
  const float rom = __fdividef(1.0f, om);
  T *= rom;  // transmittance in front of this entry
  const float wgt = alpha * T;
  const float cr = Bq.z, cg = Bq.w;
  gr[6] = fmaf(wgt, g0, gr[6]);
  gr[7] = fmaf(wgt, g1, gr[7]);
  gr[8] = fmaf(wgt, g2, gr[8]);
  const float dA = T * ((cr - S0) * g0 + (cg - S1) * g1 + (cb - S2) * g2) - Tf * rom * bgdot;
  S0 = fmaf(alpha, cr - S0, S0);
  S1 = fmaf(alpha, cg - S1, S1);
  S2 = fmaf(alpha, cb - S2, S2);
  if (raw <= kAlphaCap) {  // R6: zero gradient through the 0.99 cap
    const float gG = G * dA;
    const float q = Bq.y * gG;  // dL/dpower
    const float qs = q * 1.3862943611198906f;  // 2 ln 2 = 1 / kLScale^2
    gr[5] += gG;
    gr[0] = fmaf(-qs, A.z * u, gr[0]);
    gr[1] = fmaf(-qs, fmaf(A.w, u, Bq.x * w), gr[1]);
    const float hq = -0.5f * q;
    gr[2] = fmaf(hq * dx, dx, gr[2]);
    gr[3] = fmaf(-q * dx, dy, gr[3]);
    gr[4] = fmaf(hq * dy, dy, gr[4]);
  }
  return true;
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

template <bool kStats>
__global__ void __launch_bounds__(kThreads) k_render_bwd(
    const gs_rec* __restrict__ rec, const uint32_t* __restrict__ sorted_idx,
    const int32_t* __restrict__ range, gs_geom geo, int64_t B_lo, float bg0, float bg1, float bg2,
    const float* __restrict__ dL_dpix, const float* __restrict__ T_final,
    const int32_t* __restrict__ n_last, float* __restrict__ dL_drec, int64_t* __restrict__ tile_cost,
    int cost_mode, long long* __restrict__ stats) {
  __shared__ float4 s_a[kBatch], s_b[kBatch];
  __shared__ float s_c[kBatch];
  __shared__ uint32_t s_j[kBatch];
  __shared__ float s_g[kBatch * 9];
  __shared__ int s_max[kThreads / 32];
  __shared__ long long s_red[kThreads / 32];
  const long long t0 = clock64();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t lb = blockIdx.x, beta = B_lo + lb;
  const int64_t loc = beta % geo.per_view;
  const int tx = (int)(loc % geo.Wt), ty = (int)(loc / geo.Wt);
  const px_pair q = pair_of(tid);
  const int px = tx * 16 + q.x, py0 = ty * 16 + q.y, py1 = py0 + 1;
  const bool in0 = px < geo.W && py0 < geo.H, in1 = px < geo.W && py1 < geo.H;
  const float fpx = (float)px, fpy0 = (float)py0, fpy1 = (float)py1;
  const int64_t o0 = lb * 256 + q.p0, o1 = o0 + 16;
  const int nl0 = in0 ? n_last[o0] : 0, nl1 = in1 ? n_last[o1] : 0;
  const float Tf0 = in0 ? T_final[o0] : 1.f, Tf1 = in1 ? T_final[o1] : 1.f;
  float g00 = 0.f, g01 = 0.f, g02 = 0.f, g10 = 0.f, g11 = 0.f, g12 = 0.f;
  if (in0) {
    g00 = dL_dpix[lb * 768 + q.p0];
    g01 = dL_dpix[lb * 768 + 256 + q.p0];
    g02 = dL_dpix[lb * 768 + 512 + q.p0];
  }
  if (in1) {
    g10 = dL_dpix[lb * 768 + q.p0 + 16];
    g11 = dL_dpix[lb * 768 + 256 + q.p0 + 16];
    g12 = dL_dpix[lb * 768 + 512 + q.p0 + 16];
  }
  const float bgd0 = bg0 * g00 + bg1 * g01 + bg2 * g02, bgd1 = bg0 * g10 + bg1 * g11 + bg2 * g12;
  const int wmax = __reduce_max_sync(0xffffffffu, max(nl0, nl1));
  if (lane == 0) s_max[wid] = wmax;
  __syncthreads();
  int maxn = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; w++) maxn = max(maxn, s_max[w]);
  bool rvalid;
  const int ridx = red_index(lane, rvalid);
  const int beg = range[lb];
  float T0 = Tf0, T1 = Tf1, S00 = 0.f, S01 = 0.f, S02 = 0.f, S10 = 0.f, S11 = 0.f, S12 = 0.f;
  int ebc = 0;
  for (int bi = (maxn + kBatch - 1) / kBatch - 1; bi >= 0; bi--) {
    const int p0 = bi * kBatch;  // list position of the batch start
    const int cnt = min(kBatch, maxn - p0);
    __syncthreads();
    for (int t = tid; t < cnt; t += kThreads) {
      const uint32_t j = sorted_idx[beg + p0 + t];
      stage(rec, j, s_a, s_b, s_c, t);
      s_j[t] = j;
    }
    for (int t = tid; t < cnt * 9; t += kThreads) s_g[t] = 0.f;
    __syncthreads();
    for (int k = min(cnt, wmax - p0) - 1; k >= 0; k--) {  // warp-uniform range
      const int pos = p0 + k;
      const float4 A = s_a[k], Bq = s_b[k];
      const float cb = s_c[k];
      float gr[9];
#pragma unroll
      for (int c = 0; c < 9; c++) gr[c] = 0.f;
      bool contrib = false;
      if (pos < nl0) contrib |= bwd_px(A, Bq, cb, fpx, fpy0, T0, S00, S01, S02, g00, g01, g02, Tf0, bgd0, gr);
      if (kStats && contrib) ebc++;
      if (pos < nl1) {
        const bool c1 = bwd_px(A, Bq, cb, fpx, fpy1, T1, S10, S11, S12, g10, g11, g12, Tf1, bgd1, gr);
        if (kStats && c1) ebc++;
        contrib |= c1;
      }
      if (__any_sync(0xffffffffu, contrib)) {
        const float z = warp_reduce9(gr, lane);
        if (rvalid) atomicAdd(&s_g[k * 9 + ridx], z);
      }
    }
    __syncthreads();
    for (int t = tid; t < cnt; t += kThreads) {
      float* dst = dL_drec + (int64_t)s_j[t] * 9;
#pragma unroll
      for (int c = 0; c < 9; c++) {
        const float x = s_g[t * 9 + c];
        if (x != 0.f) atomicAdd(dst + c, x);
      }
    }
  }
  if (kStats) {
    long long a = block_sum<long long>(nl0 + nl1, s_red);
    long long b2 = block_sum<long long>(ebc, s_red);
    if (tid == 0) {
      atomicAdd((unsigned long long*)&stats[4], (unsigned long long)a);
      atomicAdd((unsigned long long*)&stats[5], (unsigned long long)b2);
    }
  }
  if (tile_cost) {
    if (cost_mode == GS_COST_WORK) {
      long long w = block_sum<long long>(nl0 + nl1, s_red);
      if (tid == 0) tile_cost[lb] += w;
    } else {
      __syncthreads();
      if (tid == 0) tile_cost[lb] += clock64() - t0;
    }
  }
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
  auto kf = stats ? k_render_fwd<true> : k_render_fwd<false>;
  kf<<<(unsigned)n_owned, kThreads, 0, (cudaStream_t)stream>>>(
      (const gs_rec*)recv_rec, sorted_idx, tile_range, geo, B_lo, bg[0], bg[1], bg[2], gt, norm, out_rgb,
      T_final, n_last, dL_dpix, loss_sum, tile_cost, cost_mode, (long long*)stats);
  GS_LAUNCH_CHECK(c, "render_fwd");
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
  const int64_t B_lo = dp_h[c->rank], n_owned = dp_h[c->rank + 1] - B_lo;
  if (n_owned == 0) return GS_OK;
  GS_REQUIRE(c, tile_range && T_final && n_last && dL_dpix, "null argument");
  gs_geom geo = gs_make_geom(&cams_h[0]);
  float bg[3] = {0.f, 0.f, 0.f};
  if (bg_h) for (int k = 0; k < 3; k++) bg[k] = bg_h[k];
  ++c->launches;
  auto kb = stats ? k_render_bwd<true> : k_render_bwd<false>;
  kb<<<(unsigned)n_owned, kThreads, 0, st>>>(
      (const gs_rec*)recv_rec, sorted_idx, tile_range, geo, B_lo, bg[0], bg[1], bg[2], dL_dpix, T_final, n_last,
      dL_drec, tile_cost, cost_mode, (long long*)stats);
  GS_LAUNCH_CHECK(c, "render_bwd");
  return GS_OK;
}
