// gs_render.cu -- A4/A5: front-to-back alpha compositing and its backward over the rank's
// owned 16x16 blocks.
//
// One CTA per owned block, one thread per pixel.  The block's depth-sorted list is staged
// through shared memory in batches of 256 records (one coalesced gather per thread: its
// sorted index, then the 48-byte record); every thread then walks the batch.  The conic is
// carried as its Cholesky factor L, prescaled by sqrt(0.5 log2 e), so the Gaussian weight is
// one MUFU.EX2 of a sum of two squares (no cancellation for thin Gaussians):
//   u = l11 dx + l21 dy, w = l22 dy, G = 2^-(u^2 + w^2) = exp(-0.5 d^T conic d).
// Early termination: a CTA stops staging once every pixel has stopped
// (__syncthreads_count), a thread stops evaluating once its T would drop below 1e-4.
// The forward fuses the L1 loss epilogue and the per-block cost counters.
// The backward walks each pixel's list back to front from n_last, reconstructs
// T_k = T_{k+1} / (1 - alpha_k), reduces the 9 record gradients of an entry across the warp
// (butterfly shuffles, only when some lane contributes), accumulates them per batch entry in
// shared memory and flushes one global atomic per (record, block, value).
#include "gs_device.cuh"
#include "gs_internal.h"

using namespace gsd;

namespace {

constexpr int kThreads = 256;

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

__global__ void __launch_bounds__(kThreads) k_render_fwd(
    const gs_rec* __restrict__ rec, const uint32_t* __restrict__ sorted_idx,
    const int32_t* __restrict__ range, gs_geom geo, int64_t B_lo, float bg0, float bg1, float bg2,
    const uint8_t* __restrict__ gt, float norm, float* __restrict__ out_rgb,
    float* __restrict__ T_final, int32_t* __restrict__ n_last, float* __restrict__ dL_dpix,
    double* __restrict__ loss_sum, int64_t* __restrict__ tile_cost, int cost_mode,
    long long* __restrict__ stats) {
  __shared__ float4 s_a[kThreads], s_b[kThreads];
  __shared__ float s_c[kThreads];
  __shared__ long long s_red[kThreads / 32];
  __shared__ double s_redd[kThreads / 32];
  const long long t0 = clock64();
  const int tid = threadIdx.x;
  const int64_t lb = blockIdx.x, beta = B_lo + lb;
  const int64_t v = beta / geo.per_view, loc = beta % geo.per_view;
  const int tx = (int)(loc % geo.Wt), ty = (int)(loc / geo.Wt);
  const int px = tx * 16 + (tid & 15), py = ty * 16 + (tid >> 4);
  const bool inside = px < geo.W && py < geo.H;
  const float fpx = (float)px, fpy = (float)py;
  const int beg = range[lb], end = range[lb + 1];
  float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
  bool done = !inside;
  int nlast = 0, ef = 0, efc = 0, estop = 0;
  for (int b0 = beg; b0 < end; b0 += kThreads) {
    if (__syncthreads_count(done) == kThreads) break;
    if (b0 + tid < end) stage(rec, sorted_idx[b0 + tid], s_a, s_b, s_c, tid);
    __syncthreads();
    const int cnt = min(kThreads, end - b0);
    if (!done) {
      for (int k = 0; k < cnt; k++) {
        const float4 A = s_a[k], Bq = s_b[k];
        float G, dx, dy, u, w;
        const float alpha = fminf(kAlphaCap, alpha_at(A.x, A.y, A.z, A.w, Bq.x, Bq.y, fpx, fpy, G, dx, dy, u, w));
        ef++;
        if (alpha < kAlphaMin) continue;
        const float Tn = T * (1.0f - alpha);
        if (Tn < kTStop) { done = true; estop = 1; break; }
        const float wgt = alpha * T;
        C0 = fmaf(wgt, Bq.z, C0);
        C1 = fmaf(wgt, Bq.w, C1);
        C2 = fmaf(wgt, s_c[k], C2);
        T = Tn;
        nlast = b0 - beg + k + 1;
        efc++;
      }
    }
  }
  const int64_t o = lb * kThreads + tid;
  double lsum = 0.0;
  if (inside) {
    T_final[o] = T;
    n_last[o] = nlast;
    const float col[3] = {fmaf(T, bg0, C0), fmaf(T, bg1, C1), fmaf(T, bg2, C2)};
    if (out_rgb)
      for (int ch = 0; ch < 3; ch++) out_rgb[lb * 768 + ch * 256 + tid] = col[ch];
    if (gt) {
      const uint8_t* g = gt + ((v * geo.H + py) * (int64_t)geo.W + px) * 3;
      for (int ch = 0; ch < 3; ch++) {
        float d = col[ch] - (float)g[ch] * (1.0f / 255.0f);
        float sg = (d > 0.f) ? 1.f : ((d < 0.f) ? -1.f : 0.f);
        if (dL_dpix) dL_dpix[lb * 768 + ch * 256 + tid] = sg * norm;
        lsum += (double)fabsf(d);
      }
    }
  } else {
    T_final[o] = 1.0f;
    n_last[o] = 0;
    if (out_rgb)
      for (int ch = 0; ch < 3; ch++) out_rgb[lb * 768 + ch * 256 + tid] = 0.f;
    if (gt && dL_dpix)
      for (int ch = 0; ch < 3; ch++) dL_dpix[lb * 768 + ch * 256 + tid] = 0.f;
  }
  if (loss_sum && gt) {
    double s = block_sum<double>(lsum, s_redd);
    if (tid == 0 && s != 0.0) atomicAdd(loss_sum, s * (double)norm);
  }
  if (stats) {
    long long a = block_sum<long long>(ef, s_red);
    long long b2 = block_sum<long long>(efc, s_red);
    long long c2 = block_sum<long long>(ef - efc - estop, s_red);
    long long d2 = block_sum<long long>(estop, s_red);
    if (tid == 0) {
      atomicAdd((unsigned long long*)&stats[0], (unsigned long long)a);
      atomicAdd((unsigned long long*)&stats[1], (unsigned long long)b2);
      atomicAdd((unsigned long long*)&stats[2], (unsigned long long)c2);
      atomicAdd((unsigned long long*)&stats[3], (unsigned long long)d2);
    }
  }
  if (tile_cost) {
    if (cost_mode == GS_COST_WORK) {
      long long w = block_sum<long long>(ef, s_red);
      if (tid == 0) tile_cost[lb] += w;
    } else {
      __syncthreads();
      if (tid == 0) tile_cost[lb] += clock64() - t0;
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_render_bwd(
    const gs_rec* __restrict__ rec, const uint32_t* __restrict__ sorted_idx,
    const int32_t* __restrict__ range, gs_geom geo, int64_t B_lo, float bg0, float bg1, float bg2,
    const float* __restrict__ dL_dpix, const float* __restrict__ T_final,
    const int32_t* __restrict__ n_last, float* __restrict__ dL_drec, int64_t* __restrict__ tile_cost,
    int cost_mode, long long* __restrict__ stats) {
  __shared__ float4 s_a[kThreads], s_b[kThreads];
  __shared__ float s_c[kThreads];
  __shared__ uint32_t s_j[kThreads];
  __shared__ float s_g[kThreads * 9];
  __shared__ int s_max[kThreads / 32];
  __shared__ long long s_red[kThreads / 32];
  const long long t0 = clock64();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t lb = blockIdx.x, beta = B_lo + lb;
  const int64_t loc = beta % geo.per_view;
  const int tx = (int)(loc % geo.Wt), ty = (int)(loc / geo.Wt);
  const int px = tx * 16 + (tid & 15), py = ty * 16 + (tid >> 4);
  const bool inside = px < geo.W && py < geo.H;
  const float fpx = (float)px, fpy = (float)py;
  const int64_t o = lb * kThreads + tid;
  const int nl = inside ? n_last[o] : 0;
  const float Tf = inside ? T_final[o] : 1.0f;
  float g0 = 0.f, g1 = 0.f, g2 = 0.f;
  if (inside) {
    g0 = dL_dpix[lb * 768 + tid];
    g1 = dL_dpix[lb * 768 + 256 + tid];
    g2 = dL_dpix[lb * 768 + 512 + tid];
  }
  const float bgdot = bg0 * g0 + bg1 * g1 + bg2 * g2;
  int m = __reduce_max_sync(0xffffffffu, nl);
  if (lane == 0) s_max[wid] = m;
  __syncthreads();
  int maxn = 0;
  for (int w = 0; w < kThreads / 32; w++) maxn = max(maxn, s_max[w]);
  const int beg = range[lb];
  float T = Tf, S0 = 0.f, S1 = 0.f, S2 = 0.f;
  int ebc = 0;
  const float kQ = 1.3862943611198906f;  // 2 ln 2 = 1 / kLScale^2
  for (int bi = (maxn + kThreads - 1) / kThreads - 1; bi >= 0; bi--) {
    const int p0 = bi * kThreads;  // list position of the batch start
    const int cnt = min(kThreads, maxn - p0);
    __syncthreads();
    if (tid < cnt) {
      const uint32_t j = sorted_idx[beg + p0 + tid];
      stage(rec, j, s_a, s_b, s_c, tid);
      s_j[tid] = j;
#pragma unroll
      for (int c = 0; c < 9; c++) s_g[tid * 9 + c] = 0.f;
    }
    __syncthreads();
    for (int k = cnt - 1; k >= 0; k--) {
      float gr[9];
#pragma unroll
      for (int c = 0; c < 9; c++) gr[c] = 0.f;
      bool contrib = false;
      if (p0 + k < nl) {
        const float4 A = s_a[k], Bq = s_b[k];
        float G, dx, dy, u, w;
        const float raw = alpha_at(A.x, A.y, A.z, A.w, Bq.x, Bq.y, fpx, fpy, G, dx, dy, u, w);
        const float alpha = fminf(kAlphaCap, raw);
        if (alpha >= kAlphaMin) {
          contrib = true;
          const float om = 1.0f - alpha;
          T = T / om;  // T_k, transmittance in front of entry k
          const float wgt = alpha * T;
          const float cr = Bq.z, cg = Bq.w, cb = s_c[k];
          gr[6] = wgt * g0;
          gr[7] = wgt * g1;
          gr[8] = wgt * g2;
          const float dA = T * ((cr - S0) * g0 + (cg - S1) * g1 + (cb - S2) * g2) - (Tf / om) * bgdot;
          S0 = alpha * cr + om * S0;
          S1 = alpha * cg + om * S1;
          S2 = alpha * cb + om * S2;
          if (raw <= kAlphaCap) {  // R6: zero gradient through the 0.99 cap
            gr[5] = G * dA;
            const float q = Bq.y * G * dA;  // dL/dpower
            const float qs = q * kQ;
            gr[0] = -qs * (A.z * u);
            gr[1] = -qs * (A.w * u + Bq.x * w);
            gr[2] = -0.5f * q * dx * dx;
            gr[3] = -q * dx * dy;
            gr[4] = -0.5f * q * dy * dy;
          }
          ebc++;
        }
      }
      if (__any_sync(0xffffffffu, contrib)) {
#pragma unroll
        for (int c = 0; c < 9; c++) {
          float x = gr[c];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
          gr[c] = x;
        }
        if (lane == 0) {
#pragma unroll
          for (int c = 0; c < 9; c++) atomicAdd(&s_g[k * 9 + c], gr[c]);
        }
      }
    }
    __syncthreads();
    if (tid < cnt) {
      float* dst = dL_drec + (int64_t)s_j[tid] * 9;
#pragma unroll
      for (int c = 0; c < 9; c++) {
        float x = s_g[tid * 9 + c];
        if (x != 0.f) atomicAdd(dst + c, x);
      }
    }
  }
  if (stats) {
    long long a = block_sum<long long>(nl, s_red);
    long long b2 = block_sum<long long>(ebc, s_red);
    if (tid == 0) {
      atomicAdd((unsigned long long*)&stats[4], (unsigned long long)a);
      atomicAdd((unsigned long long*)&stats[5], (unsigned long long)b2);
    }
  }
  if (tile_cost) {
    if (cost_mode == GS_COST_WORK) {
      long long w = block_sum<long long>(nl, s_red);
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
  GS_REQUIRE(c, tile_range && T_final && n_last, "null argument");
  GS_REQUIRE(c, !gt || b_loss >= 1, "b_loss must be >= 1 with gt");
  const int64_t B_lo = dp_h[c->rank], n_owned = dp_h[c->rank + 1] - B_lo;
  if (n_owned == 0) return GS_OK;
  GS_REQUIRE(c, n_owned < (1ll << 31), "too many owned blocks");
  gs_geom geo = gs_make_geom(&cams_h[0]);
  float bg[3] = {0.f, 0.f, 0.f};
  if (bg_h) for (int k = 0; k < 3; k++) bg[k] = bg_h[k];
  const float norm = gt ? (float)(1.0 / (3.0 * (double)geo.W * (double)geo.H * (double)b_loss)) : 0.f;
  ++c->launches;
  k_render_fwd<<<(unsigned)n_owned, kThreads, 0, (cudaStream_t)stream>>>(
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
  GS_REQUIRE(c, tile_range && T_final && n_last && dL_dpix, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  if (n_recv > 0) {
    GS_REQUIRE(c, dL_drec != nullptr, "null dL_drec");
    GS_CUDA(c, cudaMemsetAsync(dL_drec, 0, (size_t)n_recv * 9 * sizeof(float), st));
  }
  const int64_t B_lo = dp_h[c->rank], n_owned = dp_h[c->rank + 1] - B_lo;
  if (n_owned == 0) return GS_OK;
  gs_geom geo = gs_make_geom(&cams_h[0]);
  float bg[3] = {0.f, 0.f, 0.f};
  if (bg_h) for (int k = 0; k < 3; k++) bg[k] = bg_h[k];
  ++c->launches;
  k_render_bwd<<<(unsigned)n_owned, kThreads, 0, st>>>(
      (const gs_rec*)recv_rec, sorted_idx, tile_range, geo, B_lo, bg[0], bg[1], bg[2], dL_dpix, T_final, n_last,
      dL_drec, tile_cost, cost_mode, (long long*)stats);
  GS_LAUNCH_CHECK(c, "render_bwd");
  return GS_OK;
}
