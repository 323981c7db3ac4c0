// gs_loss.cu -- NEXT-1: fused L1 + D-SSIM loss, forward and backward, over the rank's owned
// 16x16 blocks ("computes the L1 and SSIM loss ... the SSIM loss measures the
// similarity between pixel windows"; "pixels windows for SSIM loss").
//
//   L = (1 - lambda) mean|x - y| + lambda (1 - mean SSIM),   SSIM over an 11x11 Gaussian
//   window (sigma 1.5), C1 = 0.01^2, C2 = 0.03^2, zero padding outside the image (R12),
// means over every pixel and channel of the view, the batch loss divided by b (like O13).
//
// With mu_x, E[x^2], E[xy] the window statistics of x at a centre p, the SSIM map S(p) has
// derivatives a = dS/dmu_x, b = dS/dE[x^2], c = dS/dE[xy], and
//   d(sum_p S)/dx(q) = (w * a)(q) + 2 x(q) (w * b)(q) + y(q) (w * c)(q)        (w symmetric).
// Two kernels, one CTA (256 threads) per owned block each:
//   k_ssim_terms: stage x, y over the block + 5-pixel halo (26x26), separable window sums of
//     (x, y, x^2, y^2, xy) at the block's 16x16 centres, S -> the block's loss share, and the
//     9 maps (a, b, c per channel) -> HBM;
//   k_ssim_grad: stage the maps over the block + 5-pixel halo, separable window sums of the
//     maps, combine with x, y and the L1 sign into dL/dpix.
// Between them a halo of maps is needed from neighbouring blocks (other ranks' ones through
// gs_halo_exchange), so each statistic is computed once per pixel instead of once per pixel
// per neighbouring block.  Both separable passes are register-blocked: a thread produces 4
// consecutive outputs of a row (column) from 14 staged inputs held in registers, so shared
// memory traffic is ~14 loads per 4 outputs instead of 11 per output; rows are padded to an
// odd stride (no bank conflicts).  All arithmetic is FP32 on the CUDA cores: 11-tap stencils
// over a few thousand values per block have no tensor-core-sized contraction, and the
// variance E[x^2] - mu^2 needs fp32 mantissas.
#include <algorithm>
#include <cmath>
#include <vector>

#include "gs_device.cuh"
#include "gs_internal.h"

using namespace gsd;

namespace {

constexpr int kThreads = 192;  // 6 warps: the vertical passes have exactly 192 items (3 x 16 x 4)
constexpr int kS = 26;        // staged side: block + 5-pixel halo each way
constexpr int kLd = 27;       // odd row stride of staged tiles
constexpr int kLdO = 17;      // odd row stride of 16-wide outputs

struct ssim_arg {
  float g[11];  // normalised 1D Gaussian, sigma 1.5 (the 2D window is g x g)
  float lambda, norm;
};

// The 3x3 neighbourhood of blocks around block (tx, ty) of view v: planes of `fpb` floats
// (the rank's own blocks, or halo slots found in the ascending halo id list), null outside
// the grid.  Threads 0..8 fill s_src.
__device__ __forceinline__ void neighbour_sources(const float* base, const float* halo, const int64_t* halo_ids,
                                                  int64_t n_halo, const gs_geom& geo, int64_t B_lo, int64_t B_hi,
                                                  int64_t v, int tx, int ty, int fpb, const float** s_src) {
  const int t = threadIdx.x;
  if (t >= 9) return;
  const int bx = tx + t % 3 - 1, by = ty + t / 3 - 1;
  const float* src = nullptr;
  if (bx >= 0 && bx < geo.Wt && by >= 0 && by < geo.Ht) {
    const int64_t nb = v * geo.per_view + (int64_t)by * geo.Wt + bx;
    if (nb >= B_lo && nb < B_hi) {
      src = base + (nb - B_lo) * fpb;
    } else {
      int64_t lo = 0, hi = n_halo;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (halo_ids[mid] < nb) lo = mid + 1; else hi = mid;
      }
      if (lo < n_halo && halo_ids[lo] == nb) src = halo + lo * fpb;
      else __trap();  // halo not supplied: a contract violation, never a silent zero
    }
  }
  s_src[t] = src;
}

// 1/x by one MUFU.RCP (x >= 1e-4 here: no denormal range fix-up needed; ~1 ulp).
__device__ __forceinline__ float rcp_fast(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Which of the 3x3 neighbour blocks holds staged coordinate i (0..25, block starts at 5).
__device__ __forceinline__ int nb_of(int i) { return i < 5 ? 0 : (i < 21 ? 1 : 2); }

// Stage `np` planes (256 floats each, plane stride 256 within a block's record of fpb floats)
// of the 26x26 neighbourhood into dst[plane][26][kLd] with 16-byte loads: the neighbourhood's
// row r spans columns 11..36 of the three blocks side by side (48 columns = 12 float4), of
// which float4s 2..9 overlap it.  Zero where there is no block (outside the grid).
__device__ __forceinline__ void stage_planes(const float* const* s_src, int np, int plane0, float* dst) {
  // loads of kU items are issued before their stores (memory-level parallelism: the staging
  // is latency-bound, each CTA waits for it before any arithmetic)
  constexpr int kU = 4;
  const int total = np * kS * 8;
  for (int base = threadIdx.x; base < total; base += kThreads * kU) {
    float4 q[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const int it = base + u * kThreads;
      q[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (it < total) {
        const int pl = it / (kS * 8), r = (it / 8) % kS, f = 2 + it % 8;
        const float* src = s_src[nb_of(r) * 3 + (f >> 2)];
        if (src) q[u] = __ldg(reinterpret_cast<const float4*>(src + (plane0 + pl) * 256 + ((r + 11) & 15) * 16 +
                                                              (f & 3) * 4));
      }
    }
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const int it = base + u * kThreads;
      if (it < total) {
        const int pl = it / (kS * 8), r = (it / 8) % kS, f = 2 + it % 8;
        const float e[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
        float* d = dst + (pl * kS + r) * kLd;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const int col = f * 4 + k - 11;
          if (col >= 0 && col < kS) d[col] = e[k];
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_ssim_terms(
    const float* __restrict__ out_rgb, const float* __restrict__ halo, const int64_t* __restrict__ halo_ids,
    int64_t n_halo, const uint8_t* __restrict__ gt, gs_geom geo, int64_t B_lo, int64_t B_hi, ssim_arg h,
    float* __restrict__ maps, double* __restrict__ loss_sum) {
  __shared__ float X[3][kS][kLd], Y[3][kS][kLd];
  __shared__ float HS[3][5][kS][kLdO];  // horizontal sums at the 16 own columns
  __shared__ const float* s_src[9];
  __shared__ double s_red[kThreads / 32];
  const int tid = threadIdx.x;
  const int64_t lb = blockIdx.x, beta = B_lo + lb;
  const int64_t v = beta / geo.per_view, loc = beta % geo.per_view;
  const int tx = (int)(loc % geo.Wt), ty = (int)(loc / geo.Wt);
  neighbour_sources(out_rgb, halo, halo_ids, n_halo, geo, B_lo, B_hi, v, tx, ty, 768, s_src);
  __syncthreads();
  // x: rendered planes (zero outside the grid; partial blocks hold zeros outside the image,
  // see gs_render_fwd's out_rgb); y: ground truth, zero outside the image
  // ground-truth bytes of the 26x26 window: every load of this thread (<= 4 pixels x 3 bytes)
  // is issued before the first use, so their latencies overlap (the per-pixel load -> convert
  // -> store chain was the kernel's top stall)
  constexpr int kGI = (kS * kS + kThreads - 1) / kThreads;
  uint8_t gb[kGI][3];
#pragma unroll
  for (int u = 0; u < kGI; u++) {
    const int t = tid + u * kThreads;
    const int i = t / kS, j = t % kS;
    const int gy = ty * 16 - 5 + i, gx = tx * 16 - 5 + j;
    const bool ok = t < kS * kS && gx >= 0 && gx < geo.W && gy >= 0 && gy < geo.H;
    const uint8_t* g = gt + ((v * geo.H + gy) * (int64_t)geo.W + gx) * 3;
#pragma unroll
    for (int c = 0; c < 3; c++) gb[u][c] = ok ? __ldg(g + c) : (uint8_t)0;
  }
  stage_planes(s_src, 3, 0, &X[0][0][0]);
#pragma unroll
  for (int u = 0; u < kGI; u++) {
    const int t = tid + u * kThreads;
    if (t < kS * kS) {
      const int i = t / kS, j = t % kS;
#pragma unroll
      for (int c = 0; c < 3; c++) Y[c][i][j] = (float)gb[u][c] * (1.0f / 255.0f);
    }
  }
  __syncthreads();
  // horizontal: item = (channel, row r, 4 output columns 4s..4s+3 <- staged cols 4s..4s+13)
  for (int it = tid; it < 3 * kS * 4; it += kThreads) {
    const int c = it / (kS * 4), r = (it / 4) % kS, s = it % 4;
    // (x, y) and (x^2, y^2) accumulate as packed fp32x2 pairs (FFMA2 with the tap weight
    // broadcast), xy as a scalar: 3 instructions per tap and output instead of 5
    float2 a01[4], a23[4];
    float a4[4];
#pragma unroll
    for (int o = 0; o < 4; o++) a01[o] = a23[o] = make_float2(0.f, 0.f), a4[o] = 0.f;
#pragma unroll
    for (int j = 0; j < 14; j++) {
      const float2 p01 = make_float2(X[c][r][4 * s + j], Y[c][r][4 * s + j]);
      const float2 p23 = __fmul2_rn(p01, p01);
      const float p4 = p01.x * p01.y;
#pragma unroll
      for (int o = 0; o < 4; o++) {
        const int k = j - o;
        if (k >= 0 && k <= 10) {
          const float2 w2 = make_float2(h.g[k], h.g[k]);
          a01[o] = __ffma2_rn(w2, p01, a01[o]);
          a23[o] = __ffma2_rn(w2, p23, a23[o]);
          a4[o] = fmaf(h.g[k], p4, a4[o]);
        }
      }
    }
#pragma unroll
    for (int o = 0; o < 4; o++) {
      HS[c][0][r][4 * s + o] = a01[o].x;
      HS[c][1][r][4 * s + o] = a01[o].y;
      HS[c][2][r][4 * s + o] = a23[o].x;
      HS[c][3][r][4 * s + o] = a23[o].y;
      HS[c][4][r][4 * s + o] = a4[o];
    }
  }
  __syncthreads();
  // vertical: item = (channel, column j, 4 output rows 4s..4s+3 <- rows 4s..4s+13) -> S, maps
  const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
  float lsum = 0.f;
  for (int it = tid; it < 3 * 16 * 4; it += kThreads) {
    const int c = it / 64, s = (it / 16) % 4, j = it % 16;
    float2 s01[4], s23[4];
    float s4[4];
#pragma unroll
    for (int o = 0; o < 4; o++) s01[o] = s23[o] = make_float2(0.f, 0.f), s4[o] = 0.f;
#pragma unroll
    for (int i = 0; i < 14; i++) {
      const float2 h01 = make_float2(HS[c][0][4 * s + i][j], HS[c][1][4 * s + i][j]);
      const float2 h23 = make_float2(HS[c][2][4 * s + i][j], HS[c][3][4 * s + i][j]);
      const float h4 = HS[c][4][4 * s + i][j];
#pragma unroll
      for (int o = 0; o < 4; o++) {
        const int k = i - o;
        if (k >= 0 && k <= 10) {
          const float2 w2 = make_float2(h.g[k], h.g[k]);
          s01[o] = __ffma2_rn(w2, h01, s01[o]);
          s23[o] = __ffma2_rn(w2, h23, s23[o]);
          s4[o] = fmaf(h.g[k], h4, s4[o]);
        }
      }
    }
    float st[4][5];
#pragma unroll
    for (int o = 0; o < 4; o++) {
      st[o][0] = s01[o].x, st[o][1] = s01[o].y, st[o][2] = s23[o].x, st[o][3] = s23[o].y, st[o][4] = s4[o];
    }
#pragma unroll
    for (int o = 0; o < 4; o++) {
      const int row = 4 * s + o, p = row * 16 + j;
      const int gy = ty * 16 + row, gx = tx * 16 + j;
      float a = 0.f, b = 0.f, cc = 0.f;
      if (gx < geo.W && gy < geo.H) {
        const float mx = st[o][0], my = st[o][1];
        const float A1 = 2.f * mx * my + C1, A2 = 2.f * (st[o][4] - mx * my) + C2;
        const float B1 = mx * mx + my * my + C1, B2 = (st[o][2] - mx * mx) + (st[o][3] - my * my) + C2;
        const float rB1 = rcp_fast(B1), rB2 = rcp_fast(B2), rB = rB1 * rB2;  // B1, B2 >= C1, C2 > 0
        const float S = A1 * A2 * rB;
        a = 2.f * my * (A2 - A1) * rB - 2.f * mx * S * (rB1 - rB2);
        b = -S * rB2;
        cc = 2.f * A1 * rB;
        const float x = X[c][row + 5][j + 5], y = Y[c][row + 5][j + 5];
        lsum += (1.f - h.lambda) * fabsf(x - y) + h.lambda * (1.f - S);
      }
      float* m = maps + lb * 2304 + c * 256 + p;  // [lb][map 0..2][channel][256]
      m[0] = a;
      m[768] = b;
      m[1536] = cc;
    }
  }
  double v2 = (double)lsum * (double)h.norm;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v2 += __shfl_xor_sync(0xffffffffu, v2, o);
  if ((tid & 31) == 0) s_red[tid >> 5] = v2;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; w++) s += s_red[w];
    if (s != 0.0) atomicAdd(loss_sum, s);
  }
}

__global__ void __launch_bounds__(kThreads) k_ssim_grad(
    const float* __restrict__ maps, const float* __restrict__ halo, const int64_t* __restrict__ halo_ids,
    int64_t n_halo, const float* __restrict__ out_rgb, const uint8_t* __restrict__ gt, gs_geom geo, int64_t B_lo,
    int64_t B_hi, ssim_arg h, float* __restrict__ dL_dpix) {
  __shared__ float M[9][kS][kLd];     // map m (a, b, c) of channel ch at index m * 3 + ch
  __shared__ float HB[9][kS][kLdO];   // horizontal sums at the 16 own columns
  __shared__ const float* s_src[9];
  const int tid = threadIdx.x;
  const int64_t lb = blockIdx.x, beta = B_lo + lb;
  const int64_t v = beta / geo.per_view, loc = beta % geo.per_view;
  const int tx = (int)(loc % geo.Wt), ty = (int)(loc / geo.Wt);
  // x and y of this thread's 4 output pixels of the vertical pass (item = tid: exactly 192
  // items), loaded before the staging so their latency hides behind it
  static_assert(3 * 16 * 4 == kThreads, "one vertical item per thread");
  float xs[4], ys[4];
  {
    const int c = tid / 64, s4 = (tid / 16) % 4, j = tid % 16;
#pragma unroll
    for (int o = 0; o < 4; o++) {
      const int row = 4 * s4 + o, p = row * 16 + j;
      const int gy = ty * 16 + row, gx = tx * 16 + j;
      const bool in = gx < geo.W && gy < geo.H;
      xs[o] = in ? __ldg(out_rgb + lb * 768 + c * 256 + p) : 0.f;
      ys[o] = in ? (float)__ldg(gt + ((v * geo.H + gy) * (int64_t)geo.W + gx) * 3 + c) * (1.0f / 255.0f) : 0.f;
    }
  }
  neighbour_sources(maps, halo, halo_ids, n_halo, geo, B_lo, B_hi, v, tx, ty, 2304, s_src);
  __syncthreads();
  stage_planes(s_src, 9, 0, &M[0][0][0]);  // maps are zero outside the image
  __syncthreads();
  // horizontal: item = (map, row r, 4 output columns)
  for (int it = tid; it < 9 * kS * 4; it += kThreads) {
    const int m = it / (kS * 4), r = (it / 4) % kS, s = it % 4;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 14; j++) {
      const float val = M[m][r][4 * s + j];
#pragma unroll
      for (int o = 0; o < 4; o++) {
        const int k = j - o;
        if (k >= 0 && k <= 10) acc[o] = fmaf(h.g[k], val, acc[o]);
      }
    }
#pragma unroll
    for (int o = 0; o < 4; o++) HB[m][r][4 * s + o] = acc[o];
  }
  __syncthreads();
  // vertical: item = (channel, column j, 4 output rows) -> dL/dpix
  for (int it = tid; it < 3 * 16 * 4; it += kThreads) {
    const int c = it / 64, s = (it / 16) % 4, j = it % 16;
    float2 w01[4];
    float w2s[4];
#pragma unroll
    for (int o = 0; o < 4; o++) w01[o] = make_float2(0.f, 0.f), w2s[o] = 0.f;
#pragma unroll
    for (int i = 0; i < 14; i++) {
      const float2 h01 = make_float2(HB[c][4 * s + i][j], HB[3 + c][4 * s + i][j]);
      const float h2 = HB[6 + c][4 * s + i][j];
#pragma unroll
      for (int o = 0; o < 4; o++) {
        const int k = i - o;
        if (k >= 0 && k <= 10) {
          w01[o] = __ffma2_rn(make_float2(h.g[k], h.g[k]), h01, w01[o]);
          w2s[o] = fmaf(h.g[k], h2, w2s[o]);
        }
      }
    }
    float w3[4][3];
#pragma unroll
    for (int o = 0; o < 4; o++) w3[o][0] = w01[o].x, w3[o][1] = w01[o].y, w3[o][2] = w2s[o];
#pragma unroll
    for (int o = 0; o < 4; o++) {
      const int row = 4 * s + o, p = row * 16 + j;
      const int gy = ty * 16 + row, gx = tx * 16 + j;
      float d = 0.f;
      if (gx < geo.W && gy < geo.H) {
        const float x = xs[o], y = ys[o];  // it == tid (one item per thread)
        const float gs = w3[o][0] + 2.f * x * w3[o][1] + y * w3[o][2];
        const float e = x - y;
        d = ((1.f - h.lambda) * (e > 0.f ? 1.f : (e < 0.f ? -1.f : 0.f)) - h.lambda * gs) * h.norm;
      }
      dL_dpix[lb * 768 + c * 256 + p] = d;
    }
  }
}

gs_status ssim_args(gs_ctx* c, const gs_camera* cams_h, int n_views, const int64_t* dp_h, float lambda,
                    int b_loss, int64_t n_halo, const float* halo, const int64_t* halo_ids, ssim_arg& h) {
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, b_loss >= 1, "b_loss must be >= 1");
  GS_REQUIRE(c, lambda >= 0.f && lambda <= 1.f, "lambda must be in [0, 1]");
  GS_REQUIRE(c, n_halo >= 0 && (n_halo == 0 || (halo && halo_ids)), "halo arguments");
  const gs_geom geo = gs_make_geom(&cams_h[0]);
  double g[11], sum = 0.0;
  for (int k = 0; k < 11; k++) {
    g[k] = std::exp(-(double)((k - 5) * (k - 5)) / (2.0 * 1.5 * 1.5));
    sum += g[k];
  }
  for (int k = 0; k < 11; k++) h.g[k] = (float)(g[k] / sum);
  h.lambda = lambda;
  h.norm = (float)(1.0 / (3.0 * (double)geo.W * (double)geo.H * (double)b_loss));
  return GS_OK;
}

}  // namespace

// Halo of rank r: blocks of the batch that are 8-neighbours (same view, inside the block
// grid) of an owned block and are not owned, ascending.  A block whose serialized
// neighbours beta - Wt - 1 and beta + Wt + 1 both lie in the owned range has all its
// neighbours owned, so only the first and last Wt + 1 owned blocks are examined.
void gs_halo_blocks(const gs_geom& geo, int64_t lo, int64_t hi, std::vector<int64_t>& out) {
  out.clear();
  if (hi <= lo) return;
  auto visit = [&](int64_t b) {
    const int64_t v = b / geo.per_view, l = b % geo.per_view;
    const int x = (int)(l % geo.Wt), y = (int)(l / geo.Wt);
    for (int dy = -1; dy <= 1; dy++)
      for (int dx = -1; dx <= 1; dx++) {
        const int nx = x + dx, ny = y + dy;
        if ((dx == 0 && dy == 0) || nx < 0 || nx >= geo.Wt || ny < 0 || ny >= geo.Ht) continue;
        const int64_t nb = v * geo.per_view + (int64_t)ny * geo.Wt + nx;
        if (nb < lo || nb >= hi) out.push_back(nb);
      }
  };
  const int64_t k = geo.Wt + 1;
  for (int64_t b = lo; b < std::min(hi, lo + k); b++) visit(b);
  for (int64_t b = std::max(lo + k, hi - k); b < hi; b++) visit(b);
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
}

extern "C" gs_status gs_halo_plan(gs_ctx* c, const gs_camera* cams_h, int n_views, const int64_t* dp_h,
                                  int64_t* halo_ids_h, int64_t cap, int64_t* n_halo_h) {
  if (!c) return GS_EINVAL;
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, n_halo_h != nullptr, "null n_halo_h");
  std::vector<int64_t> ids;
  gs_halo_blocks(gs_make_geom(&cams_h[0]), dp_h[c->rank], dp_h[c->rank + 1], ids);
  *n_halo_h = (int64_t)ids.size();
  if ((int64_t)ids.size() > cap)
    return gs_fail(c, GS_ECAPACITY, "halo capacity %lld < %lld", (long long)cap, (long long)ids.size());
  if (!ids.empty()) {
    GS_REQUIRE(c, halo_ids_h != nullptr, "null halo_ids_h");
    std::copy(ids.begin(), ids.end(), halo_ids_h);
  }
  return GS_OK;
}

extern "C" gs_status gs_ssim_terms(gs_ctx* c, const float* out_rgb, const float* halo_rgb, const int64_t* halo_ids,
                                   int64_t n_halo, const uint8_t* gt, const gs_camera* cams_h, int n_views,
                                   const int64_t* dp_h, float lambda, int b_loss, float* maps, double* loss_sum,
                                   void* stream) {
  if (!c) return GS_EINVAL;
  ssim_arg h;
  gs_status s = ssim_args(c, cams_h, n_views, dp_h, lambda, b_loss, n_halo, halo_rgb, halo_ids, h);
  if (s != GS_OK) return s;
  const int64_t B_lo = dp_h[c->rank], B_hi = dp_h[c->rank + 1], n_owned = B_hi - B_lo;
  if (n_owned == 0) return GS_OK;
  GS_REQUIRE(c, out_rgb && gt && maps && loss_sum, "null argument");
  ++c->launches;
  k_ssim_terms<<<(unsigned)n_owned, kThreads, 0, (cudaStream_t)stream>>>(
      out_rgb, halo_rgb, halo_ids, n_halo, gt, gs_make_geom(&cams_h[0]), B_lo, B_hi, h, maps, loss_sum);
  GS_LAUNCH_CHECK(c, "ssim_terms");
  return GS_OK;
}

extern "C" gs_status gs_ssim_grad(gs_ctx* c, const float* maps, const float* halo_maps, const int64_t* halo_ids,
                                  int64_t n_halo, const float* out_rgb, const uint8_t* gt, const gs_camera* cams_h,
                                  int n_views, const int64_t* dp_h, float lambda, int b_loss, float* dL_dpix,
                                  void* stream) {
  if (!c) return GS_EINVAL;
  ssim_arg h;
  gs_status s = ssim_args(c, cams_h, n_views, dp_h, lambda, b_loss, n_halo, halo_maps, halo_ids, h);
  if (s != GS_OK) return s;
  const int64_t B_lo = dp_h[c->rank], B_hi = dp_h[c->rank + 1], n_owned = B_hi - B_lo;
  if (n_owned == 0) return GS_OK;
  GS_REQUIRE(c, maps && out_rgb && gt && dL_dpix, "null argument");
  ++c->launches;
  k_ssim_grad<<<(unsigned)n_owned, kThreads, 0, (cudaStream_t)stream>>>(
      maps, halo_maps, halo_ids, n_halo, out_rgb, gt, gs_make_geom(&cams_h[0]), B_lo, B_hi, h, dL_dpix);
  GS_LAUNCH_CHECK(c, "ssim_grad");
  return GS_OK;
}
