// gs_loss.cu -- NEXT-1: fused L1 + D-SSIM loss, forward and backward, over the rank's owned
// 16x16 blocks ("computes the L1 and SSIM loss ... the SSIM loss measures the
// similarity between pixel windows"; "pixels windows for SSIM loss").
//
//   L = (1 - lambda) mean|x - y| + lambda (1 - mean SSIM),   SSIM over an 11x11 Gaussian
//   window (sigma 1.5), C1 = 0.01^2, C2 = 0.03^2, zero padding outside the image (R12),
// means over every pixel and channel of the view, the batch loss divided by b (like O13).
//
// One CTA (256 threads) per owned block.  The gradient at a pixel needs the SSIM map's
// derivatives at every centre within 5 pixels, and each of those needs the image within 5
// pixels of it, so the CTA stages the 36x36 neighbourhood (10-pixel halo) of the block: from
// the rank's own rendered blocks, from the halo buffer filled by gs_halo_exchange (blocks of
// the same view owned by other ranks), or zero outside the image.  Per channel, in shared
// memory:
//   1. separable window sums of (x, y, x^2, y^2, xy) at the 26x26 centres around the block,
//   2. S and its derivatives a = dS/dmu_x, b = dS/dE[x^2], c = dS/dE[xy] there (zero at
//      centres outside the image),
//   3. dSSIM_sum/dx = (w*a) + 2 x (w*b) + y (w*c) at the 16x16 pixels (separable again),
// fused with the L1 sign term into dL/dpix, and the block's share of L into *loss_sum.
// Every FP32 operation is on the CUDA cores: the window sums are 11-tap stencils over a few
// thousand values per block (no contraction shape worth a tensor-core tile), and the
// variance E[x^2] - mu^2 needs fp32 mantissas.
#include <algorithm>
#include <cmath>
#include <vector>

#include "gs_device.cuh"
#include "gs_internal.h"

using namespace gsd;

namespace {

constexpr int kR = 36;   // staged region (block + 10-pixel halo)
constexpr int kC = 26;   // centres whose SSIM terms the block's gradient needs (block + 5)
constexpr int kThreads = 256;

struct ssim_arg {
  float g[11];  // normalised 1D Gaussian, sigma 1.5 (the 2D window is g x g)
  float lambda, norm;
};

// Dynamic shared memory layout (floats).
constexpr int kXY = 3 * kR * kR;      // X or Y, 3 channels
constexpr int kHS = 5 * kR * kC;      // horizontal sums of the 5 products, one channel
constexpr int kM = 3 * kC * kC;       // a, b, c maps, one channel
constexpr int kHB = 3 * kC * 16;      // horizontal sums of the maps, one channel
constexpr size_t kSmem = (size_t)(2 * kXY + kHS + kM + kHB) * sizeof(float);

__global__ void __launch_bounds__(kThreads) k_loss_ssim(
    const float* __restrict__ out_rgb, const float* __restrict__ halo, const int64_t* __restrict__ halo_ids,
    int64_t n_halo, const uint8_t* __restrict__ gt, gs_geom geo, int64_t B_lo, int64_t B_hi, ssim_arg h,
    float* __restrict__ dL_dpix, double* __restrict__ loss_sum) {
  extern __shared__ float sm[];
  float* X = sm;             // [3][36][36]
  float* Y = X + kXY;        // [3][36][36]
  float* HS = Y + kXY;       // [5][36][26]
  float* M = HS + kHS;       // [3][26][26]
  float* HB = M + kM;        // [3][26][16]
  __shared__ const float* s_src[9];  // 3x3 neighbourhood of blocks: [3][256] planes or null
  __shared__ double s_red[kThreads / 32];
  const int tid = threadIdx.x;
  const int64_t lb = blockIdx.x, beta = B_lo + lb;
  const int64_t v = beta / geo.per_view, loc = beta % geo.per_view;
  const int tx = (int)(loc % geo.Wt), ty = (int)(loc / geo.Wt);
  if (tid < 9) {
    const int bx = tx + tid % 3 - 1, by = ty + tid / 3 - 1;
    const float* src = nullptr;
    if (bx >= 0 && bx < geo.Wt && by >= 0 && by < geo.Ht) {
      const int64_t nb = v * geo.per_view + (int64_t)by * geo.Wt + bx;
      if (nb >= B_lo && nb < B_hi) {
        src = out_rgb + (nb - B_lo) * 768;
      } else {  // another rank's block: its slot in the (ascending) halo id list
        int64_t lo = 0, hi = n_halo;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (halo_ids[mid] < nb) lo = mid + 1; else hi = mid;
        }
        if (lo < n_halo && halo_ids[lo] == nb) src = halo + lo * 768;
        else __trap();  // halo not supplied: a contract violation, never a silent zero
      }
    }
    s_src[tid] = src;
  }
  __syncthreads();
  // stage x (rendered) and y (ground truth) over the 36x36 region, zero outside the image
  const int gx0 = tx * 16 - 10, gy0 = ty * 16 - 10;
  for (int t = tid; t < kR * kR; t += kThreads) {
    const int i = t / kR, j = t % kR;
    const int gy = gy0 + i, gx = gx0 + j;
    float x[3] = {0.f, 0.f, 0.f}, y[3] = {0.f, 0.f, 0.f};
    if (gx >= 0 && gx < geo.W && gy >= 0 && gy < geo.H) {
      const int nbi = (i < 10 ? 0 : (i < 26 ? 1 : 2)) * 3 + (j < 10 ? 0 : (j < 26 ? 1 : 2));
      const float* src = s_src[nbi];
      const int p = (gy & 15) * 16 + (gx & 15);
      const uint8_t* g = gt + ((v * geo.H + gy) * (int64_t)geo.W + gx) * 3;
#pragma unroll
      for (int c = 0; c < 3; c++) {
        x[c] = src[c * 256 + p];
        y[c] = (float)g[c] * (1.0f / 255.0f);
      }
    }
#pragma unroll
    for (int c = 0; c < 3; c++) {
      X[c * kR * kR + t] = x[c];
      Y[c * kR * kR + t] = y[c];
    }
  }
  const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
  float lsum = 0.f;
  for (int c = 0; c < 3; c++) {
    const float* Xc = X + c * kR * kR;
    const float* Yc = Y + c * kR * kR;
    __syncthreads();
    // 1a. horizontal window sums: HS[k][i][jj], centre column jj + 5 of the region
    for (int t = tid; t < kR * kC; t += kThreads) {
      const int i = t / kC, jj = t % kC;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, s4 = 0.f;
#pragma unroll
      for (int k = 0; k < 11; k++) {
        const float x = Xc[i * kR + jj + k], y = Yc[i * kR + jj + k], w = h.g[k];
        s0 = fmaf(w, x, s0);
        s1 = fmaf(w, y, s1);
        s2 = fmaf(w * x, x, s2);
        s3 = fmaf(w * y, y, s3);
        s4 = fmaf(w * x, y, s4);
      }
      HS[0 * kR * kC + t] = s0;
      HS[1 * kR * kC + t] = s1;
      HS[2 * kR * kC + t] = s2;
      HS[3 * kR * kC + t] = s3;
      HS[4 * kR * kC + t] = s4;
    }
    __syncthreads();
    // 1b-2. vertical sums -> window statistics at centre (ii, jj) (region row ii + 5), SSIM
    //       terms; centres outside the image contribute nothing
    for (int t = tid; t < kC * kC; t += kThreads) {
      const int ii = t / kC, jj = t % kC;
      float st[5];
#pragma unroll
      for (int q = 0; q < 5; q++) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < 11; k++) s = fmaf(h.g[k], HS[q * kR * kC + (ii + k) * kC + jj], s);
        st[q] = s;
      }
      const int gy = ty * 16 - 5 + ii, gx = tx * 16 - 5 + jj;
      float a = 0.f, b = 0.f, cc = 0.f;
      if (gx >= 0 && gx < geo.W && gy >= 0 && gy < geo.H) {
        const float mx = st[0], my = st[1];
        const float A1 = 2.f * mx * my + C1, A2 = 2.f * (st[4] - mx * my) + C2;
        const float B1 = mx * mx + my * my + C1, B2 = (st[2] - mx * mx) + (st[3] - my * my) + C2;
        const float rB = 1.0f / (B1 * B2);
        const float S = A1 * A2 * rB;
        a = 2.f * my * (A2 - A1) * rB - 2.f * mx * S * (1.0f / B1 - 1.0f / B2);
        b = -S / B2;
        cc = 2.f * A1 * rB;
        if (ii >= 5 && ii < 21 && jj >= 5 && jj < 21) {  // a centre of this block
          const float x = Xc[(ii + 5) * kR + jj + 5], y = Yc[(ii + 5) * kR + jj + 5];
          lsum += (1.f - h.lambda) * fabsf(x - y) + h.lambda * (1.f - S);
        }
      }
      M[0 * kC * kC + t] = a;
      M[1 * kC * kC + t] = b;
      M[2 * kC * kC + t] = cc;
    }
    __syncthreads();
    // 3a. horizontal sums of the maps at the block's 16 columns
    for (int t = tid; t < kC * 16; t += kThreads) {
      const int ii = t / 16, j = t % 16;
#pragma unroll
      for (int q = 0; q < 3; q++) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < 11; k++) s = fmaf(h.g[k], M[q * kC * kC + ii * kC + j + k], s);
        HB[q * kC * 16 + t] = s;
      }
    }
    __syncthreads();
    // 3b. vertical sums -> dSSIM_sum/dx at pixel (i, j) of the block; fused with the L1 term
    {
      const int i = tid / 16, j = tid % 16;
      float s[3];
#pragma unroll
      for (int q = 0; q < 3; q++) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 11; k++) acc = fmaf(h.g[k], HB[q * kC * 16 + (i + k) * 16 + j], acc);
        s[q] = acc;
      }
      const float x = Xc[(i + 10) * kR + j + 10], y = Yc[(i + 10) * kR + j + 10];
      const int gy = ty * 16 + i, gx = tx * 16 + j;
      float d = 0.f;
      if (gx < geo.W && gy < geo.H) {
        const float gs = s[0] + 2.f * x * s[1] + y * s[2];
        const float e = x - y;
        d = ((1.f - h.lambda) * (e > 0.f ? 1.f : (e < 0.f ? -1.f : 0.f)) - h.lambda * gs) * h.norm;
      }
      dL_dpix[lb * 768 + c * 256 + tid] = d;
    }
  }
  // block's share of the loss
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

extern "C" gs_status gs_loss_ssim(gs_ctx* c, const float* out_rgb, const float* halo, const int64_t* halo_ids,
                                  int64_t n_halo, const uint8_t* gt, const gs_camera* cams_h, int n_views,
                                  const int64_t* dp_h, float lambda, int b_loss, float* dL_dpix, double* loss_sum,
                                  void* stream) {
  if (!c) return GS_EINVAL;
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, b_loss >= 1, "b_loss must be >= 1");
  GS_REQUIRE(c, lambda >= 0.f && lambda <= 1.f, "lambda must be in [0, 1]");
  GS_REQUIRE(c, n_halo >= 0 && (n_halo == 0 || (halo && halo_ids)), "halo arguments");
  const int64_t B_lo = dp_h[c->rank], B_hi = dp_h[c->rank + 1], n_owned = B_hi - B_lo;
  if (n_owned == 0) return GS_OK;
  GS_REQUIRE(c, out_rgb && gt && dL_dpix && loss_sum, "null argument");
  gs_geom geo = gs_make_geom(&cams_h[0]);
  ssim_arg h;
  {
    double g[11], sum = 0.0;
    for (int k = 0; k < 11; k++) {
      g[k] = std::exp(-(double)((k - 5) * (k - 5)) / (2.0 * 1.5 * 1.5));
      sum += g[k];
    }
    for (int k = 0; k < 11; k++) h.g[k] = (float)(g[k] / sum);
  }
  h.lambda = lambda;
  h.norm = (float)(1.0 / (3.0 * (double)geo.W * (double)geo.H * (double)b_loss));
  static bool attr = false;
  if (!attr) {
    GS_CUDA(c, cudaFuncSetAttribute(k_loss_ssim, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    attr = true;
  }
  ++c->launches;
  k_loss_ssim<<<(unsigned)n_owned, kThreads, kSmem, (cudaStream_t)stream>>>(out_rgb, halo, halo_ids, n_halo, gt, geo,
                                                                           B_lo, B_hi, h, dL_dpix, loss_sum);
  GS_LAUNCH_CHECK(c, "loss_ssim");
  return GS_OK;
}
