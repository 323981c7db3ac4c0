// gs_device.cuh -- device-side building blocks shared by the libgs kernels.
//
// The membership chain (O1-O8: activations, 3D covariance, camera space, mean2d, EWA 2D
// covariance, radius, tile rectangle) decides visibility, tile sets, exchange sets and sort
// keys, so it is written one correctly rounded fp32 operation at a time with explicit
// __f*_rn intrinsics (no FMA contraction, IEEE division and sqrt) in the fixed expression
// order of SURVEY §8(c) O1-O8 (reading R10).  Everything outside it may use FMA freely.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gs_internal.h"

namespace gsd {

// Compositing constants ("until a threshold opacity has been reached").
constexpr float kAlphaCap = 0.99f;
constexpr float kAlphaMin = 1.0f / 255.0f;
constexpr float kTStop = 1e-4f;
constexpr float kNear = 0.01f;
constexpr float kDilate = 0.3f;
constexpr int kBlock = 128;      // threads per CTA for Gaussian-wise kernels (project/adam)

struct gs_dcam {
  float R[9], t[3], fx, fy, cx, cy, campos[3];
};
struct gs_cams_arg {
  gs_dcam c[GS_MAX_VIEWS];
  int n;
};

inline gs_cams_arg make_cams(const gs_camera* cams_h, int n) {
  gs_cams_arg a;
  a.n = n;
  for (int v = 0; v < n; v++) {
    const gs_camera& s = cams_h[v];
    gs_dcam& d = a.c[v];
    for (int k = 0; k < 9; k++) d.R[k] = s.R[k];
    for (int k = 0; k < 3; k++) d.t[k] = s.t[k];
    d.fx = s.fx; d.fy = s.fy; d.cx = s.cx; d.cy = s.cy;
    for (int k = 0; k < 3; k++)  // camera centre c = -R^T t (host, double)
      d.campos[k] = (float)(-((double)s.R[k] * s.t[0] + (double)s.R[3 + k] * s.t[1] +
                              (double)s.R[6 + k] * s.t[2]));
  }
  return a;
}

__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float dvd(float a, float b) { return __fdiv_rn(a, b); }

// R10 exp: clamp, Cody-Waite with ln2 = 0.693359375 - 2.12194440e-4, Cephes polynomial.
__device__ __forceinline__ float exp_rn(float x) {
  if (x < -87.0f) x = -87.0f;
  if (x > 88.0f) x = 88.0f;
  float k = floorf(add(mul(x, 1.44269504088896341f), 0.5f));
  float r = sub(sub(x, mul(k, 0.693359375f)), mul(k, -2.12194440e-4f));
  float z = mul(r, r);
  float p = 1.9875691500e-4f;
  p = add(mul(p, r), 1.3981999507e-3f);
  p = add(mul(p, r), 8.3334519073e-3f);
  p = add(mul(p, r), 4.1665795894e-2f);
  p = add(mul(p, r), 1.6666665459e-1f);
  p = add(mul(p, r), 5.0000001201e-1f);
  p = add(add(mul(p, z), r), 1.0f);
  return mul(p, __int_as_float((int(k) + 127) << 23));
}

__device__ __forceinline__ int floordiv16(int v) { return v >= 0 ? v / 16 : -((-v + 15) / 16); }
__device__ __forceinline__ float clamp24(float v) {
  const float L = 16777216.0f;
  if (v > L) return L;
  if (v < -L) return -L;
  return v;
}

// O8: tile rectangle of the pixel-granular square [m - r, m + r]^2 (R1, R2).
// Returns false when it is empty (frustum cull).
__device__ __forceinline__ bool rect_of(float mx, float my, float r, int Wt, int Ht, int& tx0,
                                        int& tx1, int& ty0, int& ty1) {
  int c0 = (int)ceilf(clamp24(sub(mx, r))), c1 = (int)floorf(clamp24(add(mx, r)));
  int w0 = (int)ceilf(clamp24(sub(my, r))), w1 = (int)floorf(clamp24(add(my, r)));
  tx0 = max(0, floordiv16(c0));
  tx1 = min(Wt - 1, floordiv16(c1));
  ty0 = max(0, floordiv16(w0));
  ty1 = min(Ht - 1, floordiv16(w1));
  return tx0 <= tx1 && ty0 <= ty1;
}

// O1-O2, view independent: qbar rotation and 3D covariance (upper triangle S00..S22).
struct gs_cov3 {
  bool ok;
  float S[6];  // S00, S01, S02, S11, S12, S22
  float smax;  // largest scale (for the conservative early cull)
};

__device__ __forceinline__ gs_cov3 cov3_of(float4 ls, float4 q) {
  gs_cov3 o;
  float s0 = exp_rn(ls.x), s1 = exp_rn(ls.y), s2 = exp_rn(ls.z);
  o.smax = fmaxf(s0, fmaxf(s1, s2));
  float n2 = add(add(add(mul(q.x, q.x), mul(q.y, q.y)), mul(q.z, q.z)), mul(q.w, q.w));
  o.ok = n2 > 0.0f;
  float qn = __fsqrt_rn(n2);
  float w = dvd(q.x, qn), x = dvd(q.y, qn), y = dvd(q.z, qn), z = dvd(q.w, qn);
  float R0 = sub(1.0f, mul(2.0f, add(mul(y, y), mul(z, z))));
  float R1 = mul(2.0f, sub(mul(x, y), mul(w, z)));
  float R2 = mul(2.0f, add(mul(x, z), mul(w, y)));
  float R3 = mul(2.0f, add(mul(x, y), mul(w, z)));
  float R4 = sub(1.0f, mul(2.0f, add(mul(x, x), mul(z, z))));
  float R5 = mul(2.0f, sub(mul(y, z), mul(w, x)));
  float R6 = mul(2.0f, sub(mul(x, z), mul(w, y)));
  float R7 = mul(2.0f, add(mul(y, z), mul(w, x)));
  float R8 = sub(1.0f, mul(2.0f, add(mul(x, x), mul(y, y))));
  float M0 = mul(R0, s0), M1 = mul(R1, s1), M2 = mul(R2, s2);
  float M3 = mul(R3, s0), M4 = mul(R4, s1), M5 = mul(R5, s2);
  float M6 = mul(R6, s0), M7 = mul(R7, s1), M8 = mul(R8, s2);
  o.S[0] = add(add(mul(M0, M0), mul(M1, M1)), mul(M2, M2));
  o.S[1] = add(add(mul(M0, M3), mul(M1, M4)), mul(M2, M5));
  o.S[2] = add(add(mul(M0, M6), mul(M1, M7)), mul(M2, M8));
  o.S[3] = add(add(mul(M3, M3), mul(M4, M4)), mul(M5, M5));
  o.S[4] = add(add(mul(M3, M6), mul(M4, M7)), mul(M5, M8));
  o.S[5] = add(add(mul(M6, M6), mul(M7, M7)), mul(M8, M8));
  return o;
}

// O3-O8 for one view.
struct gs_memb {
  bool vis;
  float mx, my, depth, a, b, c, r;
  int tx0, tx1, ty0, ty1;
};

__device__ __forceinline__ gs_memb membership(const gs_cov3& cv, float X0, float X1, float X2,
                                              const gs_dcam& cam, int Wt, int Ht) {
  gs_memb o;
  o.vis = false;
  const float* W = cam.R;
  float p0 = add(add(add(mul(W[0], X0), mul(W[1], X1)), mul(W[2], X2)), cam.t[0]);
  float p1 = add(add(add(mul(W[3], X0), mul(W[4], X1)), mul(W[5], X2)), cam.t[1]);
  float p2 = add(add(add(mul(W[6], X0), mul(W[7], X1)), mul(W[8], X2)), cam.t[2]);
  if (!cv.ok || !(p2 > kNear)) return o;
  {
    // Cheap conservative pre-cull with fast reciprocals (not part of the definition; it only
    // skips Gaussians the exact chain below would reject): approximate mean and radius bound
    // with a 2% + 4 px margin, far beyond the error of the approximations.
    const float iz = __frcp_rn(p2);
    const float amx = cam.fx * p0 * iz + cam.cx, amy = cam.fy * p1 * iz + cam.cy;
    const float jf2 = (cam.fx * cam.fx + cam.fy * cam.fy) * iz * iz +
                      ((cam.fx * p0) * (cam.fx * p0) + (cam.fy * p1) * (cam.fy * p1)) * (iz * iz) * (iz * iz);
    const float rb = 3.0f * sqrtf((jf2 * cv.smax * cv.smax + kDilate) * 1.02f) + 4.0f;
    if (isfinite(rb) && isfinite(amx) && isfinite(amy) &&
        (amx + rb < 0.f || amx - rb > (float)(Wt * 16) || amy + rb < 0.f || amy - rb > (float)(Ht * 16)))
      return o;
  }
  float fxpx = mul(cam.fx, p0), fypy = mul(cam.fy, p1);
  o.mx = add(dvd(fxpx, p2), cam.cx);
  o.my = add(dvd(fypy, p2), cam.cy);
  o.depth = p2;
  {
    // Conservative early frustum cull (not part of the definition; it only skips Gaussians
    // the exact chain below would also reject): lambda_max(Sigma') <= ||J||_F^2 smax^2 + 0.3
    // (W orthonormal, Sigma = R diag(s^2) R^T), so the exact radius is <= r_ub and the exact
    // rectangle is inside the r_ub rectangle.  1% + 2 px margins absorb fp32 rounding.
    float iz = 1.0f / p2;
    float jf2 = (cam.fx * cam.fx + cam.fy * cam.fy) * iz * iz +
                (fxpx * fxpx + fypy * fypy) * (iz * iz) * (iz * iz);
    float lam_ub = (jf2 * cv.smax * cv.smax + kDilate) * 1.01f;
    float r_ub = ceilf(3.0f * sqrtf(lam_ub)) + 2.0f;
    int a0, a1, a2, a3;
    if (isfinite(r_ub) && !rect_of(o.mx, o.my, r_ub, Wt, Ht, a0, a1, a2, a3)) return o;
  }
  float pz2 = mul(p2, p2);
  float j00 = dvd(cam.fx, p2), j02 = -dvd(fxpx, pz2);
  float j11 = dvd(cam.fy, p2), j12 = -dvd(fypy, pz2);
  float T0 = add(mul(j00, W[0]), mul(j02, W[6]));
  float T1 = add(mul(j00, W[1]), mul(j02, W[7]));
  float T2 = add(mul(j00, W[2]), mul(j02, W[8]));
  float T3 = add(mul(j11, W[3]), mul(j12, W[6]));
  float T4 = add(mul(j11, W[4]), mul(j12, W[7]));
  float T5 = add(mul(j11, W[5]), mul(j12, W[8]));
  const float *S = cv.S;  // S00 S01 S02 S11 S12 S22
  float S00 = S[0], S01 = S[1], S02 = S[2], S11 = S[3], S12 = S[4], S22 = S[5];
  float U0 = add(add(mul(T0, S00), mul(T1, S01)), mul(T2, S02));
  float U1 = add(add(mul(T0, S01), mul(T1, S11)), mul(T2, S12));
  float U2 = add(add(mul(T0, S02), mul(T1, S12)), mul(T2, S22));
  float U3 = add(add(mul(T3, S00), mul(T4, S01)), mul(T5, S02));
  float U4 = add(add(mul(T3, S01), mul(T4, S11)), mul(T5, S12));
  float U5 = add(add(mul(T3, S02), mul(T4, S12)), mul(T5, S22));
  o.a = add(add(add(mul(U0, T0), mul(U1, T1)), mul(U2, T2)), kDilate);
  o.b = add(add(mul(U0, T3), mul(U1, T4)), mul(U2, T5));
  o.c = add(add(add(mul(U3, T3), mul(U4, T4)), mul(U5, T5)), kDilate);
  float det = sub(mul(o.a, o.c), mul(o.b, o.b));
  if (!(det > 0.0f)) return o;
  float mid = mul(0.5f, add(o.a, o.c));
  float disc = sub(mul(mid, mid), det);
  if (disc < 0.0f) disc = 0.0f;
  float lam = add(mid, __fsqrt_rn(disc));
  o.r = ceilf(mul(3.0f, __fsqrt_rn(lam)));
  o.vis = rect_of(o.mx, o.my, o.r, Wt, Ht, o.tx0, o.tx1, o.ty0, o.ty1);
  return o;
}

// Destination set D(i,v) (O10): ranks g with [dp[g], dp[g+1]) meeting a rectangle row.
__device__ __forceinline__ unsigned dest_mask(const gs_memb& m, int v, const gs_geom& geo,
                                              const gs_dp_arg& dp) {
  if (dp.G == 1) return 1u;
  unsigned mask = 0;
  long long base = (long long)v * geo.per_view;
  for (int ty = m.ty0; ty <= m.ty1; ty++) {
    long long lo = base + (long long)ty * geo.Wt + m.tx0, hi = base + (long long)ty * geo.Wt + m.tx1;
    // ranks g with dp[g] <= hi and dp[g+1] > lo
    for (int g = 0; g < dp.G; g++)
      if (dp.dp[g] <= hi && dp.dp[g + 1] > lo && dp.dp[g + 1] > dp.dp[g]) mask |= 1u << g;
    if (mask == (1u << dp.G) - 1u) break;
  }
  return mask;
}

// SH degree-3 real basis (3DGS convention [ext]).
__device__ __forceinline__ void sh_basis(float x, float y, float z, float Y[16]) {
  const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
  Y[0] = C0;
  Y[1] = -C1 * y;
  Y[2] = C1 * z;
  Y[3] = -C1 * x;
  float xx = x * x, yy = y * y, zz = z * z;
  Y[4] = 1.0925484305920792f * x * y;
  Y[5] = -1.0925484305920792f * y * z;
  Y[6] = 0.31539156525252005f * (2.f * zz - xx - yy);
  Y[7] = -1.0925484305920792f * x * z;
  Y[8] = 0.5462742152960396f * (xx - yy);
  Y[9] = -0.5900435899266435f * y * (3.f * xx - yy);
  Y[10] = 2.890611442640554f * x * y * z;
  Y[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
  Y[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
  Y[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy);
  Y[14] = 1.445305721320277f * z * (xx - yy);
  Y[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
}

// ex2.approx (MUFU.EX2) -- used for alpha in both render passes (identical instruction
// sequence in forward and backward).  Its relative error is pinned by gs_selftest_ex2.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// sqrt(0.5 * log2(e)): prescale of the conic's Cholesky factor so that
// 2^-(u'^2 + w'^2) = exp(-0.5 d^T conic d).
constexpr double kLScale64 = 0.84932180028801904272150283410289;

// The 64-byte record (include/gs.h GS_RECORD_BYTES): the conic's prescaled Cholesky factor
// L' = L sqrt(0.5 log2 e) (conic = L L^T) in double-float form, hi + lo, both rounded to
// nearest from fp64, and qmax = log2(255 o) rounded to nearest (alpha = o 2^-q >= 1/255 <=>
// q <= qmax).
struct __align__(16) gs_rec {
  float4 a;  // mx, my, depth, radius
  float4 b;  // l11', l21', l22' (hi), opacity
  float4 c;  // r, g, b, qmax
  float4 d;  // l11', l21', l22' (lo), meta bits (gid * 32 + view)
};

}  // namespace gsd
