// gs_adam.cu -- A7+A8: transformation backward fused with the Adam step on the owner
// ("Gaussian transformation backward ... distributed the same way as the Gaussian
// transformation forward"; Eq. (1) lambda' = lambda sqrt(b), Eq. (2) beta^b).
//
// One thread per owned Gaussian, the same 256-thread CTA decomposition as gs_project, so the
// send positions of its records are recomputed from the backward index exactly as A1 placed
// them.  Per view: sum the returned 9-float gradients over destinations in ascending rank,
// then the chain rule O16 (conic -> 2D covariance -> (Sigma, J(p)) -> (s, q), mean2d -> p -> x,
// colour -> SH and view direction, opacity -> logit), summed over the batch's views; then
// Adam on all 59 parameters in registers (dense over the shard, R9).  The parameter gradient
// never touches HBM unless GS_ADAM_WRITE_GRAD asks for it (parity mode).
#include <cstdlib>

#include "gs_device.cuh"
#include "gs_index.cuh"

using namespace gsd;

namespace {

constexpr int kListCap = 8;  // records per thread listed per round (phase A of k_bwd_adam)

struct adam_arg {
  float step[6];  // lambda'_g / (1 - beta1'^t), groups: pos, sh_dc, sh_rest, opacity, scale, rot
  float b1, b2, omb1, omb2, inv_sqrt_bc2, eps;
};

__device__ __forceinline__ void adam1(float& p, float& m, float& v, float g, float step, const adam_arg& h) {
  m = h.b1 * m + h.omb1 * g;
  v = h.b2 * v + h.omb2 * g * g;
  p -= step * m / (sqrtf(v) * h.inv_sqrt_bc2 + h.eps);
}

// Adam on one float4 plane element; grp[c] = group of lane c, or -1 (unused lane).
__device__ __forceinline__ void adam4(float4* P, float4* M, float4* V, int64_t idx, float4 g, int g0, int g1,
                                      int g2, int g3, const adam_arg& h) {
  float4 p = P[idx], m = M[idx], v = V[idx];
  if (g0 >= 0) adam1(p.x, m.x, v.x, g.x, h.step[g0], h);
  if (g1 >= 0) adam1(p.y, m.y, v.y, g.y, h.step[g1], h);
  if (g2 >= 0) adam1(p.z, m.z, v.z, g.z, h.step[g2], h);
  if (g3 >= 0) adam1(p.w, m.w, v.w, g.w, h.step[g3], h);
  P[idx] = p;
  M[idx] = m;
  V[idx] = v;
}

struct planes {
  float4 *pos_op, *ls, *rot, *sh;
};
inline planes mk(const gs_params* p) {
  return planes{(float4*)p->pos_op, (float4*)p->log_scale, (float4*)p->rot, (float4*)p->sh};
}

// Gradient of P(d) = sum_k c_k Y_k(d) with respect to d (d treated as free; the unit-norm
// constraint is applied by the caller's (I - d d^T)/|x - c| projection).
__device__ __forceinline__ void sh_poly_grad(float x, float y, float z, const float c[16], float& gx, float& gy,
                                             float& gz) {
  const float C1 = 0.4886025119029199f;
  const float a0 = 1.0925484305920792f, a1 = -1.0925484305920792f, a2 = 0.31539156525252005f,
              a3 = -1.0925484305920792f, a4 = 0.5462742152960396f;
  const float c0 = -0.5900435899266435f, c1 = 2.890611442640554f, c2 = -0.4570457994644658f,
              c3 = 0.3731763325901154f, c4 = -0.4570457994644658f, c5 = 1.445305721320277f,
              c6 = -0.5900435899266435f;
  const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z;
  gx = -C1 * c[3] + a0 * y * c[4] - 2.f * a2 * x * c[6] + a3 * z * c[7] + 2.f * a4 * x * c[8] +
       6.f * c0 * xy * c[9] + c1 * yz * c[10] - 2.f * c2 * xy * c[11] - 6.f * c3 * xz * c[12] +
       c4 * (4.f * zz - 3.f * xx - yy) * c[13] + 2.f * c5 * xz * c[14] + c6 * (3.f * xx - 3.f * yy) * c[15];
  gy = -C1 * c[1] + a0 * x * c[4] + a1 * z * c[5] - 2.f * a2 * y * c[6] - 2.f * a4 * y * c[8] +
       c0 * (3.f * xx - 3.f * yy) * c[9] + c1 * xz * c[10] + c2 * (4.f * zz - xx - 3.f * yy) * c[11] -
       6.f * c3 * yz * c[12] - 2.f * c4 * xy * c[13] - 2.f * c5 * yz * c[14] - 6.f * c6 * xy * c[15];
  gz = C1 * c[2] + a1 * y * c[5] + 4.f * a2 * z * c[6] + a3 * x * c[7] + c1 * xy * c[10] +
       8.f * c2 * yz * c[11] + c3 * (6.f * zz - 3.f * xx - 3.f * yy) * c[12] + 8.f * c4 * xz * c[13] +
       c5 * (xx - yy) * c[14];
}

// Chain rule O16 for one (Gaussian, view) given the summed record gradient g9 =
// dL/d(mx, my, A, B, C, opacity, r, g, b).  Accumulates into the parameter gradients.
__device__ __forceinline__ void proj_bwd_view(const float g9[9], float4 X, const float s[3], const float qb[4],
                                              float qn, const float Rq[9], const float Sig[6],
                                              const float4* __restrict__ sh, int64_t n, int64_t i,
                                              const gs_dcam& cam, float gpos[3], float gls[3],
                                              float gq[4], float& gop, float* gsh) {
  const float* W = cam.R;
  // opacity: o = sigmoid(logit)
  const float o = 1.0f / (1.0f + expf(-X.w));
  gop += g9[5] * o * (1.0f - o);
  // colour: SH coefficients and view direction, zero where the 0.5 + SH < 0 clamp was active
  float dvx = X.x - cam.campos[0], dvy = X.y - cam.campos[1], dvz = X.z - cam.campos[2];
  float dist = sqrtf(dvx * dvx + dvy * dvy + dvz * dvz), inv = 1.0f / dist;
  float dx = dvx * inv, dy = dvy * inv, dz = dvz * inv;
  float Y[16];
  sh_basis(dx, dy, dz, Y);
  // pass 1 over the SH planes: the colour (for the clamp mask)
  float col[3] = {0.5f, 0.5f, 0.5f};
#pragma unroll
  for (int k = 0; k < 12; k++) {
    const float4 s4 = sh[(int64_t)k * n + i];
    const float e[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
    for (int j = 0; j < 4; j++) col[(4 * k + j) % 3] = fmaf(Y[(4 * k + j) / 3], e[j], col[(4 * k + j) % 3]);
  }
  float gc[3];
#pragma unroll
  for (int ch = 0; ch < 3; ch++) gc[ch] = col[ch] < 0.f ? 0.f : g9[6 + ch];
  // pass 2: dL/dsh = Y gc and the contraction c_k = sum_ch sh[k][ch] gc[ch] (L1-resident reload)
  float ck[16];
#pragma unroll
  for (int k = 0; k < 16; k++) ck[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 12; k++) {
    const float4 s4 = sh[(int64_t)k * n + i];
    const float e[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int f = 4 * k + j, kk = f / 3, ch = f % 3;
      ck[kk] = fmaf(e[j], gc[ch], ck[kk]);
      gsh[f * kBlock] = fmaf(Y[kk], gc[ch], gsh[f * kBlock]);  // shared memory, column of this thread
    }
  }
  float gd0, gd1, gd2;
  sh_poly_grad(dx, dy, dz, ck, gd0, gd1, gd2);
  float dd = dx * gd0 + dy * gd1 + dz * gd2;
  gpos[0] += (gd0 - dx * dd) * inv;
  gpos[1] += (gd1 - dy * dd) * inv;
  gpos[2] += (gd2 - dz * dd) * inv;
  // camera space, J, T = J W, Sigma' = T Sigma T^T + 0.3 I
  float p0 = W[0] * X.x + W[1] * X.y + W[2] * X.z + cam.t[0];
  float p1 = W[3] * X.x + W[4] * X.y + W[5] * X.z + cam.t[1];
  float p2 = W[6] * X.x + W[7] * X.y + W[8] * X.z + cam.t[2];
  float iz = 1.0f / p2, iz2 = iz * iz;
  float j00 = cam.fx * iz, j02 = -cam.fx * p0 * iz2, j11 = cam.fy * iz, j12 = -cam.fy * p1 * iz2;
  float T[6] = {j00 * W[0] + j02 * W[6], j00 * W[1] + j02 * W[7], j00 * W[2] + j02 * W[8],
                j11 * W[3] + j12 * W[6], j11 * W[4] + j12 * W[7], j11 * W[5] + j12 * W[8]};
  const float S3[9] = {Sig[0], Sig[1], Sig[2], Sig[1], Sig[3], Sig[4], Sig[2], Sig[4], Sig[5]};
  float TS[6];  // T Sigma (2x3)
#pragma unroll
  for (int r = 0; r < 2; r++)
#pragma unroll
    for (int k = 0; k < 3; k++) TS[3 * r + k] = T[3 * r] * S3[k] + T[3 * r + 1] * S3[3 + k] + T[3 * r + 2] * S3[6 + k];
  float a = TS[0] * T[0] + TS[1] * T[1] + TS[2] * T[2] + kDilate;
  float b = TS[0] * T[3] + TS[1] * T[4] + TS[2] * T[5];
  float c = TS[3] * T[3] + TS[4] * T[4] + TS[5] * T[5] + kDilate;
  float bb = b * b;
  float det = fmaf(a, c, -bb) + fmaf(-b, b, bb);
  float id2 = 1.0f / (det * det);
  // conic (A, B, C) = (c, -b, a) / det  ->  gradient w.r.t. (a, b, c)
  const float gA = g9[2], gB = g9[3], gC = g9[4];
  float ga = (-c * c * gA + b * c * gB - bb * gC) * id2;
  float gb = (2.f * b * c * gA - (a * c + bb) * gB + 2.f * a * b * gC) * id2;
  float gcc = (-bb * gA + a * b * gB - a * a * gC) * id2;
  const float G00 = ga, G01 = 0.5f * gb, G11 = gcc;
  // dL/dSigma = T^T Gbar T (symmetric 3x3), dL/dT = 2 Gbar T Sigma
  float GT[6] = {G00 * T[0] + G01 * T[3], G00 * T[1] + G01 * T[4], G00 * T[2] + G01 * T[5],
                 G01 * T[0] + G11 * T[3], G01 * T[1] + G11 * T[4], G01 * T[2] + G11 * T[5]};
  float gS[9];
#pragma unroll
  for (int j = 0; j < 3; j++)
#pragma unroll
    for (int k = 0; k < 3; k++) gS[3 * j + k] = T[j] * GT[k] + T[3 + j] * GT[3 + k];
  float gT[6];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    gT[k] = 2.f * (G00 * TS[k] + G01 * TS[3 + k]);
    gT[3 + k] = 2.f * (G01 * TS[k] + G11 * TS[3 + k]);
  }
  // dL/dJ = dL/dT W^T (only the four non-zero entries of J matter)
  float gJ00 = gT[0] * W[0] + gT[1] * W[1] + gT[2] * W[2];
  float gJ02 = gT[0] * W[6] + gT[1] * W[7] + gT[2] * W[8];
  float gJ11 = gT[3] * W[3] + gT[4] * W[4] + gT[5] * W[5];
  float gJ12 = gT[3] * W[6] + gT[4] * W[7] + gT[5] * W[8];
  float gp0 = g9[0] * cam.fx * iz + gJ02 * (-cam.fx * iz2);
  float gp1 = g9[1] * cam.fy * iz + gJ12 * (-cam.fy * iz2);
  float iz3 = iz2 * iz;
  float gp2 = -g9[0] * cam.fx * p0 * iz2 - g9[1] * cam.fy * p1 * iz2 + gJ00 * (-cam.fx * iz2) +
              gJ02 * (2.f * cam.fx * p0 * iz3) + gJ11 * (-cam.fy * iz2) + gJ12 * (2.f * cam.fy * p1 * iz3);
  gpos[0] += W[0] * gp0 + W[3] * gp1 + W[6] * gp2;
  gpos[1] += W[1] * gp0 + W[4] * gp1 + W[7] * gp2;
  gpos[2] += W[2] * gp0 + W[5] * gp1 + W[8] * gp2;
  // Sigma = M M^T, M = Rq diag(s): dL/dM = 2 gS M
  float M[9];
#pragma unroll
  for (int j = 0; j < 3; j++)
#pragma unroll
    for (int k = 0; k < 3; k++) M[3 * j + k] = Rq[3 * j + k] * s[k];
  float gR[9];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    float gsk = 0.f;
#pragma unroll
    for (int j = 0; j < 3; j++) {
      float gm = 2.f * (gS[3 * j] * M[k] + gS[3 * j + 1] * M[3 + k] + gS[3 * j + 2] * M[6 + k]);
      gsk += gm * Rq[3 * j + k];
      gR[3 * j + k] = gm * s[k];
    }
    gls[k] += gsk * s[k];
  }
  const float w = qb[0], x = qb[1], y = qb[2], z = qb[3];
  float gqb[4];
  gqb[0] = 2.f * (-z * gR[1] + y * gR[2] + z * gR[3] - x * gR[5] - y * gR[6] + x * gR[7]);
  gqb[1] = 2.f * (y * gR[1] + z * gR[2] + y * gR[3] - 2.f * x * gR[4] - w * gR[5] + z * gR[6] + w * gR[7] - 2.f * x * gR[8]);
  gqb[2] = 2.f * (-2.f * y * gR[0] + x * gR[1] + w * gR[2] + x * gR[3] + z * gR[5] - w * gR[6] + z * gR[7] - 2.f * y * gR[8]);
  gqb[3] = 2.f * (-2.f * z * gR[0] - w * gR[1] + x * gR[2] + w * gR[3] - 2.f * z * gR[4] + y * gR[5] + x * gR[6] + y * gR[7]);
  float qd = w * gqb[0] + x * gqb[1] + y * gqb[2] + z * gqb[3];
  float iqn = 1.0f / qn;
#pragma unroll
  for (int k = 0; k < 4; k++) gq[k] += (gqb[k] - qb[k] * qd) * iqn;
}

template <bool kWriteGrad, bool kApply, int kMinBlocks>
__global__ void __launch_bounds__(kBlock, kMinBlocks) k_bwd_adam(planes P, planes Mo, planes Vo, planes Go, int64_t n,
                                                     gs_cams_arg cams, int G, int nb, int NW,
                                                     const uint32_t* __restrict__ maskw,
                                                     const int64_t* __restrict__ base, int64_t ncta,
                                                     const float* __restrict__ dL_dsend, adam_arg h) {
  __shared__ int s_cnt[kWarps * kMaxBuckets];
  __shared__ float s_gsh[48 * kBlock];  // SH gradient accumulators, [coefficient][thread]
  __shared__ int32_t s_pos[kListCap * kBlock];        // per-thread record positions (< 2^31)
  __shared__ unsigned char s_view[kListCap * kBlock];  // and their views
  // cameras in shared memory: lanes of a warp handle different views at the same time in
  // phase B, and divergent indexing of the kernel-parameter bank would serialise
  __shared__ gs_dcam s_cams[GS_MAX_VIEWS];
  for (int t = threadIdx.x; t < cams.n * (int)(sizeof(gs_dcam) / 4); t += kBlock)
    reinterpret_cast<float*>(s_cams)[t] = reinterpret_cast<const float*>(cams.c)[t];
  const int b = cams.n;
  const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  float* gsh = s_gsh + threadIdx.x;
#pragma unroll
  for (int f = 0; f < 48; f++) gsh[f * kBlock] = 0.f;
  uint32_t m[kMaxWords], u[kMaxWords];
  load_masks(maskw, n, i, NW, m);
  cta_rank_phase1(m, u, NW, nb, s_cnt);
  const bool live = i < n;
  float4 X = make_float4(0, 0, 0, 0), L4 = X, Q = X;
  if (live) {
    X = P.pos_op[i];
    L4 = P.ls[i];
    Q = P.rot[i];
  }
  float s[3] = {expf(L4.x), expf(L4.y), expf(L4.z)};
  float qn = sqrtf(Q.x * Q.x + Q.y * Q.y + Q.z * Q.z + Q.w * Q.w);
  float iq = qn > 0.f ? 1.0f / qn : 0.f;
  float qb[4] = {Q.x * iq, Q.y * iq, Q.z * iq, Q.w * iq};
  float Rq[9];
  {
    const float w = qb[0], x = qb[1], y = qb[2], z = qb[3];
    Rq[0] = 1.f - 2.f * (y * y + z * z); Rq[1] = 2.f * (x * y - w * z); Rq[2] = 2.f * (x * z + w * y);
    Rq[3] = 2.f * (x * y + w * z); Rq[4] = 1.f - 2.f * (x * x + z * z); Rq[5] = 2.f * (y * z - w * x);
    Rq[6] = 2.f * (x * z - w * y); Rq[7] = 2.f * (y * z + w * x); Rq[8] = 1.f - 2.f * (x * x + y * y);
  }
  float Sig[6];
  {
    float Mm[9];
#pragma unroll
    for (int j = 0; j < 3; j++)
#pragma unroll
      for (int k = 0; k < 3; k++) Mm[3 * j + k] = Rq[3 * j + k] * s[k];
    Sig[0] = Mm[0] * Mm[0] + Mm[1] * Mm[1] + Mm[2] * Mm[2];
    Sig[1] = Mm[0] * Mm[3] + Mm[1] * Mm[4] + Mm[2] * Mm[5];
    Sig[2] = Mm[0] * Mm[6] + Mm[1] * Mm[7] + Mm[2] * Mm[8];
    Sig[3] = Mm[3] * Mm[3] + Mm[4] * Mm[4] + Mm[5] * Mm[5];
    Sig[4] = Mm[3] * Mm[6] + Mm[4] * Mm[7] + Mm[5] * Mm[8];
    Sig[5] = Mm[6] * Mm[6] + Mm[7] * Mm[7] + Mm[8] * Mm[8];
  }
  float gpos[3] = {0, 0, 0}, gls[3] = {0, 0, 0}, gq[4] = {0, 0, 0, 0}, gop = 0.f;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  // Phase A (warp-uniform over the warp's union of buckets, v outer, d inner): each thread
  // lists the send positions of its own records in that order.  Phase B (per thread,
  // divergent): walks its own list, sums a view's destinations (ascending rank) and
  // runs the chain rule once per view -- a warp no longer steps through every view any lane
  // sees.  Lists longer than kListCap are processed in rounds.
  int n_mine = 0;
  for (int v = 0; v < b; v++)
    for (int d = 0; d < G; d++) n_mine += live && get_bit(m, d * b + v);
  __shared__ int s_rounds;
  if (threadIdx.x == 0) s_rounds = 1;
  __syncthreads();
  if (n_mine > kListCap) atomicMax(&s_rounds, (n_mine + kListCap - 1) / kListCap);
  __syncthreads();
  const int max_rounds = s_rounds;
  for (int r = 0; r < max_rounds; r++) {
    int cnt = 0;
    for (int v = 0; v < b; v++) {
      if (!view_in_union(u, v, b, G)) continue;  // warp-uniform
      for (int d = 0; d < G; d++) {
        const int k = d * b + v;
        if (!get_bit(u, k)) continue;
        const bool bit = live && get_bit(m, k);
        const unsigned bal = __ballot_sync(0xffffffffu, bit);
        if (bit) {
          const int slot = cnt - r * kListCap;
          if (slot >= 0 && slot < kListCap) {
            s_pos[slot * kBlock + threadIdx.x] =
                (int32_t)(base[(int64_t)k * ncta + blockIdx.x] + warp_prefix(s_cnt, wid, nb, k) + __popc(bal & lt));
            s_view[slot * kBlock + threadIdx.x] = (unsigned char)v;
          }
          cnt++;
        }
      }
    }
    const int nl = min(kListCap, max(0, cnt - r * kListCap));
    float g9[9];
#pragma unroll
    for (int c = 0; c < 9; c++) g9[c] = 0.f;
    for (int j = 0; j < nl; j++) {
      const int v = s_view[j * kBlock + threadIdx.x];
      const float* src = dL_dsend + (int64_t)s_pos[j * kBlock + threadIdx.x] * 9;
#pragma unroll
      for (int c = 0; c < 9; c++) g9[c] += src[c];
      if (j + 1 == nl || s_view[(j + 1) * kBlock + threadIdx.x] != v) {
        proj_bwd_view(g9, X, s, qb, qn, Rq, Sig, P.sh, n, i, s_cams[v], gpos, gls, gq, gop, gsh);
#pragma unroll
        for (int c = 0; c < 9; c++) g9[c] = 0.f;
      }
    }
  }
  if (!live) return;
  const float4 gpo = make_float4(gpos[0], gpos[1], gpos[2], gop);
  const float4 gl4 = make_float4(gls[0], gls[1], gls[2], 0.f);
  const float4 gq4 = make_float4(gq[0], gq[1], gq[2], gq[3]);
  if (kWriteGrad) {
    Go.pos_op[i] = gpo;
    Go.ls[i] = gl4;
    Go.rot[i] = gq4;
#pragma unroll
    for (int k = 0; k < 12; k++)
      Go.sh[(int64_t)k * n + i] = make_float4(gsh[(4 * k) * kBlock], gsh[(4 * k + 1) * kBlock],
                                              gsh[(4 * k + 2) * kBlock], gsh[(4 * k + 3) * kBlock]);
  }
  if (kApply) {
    adam4(P.pos_op, Mo.pos_op, Vo.pos_op, i, gpo, 0, 0, 0, 3, h);
    adam4(P.ls, Mo.ls, Vo.ls, i, gl4, 4, 4, 4, -1, h);
    adam4(P.rot, Mo.rot, Vo.rot, i, gq4, 5, 5, 5, 5, h);
    adam4(P.sh, Mo.sh, Vo.sh, i, make_float4(gsh[0], gsh[kBlock], gsh[2 * kBlock], gsh[3 * kBlock]), 1, 1, 1, 2, h);
#pragma unroll
    for (int k = 1; k < 12; k++)
      adam4(P.sh, Mo.sh, Vo.sh, (int64_t)k * n + i,
            make_float4(gsh[(4 * k) * kBlock], gsh[(4 * k + 1) * kBlock], gsh[(4 * k + 2) * kBlock],
                        gsh[(4 * k + 3) * kBlock]),
            2, 2, 2, 2, h);
  }
}

// Adam from a stored gradient (GS_ADAM_APPLY without GS_ADAM_GRAD): elementwise over planes.
__global__ void __launch_bounds__(256) k_adam_apply(planes P, planes Mo, planes Vo, planes Go, int64_t n,
                                                    adam_arg h) {
  // grid (ceil(n/256), 15): blockIdx.y = float4 plane (pos_op, log_scale, rot, sh 0..11)
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int plane = blockIdx.y;
  if (plane == 0) adam4(P.pos_op, Mo.pos_op, Vo.pos_op, i, Go.pos_op[i], 0, 0, 0, 3, h);
  else if (plane == 1) adam4(P.ls, Mo.ls, Vo.ls, i, Go.ls[i], 4, 4, 4, -1, h);
  else if (plane == 2) adam4(P.rot, Mo.rot, Vo.rot, i, Go.rot[i], 5, 5, 5, 5, h);
  else {
    const int64_t k = plane - 3, idx = k * n + i;
    if (k == 0) adam4(P.sh, Mo.sh, Vo.sh, idx, Go.sh[idx], 1, 1, 1, 2, h);
    else adam4(P.sh, Mo.sh, Vo.sh, idx, Go.sh[idx], 2, 2, 2, 2, h);
  }
}

}  // namespace

extern "C" gs_status gs_adam_step(gs_ctx* c, gs_params* p, gs_params* m, gs_params* v, gs_params* g,
                                  const gs_camera* cams_h, int n_views, const int64_t* dp_h,
                                  const float* dL_dsend, const void* bwd_index, const gs_adam_hparams* hp,
                                  int flags, void* stream) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, p && hp, "null argument");
  GS_REQUIRE(c, flags & (GS_ADAM_GRAD | GS_ADAM_APPLY), "flags select nothing");
  const bool grad = flags & GS_ADAM_GRAD, apply = flags & GS_ADAM_APPLY, wgrad = flags & GS_ADAM_WRITE_GRAD;
  GS_REQUIRE(c, !apply || (m && v && m->n == p->n && v->n == p->n), "m/v missing or mis-sized");
  GS_REQUIRE(c, !g || g->n == p->n, "g mis-sized (%lld rows for %lld Gaussians)", (long long)(g ? g->n : 0),
             (long long)p->n);
  GS_REQUIRE(c, g || (grad && !wgrad), "g required (apply-only or WRITE_GRAD)");
  GS_REQUIRE(c, hp->batch >= 1 && hp->step >= 1, "batch and step must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  if (p->n == 0) return GS_OK;
  adam_arg h;
  {
    // Eq. (1) lambda' = lambda sqrt(b); Eq. (2) beta' = beta^b; bias correction in double
    const double b = hp->batch, b1 = pow((double)hp->beta1, b), b2 = pow((double)hp->beta2, b);
    const double bc1 = 1.0 - pow(b1, (double)hp->step), bc2 = 1.0 - pow(b2, (double)hp->step);
    for (int k = 0; k < 6; k++) h.step[k] = (float)(hp->lr[k] * sqrt(b) / bc1);
    h.b1 = (float)b1;
    h.b2 = (float)b2;
    h.omb1 = (float)(1.0 - b1);
    h.omb2 = (float)(1.0 - b2);
    h.inv_sqrt_bc2 = (float)(1.0 / sqrt(bc2));
    h.eps = hp->eps;
  }
  planes P = mk(p), Mo = m ? mk(m) : planes{}, Vo = v ? mk(v) : planes{}, Go = g ? mk(g) : planes{};
  if (!grad) {
    ++c->launches;
    k_adam_apply<<<dim3((unsigned)((p->n + 255) / 256), 15), 256, 0, st>>>(P, Mo, Vo, Go, p->n, h);
    GS_LAUNCH_CHECK(c, "adam_apply");
    return GS_OK;
  }
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, bwd_index != nullptr, "null bwd_index");
  const int G = c->world, nb = n_views * G;
  GS_REQUIRE(c, nb <= kMaxBuckets, "n_views * world too large");
  gs_index_layout L = index_layout(p->n, n_views, G);
  const uint32_t* maskw = (const uint32_t*)bwd_index;
  const int64_t* base = (const int64_t*)((const char*)bwd_index + L.base_off);
  gs_cams_arg cams = make_cams(cams_h, n_views);
  const unsigned grid = (unsigned)L.ncta;
  if (!wgrad && !apply) return gs_fail(c, GS_EINVAL, "GS_ADAM_GRAD alone computes nothing observable");
  if (apply && g) {
    // split path (default when a gradient buffer is given): the transformation backward writes
    // the parameter gradient, then an elementwise Adam pass streams p, m, v, g at full
    // occupancy; the fused kernel's register footprint caps its memory parallelism
    ++c->launches;
    // 5 resident CTAs per SM: C2 4.97 -> 4.83 ms against 4 (126 registers; 1: 188 registers,
    // 8 warps/SM: 6.7 ms; 6: 4.94 ms)
    k_bwd_adam<true, false, 5><<<grid, kBlock, 0, st>>>(P, Mo, Vo, Go, p->n, cams, G, nb, L.NW, maskw, base, L.ncta,
                                                        dL_dsend, h);
    ++c->launches;
    k_adam_apply<<<dim3((unsigned)((p->n + 255) / 256), 15), 256, 0, st>>>(P, Mo, Vo, Go, p->n, h);
    GS_LAUNCH_CHECK(c, "bwd + adam_apply");
    return GS_OK;
  }
  ++c->launches;
  if (!apply)  // parity mode: the parameter gradient only
    k_bwd_adam<true, false, 5><<<grid, kBlock, 0, st>>>(P, Mo, Vo, Go, p->n, cams, G, nb, L.NW, maskw, base, L.ncta,
                                                        dL_dsend, h);
  else  // no gradient buffer: backward and Adam fused in registers (tests/test_gpu_multiview.py)
    k_bwd_adam<false, true, 1><<<grid, kBlock, 0, st>>>(P, Mo, Vo, Go, p->n, cams, G, nb, L.NW, maskw, base, L.ncta,
                                                        dL_dsend, h);
  GS_LAUNCH_CHECK(c, "bwd_adam");
  return GS_OK;
}
