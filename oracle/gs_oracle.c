/* gs_oracle.c -- the CPU oracle (TEST INFRASTRUCTURE; see gs_oracle.h header comment).
 *
 * Each function follows the definition it cites, written out in the paper's order and
 * notation, with no blocking, fusion or reordering: P:103 (transformation)
 * (compositing "in increasing depth ... until a threshold opacity"), P:114 (L1 loss),
 * P:190 (sparse exchange), P:215-226 (Algorithm 1), P:248-253 (Eq. 1-2), P:497 (backward).
 * The concrete formulas the paper defers to the 3DGS reference are the ones
 * SPEC.md states plus the readings R1-R11.
 *
 * Compile: gcc -O2 -fno-fast-math -ffp-contract=off -fPIC -shared (x86-64 SSE, no x87).
 */
#define _GNU_SOURCE /* qsort_r: the O11 comparator takes the record arrays as an argument */
#include "gs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ constants */
#define ALPHA_CAP 0.99
#define ALPHA_MIN (1.0 / 255.0)
#define T_STOP 1e-4
#define NEAR_Z 0.01f   /* S:179 near plane */
#define DILATE 0.3f    /* S:148 +0.3 I       */

/* Real SH basis constants, degree 0..3 (3DGS convention [ext], SURVEY §8(c) O9 list). */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* ------------------------------------------------------------------ R10 exp */
static float pow2i_f32(int k) { /* exact 2^k for k in [-126, 127] */
  union { unsigned u; float f; } v;
  v.u = (unsigned)(k + 127) << 23;
  return v.f;
}

float orc_exp_rn(float x) {
  /* R10: clamp, Cody-Waite reduction with ln2 = 0.693359375 - 2.12194440e-4, Cephes
   * degree-6 polynomial, every operation a separately rounded fp32 operation. */
  if (x < -87.0f) x = -87.0f;
  if (x > 88.0f) x = 88.0f;
  float k = floorf(x * 1.44269504088896341f + 0.5f);
  float r = (x - k * 0.693359375f) - k * (-2.12194440e-4f);
  float z = r * r;
  float p = 1.9875691500e-4f;
  p = p * r + 1.3981999507e-3f;
  p = p * r + 8.3334519073e-3f;
  p = p * r + 4.1665795894e-2f;
  p = p * r + 1.6666665459e-1f;
  p = p * r + 5.0000001201e-1f;
  p = ((p * z) + r) + 1.0f;
  return p * pow2i_f32((int)k);
}

/* ------------------------------------------------------------------ O1-O8 (fp32) */
static int floordiv16(int v) { return (v >= 0) ? v / 16 : -((-v + 15) / 16); }

static float clamp24(float v) {
  const float L = 16777216.0f;
  if (v > L) return L;
  if (v < -L) return -L;
  return v;
}

void orc_membership_f32(int64_t n, const float* pos, const float* log_scale, const float* rot,
                        const orc_camera* cam, int8_t* vis, float* mx, float* my, float* depth,
                        float* cov, int32_t* radius, int32_t* rect) {
  const int Wt = (cam->width + 15) / 16, Ht = (cam->height + 15) / 16;
  for (int64_t i = 0; i < n; i++) {
    vis[i] = 0;
    mx[i] = my[i] = depth[i] = 0.0f;
    cov[3 * i] = cov[3 * i + 1] = cov[3 * i + 2] = 0.0f;
    radius[i] = 0;
    rect[4 * i] = rect[4 * i + 2] = 0;
    rect[4 * i + 1] = rect[4 * i + 3] = -1;
    /* O1 activations: s = exp_rn(log s); qbar = q / sqrt(n2), n2 = ((ww+xx)+yy)+zz */
    float s[3];
    for (int k = 0; k < 3; k++) s[k] = orc_exp_rn(log_scale[3 * i + k]);
    const float* q = rot + 4 * i;
    float n2 = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
    if (!(n2 > 0.0f)) continue;
    float qn = sqrtf(n2);
    float w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
    /* O2: rotation matrix of qbar, M = R diag(s), Sigma = M M^T */
    float Rq[9];
    Rq[0] = 1.0f - 2.0f * (y * y + z * z);
    Rq[1] = 2.0f * (x * y - w * z);
    Rq[2] = 2.0f * (x * z + w * y);
    Rq[3] = 2.0f * (x * y + w * z);
    Rq[4] = 1.0f - 2.0f * (x * x + z * z);
    Rq[5] = 2.0f * (y * z - w * x);
    Rq[6] = 2.0f * (x * z - w * y);
    Rq[7] = 2.0f * (y * z + w * x);
    Rq[8] = 1.0f - 2.0f * (x * x + y * y);
    float M[9];
    for (int j = 0; j < 3; j++)
      for (int k = 0; k < 3; k++) M[3 * j + k] = Rq[3 * j + k] * s[k];
    float S[9];
    for (int j = 0; j < 3; j++)
      for (int k = j; k < 3; k++) {
        float v = (M[3 * j] * M[3 * k] + M[3 * j + 1] * M[3 * k + 1]) + M[3 * j + 2] * M[3 * k + 2];
        S[3 * j + k] = v;
        S[3 * k + j] = v;
      }
    /* O3: camera space p = R x + t; near plane */
    const float* X = pos + 3 * i;
    const float* W = cam->R;
    float p[3];
    for (int j = 0; j < 3; j++) p[j] = ((W[3 * j] * X[0] + W[3 * j + 1] * X[1]) + W[3 * j + 2] * X[2]) + cam->t[j];
    if (!(p[2] > NEAR_Z)) continue;
    /* O4: mean2d */
    float fxpx = cam->fx * p[0], fypy = cam->fy * p[1];
    float m_x = fxpx / p[2] + cam->cx;
    float m_y = fypy / p[2] + cam->cy;
    /* O5: EWA Sigma' = T Sigma T^T + 0.3 I with T = J W (no FOV clamp, R5) */
    float pz2 = p[2] * p[2];
    float j00 = cam->fx / p[2], j02 = -(fxpx / pz2);
    float j11 = cam->fy / p[2], j12 = -(fypy / pz2);
    float T[6];
    for (int k = 0; k < 3; k++) {
      T[k] = j00 * W[k] + j02 * W[6 + k];
      T[3 + k] = j11 * W[3 + k] + j12 * W[6 + k];
    }
    float U[6];
    for (int r = 0; r < 2; r++)
      for (int k = 0; k < 3; k++)
        U[3 * r + k] = (T[3 * r] * S[k] + T[3 * r + 1] * S[3 + k]) + T[3 * r + 2] * S[6 + k];
    float a = ((U[0] * T[0] + U[1] * T[1]) + U[2] * T[2]) + DILATE;
    float b = (U[0] * T[3] + U[1] * T[4]) + U[2] * T[5];
    float c = ((U[3] * T[3] + U[4] * T[4]) + U[5] * T[5]) + DILATE;
    /* O6: det > 0 required */
    float det = a * c - b * b;
    if (!(det > 0.0f)) continue;
    /* O7: radius = ceil(3 sqrt(lambda_max)), guard max(0, .) (R4) */
    float mid = 0.5f * (a + c);
    float disc = mid * mid - det;
    if (disc < 0.0f) disc = 0.0f;
    float lam = mid + sqrtf(disc);
    float r = ceilf(3.0f * sqrtf(lam));
    /* O8: pixel-granular rectangle (R1, R2), frustum cull when empty */
    int c0 = (int)ceilf(clamp24(m_x - r)), c1 = (int)floorf(clamp24(m_x + r));
    int w0 = (int)ceilf(clamp24(m_y - r)), w1 = (int)floorf(clamp24(m_y + r));
    int tx0 = floordiv16(c0), tx1 = floordiv16(c1), ty0 = floordiv16(w0), ty1 = floordiv16(w1);
    if (tx0 < 0) tx0 = 0;
    if (ty0 < 0) ty0 = 0;
    if (tx1 > Wt - 1) tx1 = Wt - 1;
    if (ty1 > Ht - 1) ty1 = Ht - 1;
    if (tx0 > tx1 || ty0 > ty1) continue;
    vis[i] = 1;
    mx[i] = m_x;
    my[i] = m_y;
    depth[i] = p[2];
    cov[3 * i] = a;
    cov[3 * i + 1] = b;
    cov[3 * i + 2] = c;
    radius[i] = (int32_t)(r < 16777216.0f ? r : 16777216.0f);
    rect[4 * i] = tx0;
    rect[4 * i + 1] = tx1;
    rect[4 * i + 2] = ty0;
    rect[4 * i + 3] = ty1;
  }
}

/* ------------------------------------------------------------------ O9 SH basis (fp64) */
static void sh_basis(const double d[3], double Y[16]) {
  double x = d[0], y = d[1], z = d[2];
  Y[0] = SH_C0;
  Y[1] = -SH_C1 * y;
  Y[2] = SH_C1 * z;
  Y[3] = -SH_C1 * x;
  Y[4] = SH_C2[0] * x * y;
  Y[5] = SH_C2[1] * y * z;
  Y[6] = SH_C2[2] * (2 * z * z - x * x - y * y);
  Y[7] = SH_C2[3] * x * z;
  Y[8] = SH_C2[4] * (x * x - y * y);
  Y[9] = SH_C3[0] * y * (3 * x * x - y * y);
  Y[10] = SH_C3[1] * x * y * z;
  Y[11] = SH_C3[2] * y * (4 * z * z - x * x - y * y);
  Y[12] = SH_C3[3] * z * (2 * z * z - 3 * x * x - 3 * y * y);
  Y[13] = SH_C3[4] * x * (4 * z * z - x * x - y * y);
  Y[14] = SH_C3[5] * z * (x * x - y * y);
  Y[15] = SH_C3[6] * x * (x * x - 3 * y * y);
}

/* dY_k/d(x,y,z) of the polynomial basis above (dir treated as free; the unit-norm
 * constraint is applied by the (I - d d^T)/|x-c| projection in O16).            */
static void sh_basis_grad(const double d[3], double dY[16][3]) {
  double x = d[0], y = d[1], z = d[2];
  memset(dY, 0, sizeof(double) * 48);
  dY[1][1] = -SH_C1;
  dY[2][2] = SH_C1;
  dY[3][0] = -SH_C1;
  dY[4][0] = SH_C2[0] * y; dY[4][1] = SH_C2[0] * x;
  dY[5][1] = SH_C2[1] * z; dY[5][2] = SH_C2[1] * y;
  dY[6][0] = SH_C2[2] * (-2 * x); dY[6][1] = SH_C2[2] * (-2 * y); dY[6][2] = SH_C2[2] * (4 * z);
  dY[7][0] = SH_C2[3] * z; dY[7][2] = SH_C2[3] * x;
  dY[8][0] = SH_C2[4] * (2 * x); dY[8][1] = SH_C2[4] * (-2 * y);
  dY[9][0] = SH_C3[0] * 6 * x * y; dY[9][1] = SH_C3[0] * (3 * x * x - 3 * y * y);
  dY[10][0] = SH_C3[1] * y * z; dY[10][1] = SH_C3[1] * x * z; dY[10][2] = SH_C3[1] * x * y;
  dY[11][0] = SH_C3[2] * (-2 * x * y);
  dY[11][1] = SH_C3[2] * (4 * z * z - x * x - 3 * y * y);
  dY[11][2] = SH_C3[2] * (8 * y * z);
  dY[12][0] = SH_C3[3] * (-6 * x * z);
  dY[12][1] = SH_C3[3] * (-6 * y * z);
  dY[12][2] = SH_C3[3] * (6 * z * z - 3 * x * x - 3 * y * y);
  dY[13][0] = SH_C3[4] * (4 * z * z - 3 * x * x - y * y);
  dY[13][1] = SH_C3[4] * (-2 * x * y);
  dY[13][2] = SH_C3[4] * (8 * x * z);
  dY[14][0] = SH_C3[5] * 2 * x * z; dY[14][1] = SH_C3[5] * (-2 * y * z);
  dY[14][2] = SH_C3[5] * (x * x - y * y);
  dY[15][0] = SH_C3[6] * (3 * x * x - 3 * y * y); dY[15][1] = SH_C3[6] * (-6 * x * y);
}

/* ------------------------------------------------------------------ fp64 forward state */
typedef struct {
  int vis;
  double s[3], qn, qb[4], Rq[9], M[9], Sig[9];
  double p[3], m[2], J[6], T[6], a, b, c, det, A, B, C, o;
  double campos[3], dvec[3], dist, dir[3], Y[16], rgb[3];
  int clamp;
  double radius;
  int rect[4];
} fwd64;

static void camera_centre(const orc_camera* cam, double c[3]) {
  for (int k = 0; k < 3; k++) c[k] = -((double)cam->R[k] * cam->t[0] + (double)cam->R[3 + k] * cam->t[1] +
                                      (double)cam->R[6 + k] * cam->t[2]);
}

static void forward64(const double* X, const double* ls, const double* q, double ol, const double* sh,
                      const orc_camera* cam, fwd64* f) {
  memset(f, 0, sizeof(*f));
  const int Wt = (cam->width + 15) / 16, Ht = (cam->height + 15) / 16;
  f->o = 1.0 / (1.0 + exp(-(double)ol));
  /* O1 opacity, O9 colour (computed for every Gaussian) from view direction (x - c_v)/|x - c_v| */
  camera_centre(cam, f->campos);
  for (int k = 0; k < 3; k++) f->dvec[k] = (double)X[k] - f->campos[k];
  f->dist = sqrt(f->dvec[0] * f->dvec[0] + f->dvec[1] * f->dvec[1] + f->dvec[2] * f->dvec[2]);
  for (int k = 0; k < 3; k++) f->dir[k] = f->dvec[k] / f->dist;
  sh_basis(f->dir, f->Y);
  for (int ch = 0; ch < 3; ch++) {
    double v = 0.5;
    for (int k = 0; k < 16; k++) v += f->Y[k] * sh[3 * k + ch];
    if (v < 0) {
      f->clamp |= 1 << ch;
      v = 0;
    }
    f->rgb[ch] = v;
  }
  for (int k = 0; k < 3; k++) f->s[k] = exp((double)ls[k]);
  double n2 = (double)q[0] * q[0] + (double)q[1] * q[1] + (double)q[2] * q[2] + (double)q[3] * q[3];
  if (!(n2 > 0)) return;
  f->qn = sqrt(n2);
  for (int k = 0; k < 4; k++) f->qb[k] = q[k] / f->qn;
  double w = f->qb[0], x = f->qb[1], y = f->qb[2], z = f->qb[3];
  double* R = f->Rq;
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
  for (int j = 0; j < 3; j++)
    for (int k = 0; k < 3; k++) f->M[3 * j + k] = R[3 * j + k] * f->s[k];
  for (int j = 0; j < 3; j++)
    for (int k = 0; k < 3; k++)
      f->Sig[3 * j + k] = f->M[3 * j] * f->M[3 * k] + f->M[3 * j + 1] * f->M[3 * k + 1] + f->M[3 * j + 2] * f->M[3 * k + 2];
  const float* Wc = cam->R;
  for (int j = 0; j < 3; j++)
    f->p[j] = (double)Wc[3 * j] * X[0] + (double)Wc[3 * j + 1] * X[1] + (double)Wc[3 * j + 2] * X[2] + cam->t[j];
  if (!(f->p[2] > 0.01)) return;
  double fx = cam->fx, fy = cam->fy, pz = f->p[2];
  f->m[0] = fx * f->p[0] / pz + cam->cx;
  f->m[1] = fy * f->p[1] / pz + cam->cy;
  f->J[0] = fx / pz; f->J[1] = 0; f->J[2] = -fx * f->p[0] / (pz * pz);
  f->J[3] = 0; f->J[4] = fy / pz; f->J[5] = -fy * f->p[1] / (pz * pz);
  for (int r = 0; r < 2; r++)
    for (int k = 0; k < 3; k++)
      f->T[3 * r + k] = f->J[3 * r] * Wc[k] + f->J[3 * r + 1] * Wc[3 + k] + f->J[3 * r + 2] * Wc[6 + k];
  double Sp[4] = {0, 0, 0, 0};
  for (int r = 0; r < 2; r++)
    for (int cc = 0; cc < 2; cc++)
      for (int j = 0; j < 3; j++)
        for (int k = 0; k < 3; k++) Sp[2 * r + cc] += f->T[3 * r + j] * f->Sig[3 * j + k] * f->T[3 * cc + k];
  f->a = Sp[0] + 0.3;
  f->b = Sp[1];
  f->c = Sp[3] + 0.3;
  f->det = f->a * f->c - f->b * f->b;
  if (!(f->det > 0)) return;
  f->A = f->c / f->det;
  f->B = -f->b / f->det;
  f->C = f->a / f->det;
  double mid = 0.5 * (f->a + f->c), disc = mid * mid - f->det;
  if (disc < 0) disc = 0;
  f->radius = ceil(3.0 * sqrt(mid + sqrt(disc)));
  double c0 = ceil(f->m[0] - f->radius), c1 = floor(f->m[0] + f->radius);
  double w0 = ceil(f->m[1] - f->radius), w1 = floor(f->m[1] + f->radius);
  const double L = 16777216.0;
  c0 = fmax(-L, fmin(L, c0)); c1 = fmax(-L, fmin(L, c1));
  w0 = fmax(-L, fmin(L, w0)); w1 = fmax(-L, fmin(L, w1));
  int tx0 = floordiv16((int)c0), tx1 = floordiv16((int)c1), ty0 = floordiv16((int)w0), ty1 = floordiv16((int)w1);
  if (tx0 < 0) tx0 = 0;
  if (ty0 < 0) ty0 = 0;
  if (tx1 > Wt - 1) tx1 = Wt - 1;
  if (ty1 > Ht - 1) ty1 = Ht - 1;
  if (tx0 > tx1 || ty0 > ty1) return;
  f->rect[0] = tx0; f->rect[1] = tx1; f->rect[2] = ty0; f->rect[3] = ty1;
  f->vis = 1;
}

void orc_project_f64(int64_t n, const double* pos, const double* log_scale, const double* rot,
                     const double* opac_logit, const double* sh, const orc_camera* cam,
                     double* out, int32_t* rect) {
  for (int64_t i = 0; i < n; i++) {
    fwd64 f;
    forward64(pos + 3 * i, log_scale + 3 * i, rot + 4 * i, opac_logit[i], sh + 48 * i, cam, &f);
    double* o = out + 16 * i;
    double v[16] = {(double)f.vis, f.m[0], f.m[1], f.p[2], f.a, f.b, f.c, f.A, f.B, f.C, f.o,
                    f.rgb[0], f.rgb[1], f.rgb[2], (double)f.clamp, f.radius};
    memcpy(o, v, sizeof(v));
    for (int k = 0; k < 4; k++) rect[4 * i + k] = f.vis ? f.rect[k] : (k % 2 ? -1 : 0);
  }
}

/* ------------------------------------------------------------------ O10 exchange sets */
void orc_exchange_sets(int64_t n, const int8_t* vis, const int32_t* rect, int32_t view,
                       int32_t Wt, int32_t Ht, int32_t G, const int64_t* DP, uint32_t* mask) {
  for (int64_t i = 0; i < n; i++) {
    mask[i] = 0;
    if (!vis[i]) continue;
    for (int ty = rect[4 * i + 2]; ty <= rect[4 * i + 3]; ty++)
      for (int tx = rect[4 * i]; tx <= rect[4 * i + 1]; tx++) {
        int64_t beta = (int64_t)view * Wt * Ht + (int64_t)ty * Wt + tx;
        for (int g = 0; g < G; g++)
          if (DP[g] <= beta && beta < DP[g + 1]) mask[i] |= 1u << g;
      }
  }
}

/* ------------------------------------------------------------------ O11 tile lists */
typedef struct {
  const double* f;
  const int64_t* i;
} sort_arg_t;
/* reentrant (no static state), so concurrent calls over disjoint block ranges are safe */
static int cmp_depth_gid(const void* pa, const void* pb, void* arg) {
  const sort_arg_t* s = (const sort_arg_t*)arg;
  int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  double da = s->f[10 * a + 2], db = s->f[10 * b + 2];
  if (da < db) return -1;
  if (da > db) return 1;
  int64_t ga = s->i[6 * a], gb = s->i[6 * b];
  return (ga < gb) ? -1 : (ga > gb) ? 1 : 0;
}

void orc_tile_lists(int64_t n_rec, const double* rec_f, const int64_t* rec_i, int64_t b0,
                    int64_t b1, int32_t Wt, int32_t Ht, int64_t* offsets, int64_t* entries) {
  int64_t nb = b1 - b0, per_view = (int64_t)Wt * Ht;
  int64_t* cnt = (int64_t*)calloc((size_t)nb + 1, sizeof(int64_t));
  /* membership: record (gid, v) is in block beta iff beta's view is v and beta's tile is
   * inside the record's rectangle (R2) */
  for (int64_t j = 0; j < n_rec; j++) {
    const int64_t* ri = rec_i + 6 * j;
    for (int64_t ty = ri[4]; ty <= ri[5]; ty++)
      for (int64_t tx = ri[2]; tx <= ri[3]; tx++) {
        int64_t beta = ri[1] * per_view + ty * Wt + tx;
        if (beta >= b0 && beta < b1) cnt[beta - b0]++;
      }
  }
  offsets[0] = 0;
  for (int64_t k = 0; k < nb; k++) offsets[k + 1] = offsets[k] + cnt[k];
  if (entries) {
    memset(cnt, 0, sizeof(int64_t) * (size_t)nb);
    for (int64_t j = 0; j < n_rec; j++) {
      const int64_t* ri = rec_i + 6 * j;
      for (int64_t ty = ri[4]; ty <= ri[5]; ty++)
        for (int64_t tx = ri[2]; tx <= ri[3]; tx++) {
          int64_t beta = ri[1] * per_view + ty * Wt + tx;
          if (beta >= b0 && beta < b1) entries[offsets[beta - b0] + cnt[beta - b0]++] = j;
        }
    }
    sort_arg_t sa = {rec_f, rec_i};
    for (int64_t k = 0; k < nb; k++)
      qsort_r(entries + offsets[k], (size_t)(offsets[k + 1] - offsets[k]), sizeof(int64_t), cmp_depth_gid, &sa);
  }
  free(cnt);
}

/* ------------------------------------------------------------------ O12/O13 forward */
static double sgn(double v) { return (v > 0) - (v < 0); }

/* Decision margins (DESIGN.md §2 R16, "discontinuities").  O12 takes two threshold
 * decisions per evaluated entry (alpha < 1/255: skip; T' < 1e-4: stop, "until a
 * threshold opacity has been reached").  An fp32 renderer may take either side of a decision
 * whose exact value lies within its own rounding error of the threshold; both outcomes are
 * then correct results of the method.  The oracle marks such a decision "flagged" and
 * enumerates both outcomes (orc_render_fwd paths), so a pixel is checked against every
 * result an fp32 evaluation may legitimately produce, never excluded.  The error model is
 * the first-order bound of the renderer's fp32 arithmetic as the boundary defines it
 * (include/gs.h: the conic's Cholesky factor rounded to nearest, u and w evaluated from a
 * reference point within (3.5, 7.5) px of the pixel, four rows per thread 4 px apart), with
 * u_r = 2^-24 per operation; DESIGN.md §2 R16 has the term-by-term derivation:
 *   e_q = m->cond_eps (13 |power| + 7 |u| l11 + 51 |u l21| + 39 |w| l22), cond_eps = u_r,
 *         -2 power = u^2 + w^2, u = l11 dx + l21 dy, w = l22 dy (conic = L L^T): the bound on
 *         the error of the renderer's exponent, in ln(alpha) units;
 *   skip:  flagged if |ln(255 alpha)| < m->alpha_eps + e_q + u_r |ln(255 o)| (the rounding of
 *          the threshold log2(255 o) to fp32; alpha_eps covers the fp32 opacity);
 *   stop:  flagged if |1e4 T' - 1| < m->t_eps + e_T, e_T the accumulated bound on the relative
 *          error of the fp32 product T = prod (1 - alpha_k): per composited entry
 *          e_alpha alpha / (1 - alpha) + 3 u_r, e_alpha = m->alpha_abs + e_q the relative
 *          error of an fp32 alpha = o 2^-q (alpha_abs: ex2.approx, measured on the device by
 *          gs_selftest_ex2, the opacity and the product). */
#define U_R (1.0 / 16777216.0)
typedef struct {
  double alpha_eps, t_eps, cond_eps, alpha_abs;
} orc_margins_t;

typedef struct { /* a composited entry of one pixel, front to back */
  int64_t idx;
  double T, alpha, G, dx, dy;
  int capped;
} comp_t;

/* O12 for one pixel (px, py) over the list L[0..nL), taking the alternative outcome of the
 * f-th flagged decision met (in list order) when bit f of flips is set (f < 64).  Writes the
 * colour before background C, T, n_last, counts (E_f, E_fc, E_fs, E_stop) and, if comp is
 * not NULL, the composited entries.  Returns the number of flagged decisions met; *bits
 * gets 1 (a skip decision flagged), 2 (a stop decision flagged), 4 (power > 0 met). */
static int walk_pixel(const double* rec_f, const int64_t* L, int64_t nL, double px, double py,
                      const orc_margins_t* m, uint64_t flips, double C[3], double* Tout, int32_t* nlast,
                      int64_t cnt[4], comp_t* comp, int64_t* ncomp, int* bits) {
  double T = 1.0, terr = 0.0;
  int nf = 0;
  int64_t nc = 0;
  C[0] = C[1] = C[2] = 0.0;
  *nlast = 0;
  *bits = 0;
  cnt[0] = cnt[1] = cnt[2] = cnt[3] = 0;
  for (int64_t k = 0; k < nL; k++) {
    const double* r = rec_f + 10 * L[k];
    double dx = r[0] - px, dy = r[1] - py;
    double power = -0.5 * (r[3] * dx * dx + r[5] * dy * dy) - r[4] * dx * dy;
    cnt[0]++;
    if (power > 0) { *bits |= 4; cnt[2]++; continue; }
    double G = exp(power), raw = r[6] * G, alpha = raw;
    int capped = 0;
    if (alpha > ALPHA_CAP) { alpha = ALPHA_CAP; capped = 1; }
    /* first-order bound of the renderer's fp32 exponent error, in ln(alpha) units (see
     * orc_margins_t) */
    double l11 = sqrt(r[3]), l21 = r[4] / l11, l22 = sqrt(fmax(r[5] - l21 * l21, 0.0));
    double u = l11 * dx + l21 * dy, w = l22 * dy;
    double eq = m->cond_eps * (13.0 * fabs(power) + 7.0 * fabs(u) * l11 + 51.0 * fabs(u * l21) + 39.0 * fabs(w) * l22);
    /* skip decision: alpha < 1/255, taken by the renderer as q > qmax with qmax = log2(255 o)
     * rounded to fp32 (u_r |qmax| ln 2 in ln(alpha) units) */
    int skip = alpha < ALPHA_MIN;
    if (alpha > 0 && fabs(log(alpha * 255.0)) < m->alpha_eps + eq + U_R * fabs(log(255.0 * r[6]))) {
      *bits |= 1;
      if (nf < 64 && ((flips >> nf) & 1)) skip = !skip;
      nf++;
    }
    if (skip) { cnt[2]++; continue; }
    double ea = m->alpha_abs + eq; /* relative error bound of the fp32 alpha */
    if (capped && raw * (1.0 - ea) >= ALPHA_CAP) ea = 1.1e-8; /* both sides clamp: 0.99f vs 0.99 */
    double et = terr + ea * alpha / (1.0 - alpha) + 3.0 * U_R;
    /* stop decision: T' < 1e-4 (R3: before compositing) */
    double Tn = T * (1.0 - alpha);
    int stop = Tn < T_STOP;
    if (fabs(Tn * 1e4 - 1.0) < m->t_eps + et) {
      *bits |= 2;
      if (nf < 64 && ((flips >> nf) & 1)) stop = !stop;
      nf++;
    }
    if (stop) { cnt[3] = 1; break; }
    if (comp) {
      comp[nc].idx = L[k]; comp[nc].T = T; comp[nc].alpha = alpha; comp[nc].G = G;
      comp[nc].dx = dx; comp[nc].dy = dy; comp[nc].capped = capped;
    }
    nc++;
    for (int ch = 0; ch < 3; ch++) C[ch] += alpha * T * r[7 + ch];
    T = Tn;
    terr = et;
    *nlast = (int32_t)(k + 1);
    cnt[1]++;
  }
  *Tout = T;
  if (ncomp) *ncomp = nc;
  return nf;
}

void orc_render_fwd(int64_t n_rec, const double* rec_f, const int64_t* offsets,
                    const int64_t* entries, int64_t b0, int64_t b1, int32_t W, int32_t H,
                    const double* bg, const uint8_t* gt, int32_t b_total, const double* margins,
                    double* out_c, double* out_T, int32_t* out_nlast, int32_t* flags,
                    int64_t* counts, int64_t* work, double* dl_dc, double* loss,
                    int32_t max_paths, int32_t* n_paths, uint64_t* path_flips, double* path_c,
                    double* path_T, int32_t* path_nl, int64_t* path_counts) {
  (void)n_rec;
  const orc_margins_t m = {margins[0], margins[1], margins[2], margins[3]};
  const int Wt = (W + 15) / 16, Ht = (H + 15) / 16;
  const int64_t per_view = (int64_t)Wt * Ht;
  const double norm = 1.0 / (3.0 * (double)H * (double)W * (double)b_total);
  const int P = max_paths > 0 ? max_paths : 0;
  double lsum = 0;
  uint64_t* queue = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(P > 0 ? P : 1));
  int* qnf = (int*)malloc(sizeof(int) * (size_t)(P > 0 ? P : 1));
  for (int64_t beta = b0; beta < b1; beta++) {
    int64_t kb = beta - b0, v = beta / per_view, loc = beta % per_view;
    int tx = (int)(loc % Wt), ty = (int)(loc / Wt);
    const int64_t* L = entries + offsets[kb];
    int64_t nL = offsets[kb + 1] - offsets[kb];
    work[kb] = 0;
    for (int p = 0; p < 256; p++) {
      int px = tx * 16 + p % 16, py = ty * 16 + p / 16;
      int64_t o = kb * 256 + p;
      if (P > 0) n_paths[o] = 0;
      if (px >= W || py >= H) {
        if (P > 0) { /* not rendered: the one outcome is the untouched pixel */
          int64_t po = o * P;
          n_paths[o] = 1;
          path_flips[po] = 0;
          path_c[3 * po] = path_c[3 * po + 1] = path_c[3 * po + 2] = 0;
          path_T[po] = 1;
          path_nl[po] = 0;
          for (int k = 0; k < 4; k++) path_counts[4 * po + k] = 0;
        }
        out_c[3 * o] = out_c[3 * o + 1] = out_c[3 * o + 2] = 0;
        out_T[o] = 1;
        out_nlast[o] = 0;
        flags[o] = 0;
        for (int k = 0; k < 4; k++) counts[4 * o + k] = 0;
        if (dl_dc) dl_dc[3 * o] = dl_dc[3 * o + 1] = dl_dc[3 * o + 2] = 0;
        continue;
      }
      double C[3], T;
      int32_t nlast;
      int bits;
      int nf = walk_pixel(rec_f, L, nL, px, py, &m, 0, C, &T, &nlast, counts + 4 * o, NULL, NULL, &bits);
      int flag = bits;
      for (int ch = 0; ch < 3; ch++) C[ch] += T * bg[ch];
      for (int ch = 0; ch < 3; ch++) out_c[3 * o + ch] = C[ch];
      out_T[o] = T;
      out_nlast[o] = nlast;
      if (gt) {
        const uint8_t* g = gt + (((int64_t)v * H + py) * W + px) * 3;
        for (int ch = 0; ch < 3; ch++) {
          double d = C[ch] - g[ch] / 255.0;
          lsum += fabs(d) * norm;
          if (dl_dc) dl_dc[3 * o + ch] = sgn(d) * norm;
        }
      }
      if (P > 0) {
        /* every outcome sequence of the flagged decisions: path masks in breadth-first order,
         * a child sets one more bit above its parent's highest set bit and below the number of
         * flagged decisions its parent's walk met (each distinct walk is visited once) */
        int nq = 0, head = 0;
        queue[nq] = 0; qnf[nq] = nf; nq++;
        while (head < nq) {
          uint64_t mask = queue[head];
          int pnf = qnf[head];
          int64_t po = o * P + head;
          double Cp[3], Tp;
          int32_t nlp;
          int bp;
          if (head == 0) {
            Cp[0] = C[0]; Cp[1] = C[1]; Cp[2] = C[2]; Tp = T; nlp = nlast;
            for (int k = 0; k < 4; k++) path_counts[4 * po + k] = counts[4 * o + k];
          } else {
            walk_pixel(rec_f, L, nL, px, py, &m, mask, Cp, &Tp, &nlp, path_counts + 4 * po, NULL, NULL, &bp);
            for (int ch = 0; ch < 3; ch++) Cp[ch] += Tp * bg[ch];
          }
          path_flips[po] = mask;
          for (int ch = 0; ch < 3; ch++) path_c[3 * po + ch] = Cp[ch];
          path_T[po] = Tp;
          path_nl[po] = nlp;
          int hi = -1;
          for (int b = 63; b >= 0; b--)
            if ((mask >> b) & 1) { hi = b; break; }
          for (int b = hi + 1; b < pnf && b < 64; b++) {
            if (nq >= P) { flag |= 16; break; } /* more outcome sequences than max_paths */
            uint64_t child = mask | (1ull << b);
            double Cc[3], Tc;
            int32_t nlc;
            int64_t cc[4];
            int bc;
            int cnf = walk_pixel(rec_f, L, nL, px, py, &m, child, Cc, &Tc, &nlc, cc, NULL, NULL, &bc);
            queue[nq] = child; qnf[nq] = cnf; nq++;
          }
          head++;
        }
        n_paths[o] = nq;
      }
      flags[o] = flag;
    }
    /* WORK cost (R17): the renderer walks a 16x16 block as two 8x16 halves, each until its
     * last pixel is done -- forward the half's largest E_f, backward its largest n_last */
    for (int h = 0; h < 2; h++) {
      int64_t ef = 0, nl = 0;
      for (int p = 0; p < 256; p++) {
        if ((p % 16) / 8 != h) continue;
        int64_t o = kb * 256 + p;
        if (counts[4 * o] > ef) ef = counts[4 * o];
        if (out_nlast[o] > nl) nl = out_nlast[o];
      }
      work[kb] += ef + nl;
    }
  }
  free(queue);
  free(qnf);
  if (loss) *loss += lsum;
}

/* ------------------------------------------------------------------ O14/O15 backward */
void orc_render_bwd(int64_t n_rec, const double* rec_f, const int64_t* offsets,
                    const int64_t* entries, int64_t b0, int64_t b1, int32_t W, int32_t H,
                    const double* bg, const double* dl_dc, const double* margins, const uint64_t* flips,
                    double* grad_rec) {
  (void)n_rec;
  const orc_margins_t m = {margins[0], margins[1], margins[2], margins[3]};
  const int Wt = (W + 15) / 16, Ht = (H + 15) / 16;
  const int64_t per_view = (int64_t)Wt * Ht;
  int64_t cap = 0;
  (void)Ht;
  for (int64_t kb = 0; kb < b1 - b0; kb++)
    if (offsets[kb + 1] - offsets[kb] > cap) cap = offsets[kb + 1] - offsets[kb];
  comp_t* comp = (comp_t*)malloc(sizeof(comp_t) * (size_t)(cap + 1));
  for (int64_t beta = b0; beta < b1; beta++) {
    int64_t kb = beta - b0, loc = beta % per_view;
    int tx = (int)(loc % Wt), ty = (int)(loc / Wt);
    const int64_t* L = entries + offsets[kb];
    int64_t nL = offsets[kb + 1] - offsets[kb];
    for (int p = 0; p < 256; p++) {
      int px = tx * 16 + p % 16, py = ty * 16 + p / 16;
      if (px >= W || py >= H) continue;
      const double* g = dl_dc + 3 * (kb * 256 + p);
      /* re-run O12 along the pixel's outcome path, storing the composited entries */
      double C[3], Tfinal;
      int32_t nlast;
      int64_t cnt[4], nc = 0;
      int bits;
      walk_pixel(rec_f, L, nL, px, py, &m, flips ? flips[kb * 256 + p] : 0, C, &Tfinal, &nlast, cnt, comp, &nc,
                 &bits);
      double S[3] = {0, 0, 0};
      double bgdot = bg[0] * g[0] + bg[1] * g[1] + bg[2] * g[2];
      for (int64_t e = nc - 1; e >= 0; e--) {
        const double* r = rec_f + 10 * comp[e].idx;
        double* gr = grad_rec + 9 * comp[e].idx;
        double a = comp[e].alpha, Tk = comp[e].T;
        for (int ch = 0; ch < 3; ch++) gr[6 + ch] += a * Tk * g[ch];
        double dA = Tk * ((r[7] - S[0]) * g[0] + (r[8] - S[1]) * g[1] + (r[9] - S[2]) * g[2]) -
                    (Tfinal / (1.0 - a)) * bgdot;
        for (int ch = 0; ch < 3; ch++) S[ch] = a * r[7 + ch] + (1.0 - a) * S[ch];
        if (comp[e].capped) continue;  /* R6: alpha = 0.99 constant */
        double Gk = comp[e].G;
        gr[5] += Gk * dA;
        double q = r[6] * Gk * dA;  /* dL/dpower */
        double dx = comp[e].dx, dy = comp[e].dy;
        gr[0] += q * (-(r[3] * dx + r[4] * dy));
        gr[1] += q * (-(r[4] * dx + r[5] * dy));
        gr[2] += q * (-0.5 * dx * dx);
        gr[3] += q * (-dx * dy);
        gr[4] += q * (-0.5 * dy * dy);
      }
    }
  }
  free(comp);
}

/* ------------------------------------------------------------------ O16 transformation backward */
void orc_project_bwd(int64_t n, const double* pos, const double* log_scale, const double* rot,
                     const double* opac_logit, const double* sh, int32_t n_cam,
                     const orc_camera* cams, const double* grad_rec_v, double* grad) {
  for (int64_t i = 0; i < n; i++) {
    double* gd = grad + 59 * i;
    memset(gd, 0, sizeof(double) * 59);
    for (int v = 0; v < n_cam; v++) {
      const double* gr = grad_rec_v + ((int64_t)v * n + i) * 9;
      int any = 0;
      for (int k = 0; k < 9; k++) any |= gr[k] != 0.0;
      if (!any) continue;
      const orc_camera* cam = cams + v;
      fwd64 f;
      forward64(pos + 3 * i, log_scale + 3 * i, rot + 4 * i, opac_logit[i], sh + 48 * i, cam, &f);
      if (!f.vis) continue;
      const float* Wc = cam->R;
      /* opacity: o = sigmoid(logit) */
      gd[10] += gr[5] * f.o * (1.0 - f.o);
      /* colour: SH coefficients and view direction (zero where clamped) */
      double gc[3], gdir[3] = {0, 0, 0}, dY[16][3];
      for (int ch = 0; ch < 3; ch++) gc[ch] = (f.clamp >> ch & 1) ? 0.0 : gr[6 + ch];
      sh_basis_grad(f.dir, dY);
      for (int k = 0; k < 16; k++)
        for (int ch = 0; ch < 3; ch++) {
          gd[11 + 3 * k + ch] += f.Y[k] * gc[ch];
          double sc = sh[48 * i + 3 * k + ch] * gc[ch];
          for (int j = 0; j < 3; j++) gdir[j] += sc * dY[k][j];
        }
      double dd = f.dir[0] * gdir[0] + f.dir[1] * gdir[1] + f.dir[2] * gdir[2];
      for (int j = 0; j < 3; j++) gd[j] += (gdir[j] - f.dir[j] * dd) / f.dist;
      /* conic (A,B,C) -> (a,b,c) */
      double a = f.a, b = f.b, c = f.c, d2 = f.det * f.det;
      double gA = gr[2], gB = gr[3], gC = gr[4];
      double ga = (-c * c * gA + b * c * gB - b * b * gC) / d2;
      double gb = (2 * b * c * gA - (a * c + b * b) * gB + 2 * a * b * gC) / d2;
      double gcc = (-b * b * gA + a * b * gB - a * a * gC) / d2;
      double Gb[4] = {ga, 0.5 * gb, 0.5 * gb, gcc};
      /* Sigma' = T Sigma T^T: dL/dSigma = T^T Gb T, dL/dT = 2 Gb T Sigma */
      double gS[9], gT[6];
      for (int j = 0; j < 3; j++)
        for (int k = 0; k < 3; k++) {
          double s = 0;
          for (int r = 0; r < 2; r++)
            for (int cc = 0; cc < 2; cc++) s += f.T[3 * r + j] * Gb[2 * r + cc] * f.T[3 * cc + k];
          gS[3 * j + k] = s;
        }
      for (int r = 0; r < 2; r++)
        for (int k = 0; k < 3; k++) {
          double s = 0;
          for (int cc = 0; cc < 2; cc++)
            for (int j = 0; j < 3; j++) s += Gb[2 * r + cc] * f.T[3 * cc + j] * f.Sig[3 * j + k];
          gT[3 * r + k] = 2 * s;
        }
      /* T = J W: dL/dJ = dL/dT W^T */
      double gJ[6];
      for (int r = 0; r < 2; r++)
        for (int j = 0; j < 3; j++) {
          double s = 0;
          for (int k = 0; k < 3; k++) s += gT[3 * r + k] * Wc[3 * j + k];
          gJ[3 * r + j] = s;
        }
      double fx = cam->fx, fy = cam->fy, px = f.p[0], py = f.p[1], pz = f.p[2];
      double gp[3];
      gp[0] = gr[0] * fx / pz + gJ[2] * (-fx / (pz * pz));
      gp[1] = gr[1] * fy / pz + gJ[5] * (-fy / (pz * pz));
      gp[2] = -gr[0] * fx * px / (pz * pz) - gr[1] * fy * py / (pz * pz) + gJ[0] * (-fx / (pz * pz)) +
              gJ[2] * (2 * fx * px / (pz * pz * pz)) + gJ[4] * (-fy / (pz * pz)) +
              gJ[5] * (2 * fy * py / (pz * pz * pz));
      /* p = W x + t */
      for (int j = 0; j < 3; j++) gd[j] += Wc[j] * gp[0] + Wc[3 + j] * gp[1] + Wc[6 + j] * gp[2];
      /* Sigma = M M^T: dL/dM = 2 gS M; M = Rq diag(s) */
      double gM[9];
      for (int j = 0; j < 3; j++)
        for (int k = 0; k < 3; k++) {
          double s = 0;
          for (int l = 0; l < 3; l++) s += gS[3 * j + l] * f.M[3 * l + k];
          gM[3 * j + k] = 2 * s;
        }
      double gR[9];
      for (int k = 0; k < 3; k++) {
        double gs = 0;
        for (int j = 0; j < 3; j++) {
          gs += gM[3 * j + k] * f.Rq[3 * j + k];
          gR[3 * j + k] = gM[3 * j + k] * f.s[k];
        }
        gd[3 + k] += gs * f.s[k];  /* s = exp(log s) */
      }
      double w = f.qb[0], x = f.qb[1], y = f.qb[2], z = f.qb[3];
      double gq[4];
      gq[0] = 2 * (-z * gR[1] + y * gR[2] + z * gR[3] - x * gR[5] - y * gR[6] + x * gR[7]);
      gq[1] = 2 * (y * gR[1] + z * gR[2] + y * gR[3] - 2 * x * gR[4] - w * gR[5] + z * gR[6] + w * gR[7] - 2 * x * gR[8]);
      gq[2] = 2 * (-2 * y * gR[0] + x * gR[1] + w * gR[2] + x * gR[3] + z * gR[5] - w * gR[6] + z * gR[7] - 2 * y * gR[8]);
      gq[3] = 2 * (-2 * z * gR[0] - w * gR[1] + x * gR[2] + w * gR[3] - 2 * z * gR[4] + y * gR[5] + x * gR[6] + y * gR[7]);
      double qd = w * gq[0] + x * gq[1] + y * gq[2] + z * gq[3];
      for (int k = 0; k < 4; k++) gd[6 + k] += (gq[k] - f.qb[k] * qd) / f.qn;
    }
  }
}

/* ------------------------------------------------------------------ O17 Adam (Eq. 1-2) */
void orc_adam(int64_t n, double* theta, double* m, double* v, const double* g, double lr,
              double beta1, double beta2, double eps, int32_t batch, int64_t step) {
  double lrb = lr * sqrt((double)batch);        /* Eq. (1) */
  double b1 = pow(beta1, batch), b2 = pow(beta2, batch); /* Eq. (2) */
  double bc1 = 1.0 - pow(b1, (double)step), bc2 = 1.0 - pow(b2, (double)step);
  for (int64_t k = 0; k < n; k++) {
    m[k] = b1 * m[k] + (1 - b1) * g[k];
    v[k] = b2 * v[k] + (1 - b2) * g[k] * g[k];
    theta[k] -= (lrb / bc1) * m[k] / (sqrt(v[k]) / sqrt(bc2) + eps);
  }
}

/* ------------------------------------------------------------------ O18 Algorithm 1 */
int orc_division_points(const int64_t* ET, int64_t B, int32_t G, int64_t* DP) {
  int64_t mx = 0;
  for (int64_t i = 0; i < B; i++)
    if (ET[i] > mx) mx = ET[i];
  if (B > 0 && mx > 0 && (double)B * (double)mx * (double)G >= 9.2e18) return -1;
  int64_t* CT = (int64_t*)malloc(sizeof(int64_t) * (size_t)(B > 0 ? B : 1));
  int64_t acc = 0;
  for (int64_t i = 0; i < B; i++) CT[i] = (acc += ET[i]);  /* line 1: cumsum */
  int64_t tot = B > 0 ? CT[B - 1] : 0;
  DP[0] = 0;
  for (int g = 1; g < G; g++) {
    if (tot == 0) {
      DP[g] = (int64_t)g * B / G;  /* all-zero costs: uniform split */
      continue;
    }
    /* lines 2-4: TH[g] = g * tot / G; DP[g] = right-bisect(CT, TH[g]) = #{i : CT[i] <= TH[g]},
     * evaluated as CT[i] * G <= g * tot (exact, R8) */
    int64_t c = 0;
    for (int64_t i = 0; i < B; i++)
      if (CT[i] * G <= (int64_t)g * tot) c++;
    DP[g] = c;
  }
  DP[G] = B;
  free(CT);
  return 0;
}

void orc_costs_to_et(int32_t mode, int64_t B, int32_t G, const int64_t* DP, const int64_t* cost,
                     const int64_t* npix, int64_t* et) {
  if (mode != 2) {
    for (int64_t i = 0; i < B; i++) et[i] = cost[i];
    return;
  }
  for (int g = 0; g < G; g++) {
    int64_t Cg = 0, Ng = 0;
    for (int64_t i = DP[g]; i < DP[g + 1]; i++) { Cg += cost[i]; Ng += npix[i]; }
    for (int64_t i = DP[g]; i < DP[g + 1]; i++)
      et[i] = Ng > 0 ? (int64_t)((__int128)Cg * npix[i] / Ng) : 0;
  }
}

/* A9 step 3 (R17; "uniform estimate" for images not seen yet): ET of the next
 * batch's B_next blocks from their images' history rows (hist[k] >= 0: the estimate stored
 * when that block was last rendered; -1: never rendered), an unseen block costing the rendered
 * batch's per-pixel rate times its in-image pixels, floor(rate_num * npix / rate_den), with
 * rate_num = the sum of the rendered batch's costs and rate_den its in-image pixels, or npix
 * itself while rate_num == 0. */
void orc_next_et(int64_t B_next, const int64_t* hist, const int64_t* npix, int64_t rate_num, int64_t rate_den,
                 int64_t* et) {
  for (int64_t k = 0; k < B_next; k++) {
    if (hist[k] >= 0)
      et[k] = hist[k];
    else if (rate_num > 0 && rate_den > 0)
      et[k] = (int64_t)((__int128)rate_num * npix[k] / rate_den);
    else
      et[k] = npix[k];
  }
}

/* ------------------------------------------------------------------ NEXT-1: L1 + D-SSIM */
/* P:114 "the 3DGS computes the L1 and SSIM loss by comparing the rendered image to the
 * ground truth image ... the SSIM loss measures the similarity between pixel windows";
 * S:278-282 (11x11 Gaussian window, sigma 1.5, C1 = 0.01^2, C2 = 0.03^2, mean over centres,
 * analytic gradient), S:301 (lambda = 0.2).  Readings R12: the window is the
 * normalised 1D Gaussian outer-multiplied with itself, values outside the image are zero
 * (windows are not truncated or renormalised at the border), the mean runs over every pixel
 * and channel of the image.
 *
 * For one channel and centre p, with window w and zero padding:
 *   mx = sum w x, my = sum w y, Exx = sum w x^2, Eyy = sum w y^2, Exy = sum w x y,
 *   A1 = 2 mx my + C1, A2 = 2 (Exy - mx my) + C2, B1 = mx^2 + my^2 + C1,
 *   B2 = (Exx - mx^2) + (Eyy - my^2) + C2,  S(p) = A1 A2 / (B1 B2).
 * Treating (mx, Exx, Exy) as the independent window statistics of x:
 *   dS/dmx  = (2 my A2 - 2 my A1) / (B1 B2) - S (2 mx / B1 - 2 mx / B2)
 *   dS/dExx = -S / B2,   dS/dExy = 2 A1 / (B1 B2),
 * and dmx(p)/dx(q) = w(q - p), dExx(p)/dx(q) = 2 x(q) w(q - p), dExy(p)/dx(q) = y(q) w(q - p).
 * Every window sum below is the direct 121-term double sum (no separable filtering). */
static void orc_ssim_window(double w[11][11]) {
  double g[11], s = 0.0;
  for (int k = 0; k < 11; k++) {
    const double d = (double)(k - 5);
    g[k] = exp(-d * d / (2.0 * 1.5 * 1.5));
    s += g[k];
  }
  for (int a = 0; a < 11; a++)
    for (int b = 0; b < 11; b++) w[a][b] = (g[a] / s) * (g[b] / s);
}

void orc_ssim_loss(int32_t W, int32_t H, const double* img, const double* gt, double lambda, double* loss,
                   double* ssim_mean, double* grad) {
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  const double N = 3.0 * (double)W * (double)H;
  double w[11][11];
  orc_ssim_window(w);
  const int64_t np = (int64_t)W * H;
  double* dmx = (double*)calloc((size_t)np, sizeof(double));
  double* dxx = (double*)calloc((size_t)np, sizeof(double));
  double* dxy = (double*)calloc((size_t)np, sizeof(double));
  double l1 = 0.0, ssum = 0.0;
  for (int c = 0; c < 3; c++) {
    for (int py = 0; py < H; py++)
      for (int px = 0; px < W; px++) {
        double mx = 0, my = 0, exx = 0, eyy = 0, exy = 0;
        for (int a = 0; a < 11; a++)
          for (int b = 0; b < 11; b++) {
            const int qy = py + a - 5, qx = px + b - 5;
            if (qy < 0 || qy >= H || qx < 0 || qx >= W) continue; /* zero padding */
            const double x = img[((int64_t)qy * W + qx) * 3 + c], y = gt[((int64_t)qy * W + qx) * 3 + c];
            mx += w[a][b] * x;
            my += w[a][b] * y;
            exx += w[a][b] * x * x;
            eyy += w[a][b] * y * y;
            exy += w[a][b] * x * y;
          }
        const double A1 = 2.0 * mx * my + C1, A2 = 2.0 * (exy - mx * my) + C2;
        const double B1 = mx * mx + my * my + C1, B2 = (exx - mx * mx) + (eyy - my * my) + C2;
        const double S = A1 * A2 / (B1 * B2);
        ssum += S;
        const int64_t p = (int64_t)py * W + px;
        dmx[p] = (2.0 * my * A2 - 2.0 * my * A1) / (B1 * B2) - S * (2.0 * mx / B1 - 2.0 * mx / B2);
        dxx[p] = -S / B2;
        dxy[p] = 2.0 * A1 / (B1 * B2);
      }
    for (int qy = 0; qy < H; qy++)
      for (int qx = 0; qx < W; qx++) {
        const int64_t q = (int64_t)qy * W + qx;
        const double x = img[q * 3 + c], y = gt[q * 3 + c];
        double gs = 0.0; /* d(sum_p S(p)) / dx(q) */
        for (int a = 0; a < 11; a++)
          for (int b = 0; b < 11; b++) {
            const int py = qy - (a - 5), px = qx - (b - 5); /* q = p + (a-5, b-5) */
            if (py < 0 || py >= H || px < 0 || px >= W) continue;
            const int64_t p = (int64_t)py * W + px;
            gs += w[a][b] * (dmx[p] + 2.0 * x * dxx[p] + y * dxy[p]);
          }
        const double e = x - y;
        l1 += fabs(e);
        if (grad) grad[q * 3 + c] = ((1.0 - lambda) * (e > 0 ? 1.0 : (e < 0 ? -1.0 : 0.0)) - lambda * gs) / N;
      }
  }
  free(dmx);
  free(dxx);
  free(dxy);
  if (ssim_mean) *ssim_mean = ssum / N;
  if (loss) *loss = (1.0 - lambda) * l1 / N + lambda * (1.0 - ssum / N);
}
