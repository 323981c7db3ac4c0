// gs_densify.cu -- NEXT-2: adaptive density control on the owner ("adaptive
// densification mechanism to add Gaussians"; App. A.1 "whether their scale exceeds
// a threshold ... cloning or splitting ... opacity reset"; App. A.3 "we perform this
// process locally on the GPU that stores them").
//
//   gs_densify_stats : per (Gaussian, view) the norm of the screen-space (NDC) mean gradient
//                      of the per-image loss, its count, and the largest screen radius,
//                      read through the same backward index as gs_adam_step (R13);
//   gs_densify       : clone / split / prune of the shard into new buffers (params, Adam m, v),
//                      decisions in fp32 against host-computed thresholds (bit-exact with the
//                      oracle), order [kept originals][clones][first children][second
//                      children], each in parent order (the 3DGS append order);
//   gs_opacity_reset : opacity logits clamped to logit(max_opacity), their Adam moments zeroed.
//
// One thread per Gaussian; placement by an exclusive scan of four keep flags laid out
// [4][n], so the output order is a pure function of the decisions (no atomics).
#include <cmath>

#include "gs_device.cuh"
#include "gs_index.cuh"
#include "gs_internal.h"

using namespace gsd;

namespace {

__global__ void __launch_bounds__(kBlock) k_densify_stats(int64_t n, int b, int G, int nb, int NW,
                                                          const uint32_t* __restrict__ maskw,
                                                          const int64_t* __restrict__ base, int64_t ncta,
                                                          const gs_rec* __restrict__ send_rec,
                                                          const float* __restrict__ dL_dsend, float sx, float sy,
                                                          float* __restrict__ accum, float* __restrict__ denom,
                                                          float* __restrict__ max_radius) {
  __shared__ int s_cnt[kWarps * kMaxBuckets];
  const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  uint32_t m[kMaxWords], u[kMaxWords];
  load_masks(maskw, n, i, NW, m);
  cta_rank_phase1(m, u, NW, nb, s_cnt);
  const bool live = i < n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  float acc = 0.f, cnt = 0.f, rmax = 0.f;
  for (int v = 0; v < b; v++) {
    if (!view_in_union(u, v, b, G)) continue;  // warp-uniform
    float gx = 0.f, gy = 0.f, r = 0.f;
    bool seen = false;
    for (int d = 0; d < G; d++) {  // a view's destinations in ascending rank (as gs_adam_step)
      const int k = d * b + v;
      if (!get_bit(u, k)) continue;
      const bool bit = live && get_bit(m, k);
      const unsigned bal = __ballot_sync(0xffffffffu, bit);
      if (bit) {
        const int64_t pos = base[(int64_t)k * ncta + blockIdx.x] + warp_prefix(s_cnt, wid, nb, k) + __popc(bal & lt);
        gx += dL_dsend[pos * 9 + 0];
        gy += dL_dsend[pos * 9 + 1];
        r = send_rec[pos].a.w;
        seen = true;
      }
    }
    if (seen) {
      const float nx = gx * sx, ny = gy * sy;
      acc += sqrtf(nx * nx + ny * ny);
      cnt += 1.f;
      rmax = fmaxf(rmax, r);
    }
  }
  if (!live) return;
  accum[i] += acc;
  denom[i] += cnt;
  max_radius[i] = fmaxf(max_radius[i], rmax);
}

struct dens_arg {
  float grad_thresh;   // average NDC gradient norm that selects a Gaussian
  float log_split;     // log(percent_dense * extent): max log-scale above -> split, else clone
  float logit_min_op;  // prune if opacity logit < logit(min_opacity)
  float max_screen;    // prune if max screen radius > this (<= 0: screen/world-size pruning off)
  float log_big;       // with max_screen > 0: prune if max log-scale > log(0.1 extent)
  float log_big_child; // the same test for split children: log(1.6 * 0.1 extent) on the parent
  float log_shrink;    // log(1.6): children's scale = parent's / 1.6 (3DGS 0.8 N, N = 2)
};

__device__ __forceinline__ float max3(float a, float b, float c) { return fmaxf(a, fmaxf(b, c)); }

// keep flags [4][n]: original, clone, child 0, child 1
__global__ void k_densify_classify(const float4* __restrict__ pos_op, const float4* __restrict__ ls, int64_t n,
                                   const float* __restrict__ accum, const float* __restrict__ denom,
                                   const float* __restrict__ max_radius, dens_arg a, int64_t* __restrict__ flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 po = pos_op[i], l = ls[i];
  const float dn = denom[i];
  const float avg = dn > 0.f ? __fdiv_rn(accum[i], dn) : 0.f;
  const bool sel = avg >= a.grad_thresh;
  const float lmax = max3(l.x, l.y, l.z);
  const bool big = lmax > a.log_split;
  const bool clone = sel && !big, split = sel && big;
  const bool low_op = po.w < a.logit_min_op;
  const bool prune_orig = low_op || (a.max_screen > 0.f && (max_radius[i] > a.max_screen || lmax > a.log_big));
  // clones: the parent's parameters, screen radius 0; children: the parent's opacity, scale / 1.6
  const bool prune_clone = low_op || (a.max_screen > 0.f && lmax > a.log_big);
  const bool prune_child = low_op || (a.max_screen > 0.f && lmax > a.log_big_child);
  flags[i] = (!split && !prune_orig) ? 1 : 0;
  flags[n + i] = (clone && !prune_clone) ? 1 : 0;
  flags[2 * n + i] = (split && !prune_child) ? 1 : 0;
  flags[3 * n + i] = (split && !prune_child) ? 1 : 0;
}

struct dplanes {
  const float4 *pos_op, *ls, *rot, *sh;
};
struct wplanes {
  float4 *pos_op, *ls, *rot, *sh;
};

__device__ __forceinline__ void copy_g(const dplanes& s, int64_t n, int64_t i, const wplanes& d, int64_t n2, int64_t o,
                                       float4 pos_op, float4 ls) {
  d.pos_op[o] = pos_op;
  d.ls[o] = ls;
  d.rot[o] = s.rot[i];
#pragma unroll
  for (int k = 0; k < 12; k++) d.sh[(int64_t)k * n2 + o] = s.sh[(int64_t)k * n + i];
}
__device__ __forceinline__ void zero_g(const wplanes& d, int64_t n2, int64_t o) {
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  d.pos_op[o] = z;
  d.ls[o] = z;
  d.rot[o] = z;
#pragma unroll
  for (int k = 0; k < 12; k++) d.sh[(int64_t)k * n2 + o] = z;
}

__global__ void k_densify_write(dplanes P, dplanes M, dplanes V, int64_t n, const int64_t* __restrict__ flags,
                                const int64_t* __restrict__ off, const float* __restrict__ noise, dens_arg a,
                                wplanes PO, wplanes MO, wplanes VO, int64_t n2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 po = P.pos_op[i], l = P.ls[i];
  if (flags[i]) {  // kept original, its Adam state travels with it
    const int64_t o = off[i];
    copy_g(P, n, i, PO, n2, o, po, l);
    copy_g(M, n, i, MO, n2, o, M.pos_op[i], M.ls[i]);
    copy_g(V, n, i, VO, n2, o, V.pos_op[i], V.ls[i]);
  }
  if (flags[n + i]) {  // clone: same parameters, fresh Adam state
    const int64_t o = off[n + i];
    copy_g(P, n, i, PO, n2, o, po, l);
    zero_g(MO, n2, o);
    zero_g(VO, n2, o);
  }
  if (flags[2 * n + i] || flags[3 * n + i]) {
    // children: x + R(q) (s . z_t), z_t ~ N(0, I) given (noise[i][t][3]); scale s / 1.6
    const float4 q = P.rot[i];
    const float qn = sqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
    const float iq = qn > 0.f ? 1.0f / qn : 0.f;
    const float w = q.x * iq, x = q.y * iq, y = q.z * iq, z = q.w * iq;
    const float R[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                        2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                        2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
    const float s[3] = {expf(l.x), expf(l.y), expf(l.z)};
    const float4 lc = make_float4(l.x - a.log_shrink, l.y - a.log_shrink, l.z - a.log_shrink, l.w);
    for (int t = 0; t < 2; t++) {
      if (!flags[(2 + t) * n + i]) continue;
      const float* zz = noise + (i * 2 + t) * 3;
      const float e0 = s[0] * zz[0], e1 = s[1] * zz[1], e2 = s[2] * zz[2];
      const float4 pc = make_float4(po.x + R[0] * e0 + R[1] * e1 + R[2] * e2, po.y + R[3] * e0 + R[4] * e1 + R[5] * e2,
                                    po.z + R[6] * e0 + R[7] * e1 + R[8] * e2, po.w);
      const int64_t o = off[(2 + t) * n + i];
      copy_g(P, n, i, PO, n2, o, pc, lc);
      zero_g(MO, n2, o);
      zero_g(VO, n2, o);
    }
  }
}

__global__ void k_opacity_reset(float4* __restrict__ pos_op, float4* __restrict__ m, float4* __restrict__ v,
                                int64_t n, float max_logit) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  pos_op[i].w = fminf(pos_op[i].w, max_logit);
  if (m) m[i].w = 0.f;
  if (v) v[i].w = 0.f;
}

}  // namespace

extern "C" gs_status gs_densify_stats(gs_ctx* c, const gs_camera* cams_h, int n_views, const int64_t* dp_h, int64_t n,
                                      const void* bwd_index, const void* send_rec, const float* dL_dsend, int b_loss,
                                      float* grad_accum, float* denom, float* max_radius, void* stream) {
  if (!c) return GS_EINVAL;
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, n >= 0 && b_loss >= 1, "bad size");
  if (n == 0) return GS_OK;
  GS_REQUIRE(c, bwd_index && grad_accum && denom && max_radius, "null argument");
  const int G = c->world, nb = n_views * G;
  GS_REQUIRE(c, nb <= kMaxBuckets, "n_views * world too large");
  gs_index_layout L = index_layout(n, n_views, G);
  const gs_geom geo = gs_make_geom(&cams_h[0]);
  // d(ndc)/d(pixel) = 2 / W: the NDC gradient is the pixel gradient times W / 2 (H / 2), and
  // the batch-mean loss is scaled back to one image's loss by b (R13)
  const float sx = 0.5f * (float)geo.W * (float)b_loss, sy = 0.5f * (float)geo.H * (float)b_loss;
  ++c->launches;
  k_densify_stats<<<(unsigned)L.ncta, kBlock, 0, (cudaStream_t)stream>>>(
      n, n_views, G, nb, L.NW, (const uint32_t*)bwd_index, (const int64_t*)((const char*)bwd_index + L.base_off),
      L.ncta, (const gs_rec*)send_rec, dL_dsend, sx, sy, grad_accum, denom, max_radius);
  GS_LAUNCH_CHECK(c, "densify_stats");
  return GS_OK;
}

extern "C" gs_status gs_densify(gs_ctx* c, const gs_params* p, const gs_params* m, const gs_params* v,
                                const float* grad_accum, const float* denom, const float* max_radius,
                                const float* noise, const gs_densify_cfg* cfg, gs_params* p_out, gs_params* m_out,
                                gs_params* v_out, int64_t out_cap, int64_t* counts_h, void* stream) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, p && m && v && cfg && counts_h && p_out && m_out && v_out, "null argument");
  GS_REQUIRE(c, m->n == p->n && v->n == p->n, "m/v mis-sized");
  GS_REQUIRE(c, cfg->scene_extent > 0.f && cfg->percent_dense > 0.f && cfg->min_opacity > 0.f &&
                    cfg->min_opacity < 1.f, "bad densify configuration");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = p->n;
  for (int k = 0; k < 4; k++) counts_h[k] = 0;
  if (n == 0) return GS_OK;
  GS_REQUIRE(c, grad_accum && denom && max_radius && noise, "null statistics / noise");
  dens_arg a;
  a.grad_thresh = cfg->grad_thresh;
  a.log_split = (float)std::log((double)cfg->percent_dense * (double)cfg->scene_extent);
  a.logit_min_op = (float)std::log((double)cfg->min_opacity / (1.0 - (double)cfg->min_opacity));
  a.max_screen = cfg->max_screen_size;
  a.log_big = (float)std::log(0.1 * (double)cfg->scene_extent);
  a.log_big_child = (float)std::log(1.6 * 0.1 * (double)cfg->scene_extent);
  a.log_shrink = (float)std::log(1.6);
  int64_t* flags = (int64_t*)gs_slot_get(c, SLOT_DENSIFY, (4 * n + 1) * sizeof(int64_t), st);
  int64_t* off = (int64_t*)gs_slot_get(c, SLOT_DENSIFY_OFF, (4 * n + 1) * sizeof(int64_t), st);
  if (!flags || !off) return gs_fail(c, GS_ECUDA, "densify scratch");
  ++c->launches;
  k_densify_classify<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((const float4*)p->pos_op, (const float4*)p->log_scale,
                                                                 n, grad_accum, denom, max_radius, a, flags);
  GS_CUDA(c, cudaMemsetAsync(flags + 4 * n, 0, sizeof(int64_t), st));
  gs_status s = gs_scan_i64(c, flags, off, 4 * n + 1, 0, st);
  if (s != GS_OK) return s;
  // counts: kept originals, clones, children (both), total
  int64_t h[5];
  GS_CUDA(c, cudaMemcpyAsync(&h[0], off + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaMemcpyAsync(&h[1], off + 2 * n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaMemcpyAsync(&h[2], off + 4 * n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  const int64_t n2 = h[2];
  counts_h[0] = h[0];
  counts_h[1] = h[1] - h[0];
  counts_h[2] = n2 - h[1];
  counts_h[3] = n2;
  if (n2 > out_cap) return gs_fail(c, GS_ECAPACITY, "densify output capacity %lld < %lld", (long long)out_cap,
                                   (long long)n2);
  if (n2 == 0) return GS_OK;
  GS_REQUIRE(c, p_out->pos_op && m_out->pos_op && v_out->pos_op, "null output planes");
  p_out->n = m_out->n = v_out->n = n2;  // the output planes are laid out for n2 (SH plane stride)
  auto dp_of = [](const gs_params* q) {
    return dplanes{(const float4*)q->pos_op, (const float4*)q->log_scale, (const float4*)q->rot, (const float4*)q->sh};
  };
  auto wp_of = [](gs_params* q) {
    return wplanes{(float4*)q->pos_op, (float4*)q->log_scale, (float4*)q->rot, (float4*)q->sh};
  };
  ++c->launches;
  k_densify_write<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(dp_of(p), dp_of(m), dp_of(v), n, flags, off, noise, a,
                                                              wp_of(p_out), wp_of(m_out), wp_of(v_out), n2);
  GS_LAUNCH_CHECK(c, "densify");
  return GS_OK;
}

extern "C" gs_status gs_opacity_reset(gs_ctx* c, gs_params* p, gs_params* m, gs_params* v, float max_opacity,
                                      void* stream) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, p != nullptr, "null params");
  GS_REQUIRE(c, max_opacity > 0.f && max_opacity < 1.f, "max_opacity must be in (0, 1)");
  if (p->n == 0) return GS_OK;
  const float max_logit = (float)std::log((double)max_opacity / (1.0 - (double)max_opacity));
  ++c->launches;
  k_opacity_reset<<<(unsigned)((p->n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (float4*)p->pos_op, m ? (float4*)m->pos_op : nullptr, v ? (float4*)v->pos_op : nullptr, p->n, max_logit);
  GS_LAUNCH_CHECK(c, "opacity_reset");
  return GS_OK;
}
