// gs_project.cu -- A1: EWA projection, culling, colour and exchange destinations on the
// Gaussian's owner (P:103 step 1 "each Gaussian i is transformed and projected to determine
// its position x_{v,i} ... depth_{v,i} ... radius_{v,i} ... color c_{v,i}").
//
// Two passes over the owned shard, one thread per Gaussian, 256 per CTA:
//   count: fp32 membership chain for every view, destination set D(i,v) (O10), per-CTA
//          bucket counts, bucket = (destination d, view v), and the (v,d) bitmask per Gaussian
//          (the backward index gs_adam_step reuses);
//   scan:  exclusive scan of the counts in (d, v, CTA) order -> each CTA's bucket bases;
//   write: recompute the projection, rank each Gaussian inside its CTA bucket with warp
//          ballots (thread order = gid order), write 64-byte records.
// Placement is therefore deterministic and gid-ordered within each (d, v) bucket, which the
// stable (depth, gid) order of A3 relies on; no placement atomics.
#include <cstring>

#include "gs_device.cuh"
#include "gs_index.cuh"

using namespace gsd;

namespace {

// Record destinations of k_project_write: the record at send-order position pos with
// destination d goes to d_[d][pos] (all d_ = the send buffer for gs_project; for the fused
// NEXT-3 path d_[d] = d's receive buffer + put_base[d] - send_off[d]).
constexpr int kPList = 8;  // records per thread listed per round (k_project_write)

struct gs_outs {
  gs_rec* d[GS_MAX_WORLD];
};

__global__ void __launch_bounds__(kBlock) k_project_count(
    const float4* __restrict__ pos_op, const float4* __restrict__ log_scale,
    const float4* __restrict__ rot, int64_t n, gs_cams_arg cams, gs_geom geo, gs_dp_arg dp,
    int nb, int NW, uint32_t* __restrict__ maskw, int64_t* __restrict__ cta_cnt, int64_t ncta, int64_t gid_base,
    unsigned long long* __restrict__ bad) {
  __shared__ int s_c[kMaxBuckets];
  for (int k = threadIdx.x; k < nb; k += kBlock) s_c[k] = 0;
  __syncthreads();
  int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  uint32_t m[kMaxWords];
#pragma unroll
  for (int w = 0; w < kMaxWords; w++) m[w] = 0;
  if (i < n) {
    float4 X = pos_op[i];
    const float4 ls = log_scale[i], q = rot[i];
    // a non-finite parameter is an error naming the Gaussian (lowest gid wins)
    if (!(isfinite(X.x) && isfinite(X.y) && isfinite(X.z) && isfinite(X.w) && isfinite(ls.x) && isfinite(ls.y) &&
          isfinite(ls.z) && isfinite(q.x) && isfinite(q.y) && isfinite(q.z) && isfinite(q.w)))
      atomicMin(bad, (unsigned long long)(gid_base + i));
    gs_cov3 cv = cov3_of(ls, q);
    for (int v = 0; v < cams.n; v++) {
      gs_memb mb = membership(cv, X.x, X.y, X.z, cams.c[v], geo.Wt, geo.Ht);
      if (!mb.vis) continue;
      unsigned dm = dest_mask(mb, v, geo, dp);
      while (dm) {
        int d = __ffs(dm) - 1;
        dm &= dm - 1;
        int k = d * cams.n + v;
        set_bit(m, k);
        atomicAdd(&s_c[k], 1);
      }
    }
    for (int w = 0; w < NW; w++) maskw[(int64_t)w * n + i] = m[w];
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nb; k += kBlock) cta_cnt[(int64_t)k * ncta + blockIdx.x] = s_c[k];
}

__global__ void k_gather_totals(const int64_t* base, int64_t ncta, int b, int G, int64_t* out) {
  int d = threadIdx.x;
  if (d <= G) out[d] = base[(int64_t)d * b * ncta];
}

// NEXT-3 sync-free put: the destinations' receive buffers and capacities; the record offsets
// come from the G x G count matrix on the device (this rank's copy, complete after the
// count-exchange barrier).
struct gs_devouts {
  gs_rec* recv[GS_MAX_WORLD];
  long long cap[GS_MAX_WORLD];
  const int64_t* cmat;
  int rank;
};

template <bool kDev>
__global__ void __launch_bounds__(kBlock) k_project_write(
    const float4* __restrict__ pos_op, const float4* __restrict__ log_scale,
    const float4* __restrict__ rot, const float4* __restrict__ sh, int64_t n, int64_t gid_base,
    gs_cams_arg cams, gs_geom geo, int G, int nb, int NW, const uint32_t* __restrict__ maskw,
    const int64_t* __restrict__ base, int64_t ncta, gs_outs outs, unsigned long long* __restrict__ bad,
    gs_devouts dv) {
  __shared__ int s_cnt[kWarps * kMaxBuckets];
  __shared__ gs_rec* s_out[GS_MAX_WORLD];  // kDev: destination d's base for this rank's records
  __shared__ int64_t s_pos[kPList * kBlock];  // per-thread send positions of its records
  __shared__ uint16_t s_vd[kPList * kBlock];  // and their (view, destination)
  if constexpr (kDev) {
    // every destination's records: this rank's bucket for d starts at put[d] = sum over
    // s < rank of C[s][d] in d's buffer and at soff[d] = sum over d' < d of C[rank][d'] in the
    // send order; nothing is written if any destination would overflow (every rank sees the
    // same matrix: all skip together, gs_p2p_counts reports it)
    __shared__ int s_ok;
    if (threadIdx.x == 0) s_ok = 1;
    __syncthreads();
    if ((int)threadIdx.x < G) {
      const int d = threadIdx.x;
      long long put = 0, in = 0, soff = 0;
      for (int q = 0; q < G; q++) {
        const long long x = dv.cmat[q * G + d];
        in += x;
        if (q < dv.rank) put += x;
      }
      for (int e = 0; e < d; e++) soff += dv.cmat[dv.rank * G + e];
      if (in > dv.cap[d]) s_ok = 0;
      s_out[d] = dv.recv[d] + (put - soff);
    }
    __syncthreads();
    if (!s_ok) return;
  }
  const int b = cams.n;
  int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  uint32_t m[kMaxWords], u[kMaxWords];
  load_masks(maskw, n, i, NW, m);
  cta_rank_phase1(m, u, NW, nb, s_cnt);
  // view-independent parameters
  float4 X = make_float4(0, 0, 0, 0), q = X, ls = X;
  if (i < n) {
    X = pos_op[i];
    ls = log_scale[i];
    q = rot[i];
  }
  gs_cov3 cv = cov3_of(ls, q);
  // O1 opacity, rounded to nearest from fp64 (it sets alpha and the skip threshold), and
  // log2(255 o) rounded to nearest from fp64 (a record's qmax; per Gaussian, not per view)
  const float opac = __double2float_rn(1.0 / (1.0 + exp(-(double)X.w)));
  const float qmax_o = opac > 0.f ? __double2float_rn(log2(255.0 * (double)opac)) : -1.0f;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  // Phase A (warp-uniform over the union of the warp's buckets, view outer, destination
  // inner): each lane lists the send positions of its own records in that order.  Phase B
  // (per lane, divergent): walks its own list, forms the record of each of its views once and
  // stores it at each destination's position -- a warp no longer steps through every view any
  // lane sees.  Lists longer than kPList go in rounds (warp-uniform count).
  int n_mine = 0;
  for (int w = 0; w < NW; w++) n_mine += i < n ? __popc(m[w]) : 0;
  const int rounds = (__reduce_max_sync(0xffffffffu, n_mine) + kPList - 1) / kPList;
  for (int r = 0; r < rounds; r++) {
    int cnt = 0;
    for (int v = 0; v < b; v++) {
      if (!view_in_union(u, v, b, G)) continue;  // warp-uniform
      for (int d = 0; d < G; d++) {
        const int k = d * b + v;
        if (!get_bit(u, k)) continue;  // warp-uniform
        const bool bit = i < n && get_bit(m, k);
        const unsigned bal = __ballot_sync(0xffffffffu, bit);
        if (bit) {
          const int slot = cnt - r * kPList;
          if (slot >= 0 && slot < kPList) {
            s_pos[slot * kBlock + threadIdx.x] =
                base[(int64_t)k * ncta + blockIdx.x] + warp_prefix(s_cnt, wid, nb, k) + __popc(bal & lt);
            s_vd[slot * kBlock + threadIdx.x] = (uint16_t)(v | d << 8);
          }
          cnt++;
        }
      }
    }
    const int nl = min(kPList, max(0, cnt - r * kPList));
    gs_rec rec;
    int cur = -1;
    for (int j = 0; j < nl; j++) {
      const int vd = s_vd[j * kBlock + threadIdx.x], v = vd & 0xff, d = vd >> 8;
      if (v != cur) {
        cur = v;
        const gs_dcam& cam = cams.c[v];
        gs_memb mb = membership(cv, X.x, X.y, X.z, cam, geo.Wt, geo.Ht);
        // conic = inverse of the 2D covariance (O6), carried as its Cholesky factor prescaled by
        // sqrt(0.5 log2 e) (conic = L L^T): l11 = sqrt(c / det), l21 = -b / sqrt(det c),
        // l22 = 1 / sqrt(c), evaluated in fp64 from the fp32 covariance (the products of fp32
        // values are exact in fp64) and stored as hi + lo, each rounded to nearest
        float lh[3] = {0.f, 0.f, 0.f}, ll[3] = {0.f, 0.f, 0.f};
        {
          const double a64 = mb.a, b64 = mb.b, c64 = mb.c;
          const double det = a64 * c64 - b64 * b64;
          if (det > 0.0) {
            const double sc = sqrt(c64), sd = sqrt(det);
            const double L[3] = {kLScale64 * sc / sd, -kLScale64 * b64 / (sd * sc), kLScale64 / sc};
#pragma unroll
            for (int k = 0; k < 3; k++) {
              lh[k] = __double2float_rn(L[k]);
              ll[k] = __double2float_rn(L[k] - (double)lh[k]);
            }
          }
        }
        // qmax = log2(255 o), rounded to nearest from fp64 (alpha = o 2^-q >= 1/255 <=> q <= qmax);
        // -1 (never composited) for a zero opacity or a covariance whose fp64 determinant is not
        // positive (not reachable with the 0.3 I dilation: det >= 0.09)
        const float qmax = lh[0] > 0.f ? qmax_o : -1.0f;
        // O9: colour from the view direction
        float dx = X.x - cam.campos[0], dy = X.y - cam.campos[1], dz = X.z - cam.campos[2];
        float inv = rsqrtf(dx * dx + dy * dy + dz * dz);
        float Y[16];
        sh_basis(dx * inv, dy * inv, dz * inv, Y);
        float col[3];
        col[0] = col[1] = col[2] = 0.5f;
        bool shf = true;
#pragma unroll
        for (int k = 0; k < 12; k++) {  // SH planes read only for visible (i, v)
          const float4 s4 = sh[(int64_t)k * n + i];
          shf = shf && isfinite(s4.x) && isfinite(s4.y) && isfinite(s4.z) && isfinite(s4.w);
          const float e[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
          for (int jj = 0; jj < 4; jj++)
            col[(4 * k + jj) % 3] = fmaf(Y[(4 * k + jj) / 3], e[jj], col[(4 * k + jj) % 3]);
        }
#pragma unroll
        for (int ch = 0; ch < 3; ch++) col[ch] = fmaxf(col[ch], 0.0f);
        // SH coefficients are read here only (visible Gaussians): reported by the next call's sync
        if (!shf) atomicMin(bad, (unsigned long long)(gid_base + i));
        unsigned meta = (unsigned)((gid_base + i) * 32 + v);
        rec.a = make_float4(mb.mx, mb.my, mb.depth, mb.r);
        rec.b = make_float4(lh[0], lh[1], lh[2], opac);
        rec.c = make_float4(col[0], col[1], col[2], qmax);
        rec.d = make_float4(ll[0], ll[1], ll[2], __uint_as_float(meta));
      }
      // own send buffer, or (NEXT-3) d's receive buffer
      (kDev ? s_out[d] : outs.d[d])[s_pos[j * kBlock + threadIdx.x]] = rec;
    }
  }
}

}  // namespace

// The context's non-finite word (lowest offending gid, ~0 = none), initialised on first use.
static unsigned long long* nonfinite_word(gs_ctx* c, cudaStream_t st) {
  const bool fresh = c->slot[SLOT_NONFINITE].ptr == nullptr;
  unsigned long long* w = (unsigned long long*)gs_slot_get(c, SLOT_NONFINITE, sizeof(unsigned long long), st);
  if (w && fresh && cudaMemsetAsync(w, 0xff, sizeof(unsigned long long), st) != cudaSuccess) return nullptr;
  return w;
}

extern "C" size_t gs_project_index_bytes(const gs_ctx* c, int64_t n, int n_views) {
  if (!c || n < 0 || n_views < 1) return 0;
  return index_layout(n, n_views, c->world).bytes;
}

// Counting half, device part (gs_project, gs_project_count, gs_project_put_dev): bwd_index
// masks and per-CTA bucket bases, and *tot_dev = this rank's per-destination prefix [G + 1]
// on the device.  No host sync.
static gs_status project_count_launch(gs_ctx* c, const gs_params* p, const gs_camera* cams_h, int n_views,
                                      const int64_t* dp_h, void* bwd_index, cudaStream_t st, int64_t** tot_dev) {
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, p, "null argument");
  const int G = c->world, b = n_views, nb = b * G;
  GS_REQUIRE(c, nb <= kMaxBuckets, "n_views * world = %d exceeds %d", nb, kMaxBuckets);
  int64_t* tot = (int64_t*)gs_slot_get(c, SLOT_PROJ_TMP, (GS_MAX_WORLD + 1) * sizeof(int64_t), st);
  if (!tot) return gs_fail(c, GS_ECUDA, "scratch");
  *tot_dev = tot;
  if (p->n == 0) {
    GS_CUDA(c, cudaMemsetAsync(tot, 0, (GS_MAX_WORLD + 1) * sizeof(int64_t), st));
    return GS_OK;
  }
  GS_REQUIRE(c, bwd_index && p->pos_op && p->log_scale && p->rot && p->sh, "null buffer");
  gs_index_layout L = index_layout(p->n, b, G);
  uint32_t* maskw = (uint32_t*)bwd_index;
  int64_t* base = (int64_t*)((char*)bwd_index + L.base_off);
  gs_cams_arg cams = make_cams(cams_h, n_views);
  gs_geom geo = gs_make_geom(&cams_h[0]);
  gs_dp_arg dp = gs_make_dp(c, dp_h);
  GS_CUDA(c, cudaMemsetAsync(base + (int64_t)nb * L.ncta, 0, sizeof(int64_t), st));
  unsigned long long* bad = nonfinite_word(c, st);
  if (!bad) return gs_fail(c, GS_ECUDA, "scratch");
  ++c->launches;
  k_project_count<<<(unsigned)L.ncta, kBlock, 0, st>>>(
      (const float4*)p->pos_op, (const float4*)p->log_scale, (const float4*)p->rot, p->n, cams, geo,
      dp, nb, L.NW, maskw, base, L.ncta, p->gid_base, bad);
  GS_LAUNCH_CHECK(c, "project_count");
  s = gs_scan_i64(c, base, base, (int64_t)nb * L.ncta + 1, 0, st);
  if (s != GS_OK) return s;
  ++c->launches;
  k_gather_totals<<<1, 64, 0, st>>>(base, L.ncta, b, G, tot);
  GS_LAUNCH_CHECK(c, "project totals");
  return GS_OK;
}

// The non-finite word read back with a count sync: GS_ENONFINITE naming the lowest gid (and
// the word reset) if set.
static gs_status nonfinite_result(gs_ctx* c, unsigned long long badv, cudaStream_t st) {
  if (badv == ~0ull) return GS_OK;  // this call's position / scale / rotation / opacity, or an earlier call's SH
  unsigned long long* bad = nonfinite_word(c, st);
  if (bad) GS_CUDA(c, cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
  return gs_fail(c, GS_ENONFINITE, "non-finite parameter at gid %lld", (long long)badv);
}

// Counting half with the read-back (gs_project, gs_project_count): per-destination counts to
// the host (one sync).
static gs_status project_count_phase(gs_ctx* c, const gs_params* p, const gs_camera* cams_h, int n_views,
                                     const int64_t* dp_h, int64_t* send_counts_h, void* bwd_index,
                                     cudaStream_t st, int64_t* total_h) {
  GS_REQUIRE(c, send_counts_h, "null argument");
  const int G = c->world;
  for (int d = 0; d < G; d++) send_counts_h[d] = 0;
  *total_h = 0;
  int64_t* tot = nullptr;
  gs_status s = project_count_launch(c, p, cams_h, n_views, dp_h, bwd_index, st, &tot);
  if (s != GS_OK) return s;
  if (p->n == 0) return GS_OK;
  unsigned long long* bad = nonfinite_word(c, st);
  if (!bad) return gs_fail(c, GS_ECUDA, "scratch");
  GS_CUDA(c, cudaMemcpyAsync(c->pinned, tot, (G + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaMemcpyAsync(c->pinned + GS_MAX_WORLD + 1, bad, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  s = nonfinite_result(c, (unsigned long long)c->pinned[GS_MAX_WORLD + 1], st);
  if (s != GS_OK) return s;
  for (int d = 0; d < G; d++) send_counts_h[d] = c->pinned[d + 1] - c->pinned[d];
  *total_h = c->pinned[G];
  if (*total_h >= (1ll << 31))
    return gs_fail(c, GS_ENOTSUP, "%lld records exceed int32 positions", (long long)*total_h);
  return GS_OK;
}

// Writing half: records of the counted batch to outs (see gs_outs).
static gs_status project_write_phase(gs_ctx* c, const gs_params* p, const gs_camera* cams_h, int n_views,
                                     const void* bwd_index, const gs_outs& outs, cudaStream_t st) {
  const int G = c->world, b = n_views, nb = b * G;
  gs_index_layout L = index_layout(p->n, b, G);
  const uint32_t* maskw = (const uint32_t*)bwd_index;
  const int64_t* base = (const int64_t*)((const char*)bwd_index + L.base_off);
  gs_cams_arg cams = make_cams(cams_h, n_views);
  gs_geom geo = gs_make_geom(&cams_h[0]);
  ++c->launches;
  gs_devouts dv;
  memset(&dv, 0, sizeof(dv));
  k_project_write<false><<<(unsigned)L.ncta, kBlock, 0, st>>>(
      (const float4*)p->pos_op, (const float4*)p->log_scale, (const float4*)p->rot,
      (const float4*)p->sh, p->n, p->gid_base, cams, geo, G, nb, L.NW, maskw, base, L.ncta, outs,
      nonfinite_word(c, st), dv);
  GS_LAUNCH_CHECK(c, "project_write");
  return GS_OK;
}

extern "C" gs_status gs_project(gs_ctx* c, const gs_params* p, const gs_camera* cams_h,
                                int n_views, const int64_t* dp_h, void* send_rec, int64_t send_cap,
                                int64_t* send_counts_h, void* bwd_index, void* stream) {
  if (!c) return GS_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t total = 0;
  gs_status s = project_count_phase(c, p, cams_h, n_views, dp_h, send_counts_h, bwd_index, st, &total);
  if (s != GS_OK) return s;
  if (total > send_cap)
    return gs_fail(c, GS_ECAPACITY, "send capacity %lld < %lld records", (long long)send_cap,
                   (long long)total);
  if (total == 0) return GS_OK;
  GS_REQUIRE(c, send_rec != nullptr, "null send_rec");
  gs_outs outs;
  for (int d = 0; d < GS_MAX_WORLD; d++) outs.d[d] = (gs_rec*)send_rec;
  return project_write_phase(c, p, cams_h, n_views, bwd_index, outs, st);
}

extern "C" gs_status gs_project_count(gs_ctx* c, const gs_params* p, const gs_camera* cams_h, int n_views,
                                      const int64_t* dp_h, int64_t* send_counts_h, void* bwd_index, void* stream) {
  if (!c) return GS_EINVAL;
  int64_t total = 0;
  return project_count_phase(c, p, cams_h, n_views, dp_h, send_counts_h, bwd_index, (cudaStream_t)stream, &total);
}

extern "C" gs_status gs_project_put(gs_ctx* c, const gs_params* p, const gs_camera* cams_h, int n_views,
                                    const int64_t* dp_h, const void* bwd_index, void* stream) {
  if (!c) return GS_EINVAL;
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, p, "null argument");
  GS_REQUIRE(c, c->p2p.attached && c->p2p.planned, "gs_project_put needs gs_p2p_attach and gs_p2p_plan");
  const int G = c->world, r = c->rank;
  int64_t seg[GS_MAX_WORLD + 1], put[GS_MAX_WORLD], soff[GS_MAX_WORLD + 1], own[GS_MAX_WORLD];
  s = gs_p2p_offsets(c->p2p.counts.data(), G, r, seg, put, soff, own);
  if (s != GS_OK) return gs_fail(c, s, "bad plan");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n_send = soff[G];
  if (n_send > 0) {  // zero the own gradient rows before any peer's backward adds into them
    GS_REQUIRE(c, c->p2p.dsend[r] != nullptr, "null dL/dsend");
    GS_CUDA(c, cudaMemsetAsync(c->p2p.dsend[r], 0, (size_t)n_send * 9 * sizeof(float), st));
  }
  if (p->n == 0 || n_send == 0) return GS_OK;
  GS_REQUIRE(c, bwd_index && p->pos_op && p->log_scale && p->rot && p->sh, "null buffer");
  gs_outs outs;
  for (int d = 0; d < GS_MAX_WORLD; d++) outs.d[d] = nullptr;
  for (int d = 0; d < G; d++)
    if (soff[d + 1] > soff[d]) {
      GS_REQUIRE(c, c->p2p.recv[d] != nullptr, "rank %d has no receive buffer", d);
      outs.d[d] = (gs_rec*)c->p2p.recv[d] + (put[d] - soff[d]);
    }
  return project_write_phase(c, p, cams_h, n_views, bwd_index, outs, st);
}

namespace {
// dL/dsend rows [0, n_send) of this rank zeroed for the peers' reductions, n_send from the
// device matrix (row `rank`); nothing if it exceeds the capacity (gs_p2p_counts reports it).
__global__ void k_zero_dsend(float* __restrict__ dsend, const int64_t* __restrict__ cmat, int G, int rank,
                             long long cap) {
  long long n = 0;
  for (int d = 0; d < G; d++) n += cmat[rank * G + d];
  if (n > cap) return;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < 9 * n; i += (long long)gridDim.x * blockDim.x)
    dsend[i] = 0.f;
}
}  // namespace

extern "C" gs_status gs_project_put_dev(gs_ctx* c, const gs_params* p, const gs_camera* cams_h, int n_views,
                                        const int64_t* dp_h, void* bwd_index, void* stream) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, p, "null argument");
  gs_p2p_state& P = c->p2p;
  GS_REQUIRE(c, P.attached && P.counts_ev, "gs_project_put_dev needs gs_p2p_attach and gs_p2p_attach_counts");
  const int G = c->world, r = c->rank, b = n_views, nb = b * G;
  cudaStream_t st = (cudaStream_t)stream;
  P.planned = false;
  int64_t* tot = nullptr;
  gs_status s = project_count_launch(c, p, cams_h, n_views, dp_h, bwd_index, st, &tot);
  if (s != GS_OK) return s;
  // the count matrix on every rank's device: row r to every peer, barrier, async read-back
  s = gs_p2p_counts_exchange(c, tot, st);
  if (s != GS_OK) return s;
  unsigned long long* bad = nonfinite_word(c, st);
  if (!bad) return gs_fail(c, GS_ECUDA, "scratch");
  GS_CUDA(c, cudaMemcpyAsync(c->pinned + kCountsPinned + GS_MAX_WORLD * GS_MAX_WORLD, bad, sizeof(int64_t),
                             cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaEventRecord(P.counts_ev, st));
  GS_REQUIRE(c, P.dsend[r] != nullptr, "null dL/dsend");
  ++c->launches;
  k_zero_dsend<<<148 * 4, 256, 0, st>>>(P.dsend[r], P.cmat[r], G, r, (long long)P.dsend_cap[r]);
  if (p->n > 0) {
    gs_devouts dv;
    memset(&dv, 0, sizeof(dv));
    for (int d = 0; d < G; d++) {
      dv.recv[d] = (gs_rec*)P.recv[d];
      dv.cap[d] = P.recv_cap[d];
    }
    dv.cmat = P.cmat[r];
    dv.rank = r;
    gs_index_layout L = index_layout(p->n, b, G);
    gs_outs outs;
    memset(&outs, 0, sizeof(outs));
    gs_cams_arg cams = make_cams(cams_h, n_views);
    gs_geom geo = gs_make_geom(&cams_h[0]);
    ++c->launches;
    k_project_write<true><<<(unsigned)L.ncta, kBlock, 0, st>>>(
        (const float4*)p->pos_op, (const float4*)p->log_scale, (const float4*)p->rot, (const float4*)p->sh, p->n,
        p->gid_base, cams, geo, G, nb, L.NW, (const uint32_t*)bwd_index,
        (const int64_t*)((const char*)bwd_index + L.base_off), L.ncta, outs, bad, dv);
  }
  GS_LAUNCH_CHECK(c, "project_put_dev");
  return GS_OK;
}
