// gs_exchange.cu -- A2/A6 sparse all-to-all exchanges and A9 dynamic
// pixel-tile load balancing (Algorithm 1).
//
// Exchanges are grouped NCCL point-to-point calls over NVLink/NVSwitch: only the records a
// peer's pixel partition needs cross the fabric ("sparse all-to-all"), the self
// bucket is a device-to-device copy.  The count matrix is all-gathered first (the only host
// sync of A2); A6 reuses those counts (exact transpose, no sync).
#include "gs_device.cuh"
#include "gs_internal.h"

using namespace gsd;

#ifdef GS_WITH_NCCL
#define GS_NCCL(ctx, expr)                                                                  \
  do {                                                                                      \
    ncclResult_t _r = (expr);                                                               \
    if (_r != ncclSuccess) return gs_fail((ctx), GS_ENCCL, "%s: %s", #expr, ncclGetErrorString(_r)); \
  } while (0)
#endif

// Grouped point-to-point transfer: to peer g `scount[g]` units from sbuf + soff[g],
// from peer g `rcount[g]` units into rbuf + roff[g] (unit = `unit` bytes).
static gs_status p2p_exchange(gs_ctx* c, const char* sbuf, const int64_t* soff, const int64_t* scnt,
                              char* rbuf, const int64_t* roff, const int64_t* rcnt, size_t unit,
                              cudaStream_t st) {
  const int G = c->world, r = c->rank;
  if (scnt[r] > 0 && (sbuf + soff[r] * unit) != (rbuf + roff[r] * unit))
    GS_CUDA(c, cudaMemcpyAsync(rbuf + roff[r] * unit, sbuf + soff[r] * unit, scnt[r] * unit,
                               cudaMemcpyDeviceToDevice, st));
  if (G == 1) return GS_OK;
#ifdef GS_WITH_NCCL
  if (!c->comm) return gs_fail(c, GS_EINVAL, "virtual context (no communicator): collectives unavailable");
  GS_NCCL(c, ncclGroupStart());
  for (int g = 0; g < G; g++) {
    if (g == r) continue;
    if (scnt[g] > 0) GS_NCCL(c, ncclSend(sbuf + soff[g] * unit, scnt[g] * unit, ncclChar, g, c->comm, st));
    if (rcnt[g] > 0) GS_NCCL(c, ncclRecv(rbuf + roff[g] * unit, rcnt[g] * unit, ncclChar, g, c->comm, st));
  }
  GS_NCCL(c, ncclGroupEnd());
  return GS_OK;
#else
  return gs_fail(c, GS_ENOTSUP, "built without NCCL");
#endif
}

extern "C" gs_status gs_exchange(gs_ctx* c, const void* send_rec, const int64_t* send_counts_h,
                                 void* recv_rec, int64_t recv_cap, int64_t* recv_counts_h,
                                 int64_t* n_recv_h, void* stream) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, send_counts_h && recv_counts_h && n_recv_h, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int G = c->world, r = c->rank;
  int64_t mat[GS_MAX_WORLD * GS_MAX_WORLD];
  if (G == 1) {
    mat[0] = send_counts_h[0];
  } else {
#ifdef GS_WITH_NCCL
    if (!c->comm) return gs_fail(c, GS_EINVAL, "virtual context (no communicator): collectives unavailable");
    int64_t* dbuf = (int64_t*)gs_slot_get(c, SLOT_COUNT_GATHER, (G + G * G) * sizeof(int64_t), st);
    if (!dbuf) return gs_fail(c, GS_ECUDA, "scratch");
    for (int g = 0; g < G; g++) c->pinned[g] = send_counts_h[g];
    GS_CUDA(c, cudaMemcpyAsync(dbuf, c->pinned, G * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    GS_NCCL(c, ncclAllGather(dbuf, dbuf + G, G, ncclInt64, c->comm, st));
    GS_CUDA(c, cudaMemcpyAsync(c->pinned + 64, dbuf + G, G * G * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, st));
    GS_CUDA(c, cudaStreamSynchronize(st));
    for (int k = 0; k < G * G; k++) mat[k] = c->pinned[64 + k];
#else
    return gs_fail(c, GS_ENOTSUP, "built without NCCL");
#endif
  }
  int64_t soff[GS_MAX_WORLD + 1], roff[GS_MAX_WORLD + 1], scnt[GS_MAX_WORLD], rcnt[GS_MAX_WORLD];
  if (gs_exchange_plan(mat, G, r, soff, roff) != GS_OK) return gs_fail(c, GS_EINVAL, "bad counts");
  for (int g = 0; g < G; g++) {
    scnt[g] = mat[r * G + g];
    rcnt[g] = mat[g * G + r];
    recv_counts_h[g] = rcnt[g];
  }
  *n_recv_h = roff[G];
  if (roff[G] > recv_cap)
    return gs_fail(c, GS_ECAPACITY, "recv capacity %lld < %lld", (long long)recv_cap, (long long)roff[G]);
  if (roff[G] + soff[G] == 0) return GS_OK;
  GS_REQUIRE(c, send_rec && recv_rec, "null record buffer");
  return p2p_exchange(c, (const char*)send_rec, soff, scnt, (char*)recv_rec, roff, rcnt,
                      GS_RECORD_BYTES, st);
}

extern "C" gs_status gs_exchange_grads(gs_ctx* c, const float* dL_drec, const int64_t* recv_counts_h,
                                       const int64_t* send_counts_h, float* dL_dsend, void* stream) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, recv_counts_h && send_counts_h, "null counts");
  const int G = c->world;
  int64_t soff[GS_MAX_WORLD + 1], roff[GS_MAX_WORLD + 1];
  soff[0] = roff[0] = 0;
  for (int g = 0; g < G; g++) {
    roff[g + 1] = roff[g] + recv_counts_h[g];
    soff[g + 1] = soff[g] + send_counts_h[g];
  }
  if (roff[G] + soff[G] == 0) return GS_OK;
  GS_REQUIRE(c, dL_drec && dL_dsend, "null gradient buffer");
  // transpose: what I received from s goes back to s; what I sent to d comes back from d
  return p2p_exchange(c, (const char*)dL_drec, roff, recv_counts_h, (char*)dL_dsend, soff,
                      send_counts_h, GS_GRAD_FLOATS * sizeof(float), (cudaStream_t)stream);
}

// ------------------------------------------------------------------ A9 rebalance
namespace {
struct gs_ids {
  int id[GS_MAX_VIEWS];
};

__device__ __forceinline__ int64_t block_npix(int64_t loc, const gs_geom& g) {
  int tx = (int)(loc % g.Wt), ty = (int)(loc / g.Wt);
  return (int64_t)min(16, g.W - tx * 16) * min(16, g.H - ty * 16);
}

__global__ void k_rank_sums(const int64_t* row, gs_dp_arg dp, gs_geom geo, int64_t* sums) {
  // one CTA per rank: C_g = sum of its block costs, N_g = its in-image pixels
  __shared__ long long s[2][256];
  int g = blockIdx.x;
  long long cs = 0, ns = 0;
  for (long long i = dp.dp[g] + threadIdx.x; i < dp.dp[g + 1]; i += blockDim.x) {
    cs += row[i];
    ns += block_npix(i % geo.per_view, geo);
  }
  s[0][threadIdx.x] = cs;
  s[1][threadIdx.x] = ns;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s[0][threadIdx.x] += s[0][threadIdx.x + o];
      s[1][threadIdx.x] += s[1][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sums[2 * g] = s[0][0];
    sums[2 * g + 1] = s[1][0];
  }
}

__global__ void k_costs_to_history(const int64_t* row, int64_t B, gs_geom geo, gs_ids ids, int mode,
                                   gs_dp_arg dp, const int64_t* sums, int64_t* history) {
  int64_t beta = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (beta >= B) return;
  int64_t v = beta / geo.per_view, loc = beta % geo.per_view;
  int64_t et = row[beta];
  if (mode == GS_COST_PAPER_AVG) {
    // per-pixel average of the owning rank, times the block's pixels
    int g = 0;
    while (g + 1 < dp.G && dp.dp[g + 1] <= beta) g++;
    int64_t Cg = sums[2 * g], Ng = sums[2 * g + 1];
    et = Ng > 0 ? (Cg * block_npix(loc, geo)) / Ng : 0;
  }
  history[(int64_t)ids.id[v] * geo.per_view + loc] = et;
}

__global__ void k_next_et(const int64_t* history, int64_t Bn, gs_geom geo, gs_ids ids, int64_t* et) {
  int64_t beta = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (beta >= Bn) return;
  int64_t v = beta / geo.per_view, loc = beta % geo.per_view;
  int64_t h = history[(int64_t)ids.id[v] * geo.per_view + loc];
  et[beta] = h >= 0 ? h : block_npix(loc, geo);  // unseen image: its pixel count
}

__global__ void k_division_points(const int64_t* CT, int64_t B, int G, int64_t* dp) {
  // Algorithm 1 on the inclusive prefix CT: DP[g] = #{i : CT[i] * G <= g * tot}
  int g = threadIdx.x;
  if (g > G) return;
  int64_t tot = B > 0 ? CT[B - 1] : 0;
  if (g == 0) { dp[0] = 0; return; }
  if (g == G) { dp[G] = B; return; }
  if (tot == 0) { dp[g] = (int64_t)g * B / G; return; }
  int64_t th = (int64_t)g * tot, lo = 0, hi = B;  // first i with CT[i]*G > th
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (CT[mid] * (int64_t)G <= th) lo = mid + 1; else hi = mid;
  }
  dp[g] = lo;
}
}  // namespace

extern "C" gs_status gs_rebalance(gs_ctx* c, const int64_t* owned_tile_cost, const gs_camera* cams_h,
                                  int n_views, const int64_t* dp_h, int64_t* history, int64_t n_images,
                                  int cost_mode, const gs_camera* next_cams_h, int n_next,
                                  int64_t* dp_next_h, void* stream) {
  if (!c) return GS_EINVAL;
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, next_cams_h && n_next >= 1 && n_next <= GS_MAX_VIEWS && dp_next_h && history,
             "bad next batch / null argument");
  GS_REQUIRE(c, cost_mode >= 0 && cost_mode <= 2, "cost_mode %d", cost_mode);
  for (int v = 0; v < n_next; v++)
    GS_REQUIRE(c, next_cams_h[v].width == cams_h[0].width && next_cams_h[v].height == cams_h[0].height,
               "all images must share one size");
  gs_ids ids, nids;
  for (int v = 0; v < n_views; v++) {
    GS_REQUIRE(c, cams_h[v].image_id >= 0 && cams_h[v].image_id < n_images, "image_id out of range");
    ids.id[v] = cams_h[v].image_id;
  }
  for (int v = 0; v < n_next; v++) {
    GS_REQUIRE(c, next_cams_h[v].image_id >= 0 && next_cams_h[v].image_id < n_images,
               "image_id out of range");
    nids.id[v] = next_cams_h[v].image_id;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int G = c->world, r = c->rank;
  gs_geom geo = gs_make_geom(&cams_h[0]);
  gs_dp_arg dp = gs_make_dp(c, dp_h);
  const int64_t B = geo.per_view * n_views, Bn = geo.per_view * n_next;
  int64_t* row = (int64_t*)gs_slot_get(c, SLOT_ROW, B * sizeof(int64_t), st);
  int64_t* et = (int64_t*)gs_slot_get(c, SLOT_ET, Bn * sizeof(int64_t), st);
  int64_t* ct = (int64_t*)gs_slot_get(c, SLOT_CT, Bn * sizeof(int64_t), st);
  int64_t* misc = (int64_t*)gs_slot_get(c, SLOT_MISC, (4 * GS_MAX_WORLD + 8) * sizeof(int64_t), st);
  if (!row || !et || !ct || !misc) return gs_fail(c, GS_ECUDA, "scratch");
  // 1. the whole cost row: own segment, then all-gather of the others' (allgatherv)
  int64_t cnt[GS_MAX_WORLD], off[GS_MAX_WORLD + 1];
  for (int g = 0; g < G; g++) {
    cnt[g] = dp_h[g + 1] - dp_h[g];
    off[g] = dp_h[g];
  }
  off[G] = B;
  if (cnt[r] > 0) {
    GS_REQUIRE(c, owned_tile_cost != nullptr, "null owned_tile_cost");
    GS_CUDA(c, cudaMemcpyAsync(row + off[r], owned_tile_cost, cnt[r] * sizeof(int64_t),
                               cudaMemcpyDeviceToDevice, st));
  }
  if (G > 1) {
    int64_t scnt[GS_MAX_WORLD], soff[GS_MAX_WORLD];
    for (int g = 0; g < G; g++) {
      scnt[g] = g == r ? 0 : cnt[r];
      soff[g] = off[r];
    }
    int64_t rc[GS_MAX_WORLD];
    for (int g = 0; g < G; g++) rc[g] = g == r ? 0 : cnt[g];
    s = p2p_exchange(c, (const char*)row, soff, scnt, (char*)row, off, rc, sizeof(int64_t), st);
    if (s != GS_OK) return s;
  }
  // 2. estimates of the rendered blocks -> history
  if (cost_mode == GS_COST_PAPER_AVG) {
    ++c->launches;
    k_rank_sums<<<G, 256, 0, st>>>(row, dp, geo, misc);
  }
  if (B > 0) {
    ++c->launches;
    k_costs_to_history<<<(unsigned)((B + 255) / 256), 256, 0, st>>>(row, B, geo, ids, cost_mode, dp,
                                                                     misc, history);
  }
  // 3. ET of the next batch, Algorithm 1
  ++c->launches;
  k_next_et<<<(unsigned)((Bn + 255) / 256), 256, 0, st>>>(history, Bn, geo, nids, et);
  GS_LAUNCH_CHECK(c, "rebalance");
  s = gs_scan_i64(c, et, ct, Bn, 1, st);
  if (s != GS_OK) return s;
  int64_t* ddp = misc + 2 * GS_MAX_WORLD + 2;
  ++c->launches;
  k_division_points<<<1, 64, 0, st>>>(ct, Bn, G, ddp);
  GS_LAUNCH_CHECK(c, "division_points");
  GS_CUDA(c, cudaMemcpyAsync(c->pinned, ddp, (G + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  for (int g = 0; g <= G; g++) dp_next_h[g] = c->pinned[g];
  return GS_OK;
}

// ------------------------------------------------------------------ NEXT-1 halo exchange
namespace {
__global__ void k_pack_blocks(const float* __restrict__ src, const int64_t* __restrict__ lbs, int64_t n, int fpb,
                              float* __restrict__ dst) {
  const int64_t i = blockIdx.x;
  if (i >= n) return;
  const float* s = src + lbs[i] * fpb;
  float* d = dst + i * fpb;
  for (int t = threadIdx.x; t < fpb; t += blockDim.x) d[t] = s[t];
}
}  // namespace

// Every rank's halo (gs_halo_blocks of its range) is filled by the blocks' owners: the plan
// of every peer is recomputed locally from dp (identical on every rank), so no counts are
// exchanged; blocks travel whole (fpb floats each) in ascending id order per peer.
extern "C" gs_status gs_halo_exchange(gs_ctx* c, const float* data, int fpb, const gs_camera* cams_h, int n_views,
                                      const int64_t* dp_h, float* halo, int64_t* halo_ids, int64_t halo_cap,
                                      int64_t* n_halo_h, void* stream) {
  if (!c) return GS_EINVAL;
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, n_halo_h != nullptr, "null n_halo_h");
  GS_REQUIRE(c, fpb > 0, "floats per block must be > 0");
  cudaStream_t st = (cudaStream_t)stream;
  const gs_geom geo = gs_make_geom(&cams_h[0]);
  const int G = c->world, r = c->rank;
  const int64_t lo = dp_h[r], hi = dp_h[r + 1];
  std::vector<int64_t> need;
  gs_halo_blocks(geo, lo, hi, need);
  *n_halo_h = (int64_t)need.size();
  if ((int64_t)need.size() > halo_cap)
    return gs_fail(c, GS_ECAPACITY, "halo capacity %lld < %lld", (long long)halo_cap, (long long)need.size());
  if (G == 1) return GS_OK;  // a single rank owns every block: no halo
  GS_REQUIRE(c, need.empty() || (halo && halo_ids), "null halo buffers");
  // receive side: need is ascending, owners are ascending ranges -> contiguous per peer
  std::vector<int64_t> rcnt(G, 0), roff(G, 0), scnt(G, 0), soff(G, 0), send_lb;
  for (int64_t b : need) {
    int g = 0;
    while (!(b >= dp_h[g] && b < dp_h[g + 1])) g++;
    rcnt[g]++;
  }
  for (int g = 1; g < G; g++) roff[g] = roff[g - 1] + rcnt[g - 1];
  // send side: the owned blocks in each peer's halo
  std::vector<int64_t> peer;
  for (int g = 0; g < G; g++) {
    soff[g] = (int64_t)send_lb.size();
    if (g == r) continue;
    gs_halo_blocks(geo, dp_h[g], dp_h[g + 1], peer);
    for (int64_t b : peer)
      if (b >= lo && b < hi) send_lb.push_back(b - lo);
    scnt[g] = (int64_t)send_lb.size() - soff[g];
  }
  if (!need.empty())
    GS_CUDA(c, cudaMemcpyAsync(halo_ids, need.data(), need.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  float* sbuf = nullptr;
  if (!send_lb.empty()) {
    int64_t* idx = (int64_t*)gs_slot_get(c, SLOT_HALO_IDX, send_lb.size() * sizeof(int64_t), st);
    sbuf = (float*)gs_slot_get(c, SLOT_HALO_SEND, send_lb.size() * fpb * sizeof(float), st);
    if (!idx || !sbuf) return gs_fail(c, GS_ECUDA, "halo scratch");
    GS_CUDA(c, cudaMemcpyAsync(idx, send_lb.data(), send_lb.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    ++c->launches;
    k_pack_blocks<<<(unsigned)send_lb.size(), 256, 0, st>>>(data, idx, (int64_t)send_lb.size(), fpb, sbuf);
    GS_LAUNCH_CHECK(c, "halo pack");
  }  // (pageable host sources: cudaMemcpyAsync has staged them before returning)
  return p2p_exchange(c, (const char*)sbuf, soff.data(), scnt.data(), (char*)halo, roff.data(), rcnt.data(),
                      (size_t)fpb * sizeof(float), st);
}
