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
  int64_t caps[GS_MAX_WORLD];
  if (G == 1) {
    mat[0] = send_counts_h[0];
    caps[0] = recv_cap;
  } else {
#ifdef GS_WITH_NCCL
    if (!c->comm) return gs_fail(c, GS_EINVAL, "virtual context (no communicator): collectives unavailable");
    // every rank's send counts AND receive capacity: a capacity shortfall on any rank makes
    // every rank return GS_ECAPACITY together (a lone early return would leave its peers
    // blocked in the point-to-point phase)
    const int W1 = G + 1;
    int64_t* dbuf = (int64_t*)gs_slot_get(c, SLOT_COUNT_GATHER, (W1 + G * W1) * sizeof(int64_t), st);
    if (!dbuf) return gs_fail(c, GS_ECUDA, "scratch");
    for (int g = 0; g < G; g++) c->pinned[g] = send_counts_h[g];
    c->pinned[G] = recv_cap;
    GS_CUDA(c, cudaMemcpyAsync(dbuf, c->pinned, W1 * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    GS_NCCL(c, ncclAllGather(dbuf, dbuf + W1, W1, ncclInt64, c->comm, st));
    GS_CUDA(c, cudaMemcpyAsync(c->pinned + 64, dbuf + W1, G * W1 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GS_CUDA(c, cudaStreamSynchronize(st));
    for (int a = 0; a < G; a++) {
      for (int b2 = 0; b2 < G; b2++) mat[a * G + b2] = c->pinned[64 + a * W1 + b2];
      caps[a] = c->pinned[64 + a * W1 + G];
    }
#else
    return gs_fail(c, GS_ENOTSUP, "built without NCCL");
#endif
  }
  {
    bool short_any = false;
    for (int d = 0; d < G; d++) {
      int64_t need = 0;
      for (int g = 0; g < G; g++) need += mat[g * G + d];
      short_any |= need > caps[d];
    }
    if (short_any) {
      int64_t mine = 0;
      for (int g = 0; g < G; g++) mine += (recv_counts_h[g] = mat[g * G + r]);
      *n_recv_h = mine;
      return gs_fail(c, GS_ECAPACITY, "recv capacity short on some rank (this rank: %lld for %lld)",
                     (long long)recv_cap, (long long)mine);
    }
  }
  int64_t soff[GS_MAX_WORLD + 1], roff[GS_MAX_WORLD + 1], scnt[GS_MAX_WORLD], rcnt[GS_MAX_WORLD];
  if (gs_exchange_plan(mat, G, r, soff, roff) != GS_OK) return gs_fail(c, GS_EINVAL, "bad counts");
  for (int g = 0; g < G; g++) {
    scnt[g] = mat[r * G + g];
    rcnt[g] = mat[g * G + r];
    recv_counts_h[g] = rcnt[g];
  }
  *n_recv_h = roff[G];
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

// Per-pixel rate of the batch just rendered (R17): rate[0] = sum of its block estimates,
// rate[1] = its in-image pixels (one CTA).
__global__ void k_batch_rate(const int64_t* row, int64_t B, gs_geom geo, int64_t* rate) {
  __shared__ long long s[2][256];
  long long cs = 0, ns = 0;
  for (long long i = threadIdx.x; i < B; i += blockDim.x) {
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
    rate[0] = s[0][0];
    rate[1] = s[1][0];
  }
}

// ET of the next batch: the history, or for an image never rendered the batch's per-pixel
// rate times the block's pixels, in the cost mode's own units (R17; "uniform":
// equal cost per pixel); its pixel count when no cost was recorded yet (rate[0] == 0).
__global__ void k_next_et(const int64_t* history, int64_t Bn, gs_geom geo, gs_ids ids, const int64_t* rate,
                          int64_t* et) {
  int64_t beta = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (beta >= Bn) return;
  int64_t v = beta / geo.per_view, loc = beta % geo.per_view;
  int64_t h = history[(int64_t)ids.id[v] * geo.per_view + loc];
  const int64_t npix = block_npix(loc, geo);
  et[beta] = h >= 0 ? h : (rate[0] > 0 && rate[1] > 0 ? (int64_t)(((__int128)rate[0] * npix) / rate[1]) : npix);
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
  // every argument check before the collective, so no rank can fail it alone (the checks see
  // the same arguments on every rank)
  gs_status s = gs_check_batch(c, cams_h, n_views, dp_h);
  if (s != GS_OK) return s;
  GS_REQUIRE(c, next_cams_h && n_next >= 1 && n_next <= GS_MAX_VIEWS && dp_next_h && history,
             "bad next batch / null argument");
  GS_REQUIRE(c, cost_mode >= 0 && cost_mode <= 2, "cost_mode %d", cost_mode);
  for (int v = 0; v < n_next; v++)
    GS_REQUIRE(c, next_cams_h[v].width == cams_h[0].width && next_cams_h[v].height == cams_h[0].height,
               "all images must share one size");
  for (int v = 0; v < n_views; v++)
    GS_REQUIRE(c, cams_h[v].image_id >= 0 && cams_h[v].image_id < n_images, "image_id out of range");
  for (int v = 0; v < n_next; v++)
    GS_REQUIRE(c, next_cams_h[v].image_id >= 0 && next_cams_h[v].image_id < n_images, "image_id out of range");
  cudaStream_t st = (cudaStream_t)stream;
  const int G = c->world, r = c->rank;
  gs_geom geo = gs_make_geom(&cams_h[0]);
  const int64_t B = geo.per_view * n_views;
  int64_t* row = (int64_t*)gs_slot_get(c, SLOT_ROW, B * sizeof(int64_t), st);
  if (!row) return gs_fail(c, GS_ECUDA, "scratch");
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
  return gs_rebalance_row(c, row, cams_h, n_views, dp_h, history, n_images, cost_mode, next_cams_h, n_next,
                          dp_next_h, stream);
}

extern "C" gs_status gs_rebalance_row(gs_ctx* c, const int64_t* cost_row, const gs_camera* cams_h, int n_views,
                                      const int64_t* dp_h, int64_t* history, int64_t n_images, int cost_mode,
                                      const gs_camera* next_cams_h, int n_next, int64_t* dp_next_h, void* stream) {
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
  const int G = c->world;
  gs_geom geo = gs_make_geom(&cams_h[0]);
  gs_dp_arg dp = gs_make_dp(c, dp_h);
  const int64_t B = geo.per_view * n_views, Bn = geo.per_view * n_next;
  GS_REQUIRE(c, B == 0 || cost_row != nullptr, "null cost_row");
  int64_t* et = (int64_t*)gs_slot_get(c, SLOT_ET, Bn * sizeof(int64_t), st);
  int64_t* ct = (int64_t*)gs_slot_get(c, SLOT_CT, Bn * sizeof(int64_t), st);
  int64_t* misc = (int64_t*)gs_slot_get(c, SLOT_MISC, (4 * GS_MAX_WORLD + 8) * sizeof(int64_t), st);
  if (!et || !ct || !misc) return gs_fail(c, GS_ECUDA, "scratch");
  int64_t* rate = misc + 2 * GS_MAX_WORLD;  // [2]
  int64_t* ddp = misc + 2 * GS_MAX_WORLD + 2;
  // 2. estimates of the rendered blocks -> history, and the batch's per-pixel rate
  if (cost_mode == GS_COST_PAPER_AVG) {
    ++c->launches;
    k_rank_sums<<<G, 256, 0, st>>>(cost_row, dp, geo, misc);
  }
  if (B > 0) {
    ++c->launches;
    k_costs_to_history<<<(unsigned)((B + 255) / 256), 256, 0, st>>>(cost_row, B, geo, ids, cost_mode, dp,
                                                                     misc, history);
  }
  ++c->launches;
  k_batch_rate<<<1, 256, 0, st>>>(cost_row, B, geo, rate);
  // 3. ET of the next batch, Algorithm 1
  ++c->launches;
  k_next_et<<<(unsigned)((Bn + 255) / 256), 256, 0, st>>>(history, Bn, geo, nids, rate, et);
  GS_LAUNCH_CHECK(c, "rebalance");
  s = gs_scan_i64(c, et, ct, Bn, 1, st);
  if (s != GS_OK) return s;
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

// ------------------------------------------------------------------ NEXT-2 redistribution
// Random redistribution of the Gaussians after densification ("redistribute the 3D
// Gaussians after every few densification steps"; App. B.2 "random redistribution";
// S:491-497): global index j (the rank's gid_base + local index) moves to position pi(j) of
// the new global order, rank d owning [floor(d N / G), floor((d+1) N / G)) -- sizes differ by
// at most one.  pi is a keyed bijection of [0, N) computed per element (4-round Feistel
// network on the smallest even bit width covering N, cycle-walking into [0, N); reading R15),
// so no permutation table exists anywhere and every rank agrees without communication.
namespace {
__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}
__device__ __forceinline__ uint64_t feistel_perm(uint64_t j, uint64_t N, uint32_t seed, int half) {
  const uint32_t mask = (half >= 32) ? 0xffffffffu : ((1u << half) - 1u);
  uint64_t y = j;
  do {
    uint32_t Lh = (uint32_t)(y >> half) & mask, Rh = (uint32_t)y & mask;
    for (uint32_t r = 0; r < 4; r++) {
      const uint32_t f = fmix32(seed ^ (r * 0x9e3779b9u) ^ fmix32(Rh + 0x7f4a7c15u * (r + 1))) & mask;
      const uint32_t t = Lh ^ f;
      Lh = Rh;
      Rh = t;
    }
    y = ((uint64_t)Lh << half) | Rh;
  } while (y >= N);
  return y;
}
__host__ __device__ __forceinline__ int64_t range_lo(int d, int64_t N, int G) { return (int64_t)d * N / G; }

constexpr int kRedistFloats = 184;  // [new index: 2 floats][pad 2][p 60][m 60][v 60]

struct rplanes {
  const float4 *pos_op, *ls, *rot, *sh;
};
struct wrplanes {
  float4 *pos_op, *ls, *rot, *sh;
};
__device__ __forceinline__ void put60(float* d, const rplanes& p, int64_t n, int64_t i) {
  float4* o = reinterpret_cast<float4*>(d);
  o[0] = p.pos_op[i];
  o[1] = p.ls[i];
  o[2] = p.rot[i];
#pragma unroll
  for (int k = 0; k < 12; k++) o[3 + k] = p.sh[(int64_t)k * n + i];
}
__device__ __forceinline__ void get60(const float* s, const wrplanes& p, int64_t n, int64_t i) {
  const float4* o = reinterpret_cast<const float4*>(s);
  p.pos_op[i] = o[0];
  p.ls[i] = o[1];
  p.rot[i] = o[2];
#pragma unroll
  for (int k = 0; k < 12; k++) p.sh[(int64_t)k * n + i] = o[3 + k];
}

__global__ void k_redist_count(int64_t n, int64_t base, int64_t N, uint32_t seed, int half, int G,
                               int64_t* __restrict__ counts) {
  __shared__ int s_c[GS_MAX_WORLD];
  if (threadIdx.x < GS_MAX_WORLD) s_c[threadIdx.x] = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const uint64_t y = feistel_perm((uint64_t)(base + i), (uint64_t)N, seed, half);
    int d = (int)((y * (uint64_t)G) / (uint64_t)N);
    while (d + 1 < G && range_lo(d + 1, N, G) <= (int64_t)y) d++;
    while (d > 0 && range_lo(d, N, G) > (int64_t)y) d--;
    atomicAdd(&s_c[d], 1);
  }
  __syncthreads();
  if (threadIdx.x < G && s_c[threadIdx.x]) atomicAdd((unsigned long long*)&counts[threadIdx.x], (unsigned long long)s_c[threadIdx.x]);
}

__global__ void k_redist_pack(rplanes P, rplanes M, rplanes V, int64_t n, int64_t base, int64_t N, uint32_t seed,
                              int half, int G, int64_t* __restrict__ cursor, float* __restrict__ buf) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t y = feistel_perm((uint64_t)(base + i), (uint64_t)N, seed, half);
  int d = (int)((y * (uint64_t)G) / (uint64_t)N);
  while (d + 1 < G && range_lo(d + 1, N, G) <= (int64_t)y) d++;
  while (d > 0 && range_lo(d, N, G) > (int64_t)y) d--;
  const int64_t slot = (int64_t)atomicAdd((unsigned long long*)&cursor[d], 1ull);  // any order: placement is by index
  float* rec = buf + slot * kRedistFloats;
  const int64_t local = (int64_t)y - range_lo(d, N, G);
  reinterpret_cast<int64_t*>(rec)[0] = local;
  put60(rec + 4, P, n, i);
  put60(rec + 64, M, n, i);
  put60(rec + 124, V, n, i);
}

__global__ void k_redist_unpack(const float* __restrict__ buf, int64_t n_recv, wrplanes P, wrplanes M, wrplanes V,
                                int64_t n_out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_recv) return;
  const float* rec = buf + r * kRedistFloats;
  const int64_t o = reinterpret_cast<const int64_t*>(rec)[0];
  if (o < 0 || o >= n_out) __trap();  // corrupt transfer: never a silent misplacement
  get60(rec + 4, P, n_out, o);
  get60(rec + 64, M, n_out, o);
  get60(rec + 124, V, n_out, o);
}

int feistel_half(int64_t N) {
  int k = 2;
  while (k < 64 && (1ll << k) < N) k++;
  if (k & 1) k++;
  return k / 2;
}
rplanes rp_of(const gs_params* q) {
  return rplanes{(const float4*)q->pos_op, (const float4*)q->log_scale, (const float4*)q->rot, (const float4*)q->sh};
}
wrplanes wp_of(gs_params* q) {
  return wrplanes{(float4*)q->pos_op, (float4*)q->log_scale, (float4*)q->rot, (float4*)q->sh};
}
}  // namespace

extern "C" gs_status gs_redistribute_pack(gs_ctx* c, const gs_params* p, const gs_params* m, const gs_params* v,
                                          int64_t n_total, uint64_t seed, void* send_buf, int64_t cap,
                                          int64_t* send_counts_h, void* stream) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, p && m && v && send_counts_h, "null argument");
  GS_REQUIRE(c, m->n == p->n && v->n == p->n, "m/v mis-sized");
  GS_REQUIRE(c, n_total >= p->gid_base + p->n && n_total < (1ll << 32), "n_total out of range");
  cudaStream_t st = (cudaStream_t)stream;
  const int G = c->world;
  const int64_t n = p->n;
  int64_t* cnt = (int64_t*)gs_slot_get(c, SLOT_MISC, 2 * GS_MAX_WORLD * sizeof(int64_t), st);
  if (!cnt) return gs_fail(c, GS_ECUDA, "scratch");
  GS_CUDA(c, cudaMemsetAsync(cnt, 0, 2 * GS_MAX_WORLD * sizeof(int64_t), st));
  const int half = feistel_half(n_total);
  const uint32_t sd = (uint32_t)(seed ^ (seed >> 32));
  if (n > 0) {
    ++c->launches;
    k_redist_count<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, p->gid_base, n_total, sd, half, G, cnt);
  }
  GS_CUDA(c, cudaMemcpyAsync(c->pinned, cnt, G * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  int64_t tot = 0;
  for (int g = 0; g < G; g++) {
    send_counts_h[g] = c->pinned[g];
    c->pinned[GS_MAX_WORLD + g] = tot;  // cursors = exclusive prefix
    tot += c->pinned[g];
  }
  if (tot > cap) return gs_fail(c, GS_ECAPACITY, "redistribution send capacity %lld < %lld", (long long)cap,
                                (long long)tot);
  if (n == 0) return GS_OK;
  GS_REQUIRE(c, send_buf != nullptr, "null send_buf");
  GS_CUDA(c, cudaMemcpyAsync(cnt + GS_MAX_WORLD, c->pinned + GS_MAX_WORLD, G * sizeof(int64_t),
                             cudaMemcpyHostToDevice, st));
  ++c->launches;
  k_redist_pack<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rp_of(p), rp_of(m), rp_of(v), n, p->gid_base, n_total,
                                                            sd, half, G, cnt + GS_MAX_WORLD, (float*)send_buf);
  GS_LAUNCH_CHECK(c, "redistribute pack");
  return GS_OK;
}

extern "C" gs_status gs_redistribute_unpack(gs_ctx* c, const void* recv_buf, int64_t n_recv, gs_params* p_out,
                                            gs_params* m_out, gs_params* v_out, void* stream) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, p_out && m_out && v_out, "null argument");
  GS_REQUIRE(c, n_recv == p_out->n && m_out->n == p_out->n && v_out->n == p_out->n,
             "outputs must hold exactly the received Gaussians");
  if (n_recv == 0) return GS_OK;
  GS_REQUIRE(c, recv_buf != nullptr, "null recv_buf");
  ++c->launches;
  k_redist_unpack<<<(unsigned)((n_recv + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (const float*)recv_buf, n_recv, wp_of(p_out), wp_of(m_out), wp_of(v_out), p_out->n);
  GS_LAUNCH_CHECK(c, "redistribute unpack");
  return GS_OK;
}

extern "C" int64_t gs_redistribute_record_bytes(void) { return kRedistFloats * sizeof(float); }

extern "C" gs_status gs_redistribute(gs_ctx* c, const gs_params* p, const gs_params* m, const gs_params* v,
                                     uint64_t seed, void* send_buf, int64_t send_cap, void* recv_buf,
                                     int64_t recv_cap, gs_params* p_out, gs_params* m_out, gs_params* v_out,
                                     int64_t* n_total_h, int64_t* n_out_h, void* stream) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, p && n_total_h && n_out_h, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int G = c->world, r = c->rank;
  if (G == 1) {  // nothing to move: the single shard is already the new order's owner
    *n_total_h = *n_out_h = p->n;
    return gs_fail(c, GS_ENOTSUP, "world 1: redistribution is the identity, keep the shard");
  }
#ifdef GS_WITH_NCCL
  if (!c->comm) return gs_fail(c, GS_EINVAL, "virtual context (no communicator): collectives unavailable");
  // local argument checks first: a rank returning after a collective would desynchronise them
  GS_REQUIRE(c, m && v && m->n == p->n && v->n == p->n, "m/v mis-sized");
  GS_REQUIRE(c, recv_buf == nullptr || (send_buf != nullptr || p->n == 0) && send_cap >= p->n,
             "send buffer must hold the shard");
  // shard sizes -> N and this rank's global base (every rank's gid ranges are contiguous)
  int64_t* dbuf = (int64_t*)gs_slot_get(c, SLOT_COUNT_GATHER, (G + 1) * (G + 2) * sizeof(int64_t), st);
  if (!dbuf) return gs_fail(c, GS_ECUDA, "scratch");
  c->pinned[0] = p->n;
  GS_CUDA(c, cudaMemcpyAsync(dbuf, c->pinned, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  GS_NCCL(c, ncclAllGather(dbuf, dbuf + 1, 1, ncclInt64, c->comm, st));
  GS_CUDA(c, cudaMemcpyAsync(c->pinned + 64, dbuf + 1, G * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  int64_t N = 0, base = 0;
  for (int g = 0; g < G; g++) {
    if (g == r) base = N;
    N += c->pinned[64 + g];
  }
  *n_total_h = N;
  const int64_t n_out = range_lo(r + 1, N, G) - range_lo(r, N, G);
  *n_out_h = n_out;
  if (recv_buf == nullptr) return GS_OK;  // size query (every rank passes NULL together)
  // The rank's global base comes from the gathered sizes (the caller's gid_base may be stale
  // after a densify changed the shard sizes).  Local checks that can differ between ranks are
  // agreed on before the next collective: every rank all-gathers its send counts plus a
  // status word, and all return the same error if any rank failed (no rank is left waiting).
  gs_params pb = *p;
  pb.gid_base = base;
  int64_t scnt[GS_MAX_WORLD] = {0};
  int64_t st_local = 0;
  std::string why;
  if (recv_cap < n_out) {
    st_local = GS_EINVAL;
    why = "receive capacity below the queried size";
  } else if (!(p_out && m_out && v_out && p_out->n == n_out && m_out->n == n_out && v_out->n == n_out)) {
    st_local = GS_EINVAL;
    why = "output planes not laid out for the queried size";
  } else {
    gs_status s = gs_redistribute_pack(c, &pb, m, v, N, seed, send_buf, send_cap, scnt, stream);
    if (s != GS_OK) {
      st_local = s;
      why = c->err;
      for (int g = 0; g < G; g++) scnt[g] = 0;
    }
  }
  // count matrix + status (all-gather of every rank's G send counts and its status)
  for (int g = 0; g < G; g++) c->pinned[g] = scnt[g];
  c->pinned[G] = st_local;
  GS_CUDA(c, cudaMemcpyAsync(dbuf, c->pinned, (G + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  GS_NCCL(c, ncclAllGather(dbuf, dbuf + G + 1, G + 1, ncclInt64, c->comm, st));
  GS_CUDA(c, cudaMemcpyAsync(c->pinned + 64, dbuf + G + 1, G * (G + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                             st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  for (int g = 0; g < G; g++) {
    const int64_t sg = c->pinned[64 + g * (G + 1) + G];
    if (sg != 0)
      return gs_fail(c, (gs_status)sg, "redistribution failed on rank %d%s%s", g, g == r ? ": " : "",
                     g == r ? why.c_str() : "");
  }
  int64_t soff[GS_MAX_WORLD], roff[GS_MAX_WORLD], rcnt[GS_MAX_WORLD];
  int64_t so = 0, ro = 0;
  for (int g = 0; g < G; g++) {
    soff[g] = so;
    so += scnt[g];
    rcnt[g] = c->pinned[64 + g * (G + 1) + r];
    roff[g] = ro;
    ro += rcnt[g];
  }
  if (ro != n_out) return gs_fail(c, GS_EINVAL, "redistribution counts inconsistent (%lld != %lld)", (long long)ro,
                                  (long long)n_out);
  gs_status s = p2p_exchange(c, (const char*)send_buf, soff, scnt, (char*)recv_buf, roff, rcnt, kRedistFloats * sizeof(float),
                   st);
  if (s != GS_OK) return s;
  p_out->gid_base = m_out->gid_base = v_out->gid_base = range_lo(r, N, G);
  return gs_redistribute_unpack(c, recv_buf, n_out, p_out, m_out, v_out, stream);
#else
  return gs_fail(c, GS_ENOTSUP, "built without NCCL");
#endif
}
