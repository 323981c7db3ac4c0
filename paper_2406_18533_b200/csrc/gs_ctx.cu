// gs_ctx.cu -- context, errors, scratch arena, host-only ABI functions, the int64 scan and
// the non-finite check.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <new>

#include "gs_device.cuh"
#include "gs_internal.h"

gs_status gs_fail(gs_ctx* c, gs_status s, const char* fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return s;
}

gs_status gs_cuda_check(gs_ctx* c, cudaError_t e, const char* what) {
  return gs_fail(c, GS_ECUDA, "CUDA error %s (%d) at %s", cudaGetErrorString(e), (int)e, what);
}

void* gs_slot_get(gs_ctx* c, int slot, size_t bytes, cudaStream_t st) {
  gs_slot& s = c->slot[slot];
  if (bytes == 0) bytes = 16;
  if (s.bytes >= bytes) return s.ptr;
  static const bool dbg = getenv("GS_DEBUG_SLOTS") != nullptr;
  if (dbg) fprintf(stderr, "libgs: slot %d grows %zu -> %zu bytes\n", slot, s.bytes, bytes + bytes / 2);
  if (s.ptr) {
    cudaStreamSynchronize(st);
    cudaFree(s.ptr);
    s.ptr = nullptr;
    s.bytes = 0;
  }
  // headroom against regrowth: pair and record counts drift up as training grows the
  // Gaussians (C2: +8 % pairs over 12 steps), and each regrowth of a GB-sized slot is a
  // synchronising cudaFree + cudaMalloc (15-60 ms) inside a step
  size_t want = bytes + bytes / 2;
  if (cudaMalloc(&s.ptr, want) != cudaSuccess) {
    cudaGetLastError();
    s.ptr = nullptr;
    return nullptr;
  }
  s.bytes = want;
  return s.ptr;
}

gs_status gs_check_batch(gs_ctx* c, const gs_camera* cams_h, int n_views, const int64_t* dp_h) {
  GS_REQUIRE(c, cams_h != nullptr && dp_h != nullptr, "null cameras or dp");
  GS_REQUIRE(c, n_views >= 1 && n_views <= GS_MAX_VIEWS, "n_views %d not in [1, %d]", n_views,
             GS_MAX_VIEWS);
  for (int v = 0; v < n_views; v++) {
    GS_REQUIRE(c, cams_h[v].width == cams_h[0].width && cams_h[v].height == cams_h[0].height,
               "views of one batch must share one image size (view %d)", v);
    GS_REQUIRE(c, cams_h[v].width > 0 && cams_h[v].height > 0, "empty image (view %d)", v);
  }
  gs_geom g = gs_make_geom(&cams_h[0]);
  long long B = g.per_view * n_views;
  GS_REQUIRE(c, dp_h[0] == 0 && dp_h[c->world] == B, "dp must start at 0 and end at B=%lld", B);
  for (int k = 0; k < c->world; k++)
    GS_REQUIRE(c, dp_h[k] <= dp_h[k + 1], "dp not monotone at %d", k);
  return GS_OK;
}

extern "C" {

int gs_version(void) { return 100; }

int64_t gs_launch_count(const gs_ctx* ctx) { return ctx ? ctx->launches : -1; }

const char* gs_last_error(const gs_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

gs_status gs_nccl_unique_id(uint8_t id_h[128]) {
#ifdef GS_WITH_NCCL
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return GS_ENCCL;
  static_assert(sizeof(id) == 128, "nccl id size");
  memcpy(id_h, &id, 128);
  return GS_OK;
#else
  (void)id_h;
  return GS_ENOTSUP;
#endif
}

gs_status gs_create(gs_ctx** out, int device, int rank, int world, const uint8_t* id_h) {
  if (!out || world < 1 || world > GS_MAX_WORLD || rank < 0 || rank >= world) return GS_EINVAL;
  gs_ctx* c = new (std::nothrow) gs_ctx();
  if (!c) return GS_EINVAL;
  c->device = device;
  c->rank = rank;
  c->world = world;
  *out = c;
  if (cudaSetDevice(device) != cudaSuccess) return gs_fail(c, GS_ECUDA, "cudaSetDevice(%d)", device);
  if (cudaMallocHost(&c->pinned, 8192 * sizeof(int64_t)) != cudaSuccess)
    return gs_fail(c, GS_ECUDA, "cudaMallocHost");
  if (world > 1 && id_h) {  // id_h == NULL: a "virtual" rank (no communicator; local calls only)
#ifdef GS_WITH_NCCL
    ncclUniqueId id;
    memcpy(&id, id_h, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) return gs_fail(c, GS_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
#else
    return gs_fail(c, GS_ENOTSUP, "built without NCCL");
#endif
  }
  return GS_OK;
}

void gs_destroy(gs_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (int s = 0; s < SLOT_N; s++)
    if (c->slot[s].ptr) cudaFree(c->slot[s].ptr);
  if (c->p2p.counts_ev) cudaEventDestroy(c->p2p.counts_ev);
  if (c->pinned) cudaFreeHost(c->pinned);
  for (void* q : c->p2p.opened) cudaIpcCloseMemHandle(q);
  if (c->p2p.err) cudaFree(c->p2p.err);
  for (int k = 0; k < 5; k++)
    if (c->p2p.sym[k]) cudaFree(c->p2p.sym[k]);
#ifdef GS_WITH_NCCL
  if (c->comm) ncclCommDestroy(c->comm);
#endif
  delete c;
}

gs_status gs_division_points(const int64_t* ET_h, int64_t B, int G, int64_t* DP_h) {
  // Algorithm 1: CT = cumsum(ET); TH[g] = g * CT[B-1] / G; DP = searchsorted.
  // Right bisection evaluated exactly as CT[i] * G <= g * tot (R8); DP[0] = 0, DP[G] = B.
  if (G < 1 || B < 0 || !DP_h || (B > 0 && !ET_h)) return GS_EINVAL;
  int64_t mx = 0, tot = 0;
  for (int64_t i = 0; i < B; i++) {
    if (ET_h[i] < 0) return GS_EINVAL;
    if (ET_h[i] > mx) mx = ET_h[i];
  }
  if (B > 0 && mx > 0 && (double)B * (double)mx * (double)G >= 9.2e18) return GS_EINVAL;
  for (int64_t i = 0; i < B; i++) tot += ET_h[i];
  DP_h[0] = 0;
  DP_h[G] = B;
  if (tot == 0) {
    for (int g = 1; g < G; g++) DP_h[g] = (int64_t)g * B / G;
    return GS_OK;
  }
  // one pass: CT is non-decreasing, so each threshold's count is a running pointer
  int64_t ct = 0, i = 0;
  for (int g = 1; g < G; g++) {
    const int64_t th = (int64_t)g * tot;
    while (i < B && (ct + ET_h[i]) * (int64_t)G <= th) ct += ET_h[i++];
    DP_h[g] = i;
  }
  return GS_OK;
}

gs_status gs_exchange_plan(const int64_t* counts_h, int G, int rank, int64_t* send_off_h,
                           int64_t* recv_off_h) {
  if (!counts_h || G < 1 || rank < 0 || rank >= G || !send_off_h || !recv_off_h) return GS_EINVAL;
  send_off_h[0] = recv_off_h[0] = 0;
  for (int g = 0; g < G; g++) {
    if (counts_h[rank * G + g] < 0 || counts_h[g * G + rank] < 0) return GS_EINVAL;
    send_off_h[g + 1] = send_off_h[g] + counts_h[rank * G + g];  // my bucket for dst g
    recv_off_h[g + 1] = recv_off_h[g] + counts_h[g * G + rank];  // from src g, ascending
  }
  return GS_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ int64 scan
namespace {
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;  // per thread
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* sm, int64_t& total) {
  // warp-shuffle inclusive scan, then warp totals in smem
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int64_t t = lane < (int)(blockDim.x >> 5) ? sm[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    sm[lane] = t;  // inclusive warp-total prefix
  }
  __syncthreads();
  total = sm[(blockDim.x >> 5) - 1];
  int64_t wbase = wid ? sm[wid - 1] : 0;
  __syncthreads();
  return wbase + x - v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const int64_t* in, int64_t n,
                                                              int64_t* part) {
  __shared__ int64_t sm[32];
  int64_t base = (int64_t)blockIdx.x * kScanTile, s = 0;
  for (int k = 0; k < kScanItems; k++) {
    int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  int64_t tot;
  block_excl_scan(s, sm, tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_partials(int64_t* part, int64_t nparts) {
  __shared__ int64_t sm[32];
  int64_t carry = 0;
  for (int64_t b = 0; b < nparts; b += kScanThreads) {
    int64_t i = b + threadIdx.x;
    int64_t v = i < nparts ? part[i] : 0, tot;
    int64_t ex = block_excl_scan(v, sm, tot);
    if (i < nparts) part[i] = carry + ex;
    carry += tot;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(const int64_t* in, int64_t* out,
                                                            int64_t n, const int64_t* part,
                                                            int inclusive) {
  __shared__ int64_t sm[32];
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems], s = 0;
  for (int k = 0; k < kScanItems; k++) {
    int64_t i = base + k;
    v[k] = i < n ? in[i] : 0;
    s += v[k];
  }
  int64_t tot;
  int64_t run = block_excl_scan(s, sm, tot) + part[blockIdx.x];
  for (int k = 0; k < kScanItems; k++) {
    int64_t i = base + k;
    if (inclusive) run += v[k];
    if (i < n) out[i] = run;
    if (!inclusive) run += v[k];
  }
}
}  // namespace

gs_status gs_scan_i64(gs_ctx* c, const int64_t* in, int64_t* out, int64_t n, int inclusive,
                      cudaStream_t st) {
  if (n <= 0) return GS_OK;
  int64_t nb = (n + kScanTile - 1) / kScanTile;
  int64_t* part = (int64_t*)gs_slot_get(c, SLOT_SCAN, nb * sizeof(int64_t), st);
  if (!part) return gs_fail(c, GS_ECUDA, "scan scratch alloc");
  ++c->launches;
  k_scan_reduce<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, part);
  ++c->launches;
  k_scan_partials<<<1, kScanThreads, 0, st>>>(part, nb);
  ++c->launches;
  k_scan_down<<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, n, part, inclusive);
  GS_LAUNCH_CHECK(c, "scan");
  return GS_OK;
}

// ------------------------------------------------------------------ non-finite check
namespace {
__global__ void k_check_finite(const float4* pos_op, const float4* ls, const float4* rot,
                               const float4* sh, int64_t n, int64_t gid_base,
                               unsigned long long* bad) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  auto fin4 = [](float4 v) { return isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w); };
  float4 l = ls[i];
  bool ok = fin4(pos_op[i]) && isfinite(l.x) && isfinite(l.y) && isfinite(l.z) && fin4(rot[i]);
  for (int k = 0; k < 12 && ok; k++) ok = fin4(sh[(int64_t)k * n + i]);
  if (!ok) atomicMin(bad, (unsigned long long)(gid_base + i));
}
}  // namespace

extern "C" gs_status gs_check_finite(gs_ctx* c, const gs_params* p, int64_t* bad_gid_h,
                                     void* stream) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, p && bad_gid_h, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  *bad_gid_h = -1;
  if (p->n == 0) return GS_OK;
  unsigned long long* bad = (unsigned long long*)gs_slot_get(c, SLOT_MISC, 64, st);
  if (!bad) return gs_fail(c, GS_ECUDA, "scratch");
  GS_CUDA(c, cudaMemsetAsync(bad, 0xff, 8, st));
  ++c->launches;
  k_check_finite<<<(unsigned)((p->n + 255) / 256), 256, 0, st>>>(
      (const float4*)p->pos_op, (const float4*)p->log_scale, (const float4*)p->rot,
      (const float4*)p->sh, p->n, p->gid_base, bad);
  GS_LAUNCH_CHECK(c, "check_finite");
  GS_CUDA(c, cudaMemcpyAsync(c->pinned, bad, 8, cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  unsigned long long v = (unsigned long long)c->pinned[0];
  if (v != ~0ull) {
    *bad_gid_h = (int64_t)v;
    return gs_fail(c, GS_ENONFINITE, "non-finite parameter at gid %lld", (long long)v);
  }
  return GS_OK;
}
