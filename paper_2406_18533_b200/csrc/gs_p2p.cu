// gs_p2p.cu -- NEXT-3: the sparse all-to-alls of P:190 over peer memory (NVLink 5 /
// NVSwitch on one box) instead of NCCL send/recv.  The forward exchange is fused into the
// projection's record write (gs_project_put, gs_project.cu) and the reverse exchange into the
// render backward's gradient reduction (gs_render_bwd_put, gs_render.cu); this file holds the
// plan arithmetic, the symmetric buffers, IPC mapping and the device-side barrier.
#include <algorithm>
#include <cstring>

#include "gs_device.cuh"
#include "gs_internal.h"

#define GS_NCCL_P2P(ctx, expr)                                                              \
  do {                                                                                      \
    ncclResult_t _r = (expr);                                                               \
    if (_r != ncclSuccess) return gs_fail((ctx), GS_ENCCL, "%s: %s", #expr, ncclGetErrorString(_r)); \
  } while (0)

namespace {

struct gs_p2p_flags {
  unsigned long long* p[GS_MAX_WORLD];
};

// Device-side barrier over the attached flag arrays (one CTA of G threads).  Thread d
// publishes this rank's epoch into rank d's slot [rank] (release at system scope: every
// earlier write of the stream -- the NVLink record stores or gradient reductions -- is visible
// to d before the flag), then waits until d's own slot [d] in THIS rank's array reached the
// epoch (acquire).  clock64-bounded: a peer that never arrives sets *err and the kernel ends.
__global__ void k_p2p_barrier(gs_p2p_flags f, int G, int rank, unsigned long long epoch, int* err) {
  const int d = threadIdx.x;
  if (d >= G) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f.p[d] + rank), "l"(epoch) : "memory");
  const long long t0 = clock64();
  unsigned long long v = 0;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f.p[rank] + d) : "memory");
    if (v >= epoch) break;
    if (clock64() - t0 > (long long)8000000000ll) {  // ~4 s at 2 GHz
      atomicExch(err, 1);
      break;
    }
    __nanosleep(200);
  }
  __threadfence_system();
}

}  // namespace

extern "C" gs_status gs_p2p_offsets(const int64_t* C, int G, int r, int64_t* seg, int64_t* put, int64_t* soff,
                                    int64_t* own) {
  if (!C || G < 1 || G > GS_MAX_WORLD || r < 0 || r >= G || !seg || !put || !soff || !own) return GS_EINVAL;
  for (int k = 0; k < G * G; k++)
    if (C[k] < 0) return GS_EINVAL;
  seg[0] = 0;
  for (int s = 0; s < G; s++) seg[s + 1] = seg[s] + C[(int64_t)s * G + r];
  for (int d = 0; d < G; d++) {
    int64_t b = 0;
    for (int s = 0; s < r; s++) b += C[(int64_t)s * G + d];
    put[d] = b;
  }
  soff[0] = 0;
  for (int d = 0; d < G; d++) soff[d + 1] = soff[d] + C[(int64_t)r * G + d];
  for (int s = 0; s < G; s++) {
    int64_t o = 0;
    for (int d = 0; d < r; d++) o += C[(int64_t)s * G + d];
    own[s] = o;
  }
  return GS_OK;
}

extern "C" gs_status gs_sym_alloc(gs_ctx* c, int which, size_t bytes, void** ptr_h, uint8_t handle_h[64]) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, which >= 0 && which < 5 && ptr_h, "bad argument");
  GS_CUDA(c, cudaSetDevice(c->device));
  gs_p2p_state& P = c->p2p;
  if (bytes == 0) bytes = 256;
  if (P.sym_bytes[which] < bytes) {
    if (P.sym[which]) {
      GS_CUDA(c, cudaDeviceSynchronize());
      GS_CUDA(c, cudaFree(P.sym[which]));
      P.sym[which] = nullptr;
      P.sym_bytes[which] = 0;
    }
    GS_CUDA(c, cudaMalloc(&P.sym[which], bytes));
    P.sym_bytes[which] = bytes;
    if (which == 2 || which == 3) GS_CUDA(c, cudaMemset(P.sym[which], 0, bytes));
    P.attached = false;  // peers must re-open and re-attach
  }
  *ptr_h = P.sym[which];
  if (handle_h) {
    cudaIpcMemHandle_t h;
    GS_CUDA(c, cudaIpcGetMemHandle(&h, P.sym[which]));
    static_assert(sizeof(h) == 64, "IPC handle size");
    memcpy(handle_h, &h, 64);
  }
  return GS_OK;
}

extern "C" gs_status gs_ipc_open(gs_ctx* c, const uint8_t handle_h[64], void** ptr_h) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, handle_h && ptr_h, "null argument");
  GS_CUDA(c, cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle_h, 64);
  void* q = nullptr;
  GS_CUDA(c, cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
  c->p2p.opened.push_back(q);
  *ptr_h = q;
  return GS_OK;
}

extern "C" gs_status gs_p2p_attach(gs_ctx* c, void* const* recv_h, const int64_t* recv_cap_h, void* const* dsend_h,
                                   const int64_t* dsend_cap_h, void* const* flags_h) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, recv_h && recv_cap_h && dsend_h && dsend_cap_h && flags_h, "null argument");
  gs_p2p_state& P = c->p2p;
  for (int g = 0; g < c->world; g++) {
    GS_REQUIRE(c, recv_cap_h[g] >= 0 && dsend_cap_h[g] >= 0, "negative capacity");
    P.recv[g] = recv_h[g];
    P.recv_cap[g] = recv_cap_h[g];
    P.dsend[g] = (float*)dsend_h[g];
    P.dsend_cap[g] = dsend_cap_h[g];
    P.flags[g] = (unsigned long long*)flags_h[g];
  }
  P.attached = true;
  P.planned = false;
  return GS_OK;
}

extern "C" gs_status gs_p2p_plan(gs_ctx* c, const int64_t* C, int64_t* n_recv_h) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, C && n_recv_h, "null argument");
  gs_p2p_state& P = c->p2p;
  GS_REQUIRE(c, P.attached, "gs_p2p_plan before gs_p2p_attach");
  const int G = c->world;
  int64_t seg[GS_MAX_WORLD + 1], put[GS_MAX_WORLD], soff[GS_MAX_WORLD + 1], own[GS_MAX_WORLD];
  if (gs_p2p_offsets(C, G, c->rank, seg, put, soff, own) != GS_OK) return gs_fail(c, GS_EINVAL, "bad count matrix");
  *n_recv_h = seg[G];
  P.planned = false;
  // every rank checks every rank's capacities from the same matrix: all fail together
  for (int d = 0; d < G; d++) {
    int64_t in = 0, out = 0;
    for (int s = 0; s < G; s++) in += C[(int64_t)s * G + d], out += C[(int64_t)d * G + s];
    if (in > P.recv_cap[d])
      return gs_fail(c, GS_ECAPACITY, "rank %d receives %lld records > capacity %lld", d, (long long)in,
                     (long long)P.recv_cap[d]);
    if (out > P.dsend_cap[d])
      return gs_fail(c, GS_ECAPACITY, "rank %d sends %lld records > gradient capacity %lld", d, (long long)out,
                     (long long)P.dsend_cap[d]);
  }
  P.counts.assign(C, C + (size_t)G * G);
  P.planned = true;
  return GS_OK;
}

// ------------------------------------------------------------------ device-side counts
namespace {
struct gs_ptrs64 {
  int64_t* p[GS_MAX_WORLD];
};
// This rank's row of the count matrix (tot = its per-destination prefix, G + 1 entries) into
// row `rank` of every rank's matrix (NVLink stores); visible to them after the next barrier.
__global__ void k_p2p_counts_put(const int64_t* __restrict__ tot, gs_ptrs64 cm, int G, int rank) {
  const int q = blockIdx.x, d = threadIdx.x;
  if (q < G && d < G) cm.p[q][rank * G + d] = tot[d + 1] - tot[d];
}
// The owned segment of the batch's cost row into every rank's row at [B_lo, B_lo + n).
__global__ void k_p2p_row_put(const int64_t* __restrict__ cost, int64_t n, int64_t B_lo, gs_ptrs64 rows, int G) {
  const int q = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    rows.p[q][B_lo + i] = cost[i];
}
}  // namespace

extern "C" gs_status gs_p2p_attach_counts(gs_ctx* c, void* const* cmat_h, void* const* row_h, int64_t row_cap) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, cmat_h, "null argument");
  GS_REQUIRE(c, row_cap >= 0 && (row_cap == 0 || row_h), "row pointers required with a capacity");
  gs_p2p_state& P = c->p2p;
  for (int g = 0; g < c->world; g++) {
    GS_REQUIRE(c, cmat_h[g] != nullptr, "rank %d has no count matrix", g);
    P.cmat[g] = (int64_t*)cmat_h[g];
    P.row[g] = row_cap ? (int64_t*)row_h[g] : nullptr;
  }
  P.row_cap = row_cap;
  if (!P.counts_ev) GS_CUDA(c, cudaEventCreateWithFlags(&P.counts_ev, cudaEventDisableTiming));
  return GS_OK;
}

// Device-side count exchange (gs_project_put_dev's first half): the row to every peer, the
// barrier, then an asynchronous copy of the own (now complete) matrix to pinned memory whose
// completion gs_p2p_counts waits for.
gs_status gs_p2p_counts_exchange(gs_ctx* c, const int64_t* tot_dev, cudaStream_t st) {
  gs_p2p_state& P = c->p2p;
  const int G = c->world;
  gs_ptrs64 cm;
  for (int g = 0; g < GS_MAX_WORLD; g++) cm.p[g] = g < G ? P.cmat[g] : nullptr;
  ++c->launches;
  k_p2p_counts_put<<<G, 32, 0, st>>>(tot_dev, cm, G, c->rank);
  GS_LAUNCH_CHECK(c, "p2p counts");
  gs_status s = gs_p2p_barrier(c, st);
  if (s != GS_OK) return s;
  GS_CUDA(c, cudaMemcpyAsync(c->pinned + kCountsPinned, P.cmat[c->rank], (size_t)G * G * sizeof(int64_t),
                             cudaMemcpyDeviceToHost, st));
  return GS_OK;
}

extern "C" gs_status gs_p2p_counts(gs_ctx* c, int64_t* counts_h, int64_t* n_recv_h) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, counts_h && n_recv_h, "null argument");
  gs_p2p_state& P = c->p2p;
  GS_REQUIRE(c, P.counts_ev, "gs_p2p_counts before gs_p2p_attach_counts");
  GS_CUDA(c, cudaEventSynchronize(P.counts_ev));
  const int G = c->world;
  for (int k = 0; k < G * G; k++) counts_h[k] = c->pinned[kCountsPinned + k];
  const unsigned long long badv = (unsigned long long)c->pinned[kCountsPinned + GS_MAX_WORLD * GS_MAX_WORLD];
  if (badv != ~0ull)  // the projection saw a non-finite parameter: its records are garbage
    return gs_fail(c, GS_ENONFINITE, "non-finite parameter at gid %lld", (long long)badv);
  return gs_p2p_plan(c, counts_h, n_recv_h);
}

extern "C" gs_status gs_p2p_put_costs(gs_ctx* c, const int64_t* owned_cost, const int64_t* dp_h, void* stream) {
  if (!c) return GS_EINVAL;
  gs_p2p_state& P = c->p2p;
  GS_REQUIRE(c, dp_h && P.row_cap > 0, "no cost rows attached");
  const int G = c->world;
  const int64_t lo = dp_h[c->rank], n = dp_h[c->rank + 1] - lo;
  GS_REQUIRE(c, dp_h[G] <= P.row_cap, "cost row capacity %lld < %lld blocks", (long long)P.row_cap,
             (long long)dp_h[G]);
  if (n == 0) return GS_OK;
  GS_REQUIRE(c, owned_cost != nullptr, "null owned_cost");
  gs_ptrs64 rows;
  for (int g = 0; g < GS_MAX_WORLD; g++) rows.p[g] = g < G ? P.row[g] : nullptr;
  ++c->launches;
  k_p2p_row_put<<<dim3((unsigned)std::min<int64_t>((n + 255) / 256, 148), G), 256, 0, (cudaStream_t)stream>>>(
      owned_cost, n, lo, rows, G);
  GS_LAUNCH_CHECK(c, "p2p cost row");
  return GS_OK;
}

extern "C" gs_status gs_exchange_counts(gs_ctx* c, const int64_t* send_counts_h, int64_t* all_h, void* stream) {
  if (!c) return GS_EINVAL;
  GS_REQUIRE(c, send_counts_h && all_h, "null argument");
  const int G = c->world;
  if (G == 1) {
    all_h[0] = send_counts_h[0];
    return GS_OK;
  }
#ifdef GS_WITH_NCCL
  if (!c->comm) return gs_fail(c, GS_EINVAL, "virtual context (no communicator): collectives unavailable");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t* dbuf = (int64_t*)gs_slot_get(c, SLOT_COUNT_GATHER, (G + G * G) * sizeof(int64_t), st);
  if (!dbuf) return gs_fail(c, GS_ECUDA, "scratch");
  for (int g = 0; g < G; g++) c->pinned[g] = send_counts_h[g];
  GS_CUDA(c, cudaMemcpyAsync(dbuf, c->pinned, G * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  GS_NCCL_P2P(c, ncclAllGather(dbuf, dbuf + G, G, ncclInt64, c->comm, st));
  GS_CUDA(c, cudaMemcpyAsync(c->pinned + 64, dbuf + G, G * G * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  for (int k = 0; k < G * G; k++) all_h[k] = c->pinned[64 + k];
  return GS_OK;
#else
  (void)stream;
  return gs_fail(c, GS_ENOTSUP, "built without NCCL");
#endif
}

extern "C" gs_status gs_p2p_barrier(gs_ctx* c, void* stream) {
  if (!c) return GS_EINVAL;
  gs_p2p_state& P = c->p2p;
  GS_REQUIRE(c, P.attached, "gs_p2p_barrier before gs_p2p_attach");
  const int G = c->world;
  gs_p2p_flags f;
  for (int g = 0; g < GS_MAX_WORLD; g++) f.p[g] = g < G ? P.flags[g] : nullptr;
  for (int g = 0; g < G; g++) GS_REQUIRE(c, f.p[g] != nullptr, "rank %d has no flag array", g);
  if (!P.err) {
    GS_CUDA(c, cudaMalloc(&P.err, sizeof(int)));
    GS_CUDA(c, cudaMemset(P.err, 0, sizeof(int)));
  }
  cudaStream_t st = (cudaStream_t)stream;
  ++P.epoch;
  ++c->launches;
  k_p2p_barrier<<<1, 32, 0, st>>>(f, G, c->rank, P.epoch, P.err);
  GS_LAUNCH_CHECK(c, "p2p_barrier");
  return GS_OK;
}

extern "C" gs_status gs_p2p_status(gs_ctx* c, void* stream) {
  if (!c) return GS_EINVAL;
  gs_p2p_state& P = c->p2p;
  if (!P.err) return GS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  GS_CUDA(c, cudaMemcpyAsync(c->pinned, P.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  GS_CUDA(c, cudaStreamSynchronize(st));
  if (*(int*)c->pinned) {
    GS_CUDA(c, cudaMemsetAsync(P.err, 0, sizeof(int), st));
    return gs_fail(c, GS_ECUDA, "p2p barrier timed out (a peer never arrived)");
  }
  return GS_OK;
}
