// gs_internal.h -- host-side internals of libgs (context, errors, scratch arena).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/gs.h"

#ifdef GS_WITH_NCCL
#include <nccl.h>
#endif

// A growable device arena of named slots.  Temporaries of one call live in slots; a slot
// grows (cudaFree + cudaMalloc, after a stream sync) only when a larger size is requested.
struct gs_slot {
  void* ptr = nullptr;
  size_t bytes = 0;
};

enum {
  SLOT_SCAN = 0,      // scan partials
  SLOT_PROJ_TMP,      // projection per-destination totals
  SLOT_COUNTS,        // bin_sort per-view coarse / owned-pair / record counts + view-order flag
  SLOT_CURSOR,        // bin_sort fine emission: first segment of each super-tile (int64)
  SLOT_KEYS,          // bin_sort radix keys + values (ping)
  SLOT_KEYS_TMP,      // bin_sort radix keys + values (pong)
  SLOT_LARGE,         // bin_sort first record of every emission CTA
  SLOT_ROW,           // rebalance cost row (all blocks of the batch)
  SLOT_ET,            // rebalance ET of next batch
  SLOT_CT,            // rebalance prefix sums
  SLOT_MISC,          // small counters / dp
  SLOT_COUNT_GATHER,  // exchange count matrix
  SLOT_RECTILES,      // bin_sort per-record coarse counts
  SLOT_RADIX_HIST,    // bin_sort radix per-tile digit histograms -> offsets
  SLOT_PSTART,        // bin_sort records' depth bits, then coarse-pair starts in (view, depth) order
  SLOT_HALO_SEND,     // halo exchange: packed blocks to send
  SLOT_HALO_IDX,      // halo exchange: owned-block indices to pack
  SLOT_DENSIFY,       // densify keep flags [4][n]
  SLOT_DENSIFY_OFF,   // densify output positions
  SLOT_NONFINITE,     // gs_project: lowest gid with a non-finite parameter (atomicMin word)
  SLOT_BCOUNT,        // bin_sort per-owned-block pair counts -> offsets (int64)
  SLOT_CLIST,         // bin_sort coarse lists (record indices by super-tile)
  SLOT_CRANGE,        // bin_sort coarse-list ranges per super-tile
  SLOT_RECT8,         // bin_sort packed tile rectangle + view per record
  SLOT_FSEG_CNT,      // bin_sort fine emission: per-segment block counts -> offsets
  SLOT_N
};

// NEXT-3 peer-memory exchange state (gs_p2p.cu): symmetric buffers this context allocated,
// peers' buffers opened from IPC handles, the attached per-rank pointers and the current plan.
struct gs_p2p_state {
  // own symmetric buffers: records, dL/dsend, flags, count matrices, cost rows
  void* sym[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t sym_bytes[5] = {0, 0, 0, 0, 0};
  int64_t* cmat[32] = {};                      // per rank: G x G count matrix (device counts)
  int64_t* row[32] = {};                       // per rank: the batch's cost row
  int64_t row_cap = 0;                         // cost-row capacity (blocks)
  cudaEvent_t counts_ev = nullptr;             // the own matrix is in pinned[kCountsPinned..]
  std::vector<void*> opened;                   // cudaIpcOpenMemHandle'd peer buffers
  bool attached = false, planned = false;
  void* recv[32] = {};                         // per rank: receive buffer (gs_rec)
  int64_t recv_cap[32] = {};                   // records
  float* dsend[32] = {};                       // per rank: dL/d(sent record) [n_send][9]
  int64_t dsend_cap[32] = {};                  // records
  unsigned long long* flags[32] = {};          // per rank: barrier flags [world]
  unsigned long long epoch = 0;
  int* err = nullptr;                          // device: barrier timed out
  std::vector<int64_t> counts;                 // plan: G x G, row = source
};

struct gs_ctx {
  int device = 0, rank = 0, world = 1;
  gs_p2p_state p2p;
  std::string err;
  gs_slot slot[SLOT_N];
  int64_t* pinned = nullptr;  // small pinned host mirror (>= 4096 int64)
  int64_t launches = 0;       // kernels launched through this context (gs_launch_count)
#ifdef GS_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
};

// pinned[kCountsPinned ..] holds the NEXT-3 count matrix read back asynchronously, then the
// non-finite word of the sync-free projection (gs_project_put_dev)
constexpr int kCountsPinned = 4096;
// NEXT-3 device-side count exchange (gs_p2p.cu): this rank's per-destination prefix tot_dev
// (G + 1 device int64) into every rank's matrix, barrier, async copy of the own matrix
gs_status gs_p2p_counts_exchange(gs_ctx* c, const int64_t* tot_dev, cudaStream_t st);

gs_status gs_fail(gs_ctx* c, gs_status s, const char* fmt, ...);
void* gs_slot_get(gs_ctx* c, int slot, size_t bytes, cudaStream_t st);
gs_status gs_cuda_check(gs_ctx* c, cudaError_t e, const char* what);

#define GS_CUDA(ctx, expr)                                              \
  do {                                                                  \
    cudaError_t _e = (expr);                                            \
    if (_e != cudaSuccess) return gs_cuda_check((ctx), _e, #expr);      \
  } while (0)

#define GS_LAUNCH_CHECK(ctx, what)                                       \
  do {                                                                  \
    cudaError_t _e = cudaPeekAtLastError();                             \
    if (_e != cudaSuccess) return gs_cuda_check((ctx), _e, what);       \
  } while (0)

#define GS_REQUIRE(ctx, cond, ...)                                       \
  do {                                                                  \
    if (!(cond)) return gs_fail((ctx), GS_EINVAL, __VA_ARGS__);         \
  } while (0)

// Shared validation of a batch description: equal-size views, monotone dp.
gs_status gs_check_batch(gs_ctx* c, const gs_camera* cams_h, int n_views, const int64_t* dp_h);

// Device-wide int64 exclusive (inclusive=0) or inclusive scan, in-place allowed.
gs_status gs_scan_i64(gs_ctx* c, const int64_t* in, int64_t* out, int64_t n, int inclusive,
                      cudaStream_t st);

// Kernel-side view of the batch geometry and of the rank's partition.
#define GS_MAX_WORLD 32
#define GS_MAX_VIEWS 32
struct gs_dp_arg {
  long long dp[GS_MAX_WORLD + 1];
  int G;
  int rank;
};
struct gs_geom {
  int W, H, Wt, Ht;
  long long per_view;  // Wt * Ht
};
inline gs_geom gs_make_geom(const gs_camera* c) {
  gs_geom g;
  g.W = c->width;
  g.H = c->height;
  g.Wt = (g.W + 15) / 16;
  g.Ht = (g.H + 15) / 16;
  g.per_view = (long long)g.Wt * g.Ht;
  return g;
}

// NEXT-1 halo of the owned block range [lo, hi): the not-owned 8-neighbours (same view,
// inside the grid) of owned blocks, ascending (gs_loss.cu).
void gs_halo_blocks(const gs_geom& geo, int64_t lo, int64_t hi, std::vector<int64_t>& out);
inline gs_dp_arg gs_make_dp(const gs_ctx* c, const int64_t* dp_h) {
  gs_dp_arg d;
  d.G = c->world;
  d.rank = c->rank;
  for (int g = 0; g <= GS_MAX_WORLD; g++) d.dp[g] = g <= c->world ? dp_h[g] : dp_h[c->world];
  return d;
}
