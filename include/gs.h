/* gs.h -- C ABI of libgs: the data-parallel hot path of one Grendel 3DGS training step
 * (arXiv 2406.18533), B200-native (CUDA sm_100a + NCCL over NVLink/NVSwitch).
 *
 * Citation key: P:n = PAPER.md line n (section/equation named), S:n = SPEC.md line n,
 * O1..O18 = the step definitions of SURVEY.md §8(c), R1..R11 = readings in DESIGN.md §2.
 *
 * One training step on rank r of G ranks over a batch of b views:
 *   gs_project -> gs_exchange -> gs_bin_sort -> gs_render_fwd -> gs_render_bwd
 *   -> gs_exchange_grads -> gs_adam_step -> gs_rebalance
 *
 * Conventions shared by every call
 *  - Pointers named *_h are HOST memory; every other buffer pointer is DEVICE memory on the
 *    context's device.  Device buffers are allocated and owned by the caller (PyTorch);
 *    the context owns only a growable device scratch arena for temporaries and a small
 *    pinned host mirror, both released by gs_destroy.
 *  - `stream` is a cudaStream_t passed as void*.  Calls are stream-ordered and
 *    asynchronous except where a host sync is stated (count read-backs).
 *  - Every call returns a gs_status and never throws; gs_last_error() has the message.
 *  - Views of one batch share one image size W x H; the batch's blocks are serialized as
 *    beta = v * Wt * Ht + ty * Wt + tx with Wt = ceil(W/16), Ht = ceil(H/16)
 *    ("dividing it into 16x16-pixel blocks, serializing the blocks";
 *    P:523).  Rank g owns blocks [dp_h[g], dp_h[g+1]) (dp_h[0] = 0, dp_h[G] = b*Wt*Ht).
 *  - Per-pixel buffers are block-major over the rank's owned blocks: pixel p = ly*16+lx
 *    of owned block lb = beta - dp_h[r] lives at [lb*256 + p] (per channel plane:
 *    [lb][ch][256]).  Pixels with px >= W or py >= H are not rendered (R: partial blocks).
 *  - All collective calls (gs_exchange, gs_exchange_grads, gs_rebalance) must be called by
 *    every rank in the same order.  Contexts are not re-entrant: one per rank and thread.
 */
#ifndef GS_H
#define GS_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GS_OK = 0,
  GS_EINVAL = 1,       /* invalid argument (null required pointer, bad sizes, dp not monotone...) */
  GS_ECAPACITY = 2,    /* a caller capacity is too small; *needed written; outputs invalid      */
  GS_ENONFINITE = 3,   /* a parameter is NaN/Inf (gs_check_finite)                               */
  GS_ECUDA = 4,        /* CUDA runtime error                                                      */
  GS_ENCCL = 5,        /* NCCL error                                                              */
  GS_ENOTSUP = 6       /* world > 1 requested but the library was built without NCCL              */
} gs_status;

typedef struct gs_ctx gs_ctx;

/* Pinhole camera, one per view of a batch ("Given a camera view v and the associated
 * screen space").  R is world->camera (rows: image-right, image-down, forward), row-major;
 * camera centre c = -R^T t.  Pixel (px,py) has its centre at (px,py) (R1).             */
typedef struct {
  float R[9];
  float t[3];
  float fx, fy, cx, cy;
  int32_t width, height;
  int32_t image_id; /* training-image id, indexes the rebalancer's cost history */
} gs_camera;

/* Gaussian parameters of the rank's shard (x, s, q, alpha, sh in R^48), SoA of
 * float4 planes so a warp reads 512 contiguous bytes per plane:
 *   pos_op[n]    = (x, y, z, opacity_logit)
 *   log_scale[n] = (log sx, log sy, log sz, unused)
 *   rot[n]       = (w, x, y, z), unnormalised (normalised inside O1)
 *   sh[12][n]    = plane k holds SH floats 4k..4k+3 of the 48 ((l,m)-major, rgb inner)
 * gid of element i is gid_base + i (contiguous shard).                            */
typedef struct {
  float* pos_op;
  float* log_scale;
  float* rot;
  float* sh;
  int64_t n;
  int64_t gid_base;
} gs_params;

/* Adam hyper-parameters.  lr[6] = base learning rates lambda per group
 * (pos, sh_dc, sh_rest, opacity, scale, rot) for THIS step (the position schedule is the
 * caller's); the call applies Eq. (1) lambda' = lambda sqrt(batch) and Eq. (2)
 * beta' = beta^batch itself.  step = t >= 1 (bias correction as torch.optim.Adam).      */
typedef struct {
  float lr[6];
  float beta1, beta2, eps;
  int32_t batch;
  int64_t step;
} gs_adam_hparams;

enum { GS_COST_MEASURED = 0, GS_COST_WORK = 1, GS_COST_PAPER_AVG = 2 };
enum { GS_ADAM_GRAD = 1, GS_ADAM_APPLY = 2, GS_ADAM_WRITE_GRAD = 4 };

/* Size of one projected record (A1 output / A2 payload):
 *   float4 {mx, my, depth, radius(float)}       mean2d, depth = p_z (O3-O4, O7)
 *   float4 {l11', l21', l22', opacity}          conic = L L^T (O6) as the prescaled Cholesky
 *                                               factor L' = L sqrt(0.5 log2 e), rounded to
 *                                               nearest from fp64 (hi part); opacity (O1)
 *   float4 {r, g, b, qmax}                      colour (O9); qmax = log2(255 opacity), so
 *                                               alpha >= 1/255 <=> q = |L'^T d|^2 <= qmax
 *   float4 {l11', l21', l22' (lo), meta}        L' - hi, rounded to nearest (double-float
 *                                               factor: hi + lo carries ~48 bits);
 *                                               meta = u32 gid * 32 + v
 * (R16: the renderer evaluates u = l11' dx + l21' dy and w = l22' dy in fp64 from hi + lo at
 * a reference point within (3.5, 7.5) px of each pixel, and in fp32 from hi for the offset.) */
#define GS_RECORD_BYTES 64
/* dL/d(record) as exchanged back (A6): 9 floats (mx, my, A, B, C, opacity, r, g, b) where
 * (A, B, C) is the conic [[A, B], [B, C]] and B is the scalar off-diagonal (R: #16).     */
#define GS_GRAD_FLOATS 9

/* --------------------------------------------------------------------------- context */
int gs_version(void);
/* 128-byte NCCL unique id (rank 0 calls it; the bytes are broadcast by torch.distributed).
 * Returns GS_ENOTSUP when built without NCCL.                                            */
gs_status gs_nccl_unique_id(uint8_t id_h[128]);
/* Create a context on `device` for rank/world.  world == 1 needs no id (id_h may be NULL);
 * world > 1 with an id initialises an NCCL communicator (collective over all ranks);
 * world > 1 with id_h == NULL creates a "virtual" rank without a communicator: the local
 * calls (project, bin_sort, render, adam) work on its partition, the collective calls
 * return GS_EINVAL.  (Used to test partitioned execution on one GPU.)                   */
gs_status gs_create(gs_ctx** out, int device, int rank, int world, const uint8_t* id_h);
void gs_destroy(gs_ctx* ctx);
const char* gs_last_error(const gs_ctx* ctx);
/* Number of CUDA kernels this context has launched so far (for launch accounting). */
int64_t gs_launch_count(const gs_ctx* ctx);

/* Non-finite parameter check: GS_ENONFINITE with *bad_gid_h = lowest offending
 * gid, else GS_OK and *bad_gid_h = -1.  Host sync.                                       */
gs_status gs_check_finite(gs_ctx* ctx, const gs_params* p, int64_t* bad_gid_h, void* stream);

/* --------------------------------------------------------------------------- A1 */
/* Bytes of the backward index gs_project writes and gs_adam_step reads, for n owned
 * Gaussians and n_views views at the context's world size.                               */
size_t gs_project_index_bytes(const gs_ctx* ctx, int64_t n, int n_views);

/* A1 gs_project -- EWA projection and culling on the owner (P:103 step 1; O1-O10).
 * For every owned Gaussian i and view v: the fp32 membership chain O1-O8 (visibility,
 * mean2d, depth, 2D covariance, radius, tile rectangle; bit-exact, R10), the conic's
 * Cholesky factor, opacity and SH degree-3 colour (O9), and the destination set
 * D(i,v) = ranks owning a block of the rectangle (O10; Fig. 3).  Writes one
 * record per (i, v, d in D(i,v)) into send_rec, bucketed by destination d, then view v,
 * then ascending gid (deterministic: no placement atomics).  send_counts_h[G] receives the
 * per-destination record counts (host sync).  If the total exceeds send_cap, returns
 * GS_ECAPACITY with the counts written and send_rec untouched.  bwd_index must hold
 * gs_project_index_bytes(ctx, p->n, n_views) bytes; it is read back by gs_adam_step.
 * Invisible Gaussians (behind near plane 0.01, det <= 0, empty rectangle) produce nothing.
 * A non-finite position, opacity logit, log-scale or rotation returns GS_ENONFINITE
 * with the lowest offending gid in gs_last_error, before any record is written; a non-finite
 * SH coefficient of a Gaussian visible in some view is found while its colour is evaluated and
 * reported the same way by the next gs_project / gs_project_count of the context (the check
 * rides on the count read-back: no extra sync).  gs_check_finite checks every parameter.   */
gs_status gs_project(gs_ctx* ctx, const gs_params* p, const gs_camera* cams_h, int n_views,
                     const int64_t* dp_h, void* send_rec, int64_t send_cap,
                     int64_t* send_counts_h, void* bwd_index, void* stream);

/* --------------------------------------------------------------------------- A2 */
/* A2 gs_exchange -- forward sparse all-to-all of records ("sparse all-to-all
 * communication to retrieve Gaussians intersecting with any pixels in the partition";
 * P:529).  Exchanges the G x G count matrix (NCCL all-gather, host sync), then grouped
 * ncclSend/ncclRecv.  recv_rec receives the records ordered by ascending source rank,
 * so within each view they are in ascending gid.  recv_counts_h[G] = records from each
 * source; *n_recv_h = total.  The capacities travel with the counts: if ANY rank's total
 * exceeds its recv_cap, EVERY rank returns GS_ECAPACITY (nothing transferred, each with its
 * own counts), so a retry after growing the buffer stays collective.
 * world == 1: identity; recv_rec may alias send_rec (then nothing is copied).            */
gs_status gs_exchange(gs_ctx* ctx, const void* send_rec, const int64_t* send_counts_h,
                      void* recv_rec, int64_t recv_cap, int64_t* recv_counts_h,
                      int64_t* n_recv_h, void* stream);

/* --------------------------------------------------------------------------- A3 */
/* A3 gs_bin_sort -- Z-buffer build ("iterates over intersecting Gaussians in
 * increasing depth"; App. A.2; O11).  For each received record, every owned block
 * of its view inside its tile rectangle gets the record; each block's list is sorted by
 * (depth, gid) (R7; unique keys, so the order is deterministic).  Outputs:
 *   tile_range[n_owned+1] (int32 offsets into sorted_idx), sorted_idx[n_pairs] (uint32
 *   receive indices).  *n_pairs_h = pair count (host sync).  GS_ECAPACITY if > pair_cap.
 * Depth ties keep receive order, so records of one view must arrive in ascending gid (the
 * exchange's ascending-source-rank order guarantees it).  Any view order is accepted; a
 * buffer whose views never decrease (a rank's own buckets) takes the segmented record sort. */
gs_status gs_bin_sort(gs_ctx* ctx, const void* recv_rec, int64_t n_recv, const gs_camera* cams_h,
                      int n_views, const int64_t* dp_h, uint32_t* sorted_idx, int64_t pair_cap,
                      int32_t* tile_range, int64_t* n_pairs_h, void* stream);

/* --------------------------------------------------------------------------- A4 */
/* A4 gs_render_fwd -- front-to-back alpha compositing over the owned blocks (P:106-107
 * "uses alpha-composition to combine their contributions until a threshold opacity has
 * been reached"; O12 with alpha = min(0.99, o G), skip alpha < 1/255, stop before the entry
 * that would take T below 1e-4 (R3); C += T bg).  Writes T_final[n_owned*256],
 * n_last[n_owned*256] (int32), optionally out_rgb[n_owned][3][256] (C incl. background).
 * If gt (uint8 [n_views][H][W][3], value/255) is given, fuses the L1 loss (O13):
 * dL_dpix[n_owned][3][256] = sign(C - GT) / (3 H W b_loss) and *loss_sum (device double)
 * += sum |C - GT| / (3 H W b_loss).  tile_cost[n_owned] (int64, nullable) += per-block
 * cost (MEASURED: SM cycles of the block; WORK: evaluations E_f).  stats (nullable
 * int64[8], device) += (E_f, E_fc, E_fs, E_stop, 0, 0, 0, 0) totals.
 * cull_bits (nullable, device u32[gs_cull_words(K, n_owned)], K = the lists' total length):
 * receives, for every list entry the forward staged, whether any pixel centre of each 8x16
 * half of its block may composite it (a conservative, semantics-free ellipse-box test: an
 * entry with the bit clear is a no-op for every pixel of that half).  Pass the same buffer
 * to gs_render_bwd / gs_render_bwd_put on the same lists to skip the test there; contents
 * are internal to the pair of calls.                                                       */
gs_status gs_render_fwd(gs_ctx* ctx, const void* recv_rec, const uint32_t* sorted_idx,
                        const int32_t* tile_range, const gs_camera* cams_h, int n_views,
                        const int64_t* dp_h, const float* bg_h, const uint8_t* gt, int b_loss,
                        float* out_rgb, float* T_final, int32_t* n_last, float* dL_dpix,
                        double* loss_sum, int64_t* tile_cost, int cost_mode, int64_t* stats,
                        uint32_t* cull_bits, void* stream);
/* Words of the cull_bits buffer for lists of total length n_pairs over n_owned blocks
 * (2 x (n_pairs / 32 + n_owned + 1): two halves, one bit per entry, 32-entry words aligned
 * per block).                                                                              */
int64_t gs_cull_words(int64_t n_pairs, int64_t n_owned);

/* --------------------------------------------------------------------------- A5 */
/* A5 gs_render_bwd -- backward of compositing (O14-O15).  Walks each pixel's list
 * back to front from n_last, reconstructing T, and accumulates dL/d(record) over all owned
 * pixels into dL_drec[n_recv][9] (zeroed by this call; float atomics, so summation order is
 * not deterministic).  tile_cost += cost (WORK: visited entries = n_last per pixel).
 * stats (nullable) += (0, 0, 0, 0, E_b visited, E_bc contributing, 0, 0).
 * cull_bits (nullable): the buffer gs_render_fwd filled for these same lists (sorted_idx,
 * tile_range, dp unchanged since), read instead of re-running the forward's cull test;
 * NULL: the test runs here.  Results are identical either way.                             */
gs_status gs_render_bwd(gs_ctx* ctx, const void* recv_rec, int64_t n_recv,
                        const uint32_t* sorted_idx, const int32_t* tile_range,
                        const gs_camera* cams_h, int n_views, const int64_t* dp_h,
                        const float* bg_h, const float* dL_dpix, const float* T_final,
                        const int32_t* n_last, float* dL_drec, int64_t* tile_cost, int cost_mode,
                        int64_t* stats, const uint32_t* cull_bits, void* stream);

/* --------------------------------------------------------------------------- A6 */
/* A6 gs_exchange_grads -- reverse sparse all-to-all ("A reversed all-to-all
 * communication is done during the backward pass").  Exact transpose of gs_exchange with
 * the counts it returned: dL_dsend[n_send][9] receives, in send order, the gradient each
 * record got from its renderer.  world == 1: identity (dL_dsend may alias dL_drec).      */
gs_status gs_exchange_grads(gs_ctx* ctx, const float* dL_drec, const int64_t* recv_counts_h,
                            const int64_t* send_counts_h, float* dL_dsend, void* stream);

/* --------------------------------------------------------------------------- A7 + A8 */
/* A7+A8 gs_adam_step -- transformation backward fused with Adam ("Gaussian
 * transformation backward ... distributed the same way"; Eq. (1)-(2); O16-O17).
 * flags:
 *   GS_ADAM_GRAD       compute the parameter gradient from dL_dsend (summed over the
 *                      record's destinations in ascending rank, then over views; O16)
 *   GS_ADAM_WRITE_GRAD also store that gradient into g (parity mode)
 *   GS_ADAM_APPLY      apply Adam to p, m, v (dense over all owned Gaussians, R9) using the
 *                      fused gradient (with GS_ADAM_GRAD) or the gradient stored in g.
 * With GS_ADAM_GRAD | GS_ADAM_APPLY and a non-NULL g, g is used as the gradient buffer: the
 * transformation backward writes it and an elementwise Adam pass applies it (the faster path
 * on B200); with g == NULL both happen in one fused kernel with the gradient in registers.
 * m, v, g use the same float4-plane layout as p (unused lanes ignored).  A non-NULL g must
 * have g->n == p->n; g is required for GS_ADAM_WRITE_GRAD and for GS_ADAM_APPLY without
 * GS_ADAM_GRAD (GS_EINVAL otherwise).                                                     */
gs_status gs_adam_step(gs_ctx* ctx, gs_params* p, gs_params* m, gs_params* v, gs_params* g,
                       const gs_camera* cams_h, int n_views, const int64_t* dp_h,
                       const float* dL_dsend, const void* bwd_index, const gs_adam_hparams* hp,
                       int flags, void* stream);

/* --------------------------------------------------------------------------- A9 */
/* A9 gs_rebalance -- dynamic pixel-tile load balancing (§3.2, Algorithm 1).
 * 1. all-gathers the owned per-block costs of the current batch (NCCL; every rank then holds
 *    the whole row, so every rank computes identical division points, no broadcast);
 * 2. converts costs to estimates (MEASURED/WORK: the cost; PAPER_AVG: the rank's average
 *    per-pixel cost times the block's pixels) and stores them in
 *    history[image_id][Wt*Ht] (device int64, initialise to -1 = never rendered);
 * 3. builds ET for the next batch from the history, an unseen image's blocks at the batch's
 *    per-pixel rate (R17), and runs Algorithm 1 in exact int64 (R8): CT = cumsum(ET),
 *    DP[g] = #{i : CT[i] G <= g CT[B-1]}, DP[0] = 0, DP[G] = B (uniform if all zero).
 * dp_next_h[G+1] is written on the host (host sync).                                     */
gs_status gs_rebalance(gs_ctx* ctx, const int64_t* owned_tile_cost, const gs_camera* cams_h,
                       int n_views, const int64_t* dp_h, int64_t* history, int64_t n_images,
                       int cost_mode, const gs_camera* next_cams_h, int n_next,
                       int64_t* dp_next_h, void* stream);

/* gs_rebalance_row -- the local part of gs_rebalance (steps 2-3) given the whole batch's
 * cost row cost_row[B] (device int64, B = n_views Wt Ht, the blocks of every rank): no
 * communication, so virtual contexts (world > 1 without a communicator) can run Algorithm 1
 * and tests can drive it with any row.  Unseen images of the next batch are estimated at the
 * batch's per-pixel rate sum(cost_row) / sum(in-image pixels) times the block's pixels
 * (floor), in the cost mode's own units (R17), or their pixel count while every cost is 0.
 * dp_next_h[G+1] on the host (host sync).                                               */
gs_status gs_rebalance_row(gs_ctx* ctx, const int64_t* cost_row, const gs_camera* cams_h, int n_views,
                           const int64_t* dp_h, int64_t* history, int64_t n_images, int cost_mode,
                           const gs_camera* next_cams_h, int n_next, int64_t* dp_next_h, void* stream);

/* Algorithm 1 alone, pure host function: DP_h[G+1] from ET_h[B].
 * GS_EINVAL if G < 1, B < 0, any ET < 0, or the int64 guard B*max(ET)*G < 2^63 fails.    */
gs_status gs_division_points(const int64_t* ET_h, int64_t B, int G, int64_t* DP_h);

/* Host-side exchange plan (used by gs_exchange; exported for multi-process CPU tests):
 * from the row-major G x G count matrix counts_h[src*G+dst] compute for `rank` the send
 * offsets send_off_h[G+1] and receive offsets recv_off_h[G+1] (ascending source rank).   */
gs_status gs_exchange_plan(const int64_t* counts_h, int G, int rank, int64_t* send_off_h,
                           int64_t* recv_off_h);

/* ------------------------------------------------------------------- NEXT-1 L1 + D-SSIM */
/* The loss of P:114 ("computes the L1 and SSIM loss ... SSIM loss measures the similarity
 * between pixel windows"), per view
 *   L_v = (1 - lambda) mean|x - y| + lambda (1 - mean SSIM(x, y)),
 * SSIM with an 11x11 Gaussian window (sigma 1.5, normalised 1D Gaussian squared), C1 = 0.01^2,
 * C2 = 0.03^2, zero padding outside the image (R12), means over all pixels and
 * channels; the batch loss is sum_v L_v / b_loss.  A pixel's gradient depends on the image
 * within 10 pixels, so blocks next to another rank's range need that rank's rendered blocks
 * (the halo: the not-owned 8-neighbours, same view, of owned blocks).                     */

/* gs_halo_plan -- the rank's halo block ids (ascending) into halo_ids_h[cap]; *n_halo_h = count
 * (GS_ECAPACITY if > cap, ids not written).  Empty at world 1.  Host only, no collective. */
gs_status gs_halo_plan(gs_ctx* ctx, const gs_camera* cams_h, int n_views, const int64_t* dp_h,
                       int64_t* halo_ids_h, int64_t cap, int64_t* n_halo_h);

/* gs_halo_exchange -- COLLECTIVE (every rank, same order).  data: a per-owned-block array
 * [n_owned][fpb] floats (the rendered blocks, fpb = 768, or the SSIM maps, fpb = 2304).
 * Writes halo[n_halo][fpb] and halo_ids[n_halo] (device, ascending, = gs_halo_plan) with the
 * owners' blocks; grouped NCCL point-to-point over NVLink, counts derived from dp on every
 * rank (no count exchange).  halo_cap in blocks (GS_ECAPACITY if smaller, *n_halo_h =
 * needed).  World 1: n_halo = 0.  Virtual contexts (no communicator) fail with GS_EINVAL
 * for world > 1 (tests fill the halo themselves from gs_halo_plan).                     */
gs_status gs_halo_exchange(gs_ctx* ctx, const float* data, int fpb, const gs_camera* cams_h, int n_views,
                           const int64_t* dp_h, float* halo, int64_t* halo_ids, int64_t halo_cap,
                           int64_t* n_halo_h, void* stream);

/* The loss replaces the L1 epilogue of gs_render_fwd (call it with gt = NULL and out_rgb):
 *   gs_ssim_terms -> [gs_halo_exchange of maps, world > 1] -> gs_ssim_grad.
 * gs_ssim_terms: out_rgb [n_owned][3][256] with its halo (halo_rgb [n_halo][3][256],
 * halo_ids device ascending = gs_halo_plan), gt uint8 [n_views][H][W][3] (value/255),
 * lambda in [0,1].  Writes maps[n_owned][3][3][256] (dS/dmu_x, dS/dE[x^2], dS/dE[xy] per
 * channel at each pixel, zero outside the image) and adds the owned pixels' share of the
 * batch loss sum_v L_v / b_loss to *loss_sum (device double, atomically).
 * gs_ssim_grad: maps with their halo (halo_maps [n_halo][2304]), the same out_rgb and gt;
 * writes dL_dpix[n_owned][3][256] (zero outside the image).  A halo block missing from
 * halo_ids traps the kernel (contract violation).                                       */
gs_status gs_ssim_terms(gs_ctx* ctx, const float* out_rgb, const float* halo_rgb, const int64_t* halo_ids,
                        int64_t n_halo, const uint8_t* gt, const gs_camera* cams_h, int n_views,
                        const int64_t* dp_h, float lambda, int b_loss, float* maps, double* loss_sum,
                        void* stream);
gs_status gs_ssim_grad(gs_ctx* ctx, const float* maps, const float* halo_maps, const int64_t* halo_ids,
                       int64_t n_halo, const float* out_rgb, const uint8_t* gt, const gs_camera* cams_h,
                       int n_views, const int64_t* dp_h, float lambda, int b_loss, float* dL_dpix,
                       void* stream);

/* ------------------------------------------------------------------- NEXT-2 densification */
/* Adaptive density control on the Gaussians' owner (App. A.1, App. A.3
 * "locally on the GPU that stores them"; readings R13-R14 in DESIGN.md).       */

/* gs_densify_stats -- after gs_exchange_grads of a step (before or after gs_adam_step):
 * for every (owned Gaussian i, view v) with a record, adds to grad_accum[i] the norm of the
 * screen-space mean gradient of the per-image loss, || b (W/2 dL/dmx, H/2 dL/dmy) || (NDC
 * units, the batch-mean loss scaled back by b = b_loss), adds 1 to denom[i], and raises
 * max_radius[i] to the record's screen radius.  bwd_index, send_rec and dL_dsend are the
 * step's gs_project / gs_exchange_grads buffers (same layouts); the three statistics arrays
 * are device float[n], accumulated in place.                                             */
gs_status gs_densify_stats(gs_ctx* ctx, const gs_camera* cams_h, int n_views, const int64_t* dp_h, int64_t n,
                           const void* bwd_index, const void* send_rec, const float* dL_dsend, int b_loss,
                           float* grad_accum, float* denom, float* max_radius, void* stream);

typedef struct {
  float grad_thresh;     /* average statistic selecting a Gaussian (0.0002, P's Table "(0.0002, 0.01)") */
  float percent_dense;   /* max scale <= percent_dense * extent: clone, else split (0.01)          */
  float scene_extent;    /* radius of the camera positions' bounding sphere               */
  float min_opacity;     /* prune below (0.005)                                                    */
  float max_screen_size; /* > 0: also prune max screen radius above it and max scale > 0.1 extent  */
} gs_densify_cfg;

/* gs_densify -- one densify-and-prune event on the rank's shard.  Selected = grad_accum/denom
 * >= grad_thresh (0 where denom = 0).  A selected Gaussian whose largest log-scale is <=
 * log(percent_dense * extent) is CLONED (an identical copy), otherwise SPLIT into two children
 * x + R(q)(s . z_t), log-scale - log 1.6, opacity/rotation/SH copied, the parent removed;
 * z_t = noise[i][t][0..2] (device float[n][2][3], N(0,1) draws supplied by the caller).
 * Pruned: opacity < min_opacity (all), and with max_screen_size > 0 originals whose
 * max_radius exceeds it or whose largest scale exceeds 0.1 extent (children: 1.6 * 0.1 extent
 * on the parent's scale).  New Gaussians get zero Adam moments; survivors keep theirs.
 * Output (caller-allocated planes laid out for the output count, out_cap Gaussians): kept
 * originals, clones, first children, second children, each in parent order.  counts_h[4] =
 * (kept originals, clones, children, total); GS_ECAPACITY if total > out_cap (host sync).
 * The statistics should be zeroed by the caller afterwards (they index the old shard).    */
gs_status gs_densify(gs_ctx* ctx, const gs_params* p, const gs_params* m, const gs_params* v,
                     const float* grad_accum, const float* denom, const float* max_radius, const float* noise,
                     const gs_densify_cfg* cfg, gs_params* p_out, gs_params* m_out, gs_params* v_out,
                     int64_t out_cap, int64_t* counts_h, void* stream);

/* gs_opacity_reset -- opacity logits clamped to logit(max_opacity) ("opacity reset"),
 * the opacity lanes of the Adam moments m, v zeroed (may be NULL).                      */
gs_status gs_opacity_reset(gs_ctx* ctx, gs_params* p, gs_params* m, gs_params* v, float max_opacity,
                           void* stream);

/* NEXT-2 random redistribution (App. B.2; reading R15): after
 * densification the shard sizes differ; global index j = gid_base + local index moves to
 * position pi(j) of a new global order in which rank d owns [floor(dN/G), floor((d+1)N/G)):
 * sizes differ by at most one, the multiset of Gaussians (parameters + Adam m, v) unchanged.
 * pi = 4-round Feistel bijection keyed by seed on the smallest even bit width covering N,
 * cycle-walked into [0, N) (no table; identical on every rank).  Records of
 * gs_redistribute_record_bytes() bytes: (new local index, p, m, v).                     */
int64_t gs_redistribute_record_bytes(void);

/* gs_redistribute_pack -- this rank's records grouped by destination rank (send_counts_h[G];
 * any order within a group), n_total = N.  GS_ECAPACITY (counts valid) if cap (records) is
 * smaller than the shard.  Host sync.                                                     */
gs_status gs_redistribute_pack(gs_ctx* ctx, const gs_params* p, const gs_params* m, const gs_params* v,
                               int64_t n_total, uint64_t seed, void* send_buf, int64_t cap,
                               int64_t* send_counts_h, void* stream);

/* gs_redistribute_unpack -- places n_recv received records at their new local indices of the
 * output planes (p_out->n == n_recv == the rank's new size; traps on an index outside).     */
gs_status gs_redistribute_unpack(gs_ctx* ctx, const void* recv_buf, int64_t n_recv, gs_params* p_out,
                                 gs_params* m_out, gs_params* v_out, void* stream);

/* gs_redistribute -- COLLECTIVE: all-gathers the shard sizes (p->gid_base must be the rank's
 * offset), packs, exchanges by grouped NCCL point-to-point, unpacks; sets the outputs'
 * gid_base.  Two calls: with recv_buf == NULL on every rank it only returns *n_total_h = N and
 * *n_out_h = the rank's new size; then with send_buf (>= p->n records), recv_buf (>= n_out
 * records) and output planes laid out for n_out.  A capacity below the queried size is a
 * contract violation (GS_EINVAL on that rank only).  World 1: GS_ENOTSUP (the identity).   */
gs_status gs_redistribute(gs_ctx* ctx, const gs_params* p, const gs_params* m, const gs_params* v, uint64_t seed,
                          void* send_buf, int64_t send_cap, void* recv_buf, int64_t recv_cap, gs_params* p_out,
                          gs_params* m_out, gs_params* v_out, int64_t* n_total_h, int64_t* n_out_h, void* stream);

/* ------------------------------------------------------- NEXT-3 peer-memory (NVLink) exchange */
/* NEXT-3 ("sparse all-to-all communication"): the two sparse
 * all-to-alls done by the kernels that produce the data, over peer memory (NVLink stores and
 * reductions on one NVSwitch box) instead of NCCL send/recv:
 *   forward  -- gs_project_put writes every record straight into the DESTINATION rank's
 *               receive buffer (no send buffer, no separate transfer);
 *   backward -- gs_render_bwd_put adds each record's 9 gradient sums straight into the OWNER's
 *               dL/d(sent record) buffer (no receive-side gradient buffer, no reverse transfer).
 * One step with the plan P = the G x G count matrix (row s = records rank s sends to each d):
 *   gs_project_count -> [all-gather counts: gs_exchange_counts or the caller] -> gs_p2p_plan ->
 *   gs_project_put -> gs_p2p_barrier -> gs_bin_sort / gs_render_fwd (on the receive buffer) ->
 *   gs_render_bwd_put -> gs_p2p_barrier -> gs_adam_step (on the own dL/dsend buffer).
 * Receive order is the same as gs_exchange's (ascending source rank, then the source's send
 * order), so every downstream result equals the NCCL path's (gradients up to the order of
 * float additions).  Buffers: each rank allocates its three symmetric buffers with
 * gs_sym_alloc (records, dL/dsend, barrier flags), exports their IPC handles, opens the
 * peers' with gs_ipc_open and attaches all G pointers (gs_p2p_attach).  Ranks of one process
 * (virtual ranks, tests) attach each other's pointers directly.                            */

/* gs_p2p_offsets -- pure host arithmetic of the plan for `rank` (counts_h = G x G, row s =
 * records source s sends to each destination d):
 *   recv_seg_h[G+1]  receive-buffer offset of each source's records (prefix over s of C[s][rank]);
 *   put_base_h[G]    where this rank's records for d start in d's receive buffer
 *                    (sum over s < rank of C[s][d]);
 *   send_off_h[G+1]  this rank's send order: destination buckets (prefix over d of C[rank][d]);
 *   owner_off_h[G]   position, in source s's send order, of the records s sent to this rank
 *                    (sum over d < rank of C[s][d]) -- where their gradients go.
 * GS_EINVAL on a negative count or G outside [1, 32].                                     */
gs_status gs_p2p_offsets(const int64_t* counts_h, int G, int rank, int64_t* recv_seg_h, int64_t* put_base_h,
                         int64_t* send_off_h, int64_t* owner_off_h);

/* gs_sym_alloc -- (re)allocates the context's symmetric buffer `which` (0: receive records,
 * 1: dL/dsend floats, 2: barrier flags, zeroed, 3: count matrix, 4: cost row) of at least `bytes`, returns its device
 * pointer and its 64-byte CUDA IPC handle (for the peers' gs_ipc_open).  Owned by the
 * context (freed by gs_destroy).  Growing invalidates the peers' mappings: re-exchange and
 * re-attach.                                                                               */
gs_status gs_sym_alloc(gs_ctx* ctx, int which, size_t bytes, void** dev_ptr_h, uint8_t handle_h[64]);
/* gs_ipc_open -- maps a peer's IPC handle into this process (peer access over NVLink);
 * closed by gs_destroy.                                                                    */
gs_status gs_ipc_open(gs_ctx* ctx, const uint8_t handle_h[64], void** dev_ptr_h);
/* gs_p2p_attach -- the G ranks' receive buffers (capacity in records), dL/dsend buffers
 * (capacity in records of 9 floats) and flag arrays (G uint64 each), as device pointers valid
 * in this process (entry `rank` = this rank's own).                                        */
gs_status gs_p2p_attach(gs_ctx* ctx, void* const* recv_h, const int64_t* recv_cap_h, void* const* dsend_h,
                        const int64_t* dsend_cap_h, void* const* flags_h);
/* gs_p2p_plan -- sets the step's G x G count matrix (identical on every rank); *n_recv_h =
 * records this rank receives.  GS_ECAPACITY on EVERY rank if any rank's receive or dL/dsend
 * capacity is too small (all ranks see the same matrix and capacities).                    */
gs_status gs_p2p_plan(gs_ctx* ctx, const int64_t* counts_h, int64_t* n_recv_h);
/* gs_exchange_counts -- COLLECTIVE (NCCL all-gather): counts_all_h[G x G] from each rank's
 * send_counts_h[G].  Host sync.                                                            */
gs_status gs_exchange_counts(gs_ctx* ctx, const int64_t* send_counts_h, int64_t* counts_all_h, void* stream);
/* gs_project_count -- the counting half of gs_project: writes bwd_index and send_counts_h
 * (host sync); no records.                                                                  */
gs_status gs_project_count(gs_ctx* ctx, const gs_params* p, const gs_camera* cams_h, int n_views,
                           const int64_t* dp_h, int64_t* send_counts_h, void* bwd_index, void* stream);
/* gs_project_put -- the writing half, fused with the forward exchange: after
 * gs_project_count (same arguments, same bwd_index) and gs_p2p_plan, writes each record to
 * destination d's receive buffer at put_base[d] + its index in the bucket, and zeroes this
 * rank's dL/dsend rows [0, n_send) for the backward's reductions.  Peers may read only after
 * gs_p2p_barrier.                                                                          */
gs_status gs_project_put(gs_ctx* ctx, const gs_params* p, const gs_camera* cams_h, int n_views,
                         const int64_t* dp_h, const void* bwd_index, void* stream);
/* gs_render_bwd_put -- gs_render_bwd on this rank's receive buffer with the reverse exchange
 * fused: record j from source s adds its gradient to s's dL/dsend row owner_off[s] +
 * (j - recv_seg[s]) (float reductions over NVLink).  Same other arguments as gs_render_bwd
 * (black background: no bg argument).
 * Owners may read dL/dsend only after gs_p2p_barrier.                                      */
gs_status gs_render_bwd_put(gs_ctx* ctx, const void* recv_rec, int64_t n_recv, const uint32_t* sorted_idx,
                            const int32_t* tile_range, const gs_camera* cams_h, int n_views, const int64_t* dp_h,
                            const float* dL_dpix, const float* T_final, const int32_t* n_last, int64_t* tile_cost,
                            int cost_mode, int64_t* stats, const uint32_t* cull_bits, void* stream);
/* gs_p2p_barrier -- device-side barrier over the attached flag arrays, asynchronous (no host
 * sync): one kernel writes the next epoch into every rank's flag slot for this rank
 * (system-scope release after the stream's earlier work) and waits until all ranks' slots
 * reached it (acquire).  A wait longer than ~4 s ends the kernel and records a timeout that
 * gs_p2p_status reports (no silent hang).  Virtual ranks of one process must issue it on
 * different streams.                                                                       */
gs_status gs_p2p_barrier(gs_ctx* ctx, void* stream);
/* gs_p2p_status -- GS_ECUDA if a barrier of this context timed out since the last call (and
 * clears it), else GS_OK.  Host sync on `stream`.                                         */
gs_status gs_p2p_status(gs_ctx* ctx, void* stream);

/* Sync-free variant of the forward half (no host round trip between counting and writing):
 *   gs_project_put_dev -> gs_p2p_counts -> gs_p2p_barrier -> gs_bin_sort / gs_render_fwd ->
 *   gs_render_bwd_put -> gs_p2p_put_costs -> gs_p2p_barrier -> gs_adam_step ->
 *   gs_rebalance_row (on the attached own cost row, identical on every rank).
 * The count matrix is exchanged on the devices (row stores + barrier), the record offsets are
 * computed from it inside the writing kernel, and the host reads the matrix (for the sizes
 * the downstream calls take) asynchronously while the records are being written.           */
/* gs_p2p_attach_counts -- the G ranks' count-matrix buffers (G x G int64 each, symmetric
 * buffer 3) and cost-row buffers (row_cap int64 each, symmetric buffer 4; row_cap = 0: none),
 * as device pointers valid in this process.                                                 */
gs_status gs_p2p_attach_counts(gs_ctx* ctx, void* const* cmat_h, void* const* row_h, int64_t row_cap);
/* gs_project_put_dev -- gs_project_count + the count exchange + gs_project_put without a host
 * sync: counts this rank's records per destination into bwd_index, stores the row into every
 * rank's count matrix, device barrier, then writes the records to their destinations'
 * receive buffers at offsets taken from the device matrix and zeroes the own dL/dsend rows.
 * Nothing is written if any destination's receive capacity is too small (gs_p2p_counts then
 * returns GS_ECAPACITY on every rank: grow, re-attach and call again).  Peers may read the
 * records only after the next gs_p2p_barrier.                                              */
gs_status gs_project_put_dev(gs_ctx* ctx, const gs_params* p, const gs_camera* cams_h, int n_views,
                             const int64_t* dp_h, void* bwd_index, void* stream);
/* gs_p2p_counts -- waits for the matrix read-back of the last gs_project_put_dev (host waits
 * on an event, not on the stream), copies it to counts_h[G x G] and sets the plan
 * (gs_p2p_plan: *n_recv_h, GS_ECAPACITY).  GS_ENONFINITE (lowest gid) if that projection saw
 * a non-finite parameter.                                                                   */
gs_status gs_p2p_counts(gs_ctx* ctx, int64_t* counts_h, int64_t* n_recv_h);
/* gs_p2p_put_costs -- this rank's owned cost row (dp_h[rank+1] - dp_h[rank] int64) into every
 * rank's attached cost row at [dp_h[rank], ...); complete on every rank after the next
 * gs_p2p_barrier.  GS_EINVAL if dp_h[G] exceeds the row capacity.                           */
gs_status gs_p2p_put_costs(gs_ctx* ctx, const int64_t* owned_cost, const int64_t* dp_h, void* stream);

/* --------------------------------------------------------------------------- self-check */
/* gs_selftest_ex2 -- the maximum relative error of the renderer's exp2 (ex2.approx.ftz.f32,
 * the alpha = o 2^-q of A4/A5) over every fp32 x in [lo, hi], hi <= 0, against fp64 exp2,
 * into *max_rel_err_h (host sync).  It pins the constant part of the error model the
 * oracle's transmittance margins use (R16).                                               */
gs_status gs_selftest_ex2(gs_ctx* ctx, float lo, float hi, double* max_rel_err_h, void* stream);

#ifdef __cplusplus
}
#endif
#endif
