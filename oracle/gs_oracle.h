/* gs_oracle.h -- plain, slow, obviously-correct CPU oracle for the Grendel 3DGS
 * training step (arXiv 2406.18533).  TEST INFRASTRUCTURE ONLY: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it.  It shares no code, header, table or constant generator with the CUDA
 * library (include/gs.h, paper_2406_18533_b200/csrc/).
 *
 * Citation key: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * O1..O18 = SURVEY.md §8(c) step table, R1..R11 = the readings listed in DESIGN.md.
 *
 * Precision: the membership chain O1-O8 (visibility, mean2d, depth, 2D covariance,
 * radius, tile rectangle) is evaluated in IEEE fp32, one correctly rounded operation at
 * a time, because it decides integers (tile sets, exchange sets, sort order) and the
 * task rule is that such decisions are taken in the kernel's precision (R10).  All other
 * quantities (conic, opacity, colour, compositing, loss, gradients, Adam) are fp64.
 * Built with -O2 -fno-fast-math -ffp-contract=off (no FMA contraction, no x87).
 */
#ifndef GS_ORACLE_H
#define GS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  float R[9];      /* world->camera rotation, row-major                          */
  float t[3];      /* world->camera translation; camera centre c = -R^T t          */
  float fx, fy, cx, cy;
  int32_t width, height;
} orc_camera;

/* R10: the literal fp32 exp used for s = exp(log_scale) in the membership chain. */
float orc_exp_rn(float x);

/* O1-O8 in fp32 for n Gaussians and one camera.  Outputs per Gaussian:
 * vis (0/1), mx, my, depth (=p_z), cov[3] = (a,b,c) of the dilated 2D covariance,
 * radius, rect[4] = (tx0, tx1, ty0, ty1) inclusive tile ranges.            */
void orc_membership_f32(int64_t n, const float* pos, const float* log_scale, const float* rot,
                        const orc_camera* cam, int8_t* vis, float* mx, float* my, float* depth,
                        float* cov, int32_t* radius, int32_t* rect);

/* O1-O9 entirely in fp64, fp64 parameters (used for finite-difference pins and for the continuous
 * outputs).  out[n][16] = (vis, mx, my, depth, a, b, c, A, B, C, opacity, r, g, b,
 * clampmask, radius); rect[n][4] as in O8 (computed from the fp64 values).   */
void orc_project_f64(int64_t n, const double* pos, const double* log_scale, const double* rot,
                     const double* opac_logit, const double* sh, const orc_camera* cam,
                     double* out, int32_t* rect);

/* O10: destination mask of each (Gaussian) for one view: bit g set iff some tile of
 * rect (view v) lies in [DP[g], DP[g+1]).  Brute force over the rectangle's tiles.  */
void orc_exchange_sets(int64_t n, const int8_t* vis, const int32_t* rect, int32_t view,
                       int32_t Wt, int32_t Ht, int32_t G, const int64_t* DP, uint32_t* mask);

/* O11: per-block lists for blocks [b0, b1) of the serialized batch row.
 * rec_f[n_rec][10] = (mx,my,depth,A,B,C,opacity,r,g,b); rec_i[n_rec][6] =
 * (gid, view, tx0, tx1, ty0, ty1).  offsets[b1-b0+1]; entries = record indices sorted
 * by (depth, gid).  Call with entries == NULL to get offsets only.          */
void orc_tile_lists(int64_t n_rec, const double* rec_f, const int64_t* rec_i, int64_t b0,
                    int64_t b1, int32_t Wt, int32_t Ht, int64_t* offsets, int64_t* entries);

/* O12 (+ O13 when gt != NULL): forward compositing over blocks [b0,b1).
 * Block-major outputs, pixel p = ly*16+lx of the block (the nominal outcome: every decision
 * taken on its exact fp64 side):
 *   out_c[nb][256][3], out_T[nb][256], out_nlast[nb][256] (int32),
 *   flags[nb][256] (bit0: a skip decision alpha < 1/255 within the margin, bit1: a stop
 *                   decision T' < 1e-4 within the margin, bit2: power > 0 met, bit4: more
 *                   outcome paths than max_paths),
 *   counts[nb][256][4] = (E_f, E_fc, E_fs, E_stop), work[nb] = the WORK cost (R17): over the
 *   block's two 8x16 halves (px % 16 < 8, >= 8), the sum of max E_f + max n_last of each half,
 *   dl_dc[nb][256][3] = sign(C-GT)/(3 H W b_total) (only if gt), *loss += sum |C-GT|/(3HWb).
 * margins[4] = (alpha_eps, t_eps, cond_eps, alpha_abs), see gs_oracle.c orc_margins_t.
 * max_paths > 0: every outcome path of the flagged decisions, up to max_paths per pixel
 * (path 0 = nominal): n_paths[nb][256], path_flips[nb][256][P] (bit f: the f-th flagged
 * decision takes its other outcome), path_c[nb][256][P][3] (incl. background), path_T,
 * path_nl[nb][256][P], path_counts[nb][256][P][4].
 * gt is [n_views][H][W][3] uint8 (value/255).  Out-of-image pixels are not rendered. */
void orc_render_fwd(int64_t n_rec, const double* rec_f, const int64_t* offsets,
                    const int64_t* entries, int64_t b0, int64_t b1, int32_t W, int32_t H,
                    const double* bg, const uint8_t* gt, int32_t b_total, const double* margins,
                    double* out_c, double* out_T, int32_t* out_nlast, int32_t* flags,
                    int64_t* counts, int64_t* work, double* dl_dc, double* loss,
                    int32_t max_paths, int32_t* n_paths, uint64_t* path_flips, double* path_c,
                    double* path_T, int32_t* path_nl, int64_t* path_counts);

/* O14-O15: backward of O12 given dl_dc[nb][256][3]; accumulates grad_rec[n_rec][9] =
 * dL/d(mx, my, A, B, C, opacity, r, g, b) summed over all pixels.  Each pixel follows the
 * outcome path flips[nb][256] (NULL: nominal) of orc_render_fwd with the same margins. */
void orc_render_bwd(int64_t n_rec, const double* rec_f, const int64_t* offsets,
                    const int64_t* entries, int64_t b0, int64_t b1, int32_t W, int32_t H,
                    const double* bg, const double* dl_dc, const double* margins, const uint64_t* flips,
                    double* grad_rec);

/* O16: transformation backward in fp64, summed over n_cam views.
 * grad_rec_v[n_cam][n][9] (zero rows for invisible (i,v)), out grad[n][59] =
 * (pos 3, log_scale 3, rot 4, opacity_logit 1, sh 48).                        */
void orc_project_bwd(int64_t n, const double* pos, const double* log_scale, const double* rot,
                     const double* opac_logit, const double* sh, int32_t n_cam,
                     const orc_camera* cams, const double* grad_rec_v, double* grad);

/* O17: one Adam step on n elements with Eq. (1)-(2) batch scaling.            */
void orc_adam(int64_t n, double* theta, double* m, double* v, const double* g, double lr,
              double beta1, double beta2, double eps, int32_t batch, int64_t step);

/* O18 (Algorithm 1): DP[G+1] from ET[B] in exact int64.  Returns 0, or -1
 * if the overflow guard B*max(ET)*G < 2^63 fails.                            */
int orc_division_points(const int64_t* ET, int64_t B, int32_t G, int64_t* DP);

/* A9: per-block cost -> ET for the blocks just rendered (mode 0 MEASURED / 1 WORK: the
 * cost itself; mode 2 PAPER_AVG: floor(C_g * npix_b / npix_g)).            */
void orc_costs_to_et(int32_t mode, int64_t B, int32_t G, const int64_t* DP, const int64_t* cost,
                     const int64_t* npix, int64_t* et);

/* A9 step 3 (R17): ET of the next batch from history rows (-1 = never rendered) and the
 * rendered batch's per-pixel rate rate_num / rate_den (unseen: floor(rate_num npix / rate_den),
 * or npix while rate_num == 0).                                                          */
void orc_next_et(int64_t B_next, const int64_t* hist, const int64_t* npix, int64_t rate_num, int64_t rate_den,
                 int64_t* et);

/* NEXT-1 (reading R12): L = (1-lambda) L1 + lambda (1 - SSIM) of one
 * image, img/gt [H][W][3] in [0,1]; SSIM = mean over pixels and channels of the 11x11
 * Gaussian-window (sigma 1.5) SSIM map with zero padding; grad[H][W][3] = dL/dimg (may be
 * NULL).  Direct window sums in fp64 (O(121 H W) per channel).                       */
void orc_ssim_loss(int32_t W, int32_t H, const double* img, const double* gt, double lambda, double* loss,
                   double* ssim_mean, double* grad);

#ifdef __cplusplus
}
#endif
#endif
