/*
 * oracle.h -- CPU ORACLE for the compact-3DGS-SLAM renderer hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2403_11247_b200/) never includes, links or calls it,
 * and this code includes nothing from the product (no shared headers,
 * helpers, constants or generators).
 *
 * What it is: a plain, slow, obviously-correct C11 implementation of what the
 * hot path computes, written from PAPER.md (arXiv 2403.11247) and the
 * readings recorded in DESIGN.md ("Readings" table, R1..R26).  Citations
 * below use "P:n" = /root/reference/PAPER.md line n.
 *
 * Precision policy:
 *   - every discrete decision (culls, tile rects, the per-pixel q <= k^2 test,
 *     codebook argmin, mask test) is taken in float32 "decision arithmetic"
 *     (DA): IEEE round-to-nearest single ops in the written order, fmaf only
 *     where written.  Build with -ffp-contract=off (no silent FMA contraction).
 *   - every continuous value (alpha, transmittance, images, gradients) is
 *     computed in float64.
 *
 * Parity status of each function: see DESIGN.md "Oracle pins".  No function
 * here is "parity unpinned".
 */
#ifndef CSPLAT_ORACLE_H
#define CSPLAT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Pinhole intrinsics K plus image size and near/far clip (R21). */
typedef struct { float fx, fy, cx, cy; int32_t width, height; float near_z, far_z; } or_camera;
/* World->camera [R|t], row-major 3x4 ("{R_i|t_i}"). */
typedef struct { float m[12]; } or_view;
/* Renderer constants: mask threshold eps (Eq 6; R12), alpha cap
 * (R1), transmittance cutoff (R3), 2D dilation (R5). */
typedef struct { float mask_eps, alpha_max, t_min, dilation; } or_params;
/* Gaussian map, planar SoA [k][n] (R15). */
typedef struct {
    int64_t n;
    const float *mean;      /* [3][n] world position          */
    const float *opacity;   /* [n]   opacity logit, o = sig() */
    const float *rgb;       /* [3][n] raw colour              */
    const float *log_scale; /* [3][n] log of S diagonal       */
    const float *quat;      /* [4][n] wxyz, unnormalised      */
    const float *mask;      /* [n]   mask logit m (Eq 6)      */
} or_gaussians;
/* Residual-VQ geometry codebooks (Eq 10; R16-R18). */
typedef struct {
    int32_t stages, size;          /* L, P */
    const float *scale_codes;      /* [L][P][3] log-scale codes  */
    const float *rot_codes;        /* [L][P][4] quaternion codes */
    const uint16_t *scale_idx;     /* [L][n] */
    const uint16_t *rot_idx;       /* [L][n] */
} or_codebook;

/* Projected record: 16 x 32-bit words per Gaussian (layout in DESIGN.md):
 * 0 u, 1 v, 2 ca, 3 cb+cb, 4 cc, 5 o_hat, 6 k2, 7 z_c, 8 r, 9 g, 10 b,
 * 11 gid (u32), 12 px0|py0<<16, 13 px1|py1<<16 (inclusive pixel rectangle), 14 0, 15 0.
 * Culled Gaussians: all 16 words 0 and count 0. */
#define OR_REC_WORDS 16
#define OR_TILE 16

int oracle_project(const or_gaussians *g, const or_codebook *cb, const or_camera *cam,
                   const or_view *view, const or_params *prm, uint32_t *rec, int32_t *count);

int oracle_bin_tiles(const uint32_t *rec, const int32_t *count, int64_t n, const or_camera *cam,
                     int64_t pair_capacity, uint32_t *pair_gid, uint32_t *tile_range,
                     int64_t *n_pairs);

/* Tiled forward (Eq 3-5).  flags[p]=1 marks a pixel whose termination or
 * cap decision lies within the float32-vs-float64 ambiguity window (DESIGN.md
 * "Comparison policy").  counters: [0]=E_pix (examined), [1]=E_contrib. */
int oracle_render_fwd(const uint32_t *rec, const uint32_t *pair_gid, const uint32_t *tile_range,
                      const or_camera *cam, const or_params *prm,
                      double *color, double *depth, double *sil, double *t_final,
                      int32_t *n_contrib, uint8_t *flags, int64_t *counters);

/* Per-pixel brute force over all n records (the untiled definition). */
int oracle_render_pixel(const uint32_t *rec, const int32_t *count, int64_t n, const or_camera *cam,
                        const or_params *prm, int32_t px, int32_t py, double *out6,
                        int32_t *n_composited);

/* Backward of the tiled forward, float64.  grads: 15 planes [15][n]
 * (mean3, opacity, rgb3, log_scale3, quat4, mask) then pose[6]=(omega,v).
 * accumulate2d (optional, [n][10]) receives the per-Gaussian 2D gradients
 * (u, v, ca, cb, cc, o_hat, z, r, g, b). */
int oracle_render_bwd(const or_gaussians *g, const or_codebook *cb, const or_camera *cam,
                      const or_view *view, const or_params *prm, const uint32_t *rec,
                      const uint32_t *pair_gid, const uint32_t *tile_range,
                      const double *d_color, const double *d_depth, const double *d_sil,
                      const uint8_t *pixel_weight_zero, double *grads, double *pose,
                      double *acc2d);

/* Smooth mode (float64 throughout, no alpha cap / q cutoff / termination,
 * continuous mask M = sig(m), J clamp optional): only for finite-difference
 * pins of the analytic backward.  pose_xi (optional) = (omega, v): the view
 * becomes p' = Rod(omega) (W p + t) + v. */
int oracle_smooth_render(const or_gaussians *g, const or_camera *cam, const or_view *view,
                         const double *pose_xi, const or_params *prm, int32_t clamp,
                         double *color, double *depth, double *sil);
int oracle_smooth_bwd(const or_gaussians *g, const or_camera *cam, const or_view *view,
                      const or_params *prm, int32_t clamp, const double *d_color,
                      const double *d_depth, const double *d_sil, double *grads, double *pose);

/* R-VQ greedy assignment (Eq 10).  idx [L][n] u16, recon [d][n] optional. */
int oracle_rvq_assign(const float *x, int64_t n, int32_t d, const float *codes, int32_t L,
                      int32_t P, uint16_t *idx, float *recon);

/* NEXT-2: one k-means M-step of the R-VQ codebooks for a given assignment
 * (Eq 11, reading R28).  codes_out [L][P][d], counts [L][P], loss_out [L+1]
 * = per-stage squared errors and L_r. */
int oracle_rvq_update(const float *x, int64_t n, int32_t d, const float *codes, int32_t L,
                      int32_t P, const uint16_t *idx, float *codes_out, int32_t *counts,
                      double *loss_out);

/* NEXT-2: straight-through gradient of the R-VQ decode (Eq 10 first line,
 * P:164, S_hat = sum_l C^l[i^l]; reading R31).  d_shat [d][n] = dL/dS_hat
 * (the renderer's decoded-geometry gradient); d_codes [L][P][d] (float64) =
 * sum over n with i_n^l = k of d_shat_n, for every stage l; with accumulate
 * = 0 it is overwritten.  (The STE gradient of the raw vector S is d_shat
 * itself.) */
int oracle_rvq_code_grad(const double *d_shat, int64_t n, int32_t d, const uint16_t *idx,
                         int32_t L, int32_t P, double *d_codes, int32_t accumulate);

/* NEXT-2: Fig 4 codebook initialisation of stage l ("randomly select
 * codebook initialization"; reading R32): C^l[k] = the stage-l residual
 * S_s - S_hat_s^{l-1} of the sampled vector s = sample[k] (k < P), with
 * S_hat^{l-1} the stage-order float32 sum of the codes of stages < l at the
 * indices idx[0..l-1][s] (from oracle_rvq_assign with l stages).  codes is
 * [L][P][d]; only stage l is written. */
int oracle_rvq_init_stage(const float *x, int64_t n, int32_t d, float *codes, int32_t L,
                          int32_t P, int32_t l, const uint16_t *idx, const int64_t *sample);

/* Mask prune: order-preserving compaction of survivors of
 * m > tau.  in_planes: n_planes float planes [n] each; idx planes u16 [n].
 * reset_mask: if not NaN, the mask plane (plane index mask_plane) of
 * survivors is set to it. */
int oracle_mask_prune(int64_t n, const float *mask, float mask_eps,
                      int32_t n_planes, const float *const *in_planes, float *const *out_planes,
                      int32_t n_idx_planes, const uint16_t *const *in_idx, uint16_t *const *out_idx,
                      int32_t mask_plane, float reset_mask, int32_t *keep_map, int64_t *n_kept);

/* NEXT-3: Eq 8 mask loss restricted to the frustum (d_mask accumulated) and
 * the keyframe-overlap counts of the sliding-window selection (reading R29). */
double oracle_mask_loss(const float *mask, const uint8_t *active, int64_t n, double lambda,
                        double *d_mask);
int oracle_keyframe_overlap(const float *depth, const or_camera *cam, const or_view *cur,
                            const or_view *views, int32_t K, int64_t *counts);

/* NEXT-1 tracking loss (Eq 12 gated by Eq 14, reading R27): upstream
 * gradients dL/d(colour, depth, silhouette) and loss3 = (L_t, L_c, L_d). */
int oracle_tracking_loss(const double *color, const double *depth, const double *sil,
                         const float *obs_color, const float *obs_depth, int32_t width,
                         int32_t height, double lambda_d, double gate, double *d_color,
                         double *d_depth, double *d_sil, double *loss3, uint8_t *flags);

/* NEXT-4: random-ray (8x8 patch) global BA loss of one keyframe (
 * reading R30): adds its share of (L_c, L_d, mean SSIM) to loss3 and writes
 * the upstream gradients on the patch pixels (zero elsewhere). */
int oracle_ba_patch_loss(const double *color, const double *depth, const float *obs_color,
                         const float *obs_depth, int32_t width, int32_t height,
                         const int32_t *patches, int64_t n_patches, int64_t n_rays,
                         int64_t n_valid, double lambda_d, double lambda_s, double c1,
                         double c2, double *d_color, double *d_depth, double *d_sil,
                         double *loss3);

/* Restrict oracle_render_fwd/bwd to pixel rows [row_lo, row_hi) (row_hi < 0:
 * all rows) -- used only to time a bounded CPU-baseline sample. */
void oracle_set_row_window(int32_t row_lo, int32_t row_hi);
/* OpenMP threads of the per-Gaussian, per-vector and per-pixel loops (default
 * 1).  Used ONLY by bench.py's timed CPU baseline (1 thread and
 * all cores).  Results do not depend on it except for the summation order of
 * the backward's per-thread partial sums (float64, reduced in thread order). */
void oracle_set_threads(int32_t n);
/* Flagging window of oracle_render_fwd; defaults 1e-5, 1e-6. */
void oracle_set_flag_window(double t_rel, double cap_abs);

/* DA helpers exported for pins. */
float oracle_pexp(float x);
float oracle_plog(float x);
float oracle_mask_tau(float eps);

#ifdef __cplusplus
}
#endif
#endif
