/*
 * oracle_loss.c -- ORACLE (test infrastructure, see oracle.h).
 *
 * NEXT-1: the tracking objective of Sec 3.4, Eq 12 gated by the
 * silhouette as in Eq 14, without the SIFT reprojection term
 * (out of scope).  Reading R27: per pixel p,
 *   g_p = 1[S_p > gate]            (Eq 14, gate = 0.99)
 *   v_p = 1[D_obs(p) > 0]          (R_i of Eq 12: rays with a valid depth)
 *   L_c = (1/N) sum_p g_p sum_c (C_p,c - C_obs_p,c)^2,   N = number of pixels
 *   L_d = (1/|R|) sum_p g_p v_p (D_p - D_obs_p)^2,      |R| = sum_p v_p (>= 1)
 *   L_t = L_c + lambda_1 L_d
 * Gradients (the gate is a hard threshold: no gradient through S):
 *   dL/dC_p,c = 2 g_p (C - C_obs)/N,  dL/dD_p = 2 lambda_1 g_p v_p (D - D_obs)/|R|,
 *   dL/dS_p = 0.
 * flags[p] = 1 when |S_p - gate| < 1e-5 (float32 vs float64 gate ambiguity).
 */
#include "oracle_internal.h"

/* NEXT-3 (a): the mask sparsity loss of Eq 8, L_m = (1/N) sum_n
 * Sig(m_n), restricted to the Gaussians inside the current viewing frustum
 * ("optimize only the mask within the current viewing frustum"; reading
 * R29: frustum membership = the Gaussian's projection touches the image,
 * i.e. tile count > 0 or the mask is off but the centre is in the frustum --
 * here: active[n] != 0 supplied by the caller).  d_mask[n] += lambda Sig'(m)/N_a
 * for active n (N_a = number of active); returns L_m. */
double oracle_mask_loss(const float *mask, const uint8_t *active, int64_t n, double lambda,
                        double *d_mask)
{
    int64_t na = 0;
    for (int64_t i = 0; i < n; i++) na += active[i] != 0;
    if (na == 0) return 0.0;
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) {
        if (!active[i]) continue;
        const double sg = 1.0 / (1.0 + exp(-(double)mask[i]));
        s += sg;
        d_mask[i] += lambda * sg * (1.0 - sg) / (double)na;
    }
    return s / (double)na;
}

/* NEXT-3 (b): keyframe overlap ("tallying points within the frustum of
 * each keyframe"): every valid depth pixel of the current frame is
 * back-projected, X = V_cur^-1 (D K^-1 [px, py, 1]), and counted for keyframe
 * k when V_k X has near < z < far and projects inside [0, W-1] x [0, H-1]
 * (reading R29).  counts[k] = number of such points. */
int oracle_keyframe_overlap(const float *depth, const or_camera *cam, const or_view *cur,
                            const or_view *views, int32_t K, int64_t *counts)
{
    /* float32 decision arithmetic in the written order (the counts are integers
     * compared bit-exactly with the GPU) */
    const int W = cam->width, H = cam->height;
    const float *C = cur->m;
    const float Wm1 = (float)W - 1.0f, Hm1 = (float)H - 1.0f;
    for (int k = 0; k < K; k++) counts[k] = 0;
    for (int py = 0; py < H; py++)
        for (int px = 0; px < W; px++) {
            const float d = depth[(int64_t)py * W + px];
            if (!(d > 0.0f)) continue;
            const float xn = ((float)px - cam->cx) / cam->fx, yn = ((float)py - cam->cy) / cam->fy;
            const float qx = xn * d - C[3], qy = yn * d - C[7], qz = d - C[11];
            float X[3];  /* R^T (p_c - t) */
            for (int a = 0; a < 3; a++) X[a] = (C[a] * qx + C[4 + a] * qy) + C[8 + a] * qz;
            for (int k = 0; k < K; k++) {
                const float *V = views[k].m;
                const float xc = ((V[0] * X[0] + V[1] * X[1]) + V[2] * X[2]) + V[3];
                const float yc = ((V[4] * X[0] + V[5] * X[1]) + V[6] * X[2]) + V[7];
                const float zc = ((V[8] * X[0] + V[9] * X[1]) + V[10] * X[2]) + V[11];
                if (!(zc > cam->near_z) || !(zc < cam->far_z)) continue;
                /* 0 <= fx xc/zc + cx <= W-1, multiplied through by zc > 0 */
                const float ax = cam->fx * xc, ay = cam->fy * yc;
                if (ax >= (-cam->cx) * zc && ax <= (Wm1 - cam->cx) * zc &&
                    ay >= (-cam->cy) * zc && ay <= (Hm1 - cam->cy) * zc)
                    counts[k]++;
            }
        }
    return 0;
}

int oracle_tracking_loss(const double *color, const double *depth, const double *sil,
                         const float *obs_color, const float *obs_depth, int32_t width,
                         int32_t height, double lambda_d, double gate, double *d_color,
                         double *d_depth, double *d_sil, double *loss3, uint8_t *flags)
{
    const int64_t HW = (int64_t)width * height;
    int64_t nvalid = 0;
    for (int64_t p = 0; p < HW; p++) nvalid += obs_depth[p] > 0.0f;
    const double N = (double)HW, R = (double)(nvalid > 0 ? nvalid : 1);
    double lc = 0.0, ld = 0.0;
    for (int64_t p = 0; p < HW; p++) {
        const double g = sil[p] > gate ? 1.0 : 0.0;
        const double v = obs_depth[p] > 0.0f ? 1.0 : 0.0;
        if (flags) flags[p] = fabs(sil[p] - gate) < 1e-5;
        for (int c = 0; c < 3; c++) {
            const double r = color[c * HW + p] - (double)obs_color[c * HW + p];
            lc += g * r * r;
            d_color[c * HW + p] = 2.0 * g * r / N;
        }
        const double rd = depth[p] - (double)obs_depth[p];
        ld += g * v * rd * rd;
        d_depth[p] = 2.0 * lambda_d * g * v * rd / R;
        d_sil[p] = 0.0;
    }
    loss3[1] = lc / N;
    loss3[2] = ld / R;
    loss3[0] = loss3[1] + lambda_d * loss3[2];
    return 0;
}

/* NEXT-4: the loss of the random-ray global bundle adjustment (Sec 3.4 "Global
 * Bundle Adjustment": "randomly sample a total number of N rays from
 * our global keyframe database ... a loss similar to tracking loss, and we also
 * add an SSIM loss to RGB rendering").  Reading R30: the N rays are
 * drawn as N/64 random 8x8 pixel patches (block-aligned), so that the SSIM
 * term has a window; no silhouette gate.  Over the whole sample:
 *   L_c    = (1/N) sum_rays sum_c (C - C_obs)^2                     (Eq 12)
 *   L_d    = (1/|R|) sum_{rays, D_obs > 0} (D - D_obs)^2             (Eq 12)
 *   SSIM_b = mean over the patches b and channels c of
 *            (2 mx my + C1)(2 sxy + C2) / ((mx^2 + my^2 + C1)(sx^2 + sy^2 + C2)),
 *            m, s^2, sxy the patch mean, (population) variance, covariance
 *   L_ba   = L_c + lambda_d L_d + lambda_s (1 - SSIM_b)
 * This call handles the patches of ONE keyframe and ADDS its share:
 *   loss3[0] += its part of L_c, loss3[1] += of L_d, loss3[2] += of SSIM_b,
 * with the sample-wide normalisers n_rays (= N) and n_valid (= |R|) given.
 * Gradients (written on the patch pixels, zero elsewhere):
 *   dL/dC_i = 2 (C_i - C_obs_i)/N - lambda_s/(3P) dSSIM_c/dC_i,  P = N/64,
 *   dSSIM/dx_i = (2S/64) [my/A1 + (y_i - my)/A2 - mx/B1 - (x_i - mx)/B2]
 *   (A1, A2, B1, B2 the four factors above), dL/dD_i = 2 lambda_d v_i (D - D_obs)/|R|,
 *   dL/dS = 0.  patches[b] = by * (W/8) + bx (block origin (8 bx, 8 by)). */
int oracle_ba_patch_loss(const double *color, const double *depth, const float *obs_color,
                         const float *obs_depth, int32_t width, int32_t height,
                         const int32_t *patches, int64_t n_patches, int64_t n_rays,
                         int64_t n_valid, double lambda_d, double lambda_s, double c1,
                         double c2, double *d_color, double *d_depth, double *d_sil,
                         double *loss3)
{
    const int64_t HW = (int64_t)width * height;
    const int bw = width / 8;
    const double N = (double)n_rays, R = (double)(n_valid > 0 ? n_valid : 1);
    const double P = N / 64.0;
    for (int64_t p = 0; p < HW; p++) {
        d_depth[p] = 0.0;
        d_sil[p] = 0.0;
        for (int c = 0; c < 3; c++) d_color[c * HW + p] = 0.0;
    }
    for (int64_t b = 0; b < n_patches; b++) {
        const int bx = patches[b] % bw, by = patches[b] / bw;
        int64_t pix[64];
        for (int k = 0; k < 64; k++) pix[k] = (int64_t)(8 * by + k / 8) * width + 8 * bx + k % 8;
        for (int k = 0; k < 64; k++) {  /* Eq 12 depth term */
            const int64_t p = pix[k];
            if (obs_depth[p] > 0.0f) {
                const double r = depth[p] - (double)obs_depth[p];
                loss3[1] += r * r / R;
                d_depth[p] = 2.0 * lambda_d * r / R;
            }
        }
        for (int c = 0; c < 3; c++) {
            const double *x = color + c * HW;
            const float *y = obs_color + c * HW;
            double mx = 0.0, my = 0.0;
            for (int k = 0; k < 64; k++) { mx += x[pix[k]]; my += (double)y[pix[k]]; }
            mx /= 64.0;
            my /= 64.0;
            double sxx = 0.0, syy = 0.0, sxy = 0.0;
            for (int k = 0; k < 64; k++) {
                const double dx = x[pix[k]] - mx, dy = (double)y[pix[k]] - my;
                sxx += dx * dx;
                syy += dy * dy;
                sxy += dx * dy;
            }
            sxx /= 64.0;
            syy /= 64.0;
            sxy /= 64.0;
            const double A1 = 2.0 * mx * my + c1, A2 = 2.0 * sxy + c2;
            const double B1 = mx * mx + my * my + c1, B2 = sxx + syy + c2;
            const double S = A1 * A2 / (B1 * B2);
            loss3[2] += S / (3.0 * P);
            for (int k = 0; k < 64; k++) {
                const int64_t p = pix[k];
                const double xi = x[p], yi = (double)y[p];
                const double dS = 2.0 * S / 64.0 *
                                  (my / A1 + (yi - my) / A2 - mx / B1 - (xi - mx) / B2);
                const double r = xi - yi;
                loss3[0] += r * r / N;
                d_color[c * HW + p] = 2.0 * r / N - lambda_s / (3.0 * P) * dS;
            }
        }
    }
    return 0;
}
