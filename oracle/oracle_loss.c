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
