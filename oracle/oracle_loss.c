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
