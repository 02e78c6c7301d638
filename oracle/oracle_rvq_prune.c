/*
 * oracle_rvq_prune.c -- ORACLE (test infrastructure, see oracle.h).
 *
 * a2: residual vector quantisation, Eq 10:
 *     S_hat^l = sum_{k<=l} C^k[i^k],  i^l = argmin_k || C^l[k] - (S - S_hat^{l-1}) ||^2,
 *     S_hat^0 = 0.  Greedy stage by stage; ties to the lowest index (R11/R17).
 *     Distances in DA: d_k = fma(e_{d-1}, e_{d-1}, ... fma(e_0, e_0, 0)),
 *     e_j = c_kj - r_j, r_j = x_j - S_hat^{l-1}_j (float32, stated order).
 * a9: mask prune (Fig 3): remove every Gaussian with
 *     Sig(m) <= eps (R12), keep the survivors' relative order.
 */
#include "oracle_internal.h"

int oracle_rvq_assign(const float *x, int64_t n, int32_t d, const float *codes, int32_t L,
                      int32_t P, uint16_t *idx, float *recon)
{
    if (n < 0 || d < 1 || d > 8 || L < 1 || P < 1 || P > 65536) return 1;
    for (int64_t i = 0; i < n; i++) {
        float xi[8], sh[8];
        for (int j = 0; j < d; j++) { xi[j] = x[(int64_t)j * n + i]; sh[j] = 0.0f; }
        for (int l = 0; l < L; l++) {
            float r[8];
            for (int j = 0; j < d; j++) r[j] = xi[j] - sh[j];        /* S - S_hat^{l-1} */
            const float *C = codes + (int64_t)l * P * d;
            int best = 0;
            float bestd = 0.0f;
            for (int k = 0; k < P; k++) {
                float acc = 0.0f;
                for (int j = 0; j < d; j++) {
                    float e = C[(int64_t)k * d + j] - r[j];
                    acc = fmaf(e, e, acc);
                }
                if (k == 0 || acc < bestd) { bestd = acc; best = k; } /* strict <: lowest index */
            }
            idx[(int64_t)l * n + i] = (uint16_t)best;
            for (int j = 0; j < d; j++)                                 /* S_hat^l, stage order */
                sh[j] = (l == 0) ? C[(int64_t)best * d + j] : sh[j] + C[(int64_t)best * d + j];
        }
        if (recon)
            for (int j = 0; j < d; j++) recon[(int64_t)j * n + i] = sh[j];
    }
    return 0;
}

int oracle_mask_prune(int64_t n, const float *mask, float mask_eps, int32_t n_planes,
                      const float *const *in_planes, float *const *out_planes, int32_t n_idx_planes,
                      const uint16_t *const *in_idx, uint16_t *const *out_idx, int32_t mask_plane,
                      float reset_mask, int32_t *keep_map, int64_t *n_kept)
{
    const float tau = oracle_mask_tau(mask_eps);
    int64_t k = 0;
    for (int64_t i = 0; i < n; i++) {
        int keep = mask[i] > tau;                 /* Eq 6: M = 1 iff Sig(m) > eps */
        if (keep_map) keep_map[i] = keep ? (int32_t)k : -1;
        if (!keep) continue;
        for (int p = 0; p < n_planes; p++) {
            float v = in_planes[p][i];
            if (p == mask_plane && !isnan(reset_mask)) v = reset_mask;
            out_planes[p][k] = v;
        }
        for (int p = 0; p < n_idx_planes; p++) out_idx[p][k] = in_idx[p][i];
        k++;
    }
    *n_kept = k;
    return 0;
}
