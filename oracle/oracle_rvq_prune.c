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
#include <stdlib.h>

int oracle_rvq_assign(const float *x, int64_t n, int32_t d, const float *codes, int32_t L,
                      int32_t P, uint16_t *idx, float *recon)
{
    if (n < 0 || d < 1 || d > 8 || L < 1 || P < 1 || P > 65536) return 1;
#pragma omp parallel for num_threads(or_threads()) schedule(static)
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

/* NEXT-2: one k-means M-step of the R-VQ codebooks given an assignment
 * (Eq 11; SPEC rvq_train S:308-316 as the update rule, reading
 * R28).  For every stage l and vector n: r_n = x_n - S_hat_n^{l-1} (float32,
 * stage-order sum of the assigned codes, as in oracle_rvq_assign), then
 *   sum_l[k] += r_n, cnt_l[k] += 1 for k = i_n^l,
 *   err_l    += ||r_n - C^l[i_n^l]||^2          (float64)
 * new C^l[k] = sum_l[k] / cnt_l[k] (unchanged when cnt = 0).
 * loss_out[0..L-1] = err_l, loss_out[L] = L_r = sum_l err_l / (n P). */
int oracle_rvq_update(const float *x, int64_t n, int32_t d, const float *codes, int32_t L,
                      int32_t P, const uint16_t *idx, float *codes_out, int32_t *counts,
                      double *loss_out)
{
    if (n < 0 || d < 1 || d > 8 || L < 1 || P < 1) return 1;
    double *sum = (double *)calloc((size_t)L * P * d, sizeof(double));
    for (int l = 0; l <= L; l++) loss_out[l] = 0.0;
    for (int64_t k = 0; k < (int64_t)L * P; k++) counts[k] = 0;
    for (int64_t i = 0; i < n; i++) {
        float sh[8];
        for (int j = 0; j < d; j++) sh[j] = 0.0f;
        for (int l = 0; l < L; l++) {
            const int k = idx[(int64_t)l * n + i];
            const float *c = codes + ((int64_t)l * P + k) * d;
            double e2 = 0.0;
            for (int j = 0; j < d; j++) {
                const float r = x[(int64_t)j * n + i] - sh[j];          /* S - S_hat^{l-1} */
                sum[((int64_t)l * P + k) * d + j] += r;
                const double e = (double)r - (double)c[j];
                e2 += e * e;
            }
            counts[(int64_t)l * P + k] += 1;
            loss_out[l] += e2;
            for (int j = 0; j < d; j++) sh[j] = (l == 0) ? c[j] : sh[j] + c[j];
        }
    }
    for (int64_t k = 0; k < (int64_t)L * P; k++)
        for (int j = 0; j < d; j++)
            codes_out[k * d + j] = counts[k] > 0 ? (float)(sum[k * d + j] / counts[k])
                                                 : codes[k * d + j];
    double tot = 0.0;
    for (int l = 0; l < L; l++) tot += loss_out[l];
    loss_out[L] = n > 0 ? tot / ((double)n * P) : 0.0;
    free(sum);
    return 0;
}

/* NEXT-2 STE (reading R31): Eq 10 decodes S_hat = sum_l C^l[i^l]; the
 * straight-through estimator passes dL/dS_hat to the raw vector unchanged,
 * and since S_hat is linear in every code, dL/dC^l[k] = sum of dL/dS_hat_n
 * over the vectors with i_n^l = k (each stage's chosen code receives the full
 * gradient). */
int oracle_rvq_code_grad(const double *d_shat, int64_t n, int32_t d, const uint16_t *idx,
                         int32_t L, int32_t P, double *d_codes, int32_t accumulate)
{
    if (n < 0 || d < 1 || d > 8 || L < 1 || P < 1) return 1;
    if (!accumulate)
        for (int64_t k = 0; k < (int64_t)L * P * d; k++) d_codes[k] = 0.0;
    for (int64_t i = 0; i < n; i++)
        for (int l = 0; l < L; l++) {
            const int k = idx[(int64_t)l * n + i];
            if (k >= P) continue;                         /* culled */
            for (int j = 0; j < d; j++)
                d_codes[((int64_t)l * P + k) * d + j] += d_shat[(int64_t)j * n + i];
        }
    return 0;
}

/* NEXT-2 Fig 4 (reading R32): stage l's codebook starts as the stage-l
 * residuals of P randomly sampled vectors (the sample is an input). */
int oracle_rvq_init_stage(const float *x, int64_t n, int32_t d, float *codes, int32_t L,
                          int32_t P, int32_t l, const uint16_t *idx, const int64_t *sample)
{
    if (n < 1 || d < 1 || d > 8 || L < 1 || P < 1 || l < 0 || l >= L) return 1;
    for (int k = 0; k < P; k++) {
        const int64_t s = sample[k];
        if (s < 0 || s >= n) return 1;
        float sh[8];
        for (int j = 0; j < d; j++) sh[j] = 0.0f;
        for (int m = 0; m < l; m++) {                     /* S_hat^{l-1}, stage order */
            const float *c = codes + ((int64_t)m * P + idx[(int64_t)m * n + s]) * d;
            for (int j = 0; j < d; j++) sh[j] = (m == 0) ? c[j] : sh[j] + c[j];
        }
        for (int j = 0; j < d; j++)
            codes[((int64_t)l * P + k) * d + j] = x[(int64_t)j * n + s] - sh[j];
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
