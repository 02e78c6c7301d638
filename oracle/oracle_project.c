/*
 * oracle_project.c -- ORACLE (test infrastructure, see oracle.h).
 *
 * Step a1 (mask, Eq 6-7), a2-decode (Eq 10) and a3
 * (projection, Eq 1-2) of the hot path, in float32 decision
 * arithmetic (DA), plus the float64 projection and chain rule used by the
 * backward.  The DA op order is the one written in DESIGN.md
 * "Decision arithmetic / projection"; it must be compiled with
 * -ffp-contract=off so every + - * / is a separately rounded float32 op.
 */
#include "oracle_internal.h"
#include <float.h>

/* ---------------- DA transcendentals ("DA pexp/plog") -------- */

/* exact 2^k for k in [-126, 127] */
static float or_pow2(int k) { return or_u2f((uint32_t)(k + 127) << 23); }

float oracle_pexp(float x)
{
    x = fminf(fmaxf(x, -86.0f), 88.0f);
    float k = rintf(x * 1.44269504f);
    float r = fmaf(-k, 0.693145751953125f, x);   /* Cody-Waite ln2 hi */
    r = fmaf(-k, 1.42860677e-06f, r);            /* ln2 lo            */
    float p = 1.98412698e-4f;                    /* Taylor to r^7     */
    p = fmaf(p, r, 1.38888889e-3f);
    p = fmaf(p, r, 8.33333333e-3f);
    p = fmaf(p, r, 4.16666667e-2f);
    p = fmaf(p, r, 0.166666667f);
    p = fmaf(p, r, 0.5f);
    p = fmaf(p, r, 1.0f);
    p = fmaf(p, r, 1.0f);
    return p * or_pow2((int)k);
}

float oracle_plog(float x)
{
    int e;
    float m = frexpf(x, &e);                     /* x = m 2^e, m in [0.5,1) */
    if (m < 0.707106781f) { m = m + m; e = e - 1; }
    float f = m - 1.0f;
    float s = f / (2.0f + f);
    float t = s * s;
    float p = fmaf(t, 0.111111111f, 0.142857143f);
    p = fmaf(t, p, 0.2f);
    p = fmaf(t, p, 0.333333333f);
    p = fmaf(t, p, 1.0f);
    float ef = (float)e;
    return fmaf(ef, 0.693145751953125f, fmaf(ef, 1.42860677e-06f, (s + s) * p));
}

float or_sigm(float x) { return 1.0f / (1.0f + oracle_pexp(-x)); }

/* Eq 6 test Sig(m) > eps, written m > tau with tau = fl32(ln(eps/(1-eps)))
 * computed in double (reading R12). */
float oracle_mask_tau(float eps)
{
    double e = (double)eps;
    return (float)log(e / (1.0 - e));
}

/* ---------------- R-VQ decode (Eq 10 first line) ----------------- */

void or_geometry(const or_gaussians *g, const or_codebook *cb, int64_t i, float ls[3], float q[4])
{
    int64_t n = g->n;
    if (!cb) {
        for (int k = 0; k < 3; k++) ls[k] = g->log_scale[k * n + i];
        for (int k = 0; k < 4; k++) q[k] = g->quat[k * n + i];
        return;
    }
    /* a Gaussian with any index outside [0, P) is culled --
     * reported as a NaN log-scale, which every user of the geometry culls. */
    for (int l = 0; l < cb->stages; l++)
        if (cb->scale_idx[(int64_t)l * n + i] >= (uint32_t)cb->size ||
            cb->rot_idx[(int64_t)l * n + i] >= (uint32_t)cb->size) {
            ls[0] = ls[1] = ls[2] = NAN;
            q[0] = 1.0f; q[1] = q[2] = q[3] = 0.0f;
            return;
        }
    /* S_hat^L = sum_{k=1..L} C^k[i^k], summed in stage order (R17). */
    for (int l = 0; l < cb->stages; l++) {
        uint32_t si = cb->scale_idx[(int64_t)l * n + i];
        uint32_t ri = cb->rot_idx[(int64_t)l * n + i];
        const float *sc = cb->scale_codes + ((int64_t)l * cb->size + si) * 3;
        const float *rc = cb->rot_codes + ((int64_t)l * cb->size + ri) * 4;
        for (int k = 0; k < 3; k++) ls[k] = (l == 0) ? sc[k] : ls[k] + sc[k];
        for (int k = 0; k < 4; k++) q[k] = (l == 0) ? rc[k] : q[k] + rc[k];
    }
}

/* ---------------- DA projection (a1 + a3) -------------------------------- */

static void put_rec_zero(uint32_t *r) { memset(r, 0, OR_REC_WORDS * sizeof(uint32_t)); }

int oracle_project(const or_gaussians *g, const or_codebook *cb, const or_camera *cam,
                   const or_view *view, const or_params *prm, uint32_t *rec, int32_t *count)
{
    if (!g || !cam || !view || !prm || !rec || !count) return 1;
    const int64_t n = g->n;
    const float tau = oracle_mask_tau(prm->mask_eps);
    const float fx = cam->fx, fy = cam->fy, cx = cam->cx, cy = cam->cy;
    const float Wf = (float)cam->width, Hf = (float)cam->height;
    const float *V = view->m;
    /* J clamp limits (R6), DA */
    const float lx_lo = -((cx + 0.15f * Wf) / fx);
    const float lx_hi = ((Wf - cx) + 0.15f * Wf) / fx;
    const float ly_lo = -((cy + 0.15f * Hf) / fy);
    const float ly_hi = ((Hf - cy) + 0.15f * Hf) / fy;
    const float dil = prm->dilation;

#pragma omp parallel for num_threads(or_threads()) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        uint32_t *r = rec + i * OR_REC_WORDS;
        put_rec_zero(r);
        count[i] = 0;
        float m = g->mask[i];
        if (!(m > tau)) continue;                                 /* Eq 6-7 */
        float ls[3], q[4];
        or_geometry(g, cb, i, ls, q);
        float mx = g->mean[i], my = g->mean[n + i], mz = g->mean[2 * n + i];
        float o = g->opacity[i];
        float cr = g->rgb[i], cg = g->rgb[n + i], cbl = g->rgb[2 * n + i];
        /* non-finite inputs are culled */
        if (!isfinite(mx) || !isfinite(my) || !isfinite(mz) || !isfinite(o) || !isfinite(ls[0]) ||
            !isfinite(ls[1]) || !isfinite(ls[2]) || !isfinite(q[0]) || !isfinite(q[1]) ||
            !isfinite(q[2]) || !isfinite(q[3]) || !isfinite(cr) || !isfinite(cg) || !isfinite(cbl))
            continue;
        float s0 = oracle_pexp(ls[0]), s1 = oracle_pexp(ls[1]), s2 = oracle_pexp(ls[2]);
        float oh = or_sigm(o);
        float a255 = 255.0f * oh;
        if (!(a255 > 1.0f)) continue;                             /* alpha >= 1/255 possible (R2) */
        float k2 = 2.0f * oracle_plog(a255);
        float xc = ((V[0] * mx + V[1] * my) + V[2] * mz) + V[3];
        float yc = ((V[4] * mx + V[5] * my) + V[6] * mz) + V[7];
        float zc = ((V[8] * mx + V[9] * my) + V[10] * mz) + V[11];
        if (!(zc > cam->near_z) || !(zc < cam->far_z)) continue;  /* R21 */
        float nq = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
        if (!(nq > 0.0f)) continue;
        float rn = 1.0f / sqrtf(nq);
        float w = q[0] * rn, x = q[1] * rn, y = q[2] * rn, z = q[3] * rn;
        float R[3][3];
        R[0][0] = 1.0f - 2.0f * (y * y + z * z);
        R[0][1] = 2.0f * (x * y - w * z);
        R[0][2] = 2.0f * (x * z + w * y);
        R[1][0] = 2.0f * (x * y + w * z);
        R[1][1] = 1.0f - 2.0f * (x * x + z * z);
        R[1][2] = 2.0f * (y * z - w * x);
        R[2][0] = 2.0f * (x * z - w * y);
        R[2][1] = 2.0f * (y * z + w * x);
        R[2][2] = 1.0f - 2.0f * (x * x + y * y);
        float s[3] = {s0, s1, s2};
        float M[3][3];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) M[a][b] = R[a][b] * s[b];
        float S[3][3];                                            /* Eq 1: R S S^T R^T */
        for (int a = 0; a < 3; a++)
            for (int b = a; b < 3; b++) {
                S[a][b] = (M[a][0] * M[b][0] + M[a][1] * M[b][1]) + M[a][2] * M[b][2];
                S[b][a] = S[a][b];
            }
        float iz = 1.0f / zc;
        float txz = xc * iz, tyz = yc * iz;
        float tx = fminf(fmaxf(txz, lx_lo), lx_hi) * zc;
        float ty = fminf(fmaxf(tyz, ly_lo), ly_hi) * zc;
        float J00 = fx * iz, J02 = -(fx * tx) * (iz * iz);
        float J11 = fy * iz, J12 = -(fy * ty) * (iz * iz);
        float A[2][3];                                            /* A = J W */
        for (int j = 0; j < 3; j++) {
            A[0][j] = J00 * V[j] + J02 * V[8 + j];
            A[1][j] = J11 * V[4 + j] + J12 * V[8 + j];
        }
        float B[2][3];                                            /* B = A Sigma */
        for (int a = 0; a < 2; a++)
            for (int j = 0; j < 3; j++)
                B[a][j] = (A[a][0] * S[0][j] + A[a][1] * S[1][j]) + A[a][2] * S[2][j];
        /* Eq 2: Sigma' = J W Sigma W^T J^T, plus dilation (R5) */
        float ca_ = ((B[0][0] * A[0][0] + B[0][1] * A[0][1]) + B[0][2] * A[0][2]) + dil;
        float cb_ = (B[0][0] * A[1][0] + B[0][1] * A[1][1]) + B[0][2] * A[1][2];
        float cc_ = ((B[1][0] * A[1][0] + B[1][1] * A[1][1]) + B[1][2] * A[1][2]) + dil;
        float det = ca_ * cc_ - cb_ * cb_;
        if (!(det > 0.0f)) continue;
        float con_a = cc_ / det, con_b = -cb_ / det, con_c = ca_ / det;
        float u = fx * txz + cx, v = fy * tyz + cy;
        float ex = sqrtf(k2 * ca_) + 1e-3f, ey = sqrtf(k2 * cc_) + 1e-3f;
        float X0 = ceilf(u - ex), X1 = floorf(u + ex);
        float Y0 = ceilf(v - ey), Y1 = floorf(v + ey);
        if (!(X0 <= Wf - 1.0f) || !(X1 >= 0.0f) || !(Y0 <= Hf - 1.0f) || !(Y1 >= 0.0f)) continue;
        if (!(X0 <= X1) || !(Y0 <= Y1)) continue;                 /* no pixel centre inside */
        int px0 = (int)fmaxf(X0, 0.0f), px1 = (int)fminf(X1, Wf - 1.0f);
        int py0 = (int)fmaxf(Y0, 0.0f), py1 = (int)fminf(Y1, Hf - 1.0f);
        int tx0 = px0 / OR_TILE, tx1 = px1 / OR_TILE, ty0 = py0 / OR_TILE, ty1 = py1 / OR_TILE;
        r[0] = or_f2u(u);
        r[1] = or_f2u(v);
        r[2] = or_f2u(con_a);
        r[3] = or_f2u(con_b + con_b);
        r[4] = or_f2u(con_c);
        r[5] = or_f2u(oh);
        r[6] = or_f2u(k2);
        r[7] = or_f2u(zc);
        r[8] = or_f2u(cr);
        r[9] = or_f2u(cg);
        r[10] = or_f2u(cbl);
        r[11] = (uint32_t)i;
        r[12] = (uint32_t)px0 | ((uint32_t)py0 << 16);   /* rectangle low corner  */
        r[13] = (uint32_t)px1 | ((uint32_t)py1 << 16);   /* rectangle high corner */
        count[i] = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
    }
    return 0;
}

/* ---------------- float64 projection (backward / smooth mode) ------------ */

static double sigd(double x) { return 1.0 / (1.0 + exp(-x)); }

void or_project64(const or_gaussians *g, const or_codebook *cb, const or_camera *cam,
                  const double W[3][3], const double t[3], const or_params *prm, int64_t i,
                  int mode, or_proj64 *p)
{
    const int smooth = mode & OR_MODE_SMOOTH_MASK, clamp = mode & OR_MODE_CLAMP;
    const int64_t n = g->n;
    memset(p, 0, sizeof(*p));
    float lsf[3], qf[4];
    or_geometry(g, cb, i, lsf, qf);
    p->M = smooth ? sigd((double)g->mask[i]) : 1.0;
    for (int k = 0; k < 3; k++) { p->s[k] = exp((double)lsf[k]); p->sh[k] = p->M * p->s[k]; }
    p->sig_o = sigd((double)g->opacity[i]);
    p->oh = p->M * p->sig_o;
    double qq = 0;
    for (int k = 0; k < 4; k++) qq += (double)qf[k] * (double)qf[k];
    p->qnorm = sqrt(qq);
    for (int k = 0; k < 4; k++) p->qn[k] = (double)qf[k] / p->qnorm;
    double w = p->qn[0], x = p->qn[1], y = p->qn[2], z = p->qn[3];
    double (*R)[3] = p->R;
    R[0][0] = 1 - 2 * (y * y + z * z); R[0][1] = 2 * (x * y - w * z); R[0][2] = 2 * (x * z + w * y);
    R[1][0] = 2 * (x * y + w * z); R[1][1] = 1 - 2 * (x * x + z * z); R[1][2] = 2 * (y * z - w * x);
    R[2][0] = 2 * (x * z - w * y); R[2][1] = 2 * (y * z + w * x); R[2][2] = 1 - 2 * (x * x + y * y);
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) p->Mm[a][b] = R[a][b] * p->sh[b];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
            double acc = 0;
            for (int k = 0; k < 3; k++) acc += p->Mm[a][k] * p->Mm[b][k];
            p->Sig[a][b] = acc;
        }
    memcpy(p->W, W, sizeof(p->W));
    memcpy(p->t, t, sizeof(p->t));
    double mu[3] = {g->mean[i], g->mean[n + i], g->mean[2 * n + i]};
    for (int a = 0; a < 3; a++) p->pc[a] = W[a][0] * mu[0] + W[a][1] * mu[1] + W[a][2] * mu[2] + t[a];
    double fx = cam->fx, fy = cam->fy, cx = cam->cx, cy = cam->cy;
    double X = p->pc[0], Y = p->pc[1], Z = p->pc[2];
    p->valid = (Z > cam->near_z) ? 1 : 0;
    double tx = X, ty = Y;
    if (clamp) {
        double Wd = cam->width, Hd = cam->height;
        double lxlo = -(cx + 0.15 * Wd) / fx, lxhi = (Wd - cx + 0.15 * Wd) / fx;
        double lylo = -(cy + 0.15 * Hd) / fy, lyhi = (Hd - cy + 0.15 * Hd) / fy;
        double rx = X / Z, ry = Y / Z;
        if (rx < lxlo) { p->clamp_x = 1; p->cxr = lxlo; }
        if (rx > lxhi) { p->clamp_x = 1; p->cxr = lxhi; }
        if (ry < lylo) { p->clamp_y = 1; p->cyr = lylo; }
        if (ry > lyhi) { p->clamp_y = 1; p->cyr = lyhi; }
        if (p->clamp_x) tx = p->cxr * Z;
        if (p->clamp_y) ty = p->cyr * Z;
    }
    p->J[0][0] = fx / Z; p->J[0][1] = 0; p->J[0][2] = -fx * tx / (Z * Z);
    p->J[1][0] = 0; p->J[1][1] = fy / Z; p->J[1][2] = -fy * ty / (Z * Z);
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 3; b++) {
            double acc = 0;
            for (int k = 0; k < 3; k++) acc += p->J[a][k] * W[k][b];
            p->A[a][b] = acc;
        }
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 2; b++) {
            double acc = 0;
            for (int k = 0; k < 3; k++)
                for (int l = 0; l < 3; l++) acc += p->A[a][k] * p->Sig[k][l] * p->A[b][l];
            p->S2[a][b] = acc + (a == b ? (double)prm->dilation : 0.0);
        }
    double det = p->S2[0][0] * p->S2[1][1] - p->S2[0][1] * p->S2[1][0];
    if (!(det > 0)) p->valid = 0;
    p->Q[0][0] = p->S2[1][1] / det;
    p->Q[1][1] = p->S2[0][0] / det;
    p->Q[0][1] = p->Q[1][0] = -p->S2[0][1] / det;
    p->u = fx * X / Z + cx;
    p->v = fy * Y / Z + cy;
}

/* ---------------- chain rule (a8), float64 ------------------------------- */
/* acc = dL/d(u, v, ca, cb, cc, o_hat, z, r, g, b).
 * grad15 = dL/d(mean xyz, opacity logit, rgb, log_scale xyz, quat wxyz, mask logit).
 * pose6 += dL/d(omega, v) for the left perturbation V' = Exp(xi) V (R22). */
void or_chain(const or_proj64 *p, const double acc[10], double grad15[15], double pose6[6])
{
    const double gu = acc[0], gv = acc[1], gca = acc[2], gcb = acc[3], gcc = acc[4];
    const double goh = acc[5], gz = acc[6];
    /* dL/dSigma' = -Q G_Q Q with G_Q the symmetric gradient of the conic. */
    double GQ[2][2] = {{gca, 0.5 * gcb}, {0.5 * gcb, gcc}};
    double T1[2][2], G2[2][2];
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 2; b++) T1[a][b] = p->Q[a][0] * GQ[0][b] + p->Q[a][1] * GQ[1][b];
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 2; b++) G2[a][b] = -(T1[a][0] * p->Q[0][b] + T1[a][1] * p->Q[1][b]);
    /* dL/dSigma = A^T G2 A */
    double GS[3][3];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
            double s = 0;
            for (int k = 0; k < 2; k++)
                for (int l = 0; l < 2; l++) s += p->A[k][a] * G2[k][l] * p->A[l][b];
            GS[a][b] = s;
        }
    /* dL/dA = 2 G2 A Sigma */
    double GA[2][3];
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 3; b++) {
            double s = 0;
            for (int k = 0; k < 2; k++)
                for (int l = 0; l < 3; l++) s += G2[a][k] * p->A[k][l] * p->Sig[l][b];
            GA[a][b] = 2.0 * s;
        }
    /* dL/dJ = dL/dA W^T */
    double GJ[2][3];
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 3; b++) {
            double s = 0;
            for (int k = 0; k < 3; k++) s += GA[a][k] * p->W[b][k];
            GJ[a][b] = s;
        }
    /* camera-space mean gradient */
    const double X = p->pc[0], Y = p->pc[1], Z = p->pc[2];
    const double fx = p->J[0][0] * Z, fy = p->J[1][1] * Z;
    double gpc[3];
    gpc[0] = gu * fx / Z;
    gpc[1] = gv * fy / Z;
    gpc[2] = gz - gu * fx * X / (Z * Z) - gv * fy * Y / (Z * Z);
    /* J00 = fx/Z, J11 = fy/Z */
    gpc[2] += GJ[0][0] * (-fx / (Z * Z)) + GJ[1][1] * (-fy / (Z * Z));
    /* J02 = -fx tx / Z^2 */
    if (!p->clamp_x) {
        gpc[0] += GJ[0][2] * (-fx / (Z * Z));
        gpc[2] += GJ[0][2] * (2.0 * fx * X / (Z * Z * Z));
    } else {
        gpc[2] += GJ[0][2] * (fx * p->cxr / (Z * Z));
    }
    if (!p->clamp_y) {
        gpc[1] += GJ[1][2] * (-fy / (Z * Z));
        gpc[2] += GJ[1][2] * (2.0 * fy * Y / (Z * Z * Z));
    } else {
        gpc[2] += GJ[1][2] * (fy * p->cyr / (Z * Z));
    }
    /* world mean: p_c = W mu + t */
    for (int a = 0; a < 3; a++)
        grad15[a] = p->W[0][a] * gpc[0] + p->W[1][a] * gpc[1] + p->W[2][a] * gpc[2];
    /* pose: translation part, rotation part via p_c and via W in A = J W */
    pose6[3] += gpc[0];
    pose6[4] += gpc[1];
    pose6[5] += gpc[2];
    pose6[0] += Y * gpc[2] - Z * gpc[1];
    pose6[1] += Z * gpc[0] - X * gpc[2];
    pose6[2] += X * gpc[1] - Y * gpc[0];
    double Mw[3][3];                                  /* W (dL/dA)^T J */
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
            double s = 0;
            for (int k = 0; k < 2; k++)
                for (int l = 0; l < 3; l++) s += p->W[a][l] * GA[k][l] * p->J[k][b];
            Mw[a][b] = s;
        }
    pose6[0] += Mw[1][2] - Mw[2][1];
    pose6[1] += Mw[2][0] - Mw[0][2];
    pose6[2] += Mw[0][1] - Mw[1][0];
    /* opacity: o_hat = M sig(o) (Eq 7) */
    grad15[3] = goh * p->M * p->sig_o * (1.0 - p->sig_o);
    double gM = goh * p->sig_o;
    /* colour */
    grad15[4] = acc[7];
    grad15[5] = acc[8];
    grad15[6] = acc[9];
    /* Sigma = Mm Mm^T, Mm = R diag(sh):  dL/dMm = 2 GS Mm */
    double GM[3][3];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
            double s = 0;
            for (int k = 0; k < 3; k++) s += GS[a][k] * p->Mm[k][b];
            GM[a][b] = 2.0 * s;
        }
    double gsh[3], GR[3][3];
    for (int b = 0; b < 3; b++) {
        double s = 0;
        for (int a = 0; a < 3; a++) s += p->R[a][b] * GM[a][b];
        gsh[b] = s;
    }
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) GR[a][b] = GM[a][b] * p->sh[b];
    for (int k = 0; k < 3; k++) {
        grad15[7 + k] = gsh[k] * p->M * p->s[k];   /* sh = M exp(ls) */
        gM += gsh[k] * p->s[k];
    }
    /* rotation: dR/dq for unit q = (w, x, y, z) */
    const double w = p->qn[0], x = p->qn[1], y = p->qn[2], z = p->qn[3];
    double dRw[3][3] = {{0, -2 * z, 2 * y}, {2 * z, 0, -2 * x}, {-2 * y, 2 * x, 0}};
    double dRx[3][3] = {{0, 2 * y, 2 * z}, {2 * y, -4 * x, -2 * w}, {2 * z, 2 * w, -4 * x}};
    double dRy[3][3] = {{-4 * y, 2 * x, 2 * w}, {2 * x, 0, 2 * z}, {-2 * w, 2 * z, -4 * y}};
    double dRz[3][3] = {{-4 * z, -2 * w, 2 * x}, {2 * w, -4 * z, 2 * y}, {2 * x, 2 * y, 0}};
    double gqn[4] = {0, 0, 0, 0};
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
            gqn[0] += GR[a][b] * dRw[a][b];
            gqn[1] += GR[a][b] * dRx[a][b];
            gqn[2] += GR[a][b] * dRy[a][b];
            gqn[3] += GR[a][b] * dRz[a][b];
        }
    double dot = 0;
    for (int k = 0; k < 4; k++) dot += p->qn[k] * gqn[k];
    for (int k = 0; k < 4; k++) grad15[10 + k] = (gqn[k] - p->qn[k] * dot) / p->qnorm;
    /* mask (Eq 6 straight-through): dL/dm = dL/dM * sig'(m); M = sg(..) + sig(m) */
    /* sig(m) is recovered from M only in smooth mode; the binary-mode caller
     * overwrites grad15[14] with gM * sig'(m). */
    grad15[14] = gM;
}
