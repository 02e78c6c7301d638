/*
 * oracle_render.c -- ORACLE (test infrastructure, see oracle.h).
 *
 * Steps a4/a5 (tile binning and (tile, depth) ordering, P:79-80 via the 3DGS
 * tile rasterizer the paper extends), a6 (front-to-back compositing of
 * colour, depth and silhouette, Eq 3-5) and a7/a8 (the analytic
 * backward including depth, silhouette and pose).
 *
 * Plain definitions:
 *  - bin:   every (tile, Gaussian) pair whose tile lies in the Gaussian's
 *           tile rectangle, ordered by (tile, bits(z_c), index) with qsort.
 *  - fwd:   per pixel, front-to-back over the tile list, Eq 3-5 with the
 *           readings R1 (alpha cap), R2 (q <= k^2 cutoff), R3 (termination).
 *  - pixel: the untiled definition -- all non-culled Gaussians sorted by
 *           (bits(z_c), index), no tiles at all.
 *  - bwd:   per pixel, replay the forward storing (alpha_j, T_j) for every
 *           composited entry, then the exact derivative of Eq 3-5 (suffix
 *           sums, no division), then the float64 chain rule (or_chain).
 */
#include "oracle_internal.h"
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Optional pixel-row window for the tiled forward/backward: the timed CPU
 * baseline renders a bounded sample of rows (bench.py); default = all rows. */
static int g_row_lo = 0, g_row_hi = -1;
static int g_threads = 1;
void oracle_set_threads(int32_t n) { g_threads = n < 1 ? 1 : n; }
int or_threads(void) { return g_threads; }
void oracle_set_row_window(int32_t row_lo, int32_t row_hi) { g_row_lo = row_lo; g_row_hi = row_hi; }
static int or_row_lo(int H) { return g_row_lo < 0 ? 0 : (g_row_lo > H ? H : g_row_lo); }
static int or_row_hi(int H) { return (g_row_hi < 0 || g_row_hi > H) ? H : g_row_hi; }

typedef struct { uint32_t tile, zbits, gid; } or_pair;

static int cmp_pair(const void *a, const void *b)
{
    const or_pair *x = (const or_pair *)a, *y = (const or_pair *)b;
    if (x->tile != y->tile) return x->tile < y->tile ? -1 : 1;
    if (x->zbits != y->zbits) return x->zbits < y->zbits ? -1 : 1;
    if (x->gid != y->gid) return x->gid < y->gid ? -1 : 1;
    return 0;
}

int oracle_bin_tiles(const uint32_t *rec, const int32_t *count, int64_t n, const or_camera *cam,
                     int64_t pair_capacity, uint32_t *pair_gid, uint32_t *tile_range,
                     int64_t *n_pairs)
{
    const int tiles_x = (cam->width + OR_TILE - 1) / OR_TILE;
    const int tiles_y = (cam->height + OR_TILE - 1) / OR_TILE;
    const int64_t T = (int64_t)tiles_x * tiles_y;
    int64_t total = 0;
    for (int64_t i = 0; i < n; i++) total += count[i];
    *n_pairs = total;
    if (total > pair_capacity) return 3;
    or_pair *pairs = (or_pair *)malloc((size_t)(total ? total : 1) * sizeof(or_pair));
    int64_t k = 0;
    for (int64_t i = 0; i < n; i++) {
        if (count[i] <= 0) continue;
        const uint32_t *r = rec + i * OR_REC_WORDS;
        int px0 = r[12] & 0xffff, py0 = r[12] >> 16, px1 = r[13] & 0xffff, py1 = r[13] >> 16;
        for (int ty = py0 / OR_TILE; ty <= py1 / OR_TILE; ty++)
            for (int tx = px0 / OR_TILE; tx <= px1 / OR_TILE; tx++) {
                pairs[k].tile = (uint32_t)(ty * tiles_x + tx);
                pairs[k].zbits = r[7];
                pairs[k].gid = (uint32_t)i;
                k++;
            }
    }
    qsort(pairs, (size_t)total, sizeof(or_pair), cmp_pair);
    for (int64_t j = 0; j < total; j++) pair_gid[j] = pairs[j].gid;
    int64_t j = 0;
    for (int64_t t = 0; t < T; t++) {
        tile_range[2 * t] = (uint32_t)j;
        while (j < total && pairs[j].tile == (uint32_t)t) j++;
        tile_range[2 * t + 1] = (uint32_t)j;
    }
    free(pairs);
    return 0;
}

/* The per-pixel DA q test shared by every form of the forward (R2). */
static int q_test(const uint32_t *r, int px, int py, float *q_out)
{
    float u = or_u2f(r[0]), v = or_u2f(r[1]);
    float ca = or_u2f(r[2]), cb2 = or_u2f(r[3]), cc = or_u2f(r[4]), k2 = or_u2f(r[6]);
    float dx = (float)px - u, dy = (float)py - v;
    float q = fmaf(ca * dx, dx, fmaf(cb2 * dx, dy, (cc * dy) * dy));
    *q_out = q;
    return (q >= 0.0f) && (q <= k2);
}

/* One composited entry of a pixel (kept for the backward). */
typedef struct {
    int64_t gid;
    double alpha, T, G, dx, dy, ca, cb, cc, rgb[3], z, oh;
    int capped;
} or_entry;

/* Ambiguity windows (SURVEY §8(c) policy 2): a pixel is flagged
 * when a termination test T(1-alpha) lies within FLAG_T_REL (relative) of
 * t_min, or o_hat*G within FLAG_CAP_ABS of alpha_max, because there a float32
 * evaluation may decide the other way than this float64 one.  Defaults are
 * the §8(c) values; oracle_set_flag_window() lets a test measure how many
 * pixels a wider or narrower window would flag (it does not change any
 * rendered value). */
static double FLAG_T_REL = 1e-5;
static double FLAG_CAP_ABS = 1e-6;
void oracle_set_flag_window(double t_rel, double cap_abs) { FLAG_T_REL = t_rel; FLAG_CAP_ABS = cap_abs; }

/* Composite one pixel over an ordered candidate list (Eq 3-5).  Returns the
 * number of composited entries; fills out6 = (C rgb, D, S, T_final), the
 * number examined, a flag, and (optionally) the entries. */
static int composite(const uint32_t *rec, const uint32_t *order, int64_t len, int px, int py,
                     const or_params *prm, double out6[6], int64_t *examined, int *flag,
                     int32_t *last_plus_one, or_entry *ent)
{
    double T = 1.0, C[3] = {0, 0, 0}, D = 0, S = 0;
    int ne = 0;
    int64_t ex = 0;
    *flag = 0;
    *last_plus_one = 0;
    for (int64_t j = 0; j < len; j++) {
        const uint32_t *r = rec + (int64_t)order[j] * OR_REC_WORDS;
        float q;
        ex++;
        if (!q_test(r, px, py, &q)) continue;
        double oh = or_u2f(r[5]);
        double G = exp(-0.5 * (double)q);
        double a_raw = oh * G;
        double alpha = a_raw < prm->alpha_max ? a_raw : (double)prm->alpha_max;
        if (fabs(a_raw - prm->alpha_max) < FLAG_CAP_ABS) *flag = 1;
        double test = T * (1.0 - alpha);
        if (fabs(test - prm->t_min) < FLAG_T_REL * prm->t_min) *flag = 1;
        if (test < prm->t_min) break;                        /* R3: not composited */
        double w = alpha * T;
        double rgb[3] = {or_u2f(r[8]), or_u2f(r[9]), or_u2f(r[10])};
        double z = or_u2f(r[7]);
        for (int c = 0; c < 3; c++) C[c] += rgb[c] * w;      /* Eq 3 */
        D += z * w;                                          /* Eq 4 */
        S += w;                                              /* Eq 5 */
        if (ent) {
            or_entry *e = &ent[ne];
            e->gid = order[j];
            e->alpha = alpha;
            e->T = T;
            e->G = G;
            e->capped = !(a_raw < prm->alpha_max);
            e->dx = (double)px - (double)or_u2f(r[0]);
            e->dy = (double)py - (double)or_u2f(r[1]);
            e->ca = or_u2f(r[2]);
            e->cb = 0.5 * (double)or_u2f(r[3]);
            e->cc = or_u2f(r[4]);
            for (int c = 0; c < 3; c++) e->rgb[c] = rgb[c];
            e->z = z;
            e->oh = oh;
        }
        ne++;
        T = test;
        *last_plus_one = (int32_t)(j + 1);
    }
    for (int c = 0; c < 3; c++) out6[c] = C[c];
    out6[3] = D;
    out6[4] = S;
    out6[5] = T;
    *examined = ex;
    return ne;
}

int oracle_render_fwd(const uint32_t *rec, const uint32_t *pair_gid, const uint32_t *tile_range,
                      const or_camera *cam, const or_params *prm, double *color, double *depth,
                      double *sil, double *t_final, int32_t *n_contrib, uint8_t *flags,
                      int64_t *counters)
{
    const int W = cam->width, H = cam->height;
    const int tiles_x = (W + OR_TILE - 1) / OR_TILE;
    const int64_t HW = (int64_t)W * H;
    int64_t e_pix = 0, e_con = 0;
#pragma omp parallel for num_threads(g_threads) schedule(dynamic, 1) reduction(+ : e_pix, e_con)
    for (int py = or_row_lo(H); py < or_row_hi(H); py++)
        for (int px = 0; px < W; px++) {
            int64_t t = (int64_t)(py / OR_TILE) * tiles_x + px / OR_TILE;
            uint32_t s = tile_range[2 * t], e = tile_range[2 * t + 1];
            double out6[6];
            int64_t ex;
            int flag;
            int32_t lp1;
            int ne = composite(rec, pair_gid + s, (int64_t)e - s, px, py, prm, out6, &ex, &flag,
                               &lp1, NULL);
            int64_t p = (int64_t)py * W + px;
            color[p] = out6[0];
            color[HW + p] = out6[1];
            color[2 * HW + p] = out6[2];
            depth[p] = out6[3];
            sil[p] = out6[4];
            t_final[p] = out6[5];
            n_contrib[p] = lp1;
            if (flags) flags[p] = (uint8_t)flag;
            e_pix += ex;
            e_con += ne;
        }
    if (counters) { counters[0] = e_pix; counters[1] = e_con; }
    return 0;
}

typedef struct { uint32_t zbits, gid; } or_zkey;
static int cmp_zkey(const void *a, const void *b)
{
    const or_zkey *x = (const or_zkey *)a, *y = (const or_zkey *)b;
    if (x->zbits != y->zbits) return x->zbits < y->zbits ? -1 : 1;
    if (x->gid != y->gid) return x->gid < y->gid ? -1 : 1;
    return 0;
}

int oracle_render_pixel(const uint32_t *rec, const int32_t *count, int64_t n, const or_camera *cam,
                        const or_params *prm, int32_t px, int32_t py, double *out6,
                        int32_t *n_composited)
{
    (void)cam;
    int64_t m = 0;
    for (int64_t i = 0; i < n; i++) m += count[i] > 0;
    or_zkey *keys = (or_zkey *)malloc((size_t)(m ? m : 1) * sizeof(or_zkey));
    uint32_t *order = (uint32_t *)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
    int64_t k = 0;
    for (int64_t i = 0; i < n; i++)
        if (count[i] > 0) { keys[k].zbits = rec[i * OR_REC_WORDS + 7]; keys[k].gid = (uint32_t)i; k++; }
    qsort(keys, (size_t)m, sizeof(or_zkey), cmp_zkey);
    for (int64_t j = 0; j < m; j++) order[j] = keys[j].gid;
    int64_t ex;
    int flag;
    int32_t lp1;
    int ne = composite(rec, order, m, px, py, prm, out6, &ex, &flag, &lp1, NULL);
    if (n_composited) *n_composited = ne;
    free(keys);
    free(order);
    return 0;
}

/* Exact derivative of Eq 3-5 for one pixel given its composited entries.
 * L = <gC, C> + gD D + gS S.  w_j = alpha_j T_j, T_{j+1} = T_j (1 - alpha_j).
 * dL/dalpha_j = T_j (v_j - B_j), v_j = <rgb_j, gC> + z_j gD + gS,
 * B_j = sum_{k>j} v_k alpha_k prod_{j<m<k} (1 - alpha_m)  (suffix, no division). */
static void accumulate_pixel(const or_entry *ent, int ne, const double gC[3], double gD, double gS,
                             double *acc2d)
{
    double B = 0.0;
    for (int j = ne - 1; j >= 0; j--) {
        const or_entry *e = &ent[j];
        double *a = acc2d + e->gid * 10;
        double v = e->rgb[0] * gC[0] + e->rgb[1] * gC[1] + e->rgb[2] * gC[2] + e->z * gD + gS;
        double w = e->alpha * e->T;
        double dLda = e->T * (v - B);
        a[7] += gC[0] * w;
        a[8] += gC[1] * w;
        a[9] += gC[2] * w;
        a[6] += gD * w;
        if (!e->capped) {                                 /* R23: zero subgradient when capped */
            a[5] += e->G * dLda;                          /* alpha = o_hat G */
            double dq = -0.5 * e->alpha * dLda;           /* dG/dq = -G/2    */
            a[2] += dq * e->dx * e->dx;
            a[3] += dq * 2.0 * e->dx * e->dy;
            a[4] += dq * e->dy * e->dy;
            a[0] += dq * (-2.0 * (e->ca * e->dx + e->cb * e->dy));
            a[1] += dq * (-2.0 * (e->cb * e->dx + e->cc * e->dy));
        }
        B = e->alpha * v + (1.0 - e->alpha) * B;
    }
}

static void view_to_d(const or_view *view, double W[3][3], double t[3])
{
    for (int a = 0; a < 3; a++) {
        for (int b = 0; b < 3; b++) W[a][b] = view->m[4 * a + b];
        t[a] = view->m[4 * a + 3];
    }
}

static double sigd(double x) { return 1.0 / (1.0 + exp(-x)); }

int oracle_render_bwd(const or_gaussians *g, const or_codebook *cb, const or_camera *cam,
                      const or_view *view, const or_params *prm, const uint32_t *rec,
                      const uint32_t *pair_gid, const uint32_t *tile_range, const double *d_color,
                      const double *d_depth, const double *d_sil, const uint8_t *pixel_weight_zero,
                      double *grads, double *pose, double *acc2d_out)
{
    const int64_t n = g->n;
    const int W = cam->width, H = cam->height;
    const int tiles_x = (W + OR_TILE - 1) / OR_TILE;
    const int64_t HW = (int64_t)W * H;
    int64_t maxlen = 0;
    const int64_t T_tiles = (int64_t)tiles_x * ((H + OR_TILE - 1) / OR_TILE);
    for (int64_t t = 0; t < T_tiles; t++) {
        int64_t l = (int64_t)tile_range[2 * t + 1] - tile_range[2 * t];
        if (l > maxlen) maxlen = l;
    }
    /* per-thread 2D accumulators (one with 1 thread), summed in thread order */
    const int nth = g_threads;
    double *accs = (double *)calloc((size_t)nth * (size_t)(n ? n : 1) * 10, sizeof(double));
#pragma omp parallel num_threads(nth)
    {
#ifdef _OPENMP
        const int tid = omp_get_thread_num();
#else
        const int tid = 0;
#endif
        double *acc_t = accs + (size_t)tid * (size_t)(n ? n : 1) * 10;
        or_entry *ent = (or_entry *)malloc((size_t)(maxlen ? maxlen : 1) * sizeof(or_entry));
#pragma omp for schedule(dynamic, 1)
        for (int py = or_row_lo(H); py < or_row_hi(H); py++)
            for (int px = 0; px < W; px++) {
                int64_t p = (int64_t)py * W + px;
                if (pixel_weight_zero && pixel_weight_zero[p]) continue;
                int64_t t = (int64_t)(py / OR_TILE) * tiles_x + px / OR_TILE;
                uint32_t s = tile_range[2 * t], e = tile_range[2 * t + 1];
                double out6[6];
                int64_t ex;
                int flag;
                int32_t lp1;
                int ne = composite(rec, pair_gid + s, (int64_t)e - s, px, py, prm, out6, &ex,
                                   &flag, &lp1, ent);
                double gC[3] = {d_color[p], d_color[HW + p], d_color[2 * HW + p]};
                accumulate_pixel(ent, ne, gC, d_depth[p], d_sil[p], acc_t);
            }
        free(ent);
    }
    double *acc2d = accs;
    for (int th = 1; th < nth; th++) {
        const double *a = accs + (size_t)th * (size_t)(n ? n : 1) * 10;
        for (int64_t k = 0; k < n * 10; k++) acc2d[k] += a[k];
    }
    double Wd[3][3], td[3];
    view_to_d(view, Wd, td);
    for (int k = 0; k < 6; k++) pose[k] = 0.0;
    double *pose_t = (double *)calloc((size_t)nth * 6, sizeof(double));
#pragma omp parallel num_threads(nth)
    {
#ifdef _OPENMP
        const int tid = omp_get_thread_num();
#else
        const int tid = 0;
#endif
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; i++) {
            double g15[15] = {0};
            const uint32_t *r = rec + i * OR_REC_WORDS;
            int alive = r[5] != 0u;                              /* o_hat word is 0 iff culled */
            if (alive) {
                or_proj64 pj;
                or_project64(g, cb, cam, Wd, td, prm, i, OR_MODE_CLAMP, &pj);
                or_chain(&pj, acc2d + i * 10, g15, pose_t + 6 * tid);
                double sm = sigd((double)g->mask[i]);
                g15[14] *= sm * (1.0 - sm);                      /* Eq 6 STE */
            }
            for (int k = 0; k < 15; k++) grads[k * n + i] = g15[k];
        }
    }
    for (int th = 0; th < nth; th++)
        for (int k = 0; k < 6; k++) pose[k] += pose_t[6 * th + k];
    free(pose_t);
    if (acc2d_out) memcpy(acc2d_out, acc2d, (size_t)n * 10 * sizeof(double));
    free(accs);
    return 0;
}

/* ---------------- smooth mode (FD pins only) ----------------------------- */

static void rodrigues(const double w[3], double R[3][3])
{
    double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    double K[3][3] = {{0, -w[2], w[1]}, {w[2], 0, -w[0]}, {-w[1], w[0], 0}};
    double a = th > 1e-12 ? sin(th) / th : 1.0;
    double b = th > 1e-12 ? (1.0 - cos(th)) / (th * th) : 0.5;
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double kk = 0;
            for (int k = 0; k < 3; k++) kk += K[i][k] * K[k][j];
            R[i][j] = (i == j ? 1.0 : 0.0) + a * K[i][j] + b * kk;
        }
}

typedef struct { double z; int64_t gid; } or_dkey;
static int cmp_dkey(const void *a, const void *b)
{
    const or_dkey *x = (const or_dkey *)a, *y = (const or_dkey *)b;
    if (x->z != y->z) return x->z < y->z ? -1 : 1;
    return x->gid < y->gid ? -1 : (x->gid > y->gid);
}

/* Smooth forward: float64, no alpha cap, no q cutoff, no termination, no J
 * clamp, continuous mask multiplier M = sig(m). */
static int smooth_core(const or_gaussians *g, const or_camera *cam, const or_view *view,
                       const double *xi, const or_params *prm, int clamp, double *color, double *depth,
                       double *sil, const double *d_color, const double *d_depth,
                       const double *d_sil, double *grads, double *pose)
{
    const int64_t n = g->n;
    const int W = cam->width, H = cam->height;
    const int64_t HW = (int64_t)W * H;
    double Wd[3][3], td[3];
    view_to_d(view, Wd, td);
    if (xi) {                                   /* V' = Exp(xi) V, p' = Rod(w) p + v */
        double R[3][3], W2[3][3], t2[3];
        rodrigues(xi, R);
        for (int a = 0; a < 3; a++) {
            for (int b = 0; b < 3; b++) {
                double s = 0;
                for (int k = 0; k < 3; k++) s += R[a][k] * Wd[k][b];
                W2[a][b] = s;
            }
            double s = 0;
            for (int k = 0; k < 3; k++) s += R[a][k] * td[k];
            t2[a] = s + xi[3 + a];
        }
        memcpy(Wd, W2, sizeof(Wd));
        memcpy(td, t2, sizeof(td));
    }
    or_proj64 *pj = (or_proj64 *)malloc((size_t)(n ? n : 1) * sizeof(or_proj64));
    or_dkey *keys = (or_dkey *)malloc((size_t)(n ? n : 1) * sizeof(or_dkey));
    int64_t m = 0;
    for (int64_t i = 0; i < n; i++) {
        or_project64(g, NULL, cam, Wd, td, prm, i,
                     OR_MODE_SMOOTH_MASK | (clamp ? OR_MODE_CLAMP : 0), &pj[i]);
        if (pj[i].valid) { keys[m].z = pj[i].pc[2]; keys[m].gid = i; m++; }
    }
    qsort(keys, (size_t)m, sizeof(or_dkey), cmp_dkey);
    or_entry *ent = (or_entry *)malloc((size_t)(m ? m : 1) * sizeof(or_entry));
    double *acc2d = grads ? (double *)calloc((size_t)(n ? n : 1) * 10, sizeof(double)) : NULL;
    for (int py = 0; py < H; py++)
        for (int px = 0; px < W; px++) {
            int64_t p = (int64_t)py * W + px;
            double T = 1.0, C[3] = {0, 0, 0}, D = 0, S = 0;
            for (int64_t j = 0; j < m; j++) {
                const or_proj64 *q = &pj[keys[j].gid];
                double dx = px - q->u, dy = py - q->v;
                double qq = q->Q[0][0] * dx * dx + 2 * q->Q[0][1] * dx * dy + q->Q[1][1] * dy * dy;
                double G = exp(-0.5 * qq);
                double alpha = q->oh * G;
                double rgb[3] = {g->rgb[keys[j].gid], g->rgb[n + keys[j].gid], g->rgb[2 * n + keys[j].gid]};
                double w = alpha * T;
                for (int c = 0; c < 3; c++) C[c] += rgb[c] * w;
                D += q->pc[2] * w;
                S += w;
                or_entry *e = &ent[j];
                e->gid = keys[j].gid;
                e->alpha = alpha;
                e->T = T;
                e->G = G;
                e->capped = 0;
                e->dx = dx;
                e->dy = dy;
                e->ca = q->Q[0][0];
                e->cb = q->Q[0][1];
                e->cc = q->Q[1][1];
                for (int c = 0; c < 3; c++) e->rgb[c] = rgb[c];
                e->z = q->pc[2];
                e->oh = q->oh;
                T *= (1.0 - alpha);
            }
            if (color) {
                for (int c = 0; c < 3; c++) color[c * HW + p] = C[c];
                depth[p] = D;
                sil[p] = S;
            }
            if (acc2d) {
                double gC[3] = {d_color[p], d_color[HW + p], d_color[2 * HW + p]};
                accumulate_pixel(ent, (int)m, gC, d_depth[p], d_sil[p], acc2d);
            }
        }
    if (grads) {
        for (int k = 0; k < 6; k++) pose[k] = 0.0;
        for (int64_t i = 0; i < n; i++) {
            double g15[15] = {0};
            if (pj[i].valid) {
                or_chain(&pj[i], acc2d + i * 10, g15, pose);
                double sm = sigd((double)g->mask[i]);
                g15[14] *= sm * (1.0 - sm);
            }
            for (int k = 0; k < 15; k++) grads[k * n + i] = g15[k];
        }
        free(acc2d);
    }
    free(ent);
    free(keys);
    free(pj);
    (void)prm;
    return 0;
}

int oracle_smooth_render(const or_gaussians *g, const or_camera *cam, const or_view *view,
                         const double *pose_xi, const or_params *prm, int32_t clamp,
                         double *color, double *depth, double *sil)
{
    return smooth_core(g, cam, view, pose_xi, prm, clamp, color, depth, sil, NULL, NULL, NULL, NULL, NULL);
}

int oracle_smooth_bwd(const or_gaussians *g, const or_camera *cam, const or_view *view,
                      const or_params *prm, int32_t clamp, const double *d_color,
                      const double *d_depth, const double *d_sil, double *grads, double *pose)
{
    return smooth_core(g, cam, view, NULL, prm, clamp, NULL, NULL, NULL, d_color, d_depth, d_sil, grads,
                       pose);
}
