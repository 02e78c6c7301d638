/* oracle_internal.h -- shared between the oracle's own .c files only.
 * TEST INFRASTRUCTURE (see oracle.h). */
#ifndef CSPLAT_ORACLE_INTERNAL_H
#define CSPLAT_ORACLE_INTERNAL_H
#include "oracle.h"
#include <math.h>
#include <stdint.h>
#include <string.h>

static inline float or_u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static inline uint32_t or_f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* OpenMP thread count of the timed baseline (oracle_set_threads; 1 = serial). */
int or_threads(void);

/* DA transcendentals. */
float or_sigm(float x);

/* Full float64 projection of one Gaussian: everything the backward chain and
 * the smooth-mode forward need (Eq 1-2). */
typedef struct {
    int valid;
    double M;                 /* mask multiplier (1 or sig(m))           */
    double s[3], sh[3];       /* activated scale, masked scale (Eq 7)    */
    double sig_o, oh;         /* sig(opacity), masked o_hat (Eq 7)       */
    double qn[4], qnorm;      /* normalised quaternion, |q|              */
    double R[3][3];           /* rotation from qn                        */
    double Mm[3][3];          /* R diag(sh)                              */
    double Sig[3][3];         /* Sigma = Mm Mm^T (Eq 1)                  */
    double W[3][3], t[3];     /* view rotation / translation             */
    double pc[3];             /* camera-space mean                       */
    double J[2][3];           /* projection Jacobian                     */
    int clamp_x, clamp_y;     /* J clamp active (R6)                     */
    double cxr, cyr;          /* clamp ratios when active                */
    double A[2][3];           /* J W                                     */
    double S2[2][2];          /* Sigma' = A Sigma A^T + dil I (Eq 2)     */
    double Q[2][2];           /* conic = inverse(Sigma')                 */
    double u, v;              /* pixel-space mean                        */
} or_proj64;

/* mode bits: OR_MODE_SMOOTH_MASK -> M = sig(m) (else M = 1, binary kept);
 *            OR_MODE_CLAMP       -> apply the J clamp of reading R6. */
#define OR_MODE_SMOOTH_MASK 1
#define OR_MODE_CLAMP 2
void or_project64(const or_gaussians *g, const or_codebook *cb, const or_camera *cam,
                  const double W[3][3], const double t[3], const or_params *prm,
                  int64_t i, int mode, or_proj64 *out);

/* Chain rule from the per-Gaussian 2D gradient (u, v, ca, cb, cc, o_hat, z,
 * r, g, b) to the 15 parameter gradients and the pose (omega, v). */
void or_chain(const or_proj64 *p, const double acc[10], double grad15[15], double pose6[6]);

/* Decoded (or raw) log-scale and quaternion of Gaussian i, float32 (R20). */
void or_geometry(const or_gaussians *g, const or_codebook *cb, int64_t i, float ls[3],
                 float q[4]);

#endif
