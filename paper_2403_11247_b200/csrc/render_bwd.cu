// render_bwd.cu -- a7 (backward of Eq 3-5) and a8 (per-Gaussian chain rule,
// Eq 6 straight-through mask, pose) -- the paper's "functions to manage depth,
// pose, and cumulative opacity during both forward and backward propagation"
// (P:270).  Readings R14, R20, R22, R23.
//
// a7: one CTA per tile replays the tile list back to front (TMA-streamed
// batches, as in the forward).  Per pixel, starting from T_final and
// n_contrib: T_j = T_{j+1} / (1 - alpha_j), v_j = <rgb_j, dL/dC> + z_j dL/dD +
// dL/dS, dL/dalpha_j = T_j (v_j - B_j), B_{j-1} = alpha_j v_j + (1-alpha_j) B_j.
// The ten per-(pixel, entry) partials (u, v, ca, cb, cc, o_hat, z, r, g, b)
// are summed over the warp with shuffles, then over the 8 warps through shared
// memory, and leave the CTA as three red.global.add.v4.f32 per (tile,
// Gaussian) into a [n][12] accumulator.
// a8: one thread per Gaussian maps the 2D gradient to the 15 parameter
// gradients and reduces the 6-vector pose gradient per CTA.
#include "common.cuh"

namespace csplat {

constexpr int kBB = 32;   // records per batch
constexpr int kBS = 3;    // ring depth
constexpr int kAcc = 12;  // accumulator floats per Gaussian

size_t bwd_workspace_bytes(int64_t n) { return (size_t)(n > 0 ? n : 1) * kAcc * sizeof(float); }

__global__ void __launch_bounds__(256) k_render_bwd(
    const float4 *__restrict__ pair_rec, const uint32_t *__restrict__ range, int W, int H,
    int tiles_x, float amax, const float *__restrict__ t_final,
    const int32_t *__restrict__ n_contrib, const float *__restrict__ dC,
    const float *__restrict__ dD, const float *__restrict__ dS, float *__restrict__ acc) {
  __shared__ __align__(128) float4 buf[kBS][kBB * 4];
  __shared__ __align__(16) float part[8][kBB][kAcc];
  __shared__ __align__(8) uint64_t full[kBS];
  __shared__ int s_max;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int wx0 = tx * kTile + (wid & 1) * 8, wy0 = ty * kTile + (wid >> 1) * 4;
  const int px = wx0 + (lane & 7), py = wy0 + (lane >> 3);
  const bool inside = px < W && py < H;
  const uint32_t start = range[2 * tile];
  const int64_t HW = (int64_t)W * H, p = (int64_t)py * W + px;

  float T = 1.f, gr = 0.f, gg = 0.f, gb = 0.f, gd = 0.f, gs = 0.f;
  int last = 0;
  if (inside) {
    T = t_final[p];
    last = n_contrib[p];
    gr = dC[p];
    gg = dC[HW + p];
    gb = dC[2 * HW + p];
    gd = dD[p];
    gs = dS[p];
  }
  if (tid == 0) {
    s_max = 0;
    for (int s = 0; s < kBS; s++) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  atomicMax(&s_max, last);
  __syncthreads();
  const int maxlast = s_max;
  const int nb = (maxlast + kBB - 1) / kBB;
  // batch k of the replay covers entries [lo, hi) with b = nb - 1 - k
  int issued = 0;
  auto issue = [&](int k) {
    const int b = nb - 1 - k;
    const int cnt = min(kBB, maxlast - b * kBB);
    const uint32_t bytes = (uint32_t)cnt * CSPLAT_RECORD_BYTES;
    uint64_t *bar = &full[k % kBS];
    mbar_arrive_expect_tx(bar, bytes);
    tma_load_1d(&buf[k % kBS][0], pair_rec + ((int64_t)start + (int64_t)b * kBB) * 4, bytes, bar);
  };
  if (tid == 0)
    for (; issued < min(kBS - 1, nb); issued++) issue(issued);

  const float fpx = (float)px, fpy = (float)py;
  float Bsuf = 0.f;  // B_j: suffix colour/depth/silhouette "behind" entry j
  for (int k = 0; k < nb; k++) {
    __syncthreads();  // slot of batch k-1 and part[] are free
    if (tid == 0 && issued < nb && issued <= k + kBS - 1) issue(issued++);
    mbar_wait(&full[k % kBS], (uint32_t)(k / kBS) & 1u);
    const float4 *rb = buf[k % kBS];
    const int b = nb - 1 - k;
    const int cnt = min(kBB, maxlast - b * kBB);
    for (int e = cnt - 1; e >= 0; e--) {
      const int j = b * kBB + e;
      const float4 r3 = rb[e * 4 + 3];
      const uint32_t rx = __float_as_uint(r3.x), ry = __float_as_uint(r3.y);
      float *pw = part[wid][e];
      if ((int)(rx & 0xffffu) > wx0 + 7 || (int)(rx >> 16) < wx0 ||
          (int)(ry & 0xffffu) > wy0 + 3 || (int)(ry >> 16) < wy0) {
        if (lane < 3) reinterpret_cast<float4 *>(pw)[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
        continue;
      }
      const float4 r0 = rb[e * 4 + 0];
      const float4 r1 = rb[e * 4 + 1];
      const float4 r2 = rb[e * 4 + 2];
      float v0 = 0, v1 = 0, v2 = 0, v3 = 0, v4 = 0, v5 = 0, v6 = 0, v7 = 0, v8 = 0, v9 = 0;
      bool act = false;
      if (j < last) {
        const float dx = DSUB(fpx, r0.x), dy = DSUB(fpy, r0.y);
        const float q = DFMA(DMUL(r0.z, dx), dx, DFMA(DMUL(r0.w, dx), dy, DMUL(DMUL(r1.x, dy), dy)));
        if (q >= 0.0f && q <= r1.z) {
          act = true;
          const float G = __expf(-0.5f * q);
          const float araw = r1.y * G;
          const bool capped = !(araw < amax);
          const float alpha = capped ? amax : araw;
          const float Tj = __fdividef(T, 1.0f - alpha);
          const float w = alpha * Tj;
          const float vv = fmaf(r2.x, gr, fmaf(r2.y, gg, fmaf(r2.z, gb, fmaf(r1.w, gd, gs))));
          const float dLda = Tj * (vv - Bsuf);
          v7 = gr * w;
          v8 = gg * w;
          v9 = gb * w;
          v6 = gd * w;
          if (!capped) {
            v5 = G * dLda;
            const float dq = -0.5f * alpha * dLda;
            v2 = dq * dx * dx;
            v3 = 2.0f * dq * dx * dy;
            v4 = dq * dy * dy;
            v0 = -dq * fmaf(2.0f * r0.z, dx, r0.w * dy);
            v1 = -dq * fmaf(r0.w, dx, 2.0f * r1.x * dy);
          }
          Bsuf = fmaf(alpha, vv, (1.0f - alpha) * Bsuf);
          T = Tj;
        }
      }
      if (__any_sync(0xffffffffu, act)) {
        v0 = warp_sum(v0); v1 = warp_sum(v1); v2 = warp_sum(v2); v3 = warp_sum(v3);
        v4 = warp_sum(v4); v5 = warp_sum(v5); v6 = warp_sum(v6); v7 = warp_sum(v7);
        v8 = warp_sum(v8); v9 = warp_sum(v9);
        if (lane == 0) {
          float4 *p4 = reinterpret_cast<float4 *>(pw);
          p4[0] = make_float4(v0, v1, v2, v3);
          p4[1] = make_float4(v4, v5, v6, v7);
          p4[2] = make_float4(v8, v9, 0.f, 0.f);
        }
      } else if (lane < 3) {
        reinterpret_cast<float4 *>(pw)[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    __syncthreads();
    // combine the 8 warps' partials: thread (e, c) owns float4 c of entry e
    if (tid < cnt * 3) {
      const int e = tid / 3, c = tid % 3;
      float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int w = 0; w < 8; w++) {
        const float4 t4 = reinterpret_cast<const float4 *>(part[w][e])[c];
        s4.x += t4.x; s4.y += t4.y; s4.z += t4.z; s4.w += t4.w;
      }
      if (s4.x != 0.f || s4.y != 0.f || s4.z != 0.f || s4.w != 0.f) {
        const uint32_t gid = __float_as_uint(rb[e * 4 + 2].w);
        red_add_v4(acc + (int64_t)gid * kAcc + c * 4, s4.x, s4.y, s4.z, s4.w);
      }
    }
  }
  if (tid == 0)
    for (int kk = nb; kk < issued; kk++) mbar_wait(&full[kk % kBS], (uint32_t)(kk / kBS) & 1u);
}

struct ChainConst {
  float W[9], t[3];
  float fx, fy, lx_lo, lx_hi, ly_lo, ly_hi, dil;
};

__device__ __forceinline__ uint32_t load_idx2(const void *p, int bytes, int64_t off) {
  return bytes == 1 ? (uint32_t)((const uint8_t *)p)[off] : (uint32_t)((const uint16_t *)p)[off];
}

__global__ void __launch_bounds__(256) k_chain(
    int64_t n, const int64_t *__restrict__ n_dev, const float *__restrict__ mean,
    const float *__restrict__ opac, const float *__restrict__ lsc, const float *__restrict__ quat,
    const float *__restrict__ mask, DecodeArgs dec, int use_dec, ChainConst cc,
    const float4 *__restrict__ rec4, const float4 *__restrict__ acc4, uint32_t flags,
    csplat_grads out) {
  __shared__ float red[8][6];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ne = eff_n(n, n_dev);
  float pose[6] = {0, 0, 0, 0, 0, 0};
  float g[15];
#pragma unroll
  for (int k = 0; k < 15; k++) g[k] = 0.f;
  bool alive = false;
  if (i < ne) alive = rec4[i * 4 + 1].y != 0.0f;  // o_hat word is 0 iff culled
  if (alive) {
    const float4 a0 = acc4[i * 3 + 0], a1 = acc4[i * 3 + 1], a2 = acc4[i * 3 + 2];
    const float gu = a0.x, gv = a0.y, gca = a0.z, gcb = a0.w, gcc = a1.x, goh = a1.y, gz = a1.z;
    g[4] = a1.w;  // rgb
    g[5] = a2.x;
    g[6] = a2.y;
    float ls[3], qv[4];
    if (use_dec) {
      for (int l = 0; l < dec.L; l++) {
        const uint32_t si = load_idx2(dec.scale_idx, dec.idx_bytes, (int64_t)l * n + i);
        const uint32_t ri = load_idx2(dec.rot_idx, dec.idx_bytes, (int64_t)l * n + i);
        const float *sc = dec.scale_codes + ((int64_t)l * dec.P + si) * 3;
        const float *rc = dec.rot_codes + ((int64_t)l * dec.P + ri) * 4;
        for (int k = 0; k < 3; k++) ls[k] = l ? DADD(ls[k], sc[k]) : sc[k];
        for (int k = 0; k < 4; k++) qv[k] = l ? DADD(qv[k], rc[k]) : rc[k];
      }
    } else {
      for (int k = 0; k < 3; k++) ls[k] = lsc[k * n + i];
      for (int k = 0; k < 4; k++) qv[k] = quat[k * n + i];
    }
    const float s[3] = {__expf(ls[0]), __expf(ls[1]), __expf(ls[2])};
    const float qn2 = qv[0] * qv[0] + qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3];
    const float qinv = rsqrtf(qn2);
    const float w = qv[0] * qinv, x = qv[1] * qinv, y = qv[2] * qinv, z = qv[3] * qinv;
    float R[3][3];
    R[0][0] = 1.f - 2.f * (y * y + z * z); R[0][1] = 2.f * (x * y - w * z); R[0][2] = 2.f * (x * z + w * y);
    R[1][0] = 2.f * (x * y + w * z); R[1][1] = 1.f - 2.f * (x * x + z * z); R[1][2] = 2.f * (y * z - w * x);
    R[2][0] = 2.f * (x * z - w * y); R[2][1] = 2.f * (y * z + w * x); R[2][2] = 1.f - 2.f * (x * x + y * y);
    float Mm[3][3], Sg[3][3];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) Mm[a][b] = R[a][b] * s[b];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) Sg[a][b] = Mm[a][0] * Mm[b][0] + Mm[a][1] * Mm[b][1] + Mm[a][2] * Mm[b][2];
    const float *Wm = cc.W;
    const float mu[3] = {mean[i], mean[n + i], mean[2 * n + i]};
    float pc[3];
#pragma unroll
    for (int a = 0; a < 3; a++) pc[a] = Wm[3 * a] * mu[0] + Wm[3 * a + 1] * mu[1] + Wm[3 * a + 2] * mu[2] + cc.t[a];
    const float X = pc[0], Y = pc[1], Z = pc[2];
    const float iz = 1.f / Z, iz2 = iz * iz;
    const float rxz = X * iz, ryz = Y * iz;
    const bool clx = rxz < cc.lx_lo || rxz > cc.lx_hi;
    const bool cly = ryz < cc.ly_lo || ryz > cc.ly_hi;
    const float cxr = fminf(fmaxf(rxz, cc.lx_lo), cc.lx_hi), cyr = fminf(fmaxf(ryz, cc.ly_lo), cc.ly_hi);
    const float tx = clx ? cxr * Z : X, ty = cly ? cyr * Z : Y;
    const float fx = cc.fx, fy = cc.fy;
    const float J00 = fx * iz, J02 = -fx * tx * iz2, J11 = fy * iz, J12 = -fy * ty * iz2;
    float A[2][3];
#pragma unroll
    for (int j = 0; j < 3; j++) {
      A[0][j] = J00 * Wm[j] + J02 * Wm[6 + j];
      A[1][j] = J11 * Wm[3 + j] + J12 * Wm[6 + j];
    }
    float AS[2][3];  // A Sigma
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
      for (int j = 0; j < 3; j++) AS[a][j] = A[a][0] * Sg[0][j] + A[a][1] * Sg[1][j] + A[a][2] * Sg[2][j];
    const float sa = AS[0][0] * A[0][0] + AS[0][1] * A[0][1] + AS[0][2] * A[0][2] + cc.dil;
    const float sb = AS[0][0] * A[1][0] + AS[0][1] * A[1][1] + AS[0][2] * A[1][2];
    const float sc2 = AS[1][0] * A[1][0] + AS[1][1] * A[1][1] + AS[1][2] * A[1][2] + cc.dil;
    const float idet = 1.f / (sa * sc2 - sb * sb);
    const float Q00 = sc2 * idet, Q01 = -sb * idet, Q11 = sa * idet;
    // dL/dSigma' = -Q G_Q Q, G_Q = [[gca, gcb/2], [gcb/2, gcc]]
    const float h = 0.5f * gcb;
    const float T00 = Q00 * gca + Q01 * h, T01 = Q00 * h + Q01 * gcc;
    const float T10 = Q01 * gca + Q11 * h, T11 = Q01 * h + Q11 * gcc;
    const float G00 = -(T00 * Q00 + T01 * Q01), G01 = -(T00 * Q01 + T01 * Q11);
    const float G11 = -(T10 * Q01 + T11 * Q11);
    // GA = 2 G2 A Sigma  (2x3),  GS = A^T G2 A (3x3)
    float GA[2][3], G2A[2][3];
#pragma unroll
    for (int j = 0; j < 3; j++) {
      GA[0][j] = 2.f * (G00 * AS[0][j] + G01 * AS[1][j]);
      GA[1][j] = 2.f * (G01 * AS[0][j] + G11 * AS[1][j]);
      G2A[0][j] = G00 * A[0][j] + G01 * A[1][j];
      G2A[1][j] = G01 * A[0][j] + G11 * A[1][j];
    }
    float GS[3][3];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) GS[a][b] = A[0][a] * G2A[0][b] + A[1][a] * G2A[1][b];
    // dL/dJ = GA W^T (only J00, J02, J11, J12 vary)
    const float GJ00 = GA[0][0] * Wm[0] + GA[0][1] * Wm[1] + GA[0][2] * Wm[2];
    const float GJ02 = GA[0][0] * Wm[6] + GA[0][1] * Wm[7] + GA[0][2] * Wm[8];
    const float GJ11 = GA[1][0] * Wm[3] + GA[1][1] * Wm[4] + GA[1][2] * Wm[5];
    const float GJ12 = GA[1][0] * Wm[6] + GA[1][1] * Wm[7] + GA[1][2] * Wm[8];
    float gpc[3];
    gpc[0] = gu * fx * iz;
    gpc[1] = gv * fy * iz;
    gpc[2] = gz - (gu * fx * X + gv * fy * Y) * iz2 - (GJ00 * fx + GJ11 * fy) * iz2;
    if (!clx) {
      gpc[0] -= GJ02 * fx * iz2;
      gpc[2] += GJ02 * 2.f * fx * X * iz2 * iz;
    } else {
      gpc[2] += GJ02 * fx * cxr * iz2;  // J02 = -fx c / Z
    }
    if (!cly) {
      gpc[1] -= GJ12 * fy * iz2;
      gpc[2] += GJ12 * 2.f * fy * Y * iz2 * iz;
    } else {
      gpc[2] += GJ12 * fy * cyr * iz2;
    }
#pragma unroll
    for (int a = 0; a < 3; a++) g[a] = Wm[a] * gpc[0] + Wm[3 + a] * gpc[1] + Wm[6 + a] * gpc[2];
    // pose: v, and omega via p_c and via W in A = J W (Mw = W GA^T J)
    pose[3] = gpc[0];
    pose[4] = gpc[1];
    pose[5] = gpc[2];
    pose[0] = Y * gpc[2] - Z * gpc[1];
    pose[1] = Z * gpc[0] - X * gpc[2];
    pose[2] = X * gpc[1] - Y * gpc[0];
    float Jm[2][3] = {{J00, 0.f, J02}, {0.f, J11, J12}};
    float Mw[3][3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      // (GA^T J)[l][b] = sum_k GA[k][l] J[k][b];  Mw[a][b] = sum_l W[a][l] (GA^T J)[l][b]
      const float c0 = Wm[3 * a] * GA[0][0] + Wm[3 * a + 1] * GA[0][1] + Wm[3 * a + 2] * GA[0][2];
      const float c1 = Wm[3 * a] * GA[1][0] + Wm[3 * a + 1] * GA[1][1] + Wm[3 * a + 2] * GA[1][2];
#pragma unroll
      for (int b = 0; b < 3; b++) Mw[a][b] = c0 * Jm[0][b] + c1 * Jm[1][b];
    }
    pose[0] += Mw[1][2] - Mw[2][1];
    pose[1] += Mw[2][0] - Mw[0][2];
    pose[2] += Mw[0][1] - Mw[1][0];
    // opacity (Eq 7, M = 1): o_hat = sig(o)
    const float oh = rec4[i * 4 + 1].y;
    g[3] = goh * oh * (1.f - oh);
    float gM = goh * oh;
    // Sigma = Mm Mm^T: dL/dMm = 2 GS Mm
    float GM[3][3];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) GM[a][b] = 2.f * (GS[a][0] * Mm[0][b] + GS[a][1] * Mm[1][b] + GS[a][2] * Mm[2][b]);
#pragma unroll
    for (int b = 0; b < 3; b++) {
      const float gsb = R[0][b] * GM[0][b] + R[1][b] * GM[1][b] + R[2][b] * GM[2][b];
      g[7 + b] = gsb * s[b];  // d/d log-scale
      gM += gsb * s[b];
    }
    float GR[3][3];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) GR[a][b] = GM[a][b] * s[b];
    const float gw = 2.f * (-z * GR[0][1] + y * GR[0][2] + z * GR[1][0] - x * GR[1][2] - y * GR[2][0] + x * GR[2][1]);
    const float gx = 2.f * (y * GR[0][1] + z * GR[0][2] + y * GR[1][0] - 2.f * x * GR[1][1] - w * GR[1][2] +
                            z * GR[2][0] + w * GR[2][1] - 2.f * x * GR[2][2]);
    const float gy = 2.f * (-2.f * y * GR[0][0] + x * GR[0][1] + w * GR[0][2] + x * GR[1][0] + z * GR[1][2] -
                            w * GR[2][0] + z * GR[2][1] - 2.f * y * GR[2][2]);
    const float gzq = 2.f * (-2.f * z * GR[0][0] - w * GR[0][1] + x * GR[0][2] + w * GR[1][0] - 2.f * z * GR[1][1] +
                             y * GR[1][2] + x * GR[2][0] + y * GR[2][1]);
    const float dot = w * gw + x * gx + y * gy + z * gzq;
    g[10] = (gw - w * dot) * qinv;
    g[11] = (gx - x * dot) * qinv;
    g[12] = (gy - y * dot) * qinv;
    g[13] = (gzq - z * dot) * qinv;
    // Eq 6 straight-through: dL/dm = dL/dM Sig'(m)
    const float sm = 1.f / (1.f + __expf(-mask[i]));
    g[14] = gM * sm * (1.f - sm);
  }
  if (!(flags & CSPLAT_POSE_ONLY) && i < n) {
    const bool accu = (flags & CSPLAT_ACCUMULATE) != 0;
    auto put = [&](float *plane, int k, int64_t off) {
      if (!plane) return;
      if (accu) plane[off] += g[k];
      else plane[off] = g[k];
    };
    for (int k = 0; k < 3; k++) put(out.mean, k, (int64_t)k * n + i);
    put(out.opacity, 3, i);
    for (int k = 0; k < 3; k++) put(out.rgb, 4 + k, (int64_t)k * n + i);
    for (int k = 0; k < 3; k++) put(out.log_scale, 7 + k, (int64_t)k * n + i);
    for (int k = 0; k < 4; k++) put(out.quat, 10 + k, (int64_t)k * n + i);
    put(out.mask, 14, i);
  }
  if (out.pose) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 6; k++) {
      const float v = warp_sum(pose[k]);
      if (lane == 0) red[wid][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
      float s = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w][threadIdx.x];
      atomicAdd(out.pose + threadIdx.x, s);
    }
  }
}

cudaError_t launch_render_bwd(const csplat_gaussians &g, const DecodeArgs *dec,
                              const csplat_camera &cam, const csplat_view &view,
                              const csplat_params &prm, const void *rec, const void *pair_rec,
                              const uint32_t *tile_range, const float *t_final,
                              const int32_t *n_contrib, const float *d_color, const float *d_depth,
                              const float *d_sil, uint32_t flags, const csplat_grads &out,
                              void *ws, cudaStream_t s) {
  const CamInfo ci = cam_info(cam);
  float *acc = static_cast<float *>(ws);
  cudaError_t e = cudaMemsetAsync(acc, 0, bwd_workspace_bytes(g.n), s);
  if (e != cudaSuccess) return e;
  if (out.pose && !(flags & CSPLAT_ACCUMULATE)) {
    e = cudaMemsetAsync(out.pose, 0, 6 * sizeof(float), s);
    if (e != cudaSuccess) return e;
  }
  const int T = ci.tiles_x * ci.tiles_y;
  k_render_bwd<<<T, 256, 0, s>>>(static_cast<const float4 *>(pair_rec), tile_range, ci.W, ci.H,
                                 ci.tiles_x, prm.alpha_max, t_final, n_contrib, d_color, d_depth,
                                 d_sil, acc);
  e = cudaGetLastError();
  if (e != cudaSuccess || g.n == 0) return e;
  ChainConst cc;
  for (int a = 0; a < 3; a++) {
    for (int b = 0; b < 3; b++) cc.W[3 * a + b] = view.m[4 * a + b];
    cc.t[a] = view.m[4 * a + 3];
  }
  cc.fx = cam.fx;
  cc.fy = cam.fy;
  const float Wf = (float)cam.width, Hf = (float)cam.height;
  cc.lx_lo = -((cam.cx + 0.15f * Wf) / cam.fx);
  cc.lx_hi = ((Wf - cam.cx) + 0.15f * Wf) / cam.fx;
  cc.ly_lo = -((cam.cy + 0.15f * Hf) / cam.fy);
  cc.ly_hi = ((Hf - cam.cy) + 0.15f * Hf) / cam.fy;
  cc.dil = prm.dilation;
  DecodeArgs d{};
  if (dec) d = *dec;
  const int64_t blocks = (g.n + 255) / 256;
  k_chain<<<(unsigned)blocks, 256, 0, s>>>(g.n, g.n_dev, g.mean, g.opacity, g.log_scale, g.quat,
                                           g.mask, d, dec ? 1 : 0, cc,
                                           static_cast<const float4 *>(rec),
                                           reinterpret_cast<const float4 *>(acc), flags, out);
  return cudaGetLastError();
}

}  // namespace csplat
