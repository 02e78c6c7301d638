// chain.cu -- a8: the per-Gaussian chain rule of the backward:
// the 2D gradient accumulated by k_render_bwd (u, v, conic, o_hat, z, rgb) is
// mapped through the conic inverse, Sigma' = J W Sigma W^T J^T (Eq 2), Sigma =
// R S S^T R^T (Eq 1), the quaternion normalisation, the exp/sigmoid
// activations (R15), the straight-through mask (Eq 6, R14) and the camera
// pose (left perturbation, R22).  One thread per Gaussian; the 6-vector pose
// gradient is reduced per CTA (warp shuffles, then shared memory) and added
// with 6 atomics per CTA.  HBM-bound: 48 B accumulator + ~60 B attributes +
// 64 B record in, 60 B out per Gaussian.
#include "common.cuh"

namespace csplat {

struct ChainConst {
  float W[9], t[3];
  float fx, fy, lx_lo, lx_hi, ly_lo, ly_hi, dil;
};

template <int LF>
__global__ void __launch_bounds__(256, 4) k_chain(
    int64_t n, const int64_t *__restrict__ n_dev, const float *__restrict__ mean,
    const float *__restrict__ opac, const float *__restrict__ lsc, const float *__restrict__ quat,
    const float *__restrict__ mask, DecodeArgs dec, int use_dec, ChainConst cc,
    const float4 *__restrict__ rec4, const float4 *__restrict__ acc4,
    const uint32_t *__restrict__ alive_bits, uint32_t flags, const float *__restrict__ view_dev,
    csplat_grads out) {
  if (view_dev) {  // the view lives in device memory (graph-captured pose updates)
#pragma unroll
    for (int a = 0; a < 3; a++) {
#pragma unroll
      for (int b = 0; b < 3; b++) cc.W[3 * a + b] = __ldg(view_dev + 4 * a + b);
      cc.t[a] = __ldg(view_dev + 4 * a + 3);
    }
  }
  __shared__ float red[8][6];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ne = eff_n(n, n_dev);
  float pose[6] = {0, 0, 0, 0, 0, 0};
  float g[15];
#pragma unroll
  for (int k = 0; k < 15; k++) g[k] = 0.f;
  // the backward marked every Gaussian that received a partial (alive_bits):
  // only those are visited -- a Gaussian no pixel reached has exact-zero
  // terms, so its chain and, when accumulating, its writes are skipped
  const uint32_t word = i < ne ? alive_bits[i >> 5] : 0u;  // one word per warp
  const bool alive = i < ne && ((word >> (i & 31)) & 1u);
  const int64_t j = alive ? i : 0;
  const float4 rc0 = rec4[j * 4 + 0], rc1 = rec4[j * 4 + 1];
  float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, a2 = a0;
  if (alive) {
    a0 = acc4[j * 3 + 0]; a1 = acc4[j * 3 + 1]; a2 = acc4[j * 3 + 2];
  }
  // ACCUMULATE adds into the planes with fire-and-forget reductions
  // (red.global.add: the same float add of the old value as a load + add +
  // store, in stream order -- the window's chains run in keyframe order on one
  // stream -- but the thread never waits on the old values' loads)
  if (alive) {
    // k_render_bwd accumulates the raw moments Sx, Sy, Sxx, Sxy, Syy of
    // a = alpha dL/dalpha; map them through the record's DA conic
    // (q = ca dx^2 + (2cb) dx dy + cc dy^2; render_bwd.cu, bwd_pixel_pair)
    const float cca = rc0.z, ccb = 0.5f * rc0.w, ccc = rc1.x;
    const float gu = cca * a0.x + ccb * a0.y, gv = ccb * a0.x + ccc * a0.y;
    const float gca = -0.5f * a0.z, gcb = -a0.w, gcc = -0.5f * a1.x;
    const float goh = a1.y, gz = a1.z;
    g[4] = a1.w;  // rgb
    g[5] = a2.x;
    g[6] = a2.y;
    float ls[3], qv[4];
    if (use_dec) {
      rvq_decode<LF>(dec, n, i, ls, qv, false);  // the decoded geometry the renderer saw (R20)
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
  const bool accu = (flags & CSPLAT_ACCUMULATE) != 0;
  if (!(flags & CSPLAT_POSE_ONLY) && i < n && (alive || !accu)) {
    auto put = [&](float *plane, int k, int64_t off) {
      if (!plane) return;
      if (accu) atomicAdd(plane + off, g[k]);  // result unused: RED.E.ADD.F32
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

cudaError_t launch_chain(const csplat_gaussians &g, const DecodeArgs *dec,
                         const csplat_camera &cam, const csplat_view &view,
                         const float *view_dev, const csplat_params &prm, const void *rec,
                         const float *acc, uint32_t flags, const csplat_grads &out,
                         cudaStream_t s) {
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
  auto kern = k_chain<0>;
  switch (rvq_lf(dec)) {
    case 4: kern = k_chain<4>; break;
    case 2: kern = k_chain<2>; break;
    default: break;
  }
  kern<<<(unsigned)blocks, 256, 0, s>>>(g.n, g.n_dev, g.mean, g.opacity, g.log_scale, g.quat,
                                           g.mask, d, dec ? 1 : 0, cc,
                                           static_cast<const float4 *>(rec),
                                           reinterpret_cast<const float4 *>(acc),
                                           bwd_alive_bits(const_cast<float *>(acc), g.n), flags,
                                           view_dev, out);
  return cudaGetLastError();
}

// ---- csplat_chain_views (SURVEY §8(e) multi-view window): the chain of
// Gaussian i summed over nv views.  The view-dependent part (camera-space
// mean, J, Sigma', its inverse, dL/dSigma' -> dL/dSigma, dL/dmu, the pose) runs
// per view whose accumulator is non-zero; everything after dL/dSigma
// (R, S -> quaternion, log-scale, opacity, the STE mask) is linear in the
// per-view terms, so it runs ONCE on their sum.  The Gaussian is read and
// decoded once; its gradient written once.  View v: records at rec + v n,
// accumulator at acc + v n, pose gradient at pose + 6 v.
constexpr int kMaxChainViews = 64;
constexpr int kChainViewsPerGroup = 64;  // (view groups on grid.y measured slower, §7)
struct ChainViews {
  float W[kMaxChainViews][9];
  float t[kMaxChainViews][3];
};

template <int LF>
__global__ void __launch_bounds__(256) k_chain_views(
    int64_t n, const int64_t *__restrict__ n_dev, const float *__restrict__ mean,
    const float *__restrict__ opac, const float *__restrict__ lsc, const float *__restrict__ quat,
    const float *__restrict__ mask, DecodeArgs dec, int use_dec, ChainConst cc,
    const __grid_constant__ ChainViews cv, int nv, const float4 *__restrict__ rec4,
    char *__restrict__ ws, int64_t ws_stride, int64_t bits_off, uint32_t flags,
    csplat_grads out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ne = eff_n(n, n_dev);
  const bool in = i < ne;
  const int lane = threadIdx.x & 31;
  // this CTA's group of views (grid.y): more independent warps per Gaussian
  // range -> more loads in flight; the groups' sums meet in the gradient
  // planes by atomics (RED)
  const int vbeg = blockIdx.y * kChainViewsPerGroup;
  const int vend = min(nv, vbeg + kChainViewsPerGroup);
  auto bits = [&](int v) { return reinterpret_cast<uint32_t *>(ws + v * ws_stride + bits_off); };
  auto acc_of = [&](int v) { return reinterpret_cast<float4 *>(ws + v * ws_stride); };
  // which views reached this Gaussian: the backward's bitmaps, one word per warp
  uint64_t alive = 0;
  if (in) {
    for (int v = vbeg; v < vend; v++) {
      const uint32_t word = bits(v)[i >> 5];
      if ((word >> lane) & 1u) alive |= 1ull << v;
    }
  }
  float g[15];
#pragma unroll
  for (int k = 0; k < 15; k++) g[k] = 0.f;
  // view-independent geometry (only when some view reached the Gaussian)
  float s[3] = {0.f, 0.f, 0.f}, R[3][3] = {}, Mm[3][3] = {}, Sg[3][3] = {};
  float qinv = 0.f, w = 0.f, x = 0.f, y = 0.f, z = 0.f, oh = 0.f;
  float mu[3] = {0.f, 0.f, 0.f};
  if (alive) {
    float ls[3], qv[4];
    if (use_dec) {
      rvq_decode<LF>(dec, n, i, ls, qv, false);  // the decoded geometry the renderer saw (R20)
    } else {
      for (int k = 0; k < 3; k++) ls[k] = lsc[k * n + i];
      for (int k = 0; k < 4; k++) qv[k] = quat[k * n + i];
    }
    for (int k = 0; k < 3; k++) s[k] = __expf(ls[k]);
    const float qn2 = qv[0] * qv[0] + qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3];
    qinv = rsqrtf(qn2);
    w = qv[0] * qinv; x = qv[1] * qinv; y = qv[2] * qinv; z = qv[3] * qinv;
    R[0][0] = 1.f - 2.f * (y * y + z * z); R[0][1] = 2.f * (x * y - w * z); R[0][2] = 2.f * (x * z + w * y);
    R[1][0] = 2.f * (x * y + w * z); R[1][1] = 1.f - 2.f * (x * x + z * z); R[1][2] = 2.f * (y * z - w * x);
    R[2][0] = 2.f * (x * z - w * y); R[2][1] = 2.f * (y * z + w * x); R[2][2] = 1.f - 2.f * (x * x + y * y);
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) Mm[a][b] = R[a][b] * s[b];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) Sg[a][b] = Mm[a][0] * Mm[b][0] + Mm[a][1] * Mm[b][1] + Mm[a][2] * Mm[b][2];
    mu[0] = mean[i]; mu[1] = mean[n + i]; mu[2] = mean[2 * n + i];
  }
  float GSs[3][3] = {}, goh_s = 0.f;
  for (int v = vbeg; v < vend; v++) {
    const bool av = (alive >> v) & 1ull;
    const unsigned wv = __ballot_sync(0xffffffffu, av);  // (also orders the bitmap reads above)
    if (!wv) continue;  // warp-uniform: no lane reached in view v
    float pose[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if ((flags & CSPLAT_WS_ZEROED) && lane == 0) bits(v)[i >> 5] = 0u;  // read above by all lanes
    if (av) {
      float4 *a = acc_of(v) + i * 3;
      const float4 a0 = a[0], a1 = a[1], a2 = a[2];
      if (flags & CSPLAT_WS_ZEROED) {  // leave the accumulator zero for the next use
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        a[0] = z4; a[1] = z4; a[2] = z4;
      }
      const float4 rc0 = rec4[((int64_t)v * n + i) * 4 + 0], rc1 = rec4[((int64_t)v * n + i) * 4 + 1];
      oh = rc1.y;  // the record's o_hat (DA sig(o); the same in every view)
      const float cca = rc0.z, ccb = 0.5f * rc0.w, ccc = rc1.x;
      const float gu = cca * a0.x + ccb * a0.y, gv = ccb * a0.x + ccc * a0.y;
      const float gca = -0.5f * a0.z, gcb = -a0.w, gcc = -0.5f * a1.x;
      goh_s += a1.y;
      const float gz = a1.z;
      g[4] += a1.w;  // rgb
      g[5] += a2.x;
      g[6] += a2.y;
      const float *Wm = cv.W[v];
      float pc[3];
#pragma unroll
      for (int q = 0; q < 3; q++) pc[q] = Wm[3 * q] * mu[0] + Wm[3 * q + 1] * mu[1] + Wm[3 * q + 2] * mu[2] + cv.t[v][q];
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
      float AS[2][3];
#pragma unroll
      for (int q = 0; q < 2; q++)
#pragma unroll
        for (int j = 0; j < 3; j++) AS[q][j] = A[q][0] * Sg[0][j] + A[q][1] * Sg[1][j] + A[q][2] * Sg[2][j];
      const float sa = AS[0][0] * A[0][0] + AS[0][1] * A[0][1] + AS[0][2] * A[0][2] + cc.dil;
      const float sb = AS[0][0] * A[1][0] + AS[0][1] * A[1][1] + AS[0][2] * A[1][2];
      const float sc2 = AS[1][0] * A[1][0] + AS[1][1] * A[1][1] + AS[1][2] * A[1][2] + cc.dil;
      const float idet = 1.f / (sa * sc2 - sb * sb);
      const float Q00 = sc2 * idet, Q01 = -sb * idet, Q11 = sa * idet;
      const float h = 0.5f * gcb;
      const float T00 = Q00 * gca + Q01 * h, T01 = Q00 * h + Q01 * gcc;
      const float T10 = Q01 * gca + Q11 * h, T11 = Q01 * h + Q11 * gcc;
      const float G00 = -(T00 * Q00 + T01 * Q01), G01 = -(T00 * Q01 + T01 * Q11);
      const float G11 = -(T10 * Q01 + T11 * Q11);
      float GA[2][3], G2A[2][3];
#pragma unroll
      for (int j = 0; j < 3; j++) {
        GA[0][j] = 2.f * (G00 * AS[0][j] + G01 * AS[1][j]);
        GA[1][j] = 2.f * (G01 * AS[0][j] + G11 * AS[1][j]);
        G2A[0][j] = G00 * A[0][j] + G01 * A[1][j];
        G2A[1][j] = G01 * A[0][j] + G11 * A[1][j];
      }
#pragma unroll
      for (int q = 0; q < 3; q++)
#pragma unroll
        for (int b = 0; b < 3; b++) GSs[q][b] += A[0][q] * G2A[0][b] + A[1][q] * G2A[1][b];
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
        gpc[2] += GJ02 * fx * cxr * iz2;
      }
      if (!cly) {
        gpc[1] -= GJ12 * fy * iz2;
        gpc[2] += GJ12 * 2.f * fy * Y * iz2 * iz;
      } else {
        gpc[2] += GJ12 * fy * cyr * iz2;
      }
#pragma unroll
      for (int q = 0; q < 3; q++) g[q] += Wm[q] * gpc[0] + Wm[3 + q] * gpc[1] + Wm[6 + q] * gpc[2];
      pose[3] = gpc[0];
      pose[4] = gpc[1];
      pose[5] = gpc[2];
      pose[0] = Y * gpc[2] - Z * gpc[1];
      pose[1] = Z * gpc[0] - X * gpc[2];
      pose[2] = X * gpc[1] - Y * gpc[0];
      const float Jm[2][3] = {{J00, 0.f, J02}, {0.f, J11, J12}};
      float Mw[3][3];
#pragma unroll
      for (int q = 0; q < 3; q++) {
        const float c0 = Wm[3 * q] * GA[0][0] + Wm[3 * q + 1] * GA[0][1] + Wm[3 * q + 2] * GA[0][2];
        const float c1 = Wm[3 * q] * GA[1][0] + Wm[3 * q + 1] * GA[1][1] + Wm[3 * q + 2] * GA[1][2];
#pragma unroll
        for (int b = 0; b < 3; b++) Mw[q][b] = c0 * Jm[0][b] + c1 * Jm[1][b];
      }
      pose[0] += Mw[1][2] - Mw[2][1];
      pose[1] += Mw[2][0] - Mw[0][2];
      pose[2] += Mw[0][1] - Mw[1][0];
    }
    if (out.pose) {  // view v's pose gradient: warp sums, one atomic per value and warp
#pragma unroll
      for (int k = 0; k < 6; k++) {
        const float t = warp_sum(pose[k]);
        if (lane == 0 && t != 0.f) atomicAdd(out.pose + 6 * v + k, t);
      }
    }
  }
  if (alive) {
    // opacity (Eq 7, M = 1): o_hat = sig(o)
    g[3] = goh_s * oh * (1.f - oh);
    float gM = goh_s * oh;
    float GM[3][3];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) GM[a][b] = 2.f * (GSs[a][0] * Mm[0][b] + GSs[a][1] * Mm[1][b] + GSs[a][2] * Mm[2][b]);
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
    const float sm = 1.f / (1.f + __expf(-mask[i]));  // Eq 6 straight-through
    g[14] = gM * sm * (1.f - sm);
  }
  if (alive) {  // add this view group's sum (the planes were zeroed unless accumulating)
    float *planes[15];
    int64_t offs[15];
    int k = 0;
    for (int q = 0; q < 3; q++, k++) { planes[k] = out.mean; offs[k] = (int64_t)q * n + i; }
    planes[k] = out.opacity; offs[k++] = i;
    for (int q = 0; q < 3; q++, k++) { planes[k] = out.rgb; offs[k] = (int64_t)q * n + i; }
    for (int q = 0; q < 3; q++, k++) { planes[k] = out.log_scale; offs[k] = (int64_t)q * n + i; }
    for (int q = 0; q < 4; q++, k++) { planes[k] = out.quat; offs[k] = (int64_t)q * n + i; }
    planes[k] = out.mask; offs[k++] = i;
#pragma unroll
    for (int q = 0; q < 15; q++)
      if (planes[q]) atomicAdd(planes[q] + offs[q], g[q]);
  }
}

cudaError_t launch_chain_views(const csplat_gaussians &g, const DecodeArgs *dec,
                               const csplat_camera &cam, const csplat_view *views, int nv,
                               const csplat_params &prm, const void *rec, void *ws,
                               uint32_t flags, const csplat_grads &out, cudaStream_t s) {
  const int64_t ws_stride = (int64_t)bwd_workspace_bytes(g.n);
  const int64_t bits_off = (int64_t)((char *)bwd_alive_bits(ws, g.n) - (char *)ws);
  if (out.pose && !(flags & CSPLAT_ACCUMULATE)) {
    cudaError_t e = cudaMemsetAsync(out.pose, 0, (size_t)nv * 6 * sizeof(float), s);
    if (e != cudaSuccess) return e;
  }
  if (g.n == 0 || nv == 0) return cudaSuccess;
  if (!(flags & CSPLAT_ACCUMULATE)) {  // the view groups add into zeroed planes
    float *planes[6] = {out.mean, out.opacity, out.rgb, out.log_scale, out.quat, out.mask};
    const int rows[6] = {3, 1, 3, 3, 4, 1};
    for (int k = 0; k < 6; k++)
      if (planes[k]) {
        cudaError_t e = cudaMemsetAsync(planes[k], 0, (size_t)rows[k] * g.n * sizeof(float), s);
        if (e != cudaSuccess) return e;
      }
  }
  ChainConst cc{};
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
  auto kern = k_chain_views<0>;
  switch (rvq_lf(dec)) {
    case 4: kern = k_chain_views<4>; break;
    case 2: kern = k_chain_views<2>; break;
    default: break;
  }
  for (int v0 = 0; v0 < nv; v0 += kMaxChainViews) {
    const int m = nv - v0 < kMaxChainViews ? nv - v0 : kMaxChainViews;
    ChainViews cv;
    for (int v = 0; v < m; v++)
      for (int a = 0; a < 3; a++) {
        for (int b = 0; b < 3; b++) cv.W[v][3 * a + b] = views[v0 + v].m[4 * a + b];
        cv.t[v][a] = views[v0 + v].m[4 * a + 3];
      }
    csplat_grads o = out;
    if (o.pose) o.pose += 6 * v0;
    const uint32_t fl = flags;
    const dim3 grid((unsigned)blocks, (unsigned)((m + kChainViewsPerGroup - 1) / kChainViewsPerGroup));
    kern<<<grid, 256, 0, s>>>(
        g.n, g.n_dev, g.mean, g.opacity, g.log_scale, g.quat, g.mask, d, dec ? 1 : 0, cc, cv, m,
        static_cast<const float4 *>(rec) + (int64_t)v0 * g.n * 4,
        static_cast<char *>(ws) + (int64_t)v0 * ws_stride, ws_stride, bits_off, fl, o);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace csplat
