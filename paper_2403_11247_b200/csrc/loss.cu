// loss.cu -- NEXT-1: the silhouette-gated tracking objective (Eq 12, P:194-198,
// gated as in Eq 14; reading R27) and its gradient with respect to
// the rendered colour, depth and silhouette -- the upstream of csplat_render_bwd
// in a tracking iteration.  Elementwise and HBM-bound: 9 floats read, 5
// written per pixel; two launches (valid-depth count, then loss + gradients).
#include "common.cuh"

namespace csplat {

constexpr int kLossThreads = 256;

__global__ void __launch_bounds__(kLossThreads) k_count_valid(int64_t HW,
                                                              const float *__restrict__ obs_depth,
                                                              unsigned long long *__restrict__ cnt) {
  unsigned c = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < HW;
       p += (int64_t)gridDim.x * blockDim.x)
    c += obs_depth[p] > 0.0f ? 1u : 0u;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}

__global__ void __launch_bounds__(kLossThreads) k_tracking_loss(
    int64_t HW, const float *__restrict__ color, const float *__restrict__ depth,
    const float *__restrict__ sil, const float *__restrict__ oc, const float *__restrict__ od,
    float lambda_d, float gate, const unsigned long long *__restrict__ cnt,
    float *__restrict__ dC, float *__restrict__ dD, float *__restrict__ dS,
    float *__restrict__ loss3) {
  __shared__ float red[2][kLossThreads / 32];
  const float invN = 1.0f / (float)HW;
  const unsigned long long nv = *cnt;
  const float invR = 1.0f / (float)(nv > 0 ? nv : 1);
  float lc = 0.f, ld = 0.f;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < HW;
       p += (int64_t)gridDim.x * blockDim.x) {
    const float g = sil[p] > gate ? 1.0f : 0.0f;        // Eq 14 gate (no gradient)
    const float obd = od[p];
    const float v = obd > 0.0f ? 1.0f : 0.0f;           // R_i: valid depth (Eq 12)
    const float r0 = color[p] - oc[p], r1 = color[HW + p] - oc[HW + p];
    const float r2 = color[2 * HW + p] - oc[2 * HW + p];
    lc += g * (r0 * r0 + r1 * r1 + r2 * r2);
    const float s = 2.0f * g * invN;
    dC[p] = s * r0;
    dC[HW + p] = s * r1;
    dC[2 * HW + p] = s * r2;
    const float rd = depth[p] - obd;
    ld += g * v * rd * rd;
    dD[p] = 2.0f * lambda_d * g * v * rd * invR;
    dS[p] = 0.0f;
  }
  lc = warp_sum(lc);
  ld = warp_sum(ld);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { red[0][wid] = lc; red[1][wid] = ld; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.f, b = 0.f;
    for (int w = 0; w < kLossThreads / 32; w++) { a += red[0][w]; b += red[1][w]; }
    a *= invN;
    b *= invR;
    atomicAdd(loss3 + 0, a + lambda_d * b);
    atomicAdd(loss3 + 1, a);
    atomicAdd(loss3 + 2, b);
  }
}

// NEXT-1: the device-side pose update of a tracking iteration, so a frame's
// iterations replay as one CUDA graph without a host round trip: V' = Exp(xi) V
// with xi = -(lr_rot g_omega, lr_trans g_v), the left perturbation the pose
// gradient of csplat_render_bwd is taken with (R22): p' = Rod(omega) p + v.
// One thread, float64 (the host form of tracking.apply_left).
__global__ void k_pose_step(float *__restrict__ V, const float *__restrict__ g, float lr_rot,
                            float lr_trans) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double w0 = -(double)lr_rot * g[0], w1 = -(double)lr_rot * g[1],
               w2 = -(double)lr_rot * g[2];
  const double th = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
  const double K[3][3] = {{0, -w2, w1}, {w2, 0, -w0}, {-w1, w0, 0}};
  double a = 1.0, b = 0.5;  // R = I + a K + b K^2 (Rodrigues); th -> 0: I + K
  if (th >= 1e-12) {
    a = sin(th) / th;
    b = (1.0 - cos(th)) / (th * th);
  } else {
    b = 0.0;
  }
  double R[3][3];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      double k2 = 0.0;
      for (int k = 0; k < 3; k++) k2 += K[i][k] * K[k][j];
      R[i][j] = (i == j ? 1.0 : 0.0) + a * K[i][j] + b * k2;
    }
  double out[12];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 4; j++) {
      double t = 0.0;
      for (int k = 0; k < 3; k++) t += R[i][k] * (double)V[4 * k + j];
      if (j == 3) t += -(double)lr_trans * g[3 + i];
      out[4 * i + j] = t;
    }
  for (int k = 0; k < 12; k++) V[k] = (float)out[k];
}

cudaError_t launch_pose_step(float *view_dev, const float *pose_grad, float lr_rot,
                             float lr_trans, cudaStream_t s) {
  k_pose_step<<<1, 32, 0, s>>>(view_dev, pose_grad, lr_rot, lr_trans);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- NEXT-3

__global__ void __launch_bounds__(kLossThreads) k_count_active(int64_t n,
                                                               const int64_t *__restrict__ n_dev,
                                                               const int32_t *__restrict__ count,
                                                               unsigned long long *__restrict__ na) {
  const int64_t ne = eff_n(n, n_dev);
  unsigned c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne;
       i += (int64_t)gridDim.x * blockDim.x)
    c += count[i] > 0 ? 1u : 0u;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(na, (unsigned long long)c);
}

// Eq 8 over the in-frustum Gaussians: d_mask += lambda Sig'(m)/N_a.
__global__ void __launch_bounds__(kLossThreads) k_mask_loss(
    int64_t n, const int64_t *__restrict__ n_dev, const float *__restrict__ mask,
    const int32_t *__restrict__ count, float lambda, const unsigned long long *__restrict__ na,
    float *__restrict__ d_mask, float *__restrict__ loss) {
  __shared__ float red[kLossThreads / 32];
  const int64_t ne = eff_n(n, n_dev);
  const unsigned long long a = *na;
  const float inv = a ? 1.0f / (float)a : 0.0f;
  float s = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (count[i] <= 0) continue;
    const float sg = 1.0f / (1.0f + __expf(-mask[i]));
    s += sg;
    d_mask[i] += lambda * sg * (1.0f - sg) * inv;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0 && loss) {
    float t = 0.f;
    for (int w = 0; w < kLossThreads / 32; w++) t += red[w];
    atomicAdd(loss, t * inv);
  }
}

constexpr int kMaxOverlapViews = 256;

struct OverlapConst {
  float C[12];
  float fx, fy, cx, cy, near_z, far_z, Wm1, Hm1, wcx, hcy;  // wcx = (W-1) - cx, hcy alike
  int W, H, K;
};

// P:138 keyframe overlap, float32 decision arithmetic (bit-exact counts).
__global__ void __launch_bounds__(kLossThreads) k_overlap(const float *__restrict__ depth,
                                                          OverlapConst oc,
                                                          const float *__restrict__ views,
                                                          unsigned long long *__restrict__ counts) {
  __shared__ __align__(16) float sv[kMaxOverlapViews * 12];
  __shared__ unsigned sc[kMaxOverlapViews];
  for (int t = threadIdx.x; t < oc.K * 12; t += blockDim.x) sv[t] = views[t];
  for (int t = threadIdx.x; t < oc.K; t += blockDim.x) sc[t] = 0;
  __syncthreads();
  const int64_t HW = (int64_t)oc.W * oc.H;
  const int lane = threadIdx.x & 31;
  // uniform trip count, so each (point, keyframe) test is warp-aggregated by a ballot
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < HW;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = base + threadIdx.x;
    const float d = p < HW ? depth[p] : 0.0f;
    const bool valid = d > 0.0f;
    const int px = (int)(p % oc.W), py = (int)(p / oc.W);
    const float xn = DDIV(DSUB((float)px, oc.cx), oc.fx), yn = DDIV(DSUB((float)py, oc.cy), oc.fy);
    const float qx = DSUB(DMUL(xn, d), oc.C[3]), qy = DSUB(DMUL(yn, d), oc.C[7]);
    const float qz = DSUB(d, oc.C[11]);
    float X[3];
#pragma unroll
    for (int a = 0; a < 3; a++)
      X[a] = DADD(DADD(DMUL(oc.C[a], qx), DMUL(oc.C[4 + a], qy)), DMUL(oc.C[8 + a], qz));
    if (!__any_sync(0xffffffffu, valid)) continue;
    // keyframes in chunks of 32: lane j keeps the warp's count for keyframe kb + j
    // in a register, one shared atomic per (warp, 32 keyframes)
    for (int kb = 0; kb < oc.K; kb += 32) {
      const int kn = min(32, oc.K - kb);
      unsigned cnt = 0;
      for (int j = 0; j < kn; j++) {
        const float4 *V = reinterpret_cast<const float4 *>(sv + 12 * (kb + j));
        const float4 r0 = V[0], r1 = V[1], r2 = V[2];
        const float xc = DADD(DADD(DADD(DMUL(r0.x, X[0]), DMUL(r0.y, X[1])), DMUL(r0.z, X[2])), r0.w);
        const float yc = DADD(DADD(DADD(DMUL(r1.x, X[0]), DMUL(r1.y, X[1])), DMUL(r1.z, X[2])), r1.w);
        const float zc = DADD(DADD(DADD(DMUL(r2.x, X[0]), DMUL(r2.y, X[1])), DMUL(r2.z, X[2])), r2.w);
        // 0 <= fx xc/zc + cx <= W-1 multiplied through by zc > 0 (no division)
        const float ax = DMUL(oc.fx, xc), ay = DMUL(oc.fy, yc);
        const bool in = valid && (zc > oc.near_z) && (zc < oc.far_z) &&
                        ax >= DMUL(-oc.cx, zc) && ax <= DMUL(oc.wcx, zc) &&
                        ay >= DMUL(-oc.cy, zc) && ay <= DMUL(oc.hcy, zc);
        const unsigned m = __ballot_sync(0xffffffffu, in);
        if (lane == j) cnt += (unsigned)__popc(m);
      }
      if (lane < kn && cnt) atomicAdd(sc + kb + lane, cnt);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < oc.K; t += blockDim.x)
    if (sc[t]) atomicAdd(counts + t, (unsigned long long)sc[t]);
}

cudaError_t launch_mask_loss(int64_t n, const int64_t *n_dev, const float *mask,
                             const int32_t *count, float lambda, float *d_mask, float *loss,
                             void *ws, cudaStream_t s) {
  unsigned long long *na = static_cast<unsigned long long *>(ws);
  cudaError_t e = cudaMemsetAsync(na, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  if (loss) {
    e = cudaMemsetAsync(loss, 0, sizeof(float), s);
    if (e != cudaSuccess) return e;
  }
  if (n == 0) return cudaSuccess;
  int64_t blocks = (n + kLossThreads - 1) / kLossThreads;
  if (blocks > 1184) blocks = 1184;
  k_count_active<<<(unsigned)blocks, kLossThreads, 0, s>>>(n, n_dev, count, na);
  k_mask_loss<<<(unsigned)blocks, kLossThreads, 0, s>>>(n, n_dev, mask, count, lambda, na, d_mask,
                                                        loss);
  return cudaGetLastError();
}

cudaError_t launch_overlap(const float *depth, const csplat_camera &cam, const csplat_view &cur,
                           const float *views_dev, int K, unsigned long long *counts,
                           cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)K * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  OverlapConst oc;
  for (int i = 0; i < 12; i++) oc.C[i] = cur.m[i];
  oc.fx = cam.fx; oc.fy = cam.fy; oc.cx = cam.cx; oc.cy = cam.cy;
  oc.near_z = cam.near_z; oc.far_z = cam.far_z;
  oc.Wm1 = (float)cam.width - 1.0f; oc.Hm1 = (float)cam.height - 1.0f;
  oc.W = cam.width; oc.H = cam.height; oc.K = K;
  volatile float wm1 = oc.Wm1, hm1 = oc.Hm1;  // one IEEE subtraction each, as in the oracle
  oc.wcx = wm1 - cam.cx;
  oc.hcy = hm1 - cam.cy;
  const int64_t HW = (int64_t)cam.width * cam.height;
  int64_t blocks = (HW + kLossThreads - 1) / kLossThreads;
  if (blocks > 1184) blocks = 1184;
  k_overlap<<<(unsigned)blocks, kLossThreads, 0, s>>>(depth, oc, views_dev, counts);
  return cudaGetLastError();
}

cudaError_t launch_count_valid(const float *obs_depth, int64_t HW, unsigned long long *n_valid,
                               cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(n_valid, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess || HW == 0) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (HW + kLossThreads - 1) / kLossThreads;
  if (blocks > 4LL * sms) blocks = 4LL * sms;
  k_count_valid<<<(unsigned)blocks, kLossThreads, 0, s>>>(HW, obs_depth, n_valid);
  return cudaGetLastError();
}

cudaError_t launch_tracking_loss(const float *color, const float *depth, const float *sil,
                                 const float *obs_color, const float *obs_depth, int W, int H,
                                 float lambda_d, float gate, float *d_color, float *d_depth,
                                 float *d_sil, float *loss3, void *ws, cudaStream_t s) {
  const int64_t HW = (int64_t)W * H;
  unsigned long long *cnt = static_cast<unsigned long long *>(ws);
  cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  if (loss3) {
    e = cudaMemsetAsync(loss3, 0, 3 * sizeof(float), s);
    if (e != cudaSuccess) return e;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (HW + kLossThreads - 1) / kLossThreads;
  if (blocks > 4LL * sms) blocks = 4LL * sms;
  if (blocks < 1) blocks = 1;
  k_count_valid<<<(unsigned)blocks, kLossThreads, 0, s>>>(HW, obs_depth, cnt);
  float *l3 = loss3;
  if (!l3) {  // loss value not requested: accumulate into the workspace tail
    l3 = reinterpret_cast<float *>(static_cast<char *>(ws) + 16);
    e = cudaMemsetAsync(l3, 0, 3 * sizeof(float), s);
    if (e != cudaSuccess) return e;
  }
  k_tracking_loss<<<(unsigned)blocks, kLossThreads, 0, s>>>(HW, color, depth, sil, obs_color,
                                                            obs_depth, lambda_d, gate, cnt,
                                                            d_color, d_depth, d_sil, l3);
  return cudaGetLastError();
}

}  // namespace csplat
