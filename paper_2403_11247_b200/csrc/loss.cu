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
