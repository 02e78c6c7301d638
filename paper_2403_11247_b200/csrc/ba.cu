// ba.cu -- NEXT-4: the random-ray global bundle adjustment of Sec 3.4 (P:212-215:
// "randomly sample a total number of N rays from our global keyframe database
// ... a loss similar to tracking loss, and we also add an SSIM loss to RGB
// rendering"); reading R30: the N rays are N/64 random 8x8
// patches aligned to the 8-pixel grid, so the SSIM term has a window.
//
//   k_ba_patches: per patch, the tile it lies in (a bit of the keyframe's
//                 active-tile mask, which restricts csplat_bin_tiles_active
//                 to the sampled tiles) and its valid-depth rays (|R| of Eq 12).
//   k_ba_loss:    one warp per patch, the renderers' warp layout (8 columns x
//                 4 row pairs, two vertically adjacent pixels per lane):
//                 Eq 12 colour / depth residuals, per-channel patch SSIM from
//                 warp-reduced (centred) moments, and the upstream gradients
//                 dL/dC, dL/dD of the patch pixels; loss shares by warp sums.
// Both are small and latency-bound (the sample is ~0.1% of the pixels); the
// cost of a BA iteration is the per-keyframe projection and chain.
#include "common.cuh"

namespace csplat {

constexpr int kBaThreads = 256;  // 8 patches per CTA
constexpr float kSsimC1 = 0.01f * 0.01f, kSsimC2 = 0.03f * 0.03f;  // data range 1

__global__ void __launch_bounds__(kBaThreads) k_ba_patches(const float *__restrict__ obs_depth,
                                                           int W, int H, int tiles_x,
                                                           const int32_t *__restrict__ patches,
                                                           int64_t n_patches,
                                                           uint32_t *__restrict__ tile_active,
                                                           unsigned long long *__restrict__ n_valid) {
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= n_patches) return;  // warp-uniform
  const int bw = W / 8;
  const int p = patches[b];
  if (p < 0 || p >= bw * (H / 8)) return;  // not a whole 8x8 block of the image: ignored
  const int bx = p % bw, by = p / bw;
  const int px = 8 * bx + (lane & 7), py = 8 * by + (lane >> 3) * 2;
  const int64_t q = (int64_t)py * W + px;
  const unsigned v = (obs_depth[q] > 0.0f ? 1u : 0u) + (obs_depth[q + W] > 0.0f ? 1u : 0u);
  const unsigned c = __reduce_add_sync(0xffffffffu, v);
  if (lane == 0) {
    if (c) atomicAdd(n_valid, (unsigned long long)c);
    const int tile = (8 * by / kTile) * tiles_x + 8 * bx / kTile;
    atomicOr(tile_active + (tile >> 5), 1u << (tile & 31));
  }
}

__global__ void __launch_bounds__(kBaThreads) k_ba_loss(
    const float *__restrict__ color, const float *__restrict__ depth,
    const float *__restrict__ oc, const float *__restrict__ od, int W, int H, int64_t HW,
    const int32_t *__restrict__ patches, int64_t n_patches, float inv_n, float inv_3p,
    const unsigned long long *__restrict__ n_valid, float lambda_d, float lambda_s,
    float *__restrict__ dC, float *__restrict__ dD, float *__restrict__ loss3) {
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= n_patches) return;  // warp-uniform
  const unsigned long long nv = *n_valid;
  const float inv_r = 1.0f / (float)(nv > 0 ? nv : 1ull);
  const int bw = W / 8;
  const int p = patches[b];
  if (p < 0 || p >= bw * (H / 8)) return;  // ignored, as in k_ba_patches
  const int bx = p % bw, by = p / bw;
  const int px = 8 * bx + (lane & 7), py = 8 * by + (lane >> 3) * 2;
  const int64_t q0 = (int64_t)py * W + px, q1 = q0 + W;
  float lc = 0.f, ld = 0.f, ls = 0.f;
  // Eq 12 depth term over the valid-depth rays
  {
    const float o0 = od[q0], o1 = od[q1];
    const float r0 = o0 > 0.0f ? depth[q0] - o0 : 0.0f, r1 = o1 > 0.0f ? depth[q1] - o1 : 0.0f;
    ld = (r0 * r0 + r1 * r1) * inv_r;
    const float s = 2.0f * lambda_d * inv_r;
    dD[q0] = s * r0;
    dD[q1] = s * r1;
  }
#pragma unroll
  for (int c = 0; c < 3; c++) {
    const float x0 = color[c * HW + q0], x1 = color[c * HW + q1];
    const float y0 = oc[c * HW + q0], y1 = oc[c * HW + q1];
    const float mx = warp_sum(x0 + x1) * (1.0f / 64.0f);
    const float my = warp_sum(y0 + y1) * (1.0f / 64.0f);
    const float ax0 = x0 - mx, ax1 = x1 - mx, ay0 = y0 - my, ay1 = y1 - my;
    const float sxx = warp_sum(fmaf(ax0, ax0, ax1 * ax1)) * (1.0f / 64.0f);
    const float syy = warp_sum(fmaf(ay0, ay0, ay1 * ay1)) * (1.0f / 64.0f);
    const float sxy = warp_sum(fmaf(ax0, ay0, ax1 * ay1)) * (1.0f / 64.0f);
    const float A1 = fmaf(2.0f * mx, my, kSsimC1), A2 = fmaf(2.0f, sxy, kSsimC2);
    const float B1 = fmaf(mx, mx, fmaf(my, my, kSsimC1)), B2 = sxx + syy + kSsimC2;
    const float S = (A1 * A2) / (B1 * B2);
    ls += S;  // identical on every lane: counted once below
    // dSSIM/dx_i = (2S/64) [my/A1 + (y_i - my)/A2 - mx/B1 - (x_i - mx)/B2]
    const float k = 2.0f * S * (1.0f / 64.0f);
    const float base = my / A1 - mx / B1;
    const float iA2 = 1.0f / A2, iB2 = 1.0f / B2;
    const float g0 = k * (base + ay0 * iA2 - ax0 * iB2);
    const float g1 = k * (base + ay1 * iA2 - ax1 * iB2);
    const float e0 = x0 - y0, e1 = x1 - y1;
    lc += (e0 * e0 + e1 * e1) * inv_n;
    dC[c * HW + q0] = 2.0f * e0 * inv_n - lambda_s * inv_3p * g0;
    dC[c * HW + q1] = 2.0f * e1 * inv_n - lambda_s * inv_3p * g1;
  }
  lc = warp_sum(lc);
  ld = warp_sum(ld);
  if (lane == 0) {
    atomicAdd(loss3 + 0, lc);
    atomicAdd(loss3 + 1, ld);
    atomicAdd(loss3 + 2, ls * inv_3p);
  }
}

cudaError_t launch_ba_patches(const float *obs_depth, const csplat_camera &cam,
                              const int32_t *patches, int64_t n_patches, uint32_t *tile_active,
                              unsigned long long *n_valid, cudaStream_t s) {
  const CamInfo ci = cam_info(cam);
  const int64_t T = (int64_t)ci.tiles_x * ci.tiles_y;
  cudaError_t e = cudaMemsetAsync(tile_active, 0, (size_t)((T + 31) / 32) * 4, s);
  if (e != cudaSuccess || n_patches == 0) return e;
  const int64_t blocks = (n_patches * 32 + kBaThreads - 1) / kBaThreads;
  k_ba_patches<<<(unsigned)blocks, kBaThreads, 0, s>>>(obs_depth, ci.W, ci.H, ci.tiles_x, patches,
                                                       n_patches, tile_active, n_valid);
  return cudaGetLastError();
}

cudaError_t launch_ba_loss(const float *color, const float *depth, const float *obs_color,
                           const float *obs_depth, const csplat_camera &cam,
                           const int32_t *patches, int64_t n_patches, int64_t n_rays,
                           const unsigned long long *n_valid, float lambda_d, float lambda_s,
                           float *d_color, float *d_depth, float *d_sil, float *loss3,
                           cudaStream_t s) {
  const int64_t HW = (int64_t)cam.width * cam.height;
  // upstream gradients are zero off the sampled patches
  cudaError_t e = cudaMemsetAsync(d_color, 0, (size_t)HW * 3 * sizeof(float), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_depth, 0, (size_t)HW * sizeof(float), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_sil, 0, (size_t)HW * sizeof(float), s);
  if (e != cudaSuccess || n_patches == 0) return e;
  const float inv_n = 1.0f / (float)n_rays;
  const float inv_3p = 64.0f / (3.0f * (float)n_rays);  // 1 / (3 P), P = N / 64 patches
  const int64_t blocks = (n_patches * 32 + kBaThreads - 1) / kBaThreads;
  k_ba_loss<<<(unsigned)blocks, kBaThreads, 0, s>>>(color, depth, obs_color, obs_depth, cam.width,
                                                    cam.height, HW, patches, n_patches, inv_n, inv_3p,
                                                    n_valid, lambda_d, lambda_s, d_color,
                                                    d_depth, loss3);
  return cudaGetLastError();
}

}  // namespace csplat
