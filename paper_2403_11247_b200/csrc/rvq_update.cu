// rvq_update.cu -- NEXT-2: the R-VQ codebook update (Eq 11; the
// k-means M-step of SPEC's rvq_train, reading R28): for an assignment i_n^l,
// residual r_n^l = x_n - S_hat_n^{l-1} (DA, the same stage-order sums as
// csplat_rvq_assign), new C^l[k] = mean of the residuals assigned to k (codes
// with no member keep their value), and the Eq 11 loss
// L_r = sum_l sum_n ||r_n^l - C^l[i_n^l]||^2 / (n P).
//
// One pass over the vectors: every CTA accumulates per-code residual sums,
// counts and per-stage errors in shared memory (privatised, so the global
// atomics are one per (CTA, code component)), then a tiny finalise kernel
// divides.  HBM-bound: (4 d + 2 L) bytes per vector.
#include <algorithm>

#include "common.cuh"

namespace csplat {

constexpr int kRuThreads = 256;

size_t rvq_update_workspace_bytes(int L, int P, int d) {
  return (size_t)L * P * d * 4 + (size_t)L * P * 4 + (size_t)(L + 1) * 4 + 256;
}

__device__ __forceinline__ uint32_t ru_idx(const void *p, int bytes, int64_t off) {
  return bytes == 1 ? (uint32_t)((const uint8_t *)p)[off] : (uint32_t)((const uint16_t *)p)[off];
}

template <int D, bool SMEM>
__global__ void __launch_bounds__(kRuThreads) k_rvq_accum(
    const float *__restrict__ x, int64_t n, const int64_t *__restrict__ n_dev,
    const float *__restrict__ codes, int L, int P, const void *__restrict__ idx, int idx_bytes,
    float *__restrict__ gsum, uint32_t *__restrict__ gcnt, float *__restrict__ gerr) {
  extern __shared__ float sm[];
  float *ssum = SMEM ? sm : gsum;
  uint32_t *scnt = SMEM ? reinterpret_cast<uint32_t *>(sm + L * P * D) : gcnt;
  float *serr = SMEM ? sm + L * P * D + L * P : gerr;
  if (SMEM) {
    for (int t = threadIdx.x; t < L * P * (D + 1) + L; t += blockDim.x) sm[t] = 0.0f;
    __syncthreads();
  }
  const int64_t ne = eff_n(n, n_dev);
  const int lane = threadIdx.x & 31;
  // uniform trip count: the Eq 11 error of each stage is warp-reduced before its
  // (shared) atomic instead of one same-address atomic per vector
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < ne;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool ok = i < ne;
    float sh[D];
#pragma unroll
    for (int j = 0; j < D; j++) sh[j] = 0.0f;
    for (int l = 0; l < L; l++) {
      const uint32_t k = ok ? ru_idx(idx, idx_bytes, (int64_t)l * n + i) : (uint32_t)P;
      ok = ok && k < (uint32_t)P;  // out-of-range index: the vector is skipped from here
      float e2 = 0.0f;
      if (ok) {
        const float *c = codes + ((int64_t)l * P + k) * D;
#pragma unroll
        for (int j = 0; j < D; j++) {
          const float r = DSUB(x[(int64_t)j * n + i], sh[j]);  // S - S_hat^{l-1}
          atomicAdd(ssum + ((int64_t)l * P + k) * D + j, r);
          const float e = r - c[j];
          e2 = fmaf(e, e, e2);
        }
        atomicAdd(scnt + (int64_t)l * P + k, 1u);
#pragma unroll
        for (int j = 0; j < D; j++) sh[j] = l == 0 ? c[j] : DADD(sh[j], c[j]);
      }
      if (!__any_sync(0xffffffffu, ok)) break;
      e2 = warp_sum(e2);
      if (lane == 0 && e2 != 0.0f) atomicAdd(serr + l, e2);
    }
  }
  if (SMEM) {
    __syncthreads();
    for (int t = threadIdx.x; t < L * P * D; t += blockDim.x)
      if (ssum[t] != 0.0f) atomicAdd(gsum + t, ssum[t]);
    for (int t = threadIdx.x; t < L * P; t += blockDim.x)
      if (scnt[t]) atomicAdd(gcnt + t, scnt[t]);
    for (int t = threadIdx.x; t < L; t += blockDim.x) atomicAdd(gerr + t, serr[t]);
  }
}

__global__ void k_rvq_finalize(int64_t n, const int64_t *__restrict__ n_dev, int L, int P, int D,
                               const float *__restrict__ codes, const float *__restrict__ gsum,
                               const uint32_t *__restrict__ gcnt, const float *__restrict__ gerr,
                               float *__restrict__ codes_out, int32_t *__restrict__ counts_out,
                               float *__restrict__ loss_out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < (int64_t)L * P * D) {
    const uint32_t c = gcnt[t / D];
    codes_out[t] = c ? gsum[t] / (float)c : codes[t];
  }
  if (counts_out && t < (int64_t)L * P) counts_out[t] = (int32_t)gcnt[t];
  if (loss_out && t == 0) {
    const int64_t ne = eff_n(n, n_dev);
    float tot = 0.0f;
    for (int l = 0; l < L; l++) {
      loss_out[l] = gerr[l];
      tot += gerr[l];
    }
    loss_out[L] = ne > 0 ? tot / ((float)ne * (float)P) : 0.0f;
  }
}

template <int D>
static cudaError_t run_update(const float *x, int64_t n, const int64_t *n_dev,
                              const float *codes, int L, int P, const void *idx, int idx_bytes,
                              float *codes_out, int32_t *counts_out, float *loss_out, void *ws,
                              cudaStream_t s) {
  float *gsum = static_cast<float *>(ws);
  uint32_t *gcnt = reinterpret_cast<uint32_t *>(gsum + (size_t)L * P * D);
  float *gerr = reinterpret_cast<float *>(gcnt + (size_t)L * P);
  cudaError_t e = cudaMemsetAsync(ws, 0, rvq_update_workspace_bytes(L, P, D), s);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (n + kRuThreads - 1) / kRuThreads;
  if (blocks > 2LL * sms) blocks = 2LL * sms;  // each CTA amortises its shared histogram
  if (blocks < 1) blocks = 1;
  const size_t smem = ((size_t)L * P * (D + 1) + L) * sizeof(float);
  if (n > 0) {
    if (smem <= 96 * 1024) {
      if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(k_rvq_accum<D, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
      }
      k_rvq_accum<D, true><<<(unsigned)blocks, kRuThreads, smem, s>>>(
          x, n, n_dev, codes, L, P, idx, idx_bytes, gsum, gcnt, gerr);
    } else {
      k_rvq_accum<D, false><<<(unsigned)blocks, kRuThreads, 0, s>>>(
          x, n, n_dev, codes, L, P, idx, idx_bytes, gsum, gcnt, gerr);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const int64_t tot = (int64_t)L * P * D;
  k_rvq_finalize<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(
      n, n_dev, L, P, D, codes, gsum, gcnt, gerr, codes_out, counts_out, loss_out);
  return cudaGetLastError();
}

cudaError_t launch_rvq_update(const float *x, int64_t n, const int64_t *n_dev, int d,
                              const float *codes, int L, int P, const void *idx, int idx_bytes,
                              float *codes_out, int32_t *counts_out, float *loss_out, void *ws,
                              cudaStream_t s) {
  switch (d) {
    case 1: return run_update<1>(x, n, n_dev, codes, L, P, idx, idx_bytes, codes_out, counts_out, loss_out, ws, s);
    case 2: return run_update<2>(x, n, n_dev, codes, L, P, idx, idx_bytes, codes_out, counts_out, loss_out, ws, s);
    case 3: return run_update<3>(x, n, n_dev, codes, L, P, idx, idx_bytes, codes_out, counts_out, loss_out, ws, s);
    case 4: return run_update<4>(x, n, n_dev, codes, L, P, idx, idx_bytes, codes_out, counts_out, loss_out, ws, s);
    case 5: return run_update<5>(x, n, n_dev, codes, L, P, idx, idx_bytes, codes_out, counts_out, loss_out, ws, s);
    case 6: return run_update<6>(x, n, n_dev, codes, L, P, idx, idx_bytes, codes_out, counts_out, loss_out, ws, s);
    case 7: return run_update<7>(x, n, n_dev, codes, L, P, idx, idx_bytes, codes_out, counts_out, loss_out, ws, s);
    case 8: return run_update<8>(x, n, n_dev, codes, L, P, idx, idx_bytes, codes_out, counts_out, loss_out, ws, s);
    default: return cudaErrorInvalidValue;
  }
}

// ---- NEXT-2 STE (reading R31): dL/dC^l[k] += sum over i_n^l = k of dL/dS_hat_n.
// One thread per vector: its d-vector gradient goes to every stage's chosen
// code with global vector reductions (red.global.add.v4 / .v2 / scalar), the
// L2 doing the per-code sums (C2: 150k vectors x 4 stages into 4 x 256 codes).
// HBM-bound: 4 d + L idx_bytes bytes per vector.
template <int D>
__global__ void __launch_bounds__(kRuThreads) k_rvq_code_grad(
    const float *__restrict__ g, int64_t n, const int64_t *__restrict__ n_dev, int L, int P,
    const void *__restrict__ idx, int idx_bytes, float *__restrict__ dcodes) {
  const int64_t ne = eff_n(n, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v[D];
    bool nz = false;
#pragma unroll
    for (int j = 0; j < D; j++) {
      v[j] = g[(int64_t)j * n + i];
      nz |= v[j] != 0.0f;
    }
    if (!nz) continue;  // exact zeros add nothing (Gaussians no pixel reached)
    for (int l = 0; l < L; l++) {
      const uint32_t k = ru_idx(idx, idx_bytes, (int64_t)l * n + i);
      if (k >= (uint32_t)P) continue;  // culled Gaussian
      float *dst = dcodes + ((int64_t)l * P + k) * D;
      if constexpr (D == 4) {
        red_add_v4(dst, v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int j = 0; j < D; j++) atomicAdd(dst + j, v[j]);
      }
    }
  }
}

// ---- NEXT-2 Fig 4 initialisation of stage l (reading R32): C^l[k] = the
// stage-l residual of the sampled vector s_k, with the same DA stage-order sum
// S_hat^{l-1} as csplat_rvq_assign.  One thread per code.
template <int D>
__global__ void k_rvq_init_stage(const float *__restrict__ x, int64_t n, float *__restrict__ codes,
                                 int P, int l, const void *__restrict__ idx, int idx_bytes,
                                 const int64_t *__restrict__ sample) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= P) return;
  const int64_t s = sample[k];
  float sh[D];
#pragma unroll
  for (int j = 0; j < D; j++) sh[j] = 0.0f;
  for (int m = 0; m < l; m++) {
    const uint32_t c = min(ru_idx(idx, idx_bytes, (int64_t)m * n + s), (uint32_t)(P - 1));
    const float *cp = codes + ((int64_t)m * P + c) * D;
#pragma unroll
    for (int j = 0; j < D; j++) sh[j] = m == 0 ? cp[j] : DADD(sh[j], cp[j]);
  }
#pragma unroll
  for (int j = 0; j < D; j++) codes[((int64_t)l * P + k) * D + j] = DSUB(x[(int64_t)j * n + s], sh[j]);
}

template <int D>
static cudaError_t run_code_grad(const float *g, int64_t n, const int64_t *n_dev, int L, int P,
                                 const void *idx, int idx_bytes, float *dcodes, bool accumulate,
                                 cudaStream_t s) {
  if (!accumulate) {
    cudaError_t e = cudaMemsetAsync(dcodes, 0, (size_t)L * P * D * sizeof(float), s);
    if (e != cudaSuccess) return e;
  }
  if (n == 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + kRuThreads - 1) / kRuThreads, 148 * 8);
  k_rvq_code_grad<D><<<(unsigned)blocks, kRuThreads, 0, s>>>(g, n, n_dev, L, P, idx, idx_bytes,
                                                             dcodes);
  return cudaGetLastError();
}

cudaError_t launch_rvq_code_grad(const float *g, int64_t n, const int64_t *n_dev, int d, int L,
                                 int P, const void *idx, int idx_bytes, float *dcodes,
                                 bool accumulate, cudaStream_t s) {
  switch (d) {
    case 1: return run_code_grad<1>(g, n, n_dev, L, P, idx, idx_bytes, dcodes, accumulate, s);
    case 2: return run_code_grad<2>(g, n, n_dev, L, P, idx, idx_bytes, dcodes, accumulate, s);
    case 3: return run_code_grad<3>(g, n, n_dev, L, P, idx, idx_bytes, dcodes, accumulate, s);
    case 4: return run_code_grad<4>(g, n, n_dev, L, P, idx, idx_bytes, dcodes, accumulate, s);
    case 5: return run_code_grad<5>(g, n, n_dev, L, P, idx, idx_bytes, dcodes, accumulate, s);
    case 6: return run_code_grad<6>(g, n, n_dev, L, P, idx, idx_bytes, dcodes, accumulate, s);
    case 7: return run_code_grad<7>(g, n, n_dev, L, P, idx, idx_bytes, dcodes, accumulate, s);
    case 8: return run_code_grad<8>(g, n, n_dev, L, P, idx, idx_bytes, dcodes, accumulate, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_rvq_init_stage(const float *x, int64_t n, int d, float *codes, int P, int l,
                                  const void *idx, int idx_bytes, const int64_t *sample,
                                  cudaStream_t s) {
  const unsigned blocks = (unsigned)((P + 127) / 128);
  switch (d) {
#define CSPLAT_INIT_CASE(D)                                                                   \
  case D:                                                                                     \
    k_rvq_init_stage<D><<<blocks, 128, 0, s>>>(x, n, codes, P, l, idx, idx_bytes, sample);  \
    return cudaGetLastError();
    CSPLAT_INIT_CASE(1) CSPLAT_INIT_CASE(2) CSPLAT_INIT_CASE(3) CSPLAT_INIT_CASE(4)
    CSPLAT_INIT_CASE(5) CSPLAT_INIT_CASE(6) CSPLAT_INIT_CASE(7) CSPLAT_INIT_CASE(8)
#undef CSPLAT_INIT_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace csplat
