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

}  // namespace csplat
