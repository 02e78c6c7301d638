// rvq.cu -- a2: greedy residual vector quantisation (Eq 10; R17).
//
// One thread per vector.  The whole codebook [L][P][d] is staged in shared
// memory once per CTA; within a stage every thread scans the same code k at the
// same time, so every shared-memory read is a broadcast.  Distances are the DA
// direct form (e = c - r; d = fma(e, e, d)) so the argmin is bit-exact with the
// oracle; ties go to the lowest index (strict <).  FP32-issue-bound:
// ~(2d + 2) instructions per (vector, code).
#include "common.cuh"

namespace csplat {

constexpr int kRvqThreads = 256;

template <int D>
__global__ void __launch_bounds__(kRvqThreads) k_rvq(const float *__restrict__ x, int64_t n,
                                                     const int64_t *__restrict__ n_dev,
                                                     const float *__restrict__ codes_g, int L,
                                                     int P, int smem_codes, void *__restrict__ idx,
                                                     int idx_bytes, float *__restrict__ recon) {
  extern __shared__ float sc[];
  const float *codes = codes_g;
  if (smem_codes) {
    const int total = L * P * D;
    for (int k = threadIdx.x; k < total; k += blockDim.x) sc[k] = codes_g[k];
    __syncthreads();
    codes = sc;
  }
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ne = eff_n(n, n_dev);
  if (i >= ne) return;
  float xv[D], sh[D];
#pragma unroll
  for (int j = 0; j < D; j++) {
    xv[j] = x[(int64_t)j * n + i];
    sh[j] = 0.0f;
  }
  for (int l = 0; l < L; l++) {
    float r[D];
#pragma unroll
    for (int j = 0; j < D; j++) r[j] = DSUB(xv[j], sh[j]);  // S - S_hat^{l-1}
    const float *C = codes + (int64_t)l * P * D;
    int best = 0;
    float bestd = 0.0f;
    for (int k = 0; k < P; k++) {
      float acc = 0.0f;
#pragma unroll
      for (int j = 0; j < D; j++) {
        const float e = DSUB(C[k * D + j], r[j]);
        acc = DFMA(e, e, acc);
      }
      if (k == 0 || acc < bestd) {
        bestd = acc;
        best = k;
      }
    }
    if (idx_bytes == 1)
      static_cast<uint8_t *>(idx)[(int64_t)l * n + i] = (uint8_t)best;
    else
      static_cast<uint16_t *>(idx)[(int64_t)l * n + i] = (uint16_t)best;
#pragma unroll
    for (int j = 0; j < D; j++) sh[j] = l == 0 ? C[best * D + j] : DADD(sh[j], C[best * D + j]);
  }
  if (recon)
#pragma unroll
    for (int j = 0; j < D; j++) recon[(int64_t)j * n + i] = sh[j];
}

template <int D>
static cudaError_t run_rvq(const float *x, int64_t n, const int64_t *n_dev, const float *codes,
                           int L, int P, void *idx, int idx_bytes, float *recon, cudaStream_t s) {
  const size_t bytes = (size_t)L * P * D * sizeof(float);
  const bool use_smem = bytes <= 200 * 1024;
  if (use_smem && bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_rvq<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bytes);
    if (e != cudaSuccess) return e;
  }
  const int64_t blocks = (n + kRvqThreads - 1) / kRvqThreads;
  k_rvq<D><<<(unsigned)blocks, kRvqThreads, use_smem ? bytes : 0, s>>>(
      x, n, n_dev, codes, L, P, use_smem ? 1 : 0, idx, idx_bytes, recon);
  return cudaGetLastError();
}

cudaError_t launch_rvq(const float *x, int64_t n, const int64_t *n_dev, int d, const float *codes,
                       int L, int P, void *idx, int idx_bytes, float *recon, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  switch (d) {
    case 1: return run_rvq<1>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 2: return run_rvq<2>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 3: return run_rvq<3>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 4: return run_rvq<4>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 5: return run_rvq<5>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 6: return run_rvq<6>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 7: return run_rvq<7>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 8: return run_rvq<8>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace csplat
