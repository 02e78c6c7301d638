// rvq.cu -- a2: greedy residual vector quantisation (Eq 10; R17).
//
// Each thread assigns TWO vectors at once with Blackwell's packed FP32x2
// instructions (sub/mul/fma.rn.f32x2 -> FADD2/FMUL2/FFMA2, each lane IEEE
// round-to-nearest, so the distances are bit-identical to the scalar DA form
// e = c - r; d = fma(e, e, d)).  The codebook [L][P][d] is staged in shared
// memory once per CTA and every code is read as a broadcast (ptxas folds the
// scalar code into the packed operand).  Ties go to the lowest index (strict
// <).  FP32-issue-bound: per (vector, code) ~ (2d + 6) / 2 instructions.
#include "common.cuh"

namespace csplat {

constexpr int kRvqThreads = 128;

typedef unsigned long long f2_t;  // two packed float32 lanes (lo = vector a, hi = vector b)

__device__ __forceinline__ f2_t pk2(float a, float b) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float lo2(f2_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi2(f2_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ f2_t sub2(f2_t a, f2_t b) {
  f2_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

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
  const int64_t ne = eff_n(n, n_dev);
  const int64_t ia = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (ia >= ne) return;
  const bool has_b = ia + 1 < ne;
  const int64_t ib = has_b ? ia + 1 : ia;
  float xa[D], xb[D], sa[D], sb[D];
#pragma unroll
  for (int j = 0; j < D; j++) {
    xa[j] = x[(int64_t)j * n + ia];
    xb[j] = x[(int64_t)j * n + ib];
    sa[j] = sb[j] = 0.0f;
  }
  for (int l = 0; l < L; l++) {
    f2_t r[D];
#pragma unroll
    for (int j = 0; j < D; j++) r[j] = pk2(DSUB(xa[j], sa[j]), DSUB(xb[j], sb[j]));  // S - S_hat
    const float *C = codes + (int64_t)l * P * D;
    int besta = 0, bestb = 0;
    float da = 0.0f, db = 0.0f;
#pragma unroll 4
    for (int k = 0; k < P; k++) {
      f2_t acc = 0ull;  // (+0, +0): fma(e, e, 0) = e*e exactly
#pragma unroll
      for (int j = 0; j < D; j++) {
        const float c = C[k * D + j];
        const f2_t e = sub2(pk2(c, c), r[j]);
        acc = fma2(e, e, acc);
      }
      const float a0 = lo2(acc), a1 = hi2(acc);
      if (k == 0 || a0 < da) { da = a0; besta = k; }
      if (k == 0 || a1 < db) { db = a1; bestb = k; }
    }
    if (idx_bytes == 1) {
      uint8_t *o = static_cast<uint8_t *>(idx) + (int64_t)l * n;
      o[ia] = (uint8_t)besta;
      if (has_b) o[ib] = (uint8_t)bestb;
    } else {
      uint16_t *o = static_cast<uint16_t *>(idx) + (int64_t)l * n;
      o[ia] = (uint16_t)besta;
      if (has_b) o[ib] = (uint16_t)bestb;
    }
#pragma unroll
    for (int j = 0; j < D; j++) {  // S_hat^l in stage order
      const float ca = C[besta * D + j], cb = C[bestb * D + j];
      sa[j] = l == 0 ? ca : DADD(sa[j], ca);
      sb[j] = l == 0 ? cb : DADD(sb[j], cb);
    }
  }
  if (recon) {
#pragma unroll
    for (int j = 0; j < D; j++) {
      recon[(int64_t)j * n + ia] = sa[j];
      if (has_b) recon[(int64_t)j * n + ib] = sb[j];
    }
  }
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
  const int64_t pairs = (n + 1) / 2;
  const int64_t blocks = (pairs + kRvqThreads - 1) / kRvqThreads;
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
