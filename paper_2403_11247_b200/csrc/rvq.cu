// rvq.cu -- a2: greedy residual vector quantisation (Eq 10; R17).
//
// A group of S threads (adjacent lanes) assigns TWO vectors: each thread scans
// the codes k = sub, sub + S, ... of a stage with Blackwell's packed FP32x2
// instructions (sub/fma.rn.f32x2 -> FADD2/FFMA2, each lane IEEE round-to-
// nearest, so every distance is bit-identical to the scalar DA form
// e = c - r; d = fma(e, e, d)), then the S partial argmins are merged with
// shuffles in (distance, index) lexicographic order -- exactly the result of
// the sequential strict-< scan (lowest index among equal minima).  Splitting
// the scan over S threads gives the SMs enough warps to hide the FFMA2 latency
// (one thread per vector pair left them at ~25% occupancy at 150k vectors).
// The codebook [L][P][d] is staged in shared memory once per CTA.
#include <cfloat>

#include "common.cuh"

namespace csplat {

constexpr int kRvqThreads = 256;

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

// Merge partial argmins over the S-lane group: (d, k) lexicographic minimum.
template <int S>
__device__ __forceinline__ void group_argmin(float &d, int &k) {
#pragma unroll
  for (int off = 1; off < S; off <<= 1) {
    const float od = __shfl_xor_sync(0xffffffffu, d, off);
    const int ok = __shfl_xor_sync(0xffffffffu, k, off);
    if (od < d || (od == d && ok < k)) {
      d = od;
      k = ok;
    }
  }
}

template <int D, int S, bool SMEM>
__global__ void __launch_bounds__(kRvqThreads) k_rvq(const float *__restrict__ x, int64_t n,
                                                     const int64_t *__restrict__ n_dev,
                                                     const float *__restrict__ codes_g, int L,
                                                     int P, void *__restrict__ idx,
                                                     int idx_bytes, float *__restrict__ recon) {
  extern __shared__ float sc[];
  const float *codes = codes_g;
  if constexpr (SMEM) {  // compile-time, so the code reads are LDS (not generic loads)
    const int total = L * P * D;
    for (int k = threadIdx.x; k < total; k += blockDim.x) sc[k] = codes_g[k];
    __syncthreads();
    codes = sc;
  }
  const int64_t ne = eff_n(n, n_dev);
  const int sub = threadIdx.x % S;
  const int64_t ia0 = 2 * (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / S);
  // no early exit: the whole warp must stay converged for the group shuffles
  const bool live = ia0 < ne;
  const int64_t ia = live ? ia0 : 0;
  const bool has_b = live && ia + 1 < ne;
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
    int besta = sub, bestb = sub;
    float da = FLT_MAX * 2.0f, db = FLT_MAX * 2.0f;  // +inf: NaN distances are never taken
    f2_t acc0 = 0ull;
#pragma unroll 4
    for (int k = sub; k < P; k += S) {
      f2_t acc = 0ull;  // (+0, +0): fma(e, e, 0) = e*e exactly
#pragma unroll
      for (int j = 0; j < D; j++) {
        const float c = C[k * D + j];
        const f2_t e = sub2(pk2(c, c), r[j]);
        acc = fma2(e, e, acc);
      }
      const float a0 = lo2(acc), a1 = hi2(acc);
      if (a0 < da) { da = a0; besta = k; }
      if (a1 < db) { db = a1; bestb = k; }
      if (k == sub) acc0 = acc;  // first code of this thread (k = 0 on sub 0)
    }
    // the sequential scan keeps k = 0 when d_0 is NaN (no later d compares below it)
    if (sub == 0) {
      if (lo2(acc0) != lo2(acc0)) { da = -FLT_MAX * 2.0f; besta = 0; }
      if (hi2(acc0) != hi2(acc0)) { db = -FLT_MAX * 2.0f; bestb = 0; }
    }
    group_argmin<S>(da, besta);
    group_argmin<S>(db, bestb);
    if (sub == 0 && live) {
      if (idx_bytes == 1) {
        uint8_t *o = static_cast<uint8_t *>(idx) + (int64_t)l * n;
        o[ia] = (uint8_t)besta;
        if (has_b) o[ib] = (uint8_t)bestb;
      } else {
        uint16_t *o = static_cast<uint16_t *>(idx) + (int64_t)l * n;
        o[ia] = (uint16_t)besta;
        if (has_b) o[ib] = (uint16_t)bestb;
      }
    }
#pragma unroll
    for (int j = 0; j < D; j++) {  // S_hat^l in stage order
      const float ca = C[besta * D + j], cb = C[bestb * D + j];
      sa[j] = l == 0 ? ca : DADD(sa[j], ca);
      sb[j] = l == 0 ? cb : DADD(sb[j], cb);
    }
  }
  if (recon && sub == 0 && live) {
#pragma unroll
    for (int j = 0; j < D; j++) {
      recon[(int64_t)j * n + ia] = sa[j];
      if (has_b) recon[(int64_t)j * n + ib] = sb[j];
    }
  }
}

template <int D, int S>
static cudaError_t run_rvq(const float *x, int64_t n, const int64_t *n_dev, const float *codes,
                           int L, int P, void *idx, int idx_bytes, float *recon, cudaStream_t s) {
  const size_t bytes = (size_t)L * P * D * sizeof(float);
  const int64_t threads = (n + 1) / 2 * S;
  const int64_t blocks = (threads + kRvqThreads - 1) / kRvqThreads;
  if (bytes <= 200 * 1024) {
    if (bytes > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k_rvq<D, S, true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      if (e != cudaSuccess) return e;
    }
    k_rvq<D, S, true><<<(unsigned)blocks, kRvqThreads, bytes, s>>>(x, n, n_dev, codes, L, P, idx,
                                                                  idx_bytes, recon);
  } else {  // codebooks beyond shared memory: read through L1/L2
    k_rvq<D, S, false><<<(unsigned)blocks, kRvqThreads, 0, s>>>(x, n, n_dev, codes, L, P, idx,
                                                              idx_bytes, recon);
  }
  return cudaGetLastError();
}

template <int D>
static cudaError_t run_rvq_d(const float *x, int64_t n, const int64_t *n_dev, const float *codes,
                             int L, int P, void *idx, int idx_bytes, float *recon,
                             cudaStream_t s) {
  if (P >= 16) return run_rvq<D, 4>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
  return run_rvq<D, 1>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
}

cudaError_t launch_rvq(const float *x, int64_t n, const int64_t *n_dev, int d, const float *codes,
                       int L, int P, void *idx, int idx_bytes, float *recon, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  switch (d) {
    case 1: return run_rvq_d<1>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 2: return run_rvq_d<2>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 3: return run_rvq_d<3>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 4: return run_rvq_d<4>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 5: return run_rvq_d<5>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 6: return run_rvq_d<6>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 7: return run_rvq_d<7>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    case 8: return run_rvq_d<8>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace csplat
