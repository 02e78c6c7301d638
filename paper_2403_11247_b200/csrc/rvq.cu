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
constexpr int kRvqVP = 2;  // vector pairs per thread (D <= 4): each 16-byte code load feeds 2 FFMA2 chains

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

// Resolve a block of 4 distances against the running (best, index): only when
// the block's minimum beats the running best (a handful of times per stage)
// is the lowest index of that minimum searched; ties keep the earlier index.
__device__ __forceinline__ void block_argmin4(float d0, float d1, float d2, float d3, int k0,
                                              float &best, int &bk) {
  const float m = fminf(fminf(d0, d1), fminf(d2, d3));  // NaN-ignoring, exact
  if (m < best) {
    best = m;
    bk = d0 == m ? k0 : (d1 == m ? k0 + 1 : (d2 == m ? k0 + 2 : k0 + 3));
  }
}

// Chunked variant: group lane `sub` scans the contiguous code range
// [sub*P/S, (sub+1)*P/S) of every stage (P % (8S) == 0), reading a padded,
// bank-conflict-free shared-memory copy of the codebook with 16-byte loads.
// Each thread carries VP packed vector PAIRS (2 VP vectors), so every code
// loaded from shared memory feeds VP FFMA2 chains (register blocking: the scan
// is bound by shared-memory loads and their latency at VP = 1).
constexpr int kRvqMinB = 3;    // 3 CTAs (24 warps) per SM: 80 registers, a few spills (114.8 vs 121 us)
constexpr int kRvqMinBS2 = 2;  // S = 2 (C2-sized inputs): 128 registers, in-step 106.5 -> 104.4 us
template <int D, int S, int VP>
__global__ void __launch_bounds__(kRvqThreads, S == 2 ? kRvqMinBS2 : kRvqMinB) k_rvq_chunked(
    const float *__restrict__ x, int64_t n, const int64_t *__restrict__ n_dev,
    const float *__restrict__ codes_g, int L, int P, void *__restrict__ idx, int idx_bytes,
    float *__restrict__ recon) {
  extern __shared__ __align__(128) float sc[];
  __shared__ __align__(8) uint64_t bar;
  const int chunk = P / S;                 // codes per lane
  const int cstride = chunk * D + 4;       // padded chunk (floats): distinct banks per lane
  const int lstride = S * cstride;         // one stage
  // stage the codebook with L*S 1-D TMA bulk copies (each chunk is contiguous
  // in global memory), into the padded layout
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    const uint32_t cbytes = (uint32_t)(chunk * D * sizeof(float));
    mbar_arrive_expect_tx(&bar, cbytes * L * S);
    for (int l = 0; l < L; l++)
      for (int s = 0; s < S; s++)
        tma_load_1d(sc + l * lstride + s * cstride, codes_g + ((int64_t)l * P + s * chunk) * D,
                    cbytes, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const int64_t ne = eff_n(n, n_dev);
  const int sub = threadIdx.x % S;
  // vectors i0 + 2v (lo) and i0 + 2v + 1 (hi) of pair v; groups of S lanes share them
  const int64_t i0 = 2 * VP * (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / S);
  // only whole warps may leave (group shuffles need a converged warp); this
  // drops the work of the vectors beyond the device-side count n_dev
  if (__all_sync(0xffffffffu, !(i0 < ne))) return;
  int64_t iv[2 * VP];
  bool has[2 * VP];
  float xv[2 * VP][D], sv[2 * VP][D];
#pragma unroll
  for (int u = 0; u < 2 * VP; u++) {
    has[u] = i0 + u < ne;
    iv[u] = has[u] ? i0 + u : 0;
#pragma unroll
    for (int j = 0; j < D; j++) {
      xv[u][j] = x[(int64_t)j * n + iv[u]];
      sv[u][j] = 0.0f;
    }
  }
  constexpr int kBlk = 8 / VP;  // codes per block (VP * kBlk accumulators in flight)
  for (int l = 0; l < L; l++) {
    f2_t r[VP][D];
#pragma unroll
    for (int v = 0; v < VP; v++)
#pragma unroll
      for (int j = 0; j < D; j++)  // S - S_hat
        r[v][j] = pk2(DSUB(xv[2 * v][j], sv[2 * v][j]), DSUB(xv[2 * v + 1][j], sv[2 * v + 1][j]));
    const float4 *C4 = reinterpret_cast<const float4 *>(sc + l * lstride + sub * cstride);
    const int kbase = sub * chunk;
    float dmin[2 * VP];
    int blk[2 * VP];
    f2_t acc0[VP];
#pragma unroll
    for (int u = 0; u < 2 * VP; u++) {
      dmin[u] = __int_as_float(0x7f800000);  // +inf: NaN distances are never taken
      blk[u] = 0;                            // block (of kBlk codes) of the best
    }
    // distances of the kBlk codes of block i for pair v (bit-identical whenever recomputed)
    auto block_dist = [&](int i, f2_t (&acc)[VP][kBlk]) {
      float cv[kBlk * D];
#pragma unroll
      for (int q = 0; q < kBlk * D / 4; q++) {  // kBlk * D floats as float4 loads
        const float4 t = C4[(i * D) / 4 + q];
        cv[4 * q] = t.x; cv[4 * q + 1] = t.y; cv[4 * q + 2] = t.z; cv[4 * q + 3] = t.w;
      }
#pragma unroll
      for (int c = 0; c < kBlk; c++)
#pragma unroll
        for (int v = 0; v < VP; v++) {
          acc[v][c] = 0ull;  // (+0, +0): fma(e, e, 0) = e*e exactly
#pragma unroll
          for (int j = 0; j < D; j++) {
            const float cf = cv[c * D + j];
            const f2_t e = sub2(pk2(cf, cf), r[v][j]);
            acc[v][c] = fma2(e, e, acc[v][c]);
          }
        }
    };
    // scan: track only the minimum and the block holding its first occurrence
    for (int i = 0; i < chunk; i += kBlk) {
      f2_t acc[VP][kBlk];
      block_dist(i, acc);
#pragma unroll
      for (int v = 0; v < VP; v++) {
        if (i == 0) acc0[v] = acc[v][0];
        float ma = lo2(acc[v][0]), mb = hi2(acc[v][0]);
#pragma unroll
        for (int c = 1; c < kBlk; c++) {
          ma = fminf(ma, lo2(acc[v][c]));
          mb = fminf(mb, hi2(acc[v][c]));
        }
        blk[2 * v] = ma < dmin[2 * v] ? i : blk[2 * v];  // strict: an earlier block keeps a tie
        blk[2 * v + 1] = mb < dmin[2 * v + 1] ? i : blk[2 * v + 1];
        dmin[2 * v] = fminf(dmin[2 * v], ma);
        dmin[2 * v + 1] = fminf(dmin[2 * v + 1], mb);
      }
    }
    // resolve the first code of the winning blocks that attains the minimum:
    // re-evaluate only vector u's pair in its block (bit-identical distances)
    int best[2 * VP];
#pragma unroll
    for (int u = 0; u < 2 * VP; u++) {
      const int v = u >> 1;
      float cv[kBlk * D];
#pragma unroll
      for (int q = 0; q < kBlk * D / 4; q++) {
        const float4 t = C4[(blk[u] * D) / 4 + q];
        cv[4 * q] = t.x; cv[4 * q + 1] = t.y; cv[4 * q + 2] = t.z; cv[4 * q + 3] = t.w;
      }
      best[u] = kbase + blk[u];
#pragma unroll
      for (int c = kBlk - 1; c >= 0; c--) {
        f2_t a = 0ull;
#pragma unroll
        for (int j = 0; j < D; j++) {
          const float cf = cv[c * D + j];
          const f2_t e = sub2(pk2(cf, cf), r[v][j]);
          a = fma2(e, e, a);
        }
        const float d = (u & 1) ? hi2(a) : lo2(a);
        if (d == dmin[u]) best[u] = kbase + blk[u] + c;
      }
    }
#pragma unroll
    for (int u = 0; u < 2 * VP; u++) {
      // the sequential scan keeps k = 0 when d_0 is NaN (no later d compares below it)
      if (sub == 0) {
        const float d0 = (u & 1) ? hi2(acc0[u >> 1]) : lo2(acc0[u >> 1]);
        if (d0 != d0) { dmin[u] = -__int_as_float(0x7f800000); best[u] = 0; }
      }
      group_argmin<S>(dmin[u], best[u]);
      if (sub == 0 && has[u]) {
        if (idx_bytes == 1) static_cast<uint8_t *>(idx)[(int64_t)l * n + iv[u]] = (uint8_t)best[u];
        else static_cast<uint16_t *>(idx)[(int64_t)l * n + iv[u]] = (uint16_t)best[u];
      }
      const float *Cl = sc + l * lstride;
      const int bs = best[u] / chunk, bi = best[u] - bs * chunk;
#pragma unroll
      for (int j = 0; j < D; j++) {  // S_hat^l in stage order
        const float c = Cl[bs * cstride + bi * D + j];
        sv[u][j] = l == 0 ? c : DADD(sv[u][j], c);
      }
    }
  }
  if (recon && sub == 0) {
#pragma unroll
    for (int u = 0; u < 2 * VP; u++)
      if (has[u])
#pragma unroll
        for (int j = 0; j < D; j++) recon[(int64_t)j * n + iv[u]] = sv[u][j];
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

// k_rvq_chunked with S lanes per vector group; false if the shape does not fit
// (P % (8 S), shared memory, 16-byte aligned codebook for the TMA copies)
template <int D, int S>
static bool try_chunked(const float *x, int64_t n, const int64_t *n_dev, const float *codes,
                        int L, int P, void *idx, int idx_bytes, float *recon, cudaStream_t s,
                        cudaError_t &err) {
  constexpr int VP = D <= 4 ? kRvqVP : 1;  // vector pairs per thread
  const size_t chunked_bytes = (size_t)L * S * ((P / S) * D + 4) * sizeof(float);
  if (!(P % (8 * S) == 0 && chunked_bytes <= 200 * 1024 &&
        (reinterpret_cast<uintptr_t>(codes) & 15u) == 0))
    return false;
  if (chunked_bytes > 48 * 1024) {
    err = cudaFuncSetAttribute(k_rvq_chunked<D, S, VP>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chunked_bytes);
    if (err != cudaSuccess) return true;
  }
  const int64_t threads = (n + 2 * VP - 1) / (2 * VP) * S;
  const int64_t blocks = (threads + kRvqThreads - 1) / kRvqThreads;
  k_rvq_chunked<D, S, VP><<<(unsigned)blocks, kRvqThreads, chunked_bytes, s>>>(
      x, n, n_dev, codes, L, P, idx, idx_bytes, recon);
  err = cudaGetLastError();
  return true;
}

// Lanes per vector group: splitting a stage's code scan over S lanes buys
// warps for latency hiding but costs a log2(S)-level merge per vector and
// stage.  Measured (B200, 4 x 256, scale / rotation): at C2's 150k vectors S = 2
// beats S = 4 (50.9 / 60.0 vs 56.4 / 65.9 us) and S = 1 (52.6 / 68.7); at C4's
// 1M, with warps to spare, S = 1 wins (259 / 329 vs 280 / 343 us at S = 2).
constexpr int64_t kRvqS1MinN = 400000;
template <int D>
static cudaError_t run_rvq_d(const float *x, int64_t n, const int64_t *n_dev, const float *codes,
                             int L, int P, void *idx, int idx_bytes, float *recon,
                             cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  if (n >= kRvqS1MinN && try_chunked<D, 1>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s, e))
    return e;
  if (try_chunked<D, 2>(x, n, n_dev, codes, L, P, idx, idx_bytes, recon, s, e)) return e;
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
