// common.cuh -- internal helpers of libcsplat (sm_100a).  Not part of the ABI.
//
// Decision arithmetic (DA): every value that feeds a discrete
// decision is computed with the explicitly rounded intrinsics below, which
// nvcc never contracts into FMAs or reassociates.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "csplat.h"
#include <cuda.h>

namespace csplat {

constexpr int kTile = CSPLAT_TILE;
constexpr int kRecWords = 16;

#define DADD __fadd_rn
#define DSUB __fsub_rn
#define DMUL __fmul_rn
#define DDIV __fdiv_rn
#define DFMA __fmaf_rn
#define DSQRT __fsqrt_rn

// exact 2^k for k in [-126, 127]
__device__ __forceinline__ float da_pow2(int k) { return __int_as_float((k + 127) << 23); }

// DA exp (DESIGN.md §3 "pexp")
__device__ __forceinline__ float da_pexp(float x) {
  x = fminf(fmaxf(x, -86.0f), 88.0f);
  const float k = rintf(DMUL(x, 1.44269504f));
  float r = DFMA(-k, 0.693145751953125f, x);
  r = DFMA(-k, 1.42860677e-06f, r);
  float p = 1.98412698e-4f;
  p = DFMA(p, r, 1.38888889e-3f);
  p = DFMA(p, r, 8.33333333e-3f);
  p = DFMA(p, r, 4.16666667e-2f);
  p = DFMA(p, r, 0.166666667f);
  p = DFMA(p, r, 0.5f);
  p = DFMA(p, r, 1.0f);
  p = DFMA(p, r, 1.0f);
  return DMUL(p, da_pow2((int)k));
}

// DA log for normal positive x (DESIGN.md §3 "plog"); frexp done on the bits.
__device__ __forceinline__ float da_plog(float x) {
  const uint32_t b = __float_as_uint(x);
  int e = (int)((b >> 23) & 0xffu) - 126;
  float m = __uint_as_float((b & 0x807fffffu) | (126u << 23));  // [0.5, 1)
  if (m < 0.707106781f) {
    m = DADD(m, m);
    e = e - 1;
  }
  const float f = DSUB(m, 1.0f);
  const float s = DDIV(f, DADD(2.0f, f));
  const float t = DMUL(s, s);
  float p = DFMA(t, 0.111111111f, 0.142857143f);
  p = DFMA(t, p, 0.2f);
  p = DFMA(t, p, 0.333333333f);
  p = DFMA(t, p, 1.0f);
  const float ef = (float)e;
  return DFMA(ef, 0.693145751953125f, DFMA(ef, 1.42860677e-06f, DMUL(DADD(s, s), p)));
}

__device__ __forceinline__ float da_sigm(float x) {
  return DDIV(1.0f, DADD(1.0f, da_pexp(-x)));
}

// Per-pixel DA q of a record ("per pixel").
__device__ __forceinline__ float da_q(float px, float py, float u, float v, float ca, float cb2,
                                      float cc) {
  const float dx = DSUB(px, u), dy = DSUB(py, v);
  return DFMA(DMUL(ca, dx), dx, DFMA(DMUL(cb2, dx), dy, DMUL(DMUL(cc, dy), dy)));
}

// The DA contribution test 0 <= q <= k2 as ONE unsigned
// compare of the bit patterns: for k2 >= +0 finite, non-negative floats order
// like their bits, a negative q or a NaN has bits above k2's, and the DA q is
// never -0 (its last term (cc dy) dy is >= +0 and an exact-zero sum rounds to
// +0), so this equals the two float comparisons bit for bit.
__device__ __forceinline__ bool da_in_range(float q, float k2) {
  return __float_as_uint(q) <= __float_as_uint(k2);
}

__device__ __forceinline__ int64_t eff_n(int64_t n, const int64_t *n_dev) {
  if (!n_dev) return n;
  const int64_t m = *n_dev;
  return m < n ? (m < 0 ? 0 : m) : n;
}

// --- Blackwell async-copy plumbing (TMA bulk copies + mbarriers) ----------

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint: the waiting warp is parked (it resumes when
// the phase completes or after ~ns) instead of re-issuing the probe, so a warp
// blocked on a slow partner does not take issue slots from the working warps.
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t *bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}
constexpr uint32_t kMbarSleepNs = 20000;  // suspend-time hint (an upper bound)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait_hint(bar, parity, kMbarSleepNs)) {
  }
}
// 1-D TMA bulk copy global -> shared, completion signalled on `bar`.
__device__ __forceinline__ void tma_load_1d(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// generic-proxy shared-memory writes ordered before later async-proxy (TMA)
// accesses of the same locations
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}


// pair_gid entries: the Gaussian index in bits 0-27, the pair's 8x8-block
// cull mask (block_mask) in bits 28-31 (csplat.h, csplat_bin_tiles)
constexpr int kPairMaskShift = 28;
constexpr uint32_t kPairGidMask = (1u << kPairMaskShift) - 1u;

// The record table as a 2-D TMA tensor for tile::gather4 loads: rows of 16
// u32 words (one 64-byte record per Gaussian), 2^28 rows (every index a pair
// entry can name; the entries only name Gaussians < n), box = 16 x 1.  Encoded
// on the host per call (rec_tensor_map, record_tmap.cu).
cudaError_t rec_tensor_map(const void *rec, CUtensorMap *out);

// The renderers' producer warp, one batch of a tile's list into ring slot
// `slot` (128-byte aligned): lane l holds entry l (Gaussian index | block mask
// << 28) and stores its mask into msk[l]; lanes j < ceil(cnt / 4) each gather
// the records of entries 4j .. 4j+3 with one tile::gather4 TMA load (4 rows x
// 64 B, rows past the batch repeat its last entry); all 32 lanes arrive on
// `full` (init count 32; lane 0 arms it with the bytes), so the phase
// completes once every mask is stored and every record has landed.
__device__ __forceinline__ void gather_batch(float4 *slot, uint32_t *msk, const CUtensorMap *tmap,
                                             uint32_t entry, int lane, int cnt, uint64_t *full) {
  const int last = cnt - 1;
  const uint32_t gid = entry & kPairGidMask;
  uint32_t r[4];
#pragma unroll
  for (int q = 0; q < 4; q++) r[q] = __shfl_sync(0xffffffffu, gid, min(4 * (lane & 7) + q, last));
  const int nreq = (cnt + 3) >> 2;
  if (lane < cnt) msk[lane] = entry >> kPairMaskShift;
  if (lane < nreq) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(slot + lane * 16)),
        "l"(tmap), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(smem_u32(full))
        : "memory");
  }
  if (lane == 0) mbar_arrive_expect_tx(full, (uint32_t)nreq * 4u * CSPLAT_RECORD_BYTES);
  else mbar_arrive(full);
}

__device__ __forceinline__ void red_add_v4(float *addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

// Packed float32 pairs (PTX .f32x2 -> FADD2/FMUL2/FFMA2 on sm_100a): each lane
// of the pair is an IEEE round-to-nearest operation, bit-identical to the
// scalar __f*_rn form; one issue slot does both.
typedef unsigned long long f2_t;  // lo = first lane, hi = second lane

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
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// --- host-side launchers (defined in the .cu files) -------------------------

struct CamInfo {
  int W, H, tiles_x, tiles_y;
};
inline CamInfo cam_info(const csplat_camera &c) {
  CamInfo i;
  i.W = c.width;
  i.H = c.height;
  i.tiles_x = (c.width + kTile - 1) / kTile;
  i.tiles_y = (c.height + kTile - 1) / kTile;
  return i;
}

struct DecodeArgs {
  int L, P, idx_bytes;
  const float *scale_codes, *rot_codes;
  const void *scale_idx, *rot_idx;
  uint32_t *status;  // optional: CSPLAT_STATUS_CODE_INDEX is OR-ed in (csplat.h)
};

__device__ __forceinline__ uint32_t load_rvq_idx(const void *p, int bytes, int64_t off) {
  return bytes == 1 ? (uint32_t)__ldg((const uint8_t *)p + off)
                    : (uint32_t)__ldg((const uint16_t *)p + off);
}

// a Gaussian with a codebook index >= P is culled (its decoded
// log-scale becomes NaN, which the projection's non-finite test culls, as
// the oracle does) and the codebook's status word gets CSPLAT_STATUS_CODE_INDEX;
// the gathers use a clamped index so nothing is read outside the codebook.
// Only a live Gaussian (i < n, mask on: `report`) sets the bit; index planes
// beyond the live count may hold anything.
__device__ __forceinline__ void rvq_flag_bad(const DecodeArgs &dec, bool bad, bool report,
                                             float (&ls)[3]) {
  if (bad) {
    ls[0] = __int_as_float(0x7fc00000);
    if (report && dec.status) atomicOr(dec.status, CSPLAT_STATUS_CODE_INDEX);
  }
}

// Eq 10 decode (R17, R20): S_hat^L = sum_l C^l[i^l], summed in stage order, of
// Gaussian i's log-scale and quaternion.  LF > 0 = the stage count known at
// compile time: all 2 LF index loads are issued first, then all code gathers,
// so a thread waits for two memory round trips instead of 2 L dependent ones.
template <int LF>
__device__ __forceinline__ void rvq_decode(const DecodeArgs &dec, int64_t n, int64_t i,
                                           float (&ls)[3], float (&qv)[4], bool report) {
  const float4 *rot4 = reinterpret_cast<const float4 *>(dec.rot_codes);
  const uint32_t Pm1 = (uint32_t)(dec.P - 1);
  if constexpr (LF > 0) {
    uint32_t si[LF], ri[LF];
#pragma unroll
    for (int l = 0; l < LF; l++) {
      si[l] = load_rvq_idx(dec.scale_idx, dec.idx_bytes, (int64_t)l * n + i);
      ri[l] = load_rvq_idx(dec.rot_idx, dec.idx_bytes, (int64_t)l * n + i);
    }
    uint32_t mx = 0;
#pragma unroll
    for (int l = 0; l < LF; l++) mx = max(mx, max(si[l], ri[l]));
    float s[LF][3];
    float4 r[LF];
#pragma unroll
    for (int l = 0; l < LF; l++) {
      const float *sc = dec.scale_codes + ((int64_t)l * dec.P + min(si[l], Pm1)) * 3;
      s[l][0] = __ldg(sc); s[l][1] = __ldg(sc + 1); s[l][2] = __ldg(sc + 2);
      r[l] = __ldg(rot4 + ((int64_t)l * dec.P + min(ri[l], Pm1)));
    }
    ls[0] = s[0][0]; ls[1] = s[0][1]; ls[2] = s[0][2];
    qv[0] = r[0].x; qv[1] = r[0].y; qv[2] = r[0].z; qv[3] = r[0].w;
#pragma unroll
    for (int l = 1; l < LF; l++) {
      ls[0] = DADD(ls[0], s[l][0]); ls[1] = DADD(ls[1], s[l][1]); ls[2] = DADD(ls[2], s[l][2]);
      qv[0] = DADD(qv[0], r[l].x); qv[1] = DADD(qv[1], r[l].y);
      qv[2] = DADD(qv[2], r[l].z); qv[3] = DADD(qv[3], r[l].w);
    }
    rvq_flag_bad(dec, mx > Pm1, report, ls);
  } else {
    bool bad = false;
    for (int l = 0; l < dec.L; l++) {
      const uint32_t si = load_rvq_idx(dec.scale_idx, dec.idx_bytes, (int64_t)l * n + i);
      const uint32_t ri = load_rvq_idx(dec.rot_idx, dec.idx_bytes, (int64_t)l * n + i);
      bad |= (si > Pm1) | (ri > Pm1);
      const float *sc = dec.scale_codes + ((int64_t)l * dec.P + min(si, Pm1)) * 3;
      const float4 rc = __ldg(rot4 + ((int64_t)l * dec.P + min(ri, Pm1)));
      const float s0 = __ldg(sc), s1 = __ldg(sc + 1), s2 = __ldg(sc + 2);
      if (l == 0) {
        ls[0] = s0; ls[1] = s1; ls[2] = s2;
        qv[0] = rc.x; qv[1] = rc.y; qv[2] = rc.z; qv[3] = rc.w;
      } else {
        ls[0] = DADD(ls[0], s0); ls[1] = DADD(ls[1], s1); ls[2] = DADD(ls[2], s2);
        qv[0] = DADD(qv[0], rc.x); qv[1] = DADD(qv[1], rc.y);
        qv[2] = DADD(qv[2], rc.z); qv[3] = DADD(qv[3], rc.w);
      }
    }
    rvq_flag_bad(dec, bad, report, ls);
  }
}

// the compile-time stage count for rvq_decode (0 = a runtime loop)
inline int rvq_lf(const DecodeArgs *dec) {
  return dec ? (dec->L == 4 ? 4 : (dec->L == 2 ? 2 : 0)) : 0;
}

cudaError_t launch_project(const csplat_gaussians &g, const DecodeArgs *dec,
                           const csplat_camera &cam, const csplat_view &view,
                           const float *view_dev, float tau, float dilation, void *rec,
                           int32_t *count, cudaStream_t s);

// csplat_project_bin: the projection with the bucket pass fused in, then the
// per-tile sort (same outputs as launch_project + launch_bin)
cudaError_t launch_project_bin(const csplat_gaussians &g, const DecodeArgs *dec,
                               const csplat_camera &cam, const csplat_view &view,
                               const float *view_dev, float tau, float dilation, void *rec,
                               int32_t *count, int64_t cap, const uint32_t *tile_active,
                               uint32_t *pair_gid, uint32_t *tile_range,
                               int64_t *n_pairs_dev, void *ws, cudaStream_t s);

size_t bin_workspace_bytes(int64_t n, int64_t cap, const csplat_camera &cam);
// Cull hint for the renderers: bit w (w = 0..3, x half = w & 1, y half = w >> 1)
// of a (tile, Gaussian) pair's block mask is set unless the Gaussian provably has
// alpha < 1/255 over the whole 8x8 pixel block w of the tile, i.e. unless the
// minimum of q(dx, dy) = ca dx^2 + (2cb) dx dy + cc dy^2 over the block's
// rectangle exceeds k^2 by more than a rounding margin (the renderers skip a
// pixel when q > k^2).  The minimum of the convex q over a box
// that does not contain the centre lies on a box edge that faces the centre,
// so at most two 1-D clamped minimisations per block.  The margin covers the
// float32 evaluation of q at any pixel of the block, so a
// cleared bit never skips a pixel the per-pixel test would have composited.
// The conic, extent and edge slopes of one (tile, Gaussian) pair's box tests
// (the bucket pass fills it from the owner lane's PairSrc, bin_dev.cuh).
struct BoxConic {
  float u, v, ca, cb2, cc, k2, sx, sy;
  int rx0, ry0, rx1, ry1;
  bool conic_ok;
};
// The mask over a tile's four 8x8 blocks, branch-free (the bucket pass runs it
// for 32 different pairs per warp, where per-block branches diverge).
// Per block: the rectangle cull, then the minimum of q over the block (0 when
// the block holds the centre, else the clamped minimisations on the one or two
// edges facing the centre, the edge offsets shared between the blocks and both
// probes evaluated and selected), kept unless it exceeds k^2 + margin.  The
// edge slopes sx, sy: on a vertical edge at dx = e the convex q is least at
// dy = -cb2 e / (2 cc) (horizontal edges alike); any rounding of this location
// only moves the probe along the edge, which can raise q by at most
// cc (location error)^2 -- far below the margin.
__device__ __forceinline__ uint32_t block_mask_c(const BoxConic &c, int X0, int Y0) {
  const float inf = __int_as_float(0x7f800000);
  float ex[4], ey[4];  // offsets of the block edges X0, X0+7, X0+8, X0+15 (y alike)
#pragma unroll
  for (int e = 0; e < 4; e++) {
    ex[e] = (float)(X0 + (e >> 1) * 8 + (e & 1) * 7) - c.u;
    ey[e] = (float)(Y0 + (e >> 1) * 8 + (e & 1) * 7) - c.v;
  }
  uint32_t m = 0;
#pragma unroll
  for (int w = 0; w < 4; w++) {
    const int hx = w & 1, hy = w >> 1;
    const int bx0 = X0 + hx * 8, by0 = Y0 + hy * 8;
    const bool rect = !(c.rx1 < bx0 || c.rx0 > bx0 + 7 || c.ry1 < by0 || c.ry0 > by0 + 7);
    const float dx0 = ex[2 * hx], dx1 = ex[2 * hx + 1];
    const float dy0 = ey[2 * hy], dy1 = ey[2 * hy + 1];
    const bool ox = dx0 > 0.0f || dx1 < 0.0f, oy = dy0 > 0.0f || dy1 < 0.0f;
    // near vertical edge, dy clamped to the block
    const float exn = dx0 > 0.0f ? dx0 : dx1;
    const float dyv = fminf(fmaxf(c.sy * exn, dy0), dy1);
    const float qv = c.ca * exn * exn + c.cb2 * exn * dyv + c.cc * dyv * dyv;
    // near horizontal edge
    const float eyn = dy0 > 0.0f ? dy0 : dy1;
    const float dxh = fminf(fmaxf(c.sx * eyn, dx0), dx1);
    const float qh = c.ca * dxh * dxh + c.cb2 * dxh * eyn + c.cc * eyn * eyn;
    const float qmin = (ox || oy) ? fminf(ox ? qv : inf, oy ? qh : inf) : 0.0f;
    const float DX = fmaxf(fabsf(dx0), fabsf(dx1)), DY = fmaxf(fabsf(dy0), fabsf(dy1));
    const float margin = 0.01f + 2e-5f * (c.ca * DX * DX + fabsf(c.cb2) * DX * DY + c.cc * DY * DY);
    const bool hit = rect && (!c.conic_ok || !(qmin > c.k2 + margin));  // NaN keeps the block
    m |= hit ? 1u << w : 0u;
  }
  return m;
}
// NEXT-2 (rvq_update.cu): the STE code gradient and the Fig 4 stage init
cudaError_t launch_rvq_code_grad(const float *g, int64_t n, const int64_t *n_dev, int d, int L,
                                 int P, const void *idx, int idx_bytes, float *dcodes,
                                 bool accumulate, cudaStream_t s);
cudaError_t launch_rvq_init_stage(const float *x, int64_t n, int d, float *codes, int P, int l,
                                  const void *idx, int idx_bytes, const int64_t *sample,
                                  cudaStream_t s);
// multi-view (SURVEY §8(e) window): projection (+ bucket + batched sort) of nv
// views reading each Gaussian once (project.cu), the chain summed over views
// (chain.cu)
cudaError_t launch_project_views(const csplat_gaussians &g, const DecodeArgs *dec,
                                 const csplat_camera &cam, const csplat_view *views, int nv,
                                 float tau, float dilation, void *rec, int32_t *count,
                                 void *ws, int64_t ws_stride, int64_t cap,
                                 const uint32_t *active, int64_t active_stride,
                                 uint32_t *pair_gid, uint32_t *tile_range, int64_t *n_pairs_dev,
                                 const int32_t *tile_lists, int64_t list_stride, int max_list,
                                 cudaStream_t s);
cudaError_t launch_chain_views(const csplat_gaussians &g, const DecodeArgs *dec,
                               const csplat_camera &cam, const csplat_view *views, int nv,
                               const csplat_params &prm, const void *rec, void *ws,
                               uint32_t flags, const csplat_grads &out, cudaStream_t s);
// the calling thread's fork streams / events of the composed calls (project.cu)
void release_thread_fork_resources();
cudaError_t launch_bin(const void *rec, const int32_t *count, int64_t n, const csplat_camera &cam,
                       int64_t cap, const uint32_t *tile_active, uint32_t *pair_gid, uint32_t *tile_range, int64_t *n_pairs_dev, void *ws,
                       cudaStream_t s);

cudaError_t launch_pose_step(float *view_dev, const float *pose_grad, float lr_rot,
                             float lr_trans, cudaStream_t s);

cudaError_t launch_ba_patches(const float *obs_depth, const csplat_camera &cam,
                              const int32_t *patches, int64_t n_patches, uint32_t *tile_active,
                              unsigned long long *n_valid, cudaStream_t s);
cudaError_t launch_ba_loss(const float *color, const float *depth, const float *obs_color,
                           const float *obs_depth, const csplat_camera &cam,
                           const int32_t *patches, int64_t n_patches, int64_t n_rays,
                           const unsigned long long *n_valid, float lambda_d, float lambda_s,
                           float *d_color, float *d_depth, float *d_sil, float *loss3,
                           cudaStream_t s);

// tiles [tile0, tile0 + ntiles) only (ntiles < 0: to the last tile)
cudaError_t launch_render_fwd(const void *rec, const uint32_t *pair_gid,
                              const uint32_t *tile_range,
                              const csplat_camera &cam, const csplat_params &prm, float *color,
                              float *depth, float *sil, float *t_final, int32_t *n_contrib,
                              cudaStream_t s, int tile0 = 0, int ntiles = -1,
                              const int32_t *list = nullptr);

// csplat_project_bin_render: projection + bucket, then the per-tile sort and
// the forward in tile chunks, the sort of chunk c+1 overlapping the forward
// of chunk c on two library streams forked from / joined into s
cudaError_t launch_project_bin_render(const csplat_gaussians &g, const DecodeArgs *dec,
                                      const csplat_camera &cam, const csplat_view &view,
                                      const float *view_dev, float tau, float dilation,
                                      const csplat_params &prm, void *rec, int32_t *count,
                                      int64_t cap, uint32_t *pair_gid,
                                      uint32_t *tile_range, int64_t *n_pairs_dev, void *ws,
                                      float *color, float *depth, float *sil, float *t_final,
                                      int32_t *n_contrib, cudaStream_t s);

size_t bwd_workspace_bytes(int64_t n);
// the render_bwd workspace's bitmap of Gaussians that received partials
uint32_t *bwd_alive_bits(void *ws, int64_t n);
struct TrackingLoss;
cudaError_t bwd_prep(const csplat_gaussians &g, uint32_t flags, const csplat_grads &out,
                     void *ws, const TrackingLoss *loss, cudaStream_t s);
cudaError_t launch_render_bwd_tiles(const csplat_camera &cam, const TrackingLoss *loss,
                                    const csplat_params &prm, const void *rec,
                                    const uint32_t *pair_gid, const uint32_t *tile_range, const float *t_final,
                                    const int32_t *n_contrib, const float *d_color,
                                    const float *d_depth, const float *d_sil, void *ws,
                                    int64_t n, cudaStream_t s, int tile0, int ntiles,
                                    const int32_t *list = nullptr);

// csplat_render_step: a3 .. a8 for one view -- projection + bucket, then per
// tile chunk (on its own library stream) the sort, the forward and the
// backward kernel, joined, then the per-Gaussian chain
struct StepBwd {
  const float *d_color, *d_depth, *d_sil;  // upstream (loss == nullptr)
  uint32_t flags;
  csplat_grads out;
  void *ws;
  const TrackingLoss *loss;                // NEXT-1: upstream formed in the backward
};
cudaError_t launch_render_step(const csplat_gaussians &g, const DecodeArgs *dec,
                               const csplat_camera &cam, const csplat_view &view,
                               const float *view_dev, float tau, float dilation,
                               const csplat_params &prm, void *rec, int32_t *count, int64_t cap,
                               uint32_t *pair_gid, uint32_t *tile_range,
                               int64_t *n_pairs_dev, void *ws, float *color, float *depth,
                               float *sil, float *t_final, int32_t *n_contrib,
                               const StepBwd *bwd, cudaStream_t s);
cudaError_t launch_chain(const csplat_gaussians &g, const DecodeArgs *dec,
                         const csplat_camera &cam, const csplat_view &view,
                         const float *view_dev, const csplat_params &prm, const void *rec,
                         const float *acc, uint32_t flags, const csplat_grads &out,
                         cudaStream_t s);
struct TrackingLoss {  // NEXT-1 loss-fused backward (render_bwd.cu)
  const float *color, *depth, *sil, *obs_color, *obs_depth;
  const unsigned long long *n_valid;
  float lambda_d, gate;
  float *loss3;
};
cudaError_t launch_count_valid(const float *obs_depth, int64_t HW, unsigned long long *n_valid,
                               cudaStream_t s);
cudaError_t launch_render_bwd(const csplat_gaussians &g, const DecodeArgs *dec,
                              const csplat_camera &cam, const csplat_view &view,
                              const float *view_dev, const TrackingLoss *loss,
                              const csplat_params &prm, const void *rec, const uint32_t *pair_gid,
                              const uint32_t *tile_range, const float *t_final,
                              const int32_t *n_contrib, const float *d_color, const float *d_depth,
                              const float *d_sil, uint32_t flags, const csplat_grads &out,
                              void *ws, cudaStream_t s, const int32_t *list = nullptr,
                              int max_tiles = 0);

cudaError_t launch_rvq(const float *x, int64_t n, const int64_t *n_dev, int d, const float *codes,
                       int L, int P, void *idx, int idx_bytes, float *recon, cudaStream_t s);

cudaError_t launch_tracking_loss(const float *color, const float *depth, const float *sil,
                                 const float *obs_color, const float *obs_depth, int W, int H,
                                 float lambda_d, float gate, float *d_color, float *d_depth,
                                 float *d_sil, float *loss3, void *ws, cudaStream_t s);

cudaError_t launch_mask_loss(int64_t n, const int64_t *n_dev, const float *mask,
                             const int32_t *count, float lambda, float *d_mask, float *loss,
                             void *ws, cudaStream_t s);
cudaError_t launch_overlap(const float *depth, const csplat_camera &cam, const csplat_view &cur,
                           const float *views_dev, int K, unsigned long long *counts,
                           cudaStream_t s);

size_t rvq_update_workspace_bytes(int L, int P, int d);
cudaError_t launch_rvq_update(const float *x, int64_t n, const int64_t *n_dev, int d,
                              const float *codes, int L, int P, const void *idx, int idx_bytes,
                              float *codes_out, int32_t *counts_out, float *loss_out, void *ws,
                              cudaStream_t s);

size_t prune_workspace_bytes(int64_t n);
cudaError_t launch_prune(const csplat_gaussians &in, const DecodeArgs *idx, float tau,
                         float reset, const csplat_gaussians_out &out, void *out_sidx,
                         void *out_ridx, int32_t *keep_map, int64_t *n_kept, void *ws,
                         cudaStream_t s);

}  // namespace csplat
