// quad.cuh -- the per-4x4-block entry lists and the replay of the block-list
// backward (k_render_bwd_quad, render_bwd.cu).
//
// A CTA of two warps takes one 16x16 tile.  Its sixteen 4x4 pixel blocks each
// get their own list of the tile's entries; the four lanes of a QUAD (lane / 4
// of a warp) own one block (quad lane q: column q of the block, i.e. two
// vertically adjacent pixel pairs) and walk its list.  An entry is listed for a
// block when the record's pixel rectangle (the k^2-ellipse's bounding box, §4)
// overlaps the block and the 8x8 block around it has its bit in the pair entry
// (block_mask_c, the bucket pass's conservative ellipse test): a superset of the
// entries any of the block's pixels composites, so skipping the others is
// result-invariant.  The tile list is taken in chunks of kChunk entries.
#pragma once
#include "common.cuh"

namespace csplat {

constexpr int kAcc = 12;          // backward accumulator floats per Gaussian
constexpr int kV = 10;            // backward partials per (pixel, entry)

__device__ __forceinline__ float ex2_approx_b(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

namespace quad {

constexpr int kPW = 2;                    // warps per CTA (16x8 pixels each)
constexpr int kThreads = kPW * 32;
constexpr int kNB = 16;                   // 4x4 blocks (quads) per tile
constexpr int kChunk = 256;               // list entries per gather

struct Lists {
  float4 rec[kChunk + 1][4];              // the chunk's records (+ a zero record)
  uint16_t m16[kChunk];                   // the entries' 4x4-block masks
  uint32_t bits[kNB][kChunk / 32];        // per block: its entries as bit words
  uint8_t lst[kNB][kChunk];               // per block: its entries (chunk index)
  int nitems[kNB];
};

// quad geometry of a lane: block B = qy * 4 + qx of the tile, its pixel column
// px and its first pixel row by
struct Geo {
  int r, ri, B, px, by;
};
__device__ __forceinline__ Geo geo(int tx, int ty, int wid, int lane) {
  Geo g;
  g.r = lane >> 2;
  g.ri = lane & 3;
  g.B = wid * 8 + g.r;
  g.px = tx * kTile + (g.r & 3) * 4 + g.ri;
  g.by = ty * kTile + wid * 8 + (g.r >> 2) * 4;
  return g;
}

// the 4x4 blocks (bit qy * 4 + qx) the record's pixel rectangle (word 12-13)
// overlaps, inside the 8x8 blocks flagged in the pair entry
__device__ __forceinline__ uint32_t mask16(uint32_t entry, const uint4 &w3, int X0, int Y0) {
  const int rx0 = (int)(w3.x & 0xffffu) - X0, ry0 = (int)(w3.x >> 16) - Y0;
  const int rx1 = (int)(w3.y & 0xffffu) - X0, ry1 = (int)(w3.y >> 16) - Y0;
  const int cx0 = max(rx0, 0) >> 2, cx1 = min(rx1, kTile - 1) >> 2;
  const int cy0 = max(ry0, 0) >> 2, cy1 = min(ry1, kTile - 1) >> 2;
  if (cx0 > cx1 || cy0 > cy1) return 0u;
  const uint32_t cols = (0xfu >> (3 - cx1)) & (0xfu << cx0);
  // bit 4 qy for the block rows cy0 <= qy <= cy1
  const uint32_t rowspread = (0x1111u >> (12 - 4 * cy1)) & (0x1111u << (4 * cy0));
  const uint32_t m8 = entry >> kPairMaskShift;
  const uint32_t m8x = ((m8 & 1u) ? 0x0033u : 0u) | ((m8 & 2u) ? 0x00ccu : 0u) |
                       ((m8 & 4u) ? 0x3300u : 0u) | ((m8 & 8u) ? 0xcc00u : 0u);
  return cols * rowspread & m8x;
}

// the 4x4 blocks of m whose pixels the record's k^2-ellipse can reach: per
// band of block rows the ellipse's x-extent over the band, from the concave
// right boundary x_r(dy) = (-cb2 dy + sqrt(4 ca K - det dy^2)) / (2 ca) at the
// clamp of its maximiser (the ellipse's rightmost point; the convex left
// boundary alike), with K = k^2 + the 8x8 mask's margin over the whole tile
// (so the float q <= k^2 test of any kept pixel lies inside),
// the band widened by 0.25 px and the extent by 0.25 px + 0.2% against the
// float evaluation here.  A dropped (block, entry) has q > k^2 at every pixel
// of the block: its replay would change no state and add exact zeros.  Records
// whose conic is not clearly positive definite keep m.
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t ellipse16(uint32_t m, const float4 &a0, const float4 &a1,
                                              int X0, int Y0) {
  const float u = a0.x, v = a0.y, ca = a0.z, cb2 = a0.w, cc = a1.x;
  const float det = 4.0f * ca * cc - cb2 * cb2;
  const float DX = fmaxf(fabsf((float)X0 - u), fabsf((float)(X0 + kTile - 1) - u));
  const float DY = fmaxf(fabsf((float)Y0 - v), fabsf((float)(Y0 + kTile - 1) - v));
  const float K = a1.z + 0.01f + 2e-5f * (ca * DX * DX + fabsf(cb2) * DX * DY + cc * DY * DY);
  const bool ok = ca > 0.0f && cc > 0.0f && det > 4e-3f * ca * cc && K < 3.0e38f;
  const float rdet = rcp_approx(fmaxf(det, 1e-30f));
  const float ye = sqrt_approx(4.0f * ca * K * rdet), xe = sqrt_approx(4.0f * cc * K * rdet);
  const float dyr = -cb2 * xe * rcp_approx(2.0f * cc);  // dy of the rightmost point (leftmost: -dyr)
  const float i2a = rcp_approx(2.0f * ca), fourcak = 4.0f * ca * K;
  const float sx = 0.25f + 2e-3f * xe;
  const float cu = (u - (float)X0) * 0.25f;
  uint32_t out = 0;
#pragma unroll
  for (int qy = 0; qy < 4; qy++) {
    const float y0 = (float)(Y0 + 4 * qy) - v - 0.25f, y1 = y0 + 3.5f;
    const float a = fmaxf(y0, -ye), b = fminf(y1, ye);
    const float dR = fminf(fmaxf(dyr, a), b), dL = fminf(fmaxf(-dyr, a), b);
    const float sR = sqrt_approx(fmaxf(fourcak - det * dR * dR, 0.0f));
    const float sL = sqrt_approx(fmaxf(fourcak - det * dL * dL, 0.0f));
    const float xR = (sR - cb2 * dR) * i2a + sx, xL = (-sL - cb2 * dL) * i2a - sx;
    // the band's block columns qx with X0 + 4 qx - u <= xR and X0 + 4 qx + 3 - u
    // >= xL, as an integer range (widened by 1e-3 block against the rounding
    // of the scaled bounds: a superset of the per-column tests)
    const int hiq = min(__float2int_rd(fmaf(xR, 0.25f, cu) + 1e-3f), 3);
    const int loq = max(__float2int_ru(fmaf(xL, 0.25f, cu - 0.75f) - 1e-3f), 0);
    const uint32_t cols = (loq <= hiq && a <= b) ? (0xfu >> (3 - hiq)) & (0xfu << loq) : 0u;
    out |= cols << (4 * qy);
  }
  return ok ? (m & out) : m;
}

// the chunk [c0, c0 + len) of the tile list starting at `start`: records to
// L.rec (cp.async, no register staging), 4x4 masks to L.m16, and (backward)
// the reached-Gaussian bits.  Ends with a CTA barrier.
// need8: the 8x8 blocks some pixel of which still needs entries (entries whose
// pair-entry mask misses all of them are not copied: their m16 is 0)
__device__ __forceinline__ void gather(Lists &L, const float4 *__restrict__ recs,
                                       const uint32_t *__restrict__ pair_gid, uint32_t start,
                                       int c0, int len, int X0, int Y0,
                                       uint32_t *__restrict__ alive, int tid,
                                       uint32_t need8 = 0xfu) {
  constexpr int kPer = kChunk / kThreads;
  uint32_t ent[kPer];
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    const int i = tid + k * kThreads;
    ent[k] = i < len ? pair_gid[start + c0 + i] : 0u;
  }
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    const int i = tid + k * kThreads;
    if (i >= len || !((ent[k] >> kPairMaskShift) & need8)) continue;
    const float4 *src = recs + (size_t)(ent[k] & kPairGidMask) * 4;
#pragma unroll
    for (int q = 0; q < 4; q++)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&L.rec[i][q])),
                   "l"(src + q)
                   : "memory");
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
  if (tid < 4) L.rec[kChunk][tid] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    const int i = tid + k * kThreads;
    if (i >= len) continue;
    uint32_t m = 0;
    if ((ent[k] >> kPairMaskShift) & need8) {
      const uint4 w3 = *reinterpret_cast<const uint4 *>(&L.rec[i][3]);
      m = mask16(ent[k], w3, X0, Y0);
      m = ellipse16(m, L.rec[i][0], L.rec[i][1], X0, Y0);
    }
    L.m16[i] = (uint16_t)m;
    if (alive && m) {
      const uint32_t gid = ent[k] & kPairGidMask;
      atomicOr(alive + (gid >> 5), 1u << (gid & 31));  // the chain visits this Gaussian
    }
  }
  __syncthreads();
}

// the warp's eight blocks' lists from L.m16 (after gather), in the backward's
// replay order (descending chunk index); entries at list position >= lim[B]
// are left out (a block whose pixels all finished before an entry has nothing
// to replay).  Two steps: (1) per 32 entries one ballot per block gives the
// block's bit word (lane rr keeps block rr's); (2) each quad compacts its own
// block's words -- lane q the words 2q, 2q + 1, at the offset of the set bits
// in the higher words (a suffix sum over the quad) -- highest bit first.
// (The one-pass form -- a ballot + popc prefix + shuffled running count per
// block and 32 entries -- spent 12 % of the kernel's warp samples here; the
// C2 kernel time did not change, the C3 tracking iteration 0.160 -> 0.158 ms.)
__device__ __forceinline__ void build_lists(Lists &L, int c0, int len, const int *lim, int wid,
                                            int lane) {
  const int nw = (len + 31) >> 5;
  for (int k = 0; k < nw; k++) {
    const int i = 32 * k + lane;
    const uint32_t m = i < len ? (uint32_t)L.m16[i] >> (wid * 8) : 0u;
    uint32_t mine = 0;
#pragma unroll
    for (int rr = 0; rr < 8; rr++) {
      const uint32_t bal = __ballot_sync(0xffffffffu, (m >> rr) & 1u);
      mine = lane == rr ? bal : mine;
    }
    if (lane < 8) L.bits[wid * 8 + lane][k] = mine;
  }
  __syncwarp();
  const int ri = lane & 3, B = wid * 8 + (lane >> 2);
  const int s = min(len, lim[B] - c0);  // the block's entries are i < s
  uint32_t w[2];
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int k = 2 * ri + h, rem = s - 32 * k;
    w[h] = rem <= 0 ? 0u : (rem >= 32 ? L.bits[B][k] : L.bits[B][k] & ((1u << rem) - 1u));
  }
  const int c = __popc(w[0]) + __popc(w[1]);
  int suf = c;  // the set bits in this lane's and the higher lanes' words
  int t = __shfl_down_sync(0xffffffffu, suf, 1);
  if (ri < 3) suf += t;
  t = __shfl_down_sync(0xffffffffu, suf, 2);
  if (ri < 2) suf += t;
  int pos = suf - c;
  uint8_t *lst = L.lst[B];
#pragma unroll
  for (int h = 1; h >= 0; h--) {
    uint32_t x = w[h];
    const int base = 32 * (2 * ri + h);
    while (x) {
      const int b = 31 - __clz(x);
      x ^= 1u << b;
      lst[pos++] = (uint8_t)(base + b);
    }
  }
  if (ri == 0) L.nitems[B] = suf;
  __syncwarp();
}

// ---- the replay (render_bwd.cu's header comment): quad lane q's two pixel
// pairs, the per-entry pieces, the quad reduction, and one chunk's walk
// one pixel pair's replay state and upstream (registers of its lane)
struct QPair {
  f2_t T, B, FPY, GR, GG, GB, GD, GS;
  int last0, last1;
};

// a pixel pair's partial terms of one entry (f32x2, summed over the quad's pixels)
struct QTerms {
  f2_t AV, TT, T2, GDL, WD, WR, WG, WB;
};

// one entry at one pixel pair in two pieces, so two entries can interleave: the front (q, the
// validity, G, alpha, 1 / (1 - alpha), v -- independent of the replay state)
// and the state update with the partial terms
struct QFront {
  f2_t DY, G, AL, RC, VV;
  bool nc0, nc1;
};
__device__ __forceinline__ QFront pair_front(const QPair &P, int j, float dx, float cadx,
                                             float cbdx, const float4 &r0, const float4 &r1,
                                             const float4 &r2, float amax) {
  QFront f;
  f.DY = sub2(P.FPY, pk2(r0.y, r0.y));
  const f2_t Y = mul2(mul2(pk2(r1.x, r1.x), f.DY), f.DY);
  const f2_t X = fma2(pk2(cbdx, cbdx), f.DY, Y);
  const f2_t Q = fma2(pk2(cadx, cadx), pk2(dx, dx), X);
  const float q0 = lo2(Q), q1 = hi2(Q);
  const bool val0 = (j < P.last0) & da_in_range(q0, r1.z);
  const bool val1 = (j < P.last1) & da_in_range(q1, r1.z);
  const f2_t QM = pk2(val0 ? q0 : __int_as_float(0x7f800000), val1 ? q1 : __int_as_float(0x7f800000));
  const f2_t QE = mul2(QM, pk2(-0.72134752f, -0.72134752f));
  f.G = pk2(ex2_approx_b(lo2(QE)), ex2_approx_b(hi2(QE)));
  const f2_t AR = mul2(pk2(r1.y, r1.y), f.G);
  f.AL = pk2(fminf(amax, lo2(AR)), fminf(amax, hi2(AR)));  // R1
  f.nc0 = lo2(AR) < amax;
  f.nc1 = hi2(AR) < amax;
  const f2_t OM = sub2(pk2(1.0f, 1.0f), f.AL);
  float rc0, rc1;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc0) : "f"(lo2(OM)));  // alpha <= alpha_max < 1
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc1) : "f"(hi2(OM)));
  f.RC = pk2(rc0, rc1);
  f.VV = fma2(pk2(r2.x, r2.x), P.GR,
              fma2(pk2(r2.y, r2.y), P.GG,
                   fma2(pk2(r2.z, r2.z), P.GB, fma2(pk2(r1.w, r1.w), P.GD, P.GS))));
  return f;
}
__device__ __forceinline__ QTerms pair_state(QPair &P, const QFront &f) {
  P.T = mul2(P.T, f.RC);
  const f2_t VB = sub2(f.VV, P.B);
  P.B = fma2(f.AL, VB, P.B);
  QTerms o;
  const f2_t W = mul2(f.AL, P.T);
  const f2_t D0 = mul2(P.T, VB);
  const f2_t DL = pk2(f.nc0 ? lo2(D0) : 0.0f, f.nc1 ? hi2(D0) : 0.0f);  // R23
  o.AV = mul2(f.AL, DL);
  o.GDL = mul2(f.G, DL);
  o.TT = mul2(o.AV, f.DY);
  o.T2 = mul2(o.TT, f.DY);
  o.WD = mul2(W, P.GD);
  o.WR = mul2(W, P.GR);
  o.WG = mul2(W, P.GG);
  o.WB = mul2(W, P.GB);
  return o;
}
// the quad's ten sums of one entry's terms over its four lanes (transposed
// shuffle reduction) into the accumulator
__device__ __forceinline__ void quad_flush(const QTerms &a, float dx, bool hi, int ri, bool act,
                                           float *dst) {
  float v[kV];
  const float sav = lo2(a.AV) + hi2(a.AV), stt = lo2(a.TT) + hi2(a.TT);
  v[0] = dx * sav;
  v[1] = stt;
  v[2] = dx * v[0];
  v[3] = dx * stt;
  v[4] = lo2(a.T2) + hi2(a.T2);
  v[5] = lo2(a.GDL) + hi2(a.GDL);
  v[6] = lo2(a.WD) + hi2(a.WD);
  v[7] = lo2(a.WR) + hi2(a.WR);
  v[8] = lo2(a.WG) + hi2(a.WG);
  v[9] = lo2(a.WB) + hi2(a.WB);
  // lanes 0-1 keep (v0 v1 v2 v3 v8), lanes 2-3 (v4 v5 v6 v7 v9); then a
  // butterfly over the lane pair
  float x[5];
#pragma unroll
  for (int k = 0; k < 5; k++) {
    const float s1 = k < 4 ? v[k] : v[8], s2 = k < 4 ? v[4 + k] : v[9];
    const float keep = hi ? s2 : s1, send = hi ? s1 : s2;
    x[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
#pragma unroll
  for (int k = 0; k < 5; k++) x[k] += __shfl_xor_sync(0xffffffffu, x[k], 1);
  const float v9 = __shfl_xor_sync(0xffffffffu, x[4], 2);  // lane 1 <- lane 3's v9
  // one 16-byte reduction per lane, a single branch (one v4 + one v2 behind
  // two branches measured 141 vs 133 us at C2): lanes 0 and 2 add slots 0-3 /
  // 4-7, lane 1 slots 8-11 (the last two sums and +0 into the two padding
  // slots, which nothing reads); lane 3 none
  const bool odd = ri & 1;
  float *d = dst + (odd ? 8 : (hi ? 4 : 0));
  const float y0 = odd ? x[4] : x[0], y1 = odd ? v9 : x[1], y2 = odd ? 0.f : x[2],
              y3 = odd ? 0.f : x[3];
  if (act && ri != 3) red_add_v4(d, y0, y1, y2, y3);
}
__device__ __forceinline__ QTerms qadd(const QTerms &a, const QTerms &b) {
  QTerms o;
  o.AV = add2(a.AV, b.AV); o.TT = add2(a.TT, b.TT); o.T2 = add2(a.T2, b.T2);
  o.GDL = add2(a.GDL, b.GDL); o.WD = add2(a.WD, b.WD); o.WR = add2(a.WR, b.WR);
  o.WG = add2(a.WG, b.WG); o.WB = add2(a.WB, b.WB);
  return o;
}


// the quad walks its block's list of the chunk [c0, ...) (L, back to front),
// two entries per iteration: both fronts, the two state updates in list order,
// both partial sums -- the independent halves interleave
__device__ __forceinline__ void replay_chunk(const Lists &L, QPair (&P)[2], int B, int ri, int c0,
                                             float fpx, float amax, float *__restrict__ accg) {
  const int nr = L.nitems[B];
  const int nmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)nr);
  const uint8_t *lst = L.lst[B];
  const bool hi = ri >= 2;
  for (int e = 0; e < nmax; e += 2) {
    // past its list a quad replays the zero record with j beyond every pixel's
    // last contributor: no state change, exact zero partials
    const bool actA = e < nr, actB = e + 1 < nr;
    const int iA = actA ? (int)lst[e] : kChunk, iB = actB ? (int)lst[e + 1] : kChunk;
    const float4 a0 = L.rec[iA][0], a1 = L.rec[iA][1], a2 = L.rec[iA][2];
    const float4 b0 = L.rec[iB][0], b1 = L.rec[iB][1], b2 = L.rec[iB][2];
    const int jA = actA ? c0 + iA : 0x7fffffff, jB = actB ? c0 + iB : 0x7fffffff;
    const float dxA = DSUB(fpx, a0.x), dxB = DSUB(fpx, b0.x);
    const QFront fA0 = pair_front(P[0], jA, dxA, DMUL(a0.z, dxA), DMUL(a0.w, dxA), a0, a1, a2, amax);
    const QFront fA1 = pair_front(P[1], jA, dxA, DMUL(a0.z, dxA), DMUL(a0.w, dxA), a0, a1, a2, amax);
    const QFront fB0 = pair_front(P[0], jB, dxB, DMUL(b0.z, dxB), DMUL(b0.w, dxB), b0, b1, b2, amax);
    const QFront fB1 = pair_front(P[1], jB, dxB, DMUL(b0.z, dxB), DMUL(b0.w, dxB), b0, b1, b2, amax);
    const QTerms tA0 = pair_state(P[0], fA0), tA1 = pair_state(P[1], fA1);
    const QTerms tB0 = pair_state(P[0], fB0), tB1 = pair_state(P[1], fB1);
    quad_flush(qadd(tA0, tA1), dxA, hi, ri, actA, accg + (int64_t)__float_as_uint(a2.w) * kAcc);
    quad_flush(qadd(tB0, tB1), dxB, hi, ri, actB, accg + (int64_t)__float_as_uint(b2.w) * kAcc);
  }
}

}  // namespace quad
}  // namespace csplat
