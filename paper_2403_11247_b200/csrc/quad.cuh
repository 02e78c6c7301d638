// quad.cuh -- the per-4x4-block entry lists of the block-list backward
// (k_render_bwd_quad, render_bwd.cu).
//
// A CTA of two warps takes one 16x16 tile.  Its sixteen 4x4 pixel blocks each
// get their own list of the tile's entries; the four lanes of a QUAD (lane / 4
// of a warp) own one block (quad lane q: column q of the block, i.e. two
// vertically adjacent pixel pairs) and walk its list.  An entry is listed for a
// block when the record's pixel rectangle (the k^2-ellipse's bounding box, §4)
// overlaps the block and the 8x8 block around it has its bit in the pair entry
// (block_mask, the sort's conservative ellipse test): a superset of the
// entries any of the block's pixels composites, so skipping the others is
// result-invariant.  The tile list is taken in chunks of kChunk entries.
#pragma once
#include "common.cuh"

namespace csplat {
namespace quad {

constexpr int kPW = 2;                    // warps per CTA (16x8 pixels each)
constexpr int kThreads = kPW * 32;
constexpr int kNB = 16;                   // 4x4 blocks (quads) per tile
constexpr int kChunk = 256;               // list entries per gather

struct Lists {
  float4 rec[kChunk + 1][4];              // the chunk's records (+ a zero record)
  uint16_t m16[kChunk];                   // the entries' 4x4-block masks
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
  const uint32_t rows = (0xfu >> (3 - cy1)) & (0xfu << cy0);
  uint32_t rowspread = 0;
#pragma unroll
  for (int q = 0; q < 4; q++) rowspread |= ((rows >> q) & 1u) << (4 * q);
  const uint32_t m8 = entry >> kPairMaskShift;
  const uint32_t m8x = ((m8 & 1u) ? 0x0033u : 0u) | ((m8 & 2u) ? 0x00ccu : 0u) |
                       ((m8 & 4u) ? 0x3300u : 0u) | ((m8 & 8u) ? 0xcc00u : 0u);
  return cols * rowspread & m8x;
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
// to replay)
__device__ __forceinline__ void build_lists(Lists &L, int c0, int len, const int *lim, int wid,
                                            int lane) {
  int cnt = 0;  // lane rr < 8: block 8 wid + rr's count
  const int rounds = (len + 31) / 32;
  for (int k = 0; k < rounds; k++) {
    const int i = len - 32 * (k + 1) + lane;
    const uint32_t m = i >= 0 ? L.m16[i] : 0u;
#pragma unroll
    for (int rr = 0; rr < 8; rr++) {
      const int B = wid * 8 + rr;
      const bool sel = ((m >> B) & 1u) && c0 + i < lim[B];
      const uint32_t bal = __ballot_sync(0xffffffffu, sel);
      const int before = __shfl_sync(0xffffffffu, cnt, rr);
      if (sel) L.lst[B][before + __popc(bal >> lane >> 1)] = (uint8_t)i;
      if (lane == rr) cnt += __popc(bal);
    }
  }
  if (lane < 8) L.nitems[wid * 8 + lane] = cnt;
  __syncwarp();
}

}  // namespace quad
}  // namespace csplat
