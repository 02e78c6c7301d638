// bin_dev.cuh -- the a4 bucket pass's device pieces, shared by the stand-alone
// bucket kernel (bin.cu) and the fused projection + bucket kernel (project.cu,
// csplat_project_bin): the workspace layout, the warp-cooperative expansion of
// 32 Gaussians' tile rectangles and the bucket insert.  See bin.cu.
#pragma once
#include "common.cuh"

namespace csplat {

constexpr int kBucketCap = 512;    // bucket slots per tile; later pairs go to the overflow list
// the tiles' cursors are kCurStride words apart: the bucket pass's ~174
// atomics per tile (C2) then do not share an L2 sector with 7 other tiles'
// (stride 1 -> 8: C2 stand-alone bin 44 -> 42 us, fused projection + bucket
// pass 50.2 -> 48.1 us; 32 no further change)
constexpr int kCurStride = 8;

struct BinWs {
  uint32_t *cur;                     // [T][kCurStride] pairs per tile (atomic cursor, word 0)
  uint32_t *ovf_n;                   // overflow-list length
  unsigned long long *status;        // [T] each tile's (list position's) output offset (k_tile_scan)
  unsigned long long *bucket;        // [T][kBucketCap] keys
  uint32_t *ovf_tile;                // [cap] tile of each overflow entry
  unsigned long long *ovf_key;       // [cap] its key
  unsigned long long *keys;          // [cap] global-memory sort scratch (tiles > kCtaCap)
  // ovf_n[1]: CTAs of the bucket pass that finished (the last one runs the
  // offset scan, tile_scan_cta); zeroed with the head
};

BinWs bin_carve(void *ws, int64_t cap, int64_t T);
// the workspace of view v of a batched call: every region offset by v * stride bytes
__host__ __device__ __forceinline__ BinWs ws_at(BinWs w, int64_t off) {
  auto mv = [off](auto *p) { return reinterpret_cast<decltype(p)>(reinterpret_cast<char *>(p) + off); };
  w.cur = mv(w.cur); w.ovf_n = mv(w.ovf_n); w.status = mv(w.status); w.bucket = mv(w.bucket);
  w.ovf_tile = mv(w.ovf_tile); w.ovf_key = mv(w.ovf_key); w.keys = mv(w.keys);
  return w;
}
// bytes of the head (cursors, overflow length, offset words) bin_reset zeroes
size_t bin_head_bytes(int64_t T);
// zero the cursors, the overflow length and the offset words (one memset)
cudaError_t bin_reset(const BinWs &w, int64_t T, cudaStream_t s);
// a5 offsets: the exclusive scan of the pair counts of nv views' tiles (view v's
// workspace at + v ws_stride bytes; list: per view a tile list as below, the
// scan then runs over its positions) -- after the bucket pass, before the sort
cudaError_t launch_tile_scan(const BinWs &w, int64_t T, int nv, int64_t ws_stride,
                             const int32_t *list, int64_t list_stride, cudaStream_t s);
// a5: k_sort_tiles over the buckets filled by k_bucket or the fused projection,
// after launch_tile_scan (tiles [tile0, tile0 + ntiles) only, ntiles < 0 = to
// the end: every tile reads only its own offset, so any split of the tiles
// into launches is valid).  narrow: the register sort on 32-bit keys
// (warp_sort_emit32) instead of the 64-bit keys -- the same order bit for bit
cudaError_t launch_sort_tiles(const BinWs &w, int64_t T, int tiles_x, int64_t cap,
                              const void *rec, uint32_t *pair_gid,
                              uint32_t *tile_range, int64_t *n_pairs_dev, cudaStream_t s,
                              int64_t tile0 = 0, int64_t ntiles = -1, bool narrow = true);
// the same over nv views at once (grid.y = view): view v's workspace at
// + v ws_stride bytes, records + v rec_stride (uint4 units), pair_gid + v
// gid_stride, tile_range + v range_stride, n_pairs_dev + v
// list (optional): per view a device tile list {count, tile_0 < tile_1 < ...}
// at list + v list_stride -- only those tiles are sorted (their buckets hold
// every pair: the bucket pass saw only those tiles), the offsets scan the list
// positions, and the other tiles' ranges must be empty (zeroed by the caller)
struct SortViews {
  int64_t ws_stride, rec_stride, gid_stride, range_stride;
  const int32_t *list;
  int64_t list_stride;
};
cudaError_t launch_sort_tiles_views(const BinWs &w, int64_t nctas, int64_t T, int tiles_x,
                                    int64_t cap, const void *rec, uint32_t *pair_gid,
                                    uint32_t *tile_range, int64_t *n_pairs_dev,
                                    const SortViews &sv, int nv, cudaStream_t s);

// a5 offsets: the exclusive scan of the T cursors (the tiles' pair counts, or
// of list positions' counts) into the offset words, by one whole CTA
// (blockDim.x a multiple of 32, <= 1024)
__device__ __forceinline__ void tile_scan_cta(const BinWs &w, int64_t npos,
                                              const int32_t *__restrict__ list) {
  constexpr int kPer = 4;
  __shared__ unsigned long long wsum[32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
  const int64_t step = (int64_t)blockDim.x * kPer;
  unsigned long long carry = 0;
  for (int64_t base = 0; base < npos; base += step) {
    uint32_t c[kPer];
    unsigned long long own = 0;
#pragma unroll
    for (int k = 0; k < kPer; k++) {
      const int64_t p = base + (int64_t)t * kPer + k;
      c[k] = p < npos ? *(volatile uint32_t *)&w.cur[(list ? list[1 + p] : p) * kCurStride] : 0u;
      own += c[k];
    }
    unsigned long long inc = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      unsigned long long v = lane < nw ? wsum[lane] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      wsum[lane] = v;
    }
    __syncthreads();
    unsigned long long ex = carry + (wid > 0 ? wsum[wid - 1] : 0ull) + inc - own;
#pragma unroll
    for (int k = 0; k < kPer; k++) {
      const int64_t p = base + (int64_t)t * kPer + k;
      if (p < npos) w.status[p] = ex;
      ex += c[k];
    }
    carry += wsum[nw - 1];
    __syncthreads();  // wsum is rewritten by the next round
  }
}
// The end of a bucket-pass kernel: the CTA that finishes last (every other
// CTA's cursor atomics are visible after its fence and ticket) runs the offset
// scan, so the sort needs no separate scan launch.  Block-uniform; all threads.
__device__ __forceinline__ void bucket_pass_done(const BinWs &w, int64_t T) {
  __shared__ bool last;
  __syncthreads();
  // (acq_rel, not the sequentially consistent __threadfence: the barrier
  // orders the CTA's cursor atomics before thread 0's cumulative release)
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    last = atomicAdd(w.ovf_n + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    tile_scan_cta(w, T, nullptr);
  }
}

// What a Gaussian contributes to the bucket pass: its pair count c, its pixel
// rectangle corners rx, ry (record words 12, 13), bits(z_c) zb, and the conic
// and extent the pairs' 8x8-block cull masks need (block_mask_c, DESIGN.md §4:
// the sort used to gather the record per pair for it).
struct PairSrc {
  int c;
  uint32_t rx, ry, zb;
  float u, v, ca, cb2, cc, k2;
};
__device__ __forceinline__ PairSrc pair_src_none() {
  PairSrc s;
  s.c = 0; s.rx = s.ry = s.zb = 0u;
  s.u = s.v = s.ca = s.cb2 = s.cc = s.k2 = 0.f;
  return s;
}
// from a record (words 0-7, 12-13) and its pair count
__device__ __forceinline__ PairSrc pair_src_rec(int c, const uint4 &r0, const uint4 &r1,
                                                const uint4 &r3) {
  PairSrc s;
  s.c = c; s.rx = r3.x; s.ry = r3.y; s.zb = r1.w;
  s.u = __uint_as_float(r0.x); s.v = __uint_as_float(r0.y);
  s.ca = __uint_as_float(r0.z); s.cb2 = __uint_as_float(r0.w);
  s.cc = __uint_as_float(r1.x); s.k2 = __uint_as_float(r1.z);
  return s;
}

// Warp-cooperative expansion of 32 Gaussians' tile rectangles into the
// tiles' buckets.  Lane l holds Gaussian base + l's PairSrc; all 32 lanes must
// be converged on entry.  The warp's pairs are spread over its lanes in rounds
// of 32 (a warp scan of the counts, the owner lane by binary search, so one big
// rectangle does not serialise a lane); per pair the 8x8-block cull mask from
// the owner's conic and the key bits(z_c) << 32 | gid << 4 | mask (the (tile,
// bits(z_c), gid) order; gids are unique, so the mask bits never decide, and
// the sort emits the pair entry without touching the record).  Each pair takes
// the slot its tile's atomic cursor returns, or the shared overflow list once
// the tile's bucket is full; with an active-tile mask (NEXT-4) only the pairs
// of sampled tiles.  (Several rounds' cursor atomics issued before their
// stores measured slower: the pass is not bound by the atomics' round trips.)
__device__ __forceinline__ void expand_warp_bucket(int64_t base, const PairSrc &src, int tiles_x,
                                                   const BinWs &w, int64_t cap,
                                                   const uint32_t *__restrict__ active) {
  const int lane = threadIdx.x & 31;
  const int c = src.c;
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int excl = incl - c;
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  // the edge minimisers' slopes of the box test, once per Gaussian
  const bool ok = src.ca > 0.0f && src.cc > 0.0f;
  const float sy = ok ? -src.cb2 / (2.0f * src.cc) : 0.0f;
  const float sx = ok ? -src.cb2 / (2.0f * src.ca) : 0.0f;
  for (int kb = 0; kb < total; kb += 32) {
    const int k = kb + lane;
    int owner = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int cand = owner + step;
      const int e = __shfl_sync(0xffffffffu, excl, cand & 31);
      if (cand < 32 && e <= k) owner = cand;
    }
    const int oe = __shfl_sync(0xffffffffu, excl, owner);
    const uint32_t orx = __shfl_sync(0xffffffffu, src.rx, owner);
    const uint32_t ory = __shfl_sync(0xffffffffu, src.ry, owner);
    const uint32_t ozb = __shfl_sync(0xffffffffu, src.zb, owner);
    BoxConic bc;
    bc.u = __shfl_sync(0xffffffffu, src.u, owner);
    bc.v = __shfl_sync(0xffffffffu, src.v, owner);
    bc.ca = __shfl_sync(0xffffffffu, src.ca, owner);
    bc.cb2 = __shfl_sync(0xffffffffu, src.cb2, owner);
    bc.cc = __shfl_sync(0xffffffffu, src.cc, owner);
    bc.k2 = __shfl_sync(0xffffffffu, src.k2, owner);
    bc.sx = __shfl_sync(0xffffffffu, sx, owner);
    bc.sy = __shfl_sync(0xffffffffu, sy, owner);
    if (k >= total) continue;
    // rx = px0 | py0 << 16 (low corner), ry = px1 | py1 << 16 (high corner)
    bc.rx0 = (int)(orx & 0xffffu); bc.ry0 = (int)(orx >> 16);
    bc.rx1 = (int)(ory & 0xffffu); bc.ry1 = (int)(ory >> 16);
    bc.conic_ok = bc.ca > 0.0f && bc.cc > 0.0f;
    const int tx0 = bc.rx0 / kTile, tx1 = bc.rx1 / kTile;
    const int ty0 = bc.ry0 / kTile;
    const int wd = tx1 - tx0 + 1;
    const int li = k - oe;
    const int ty = ty0 + li / wd, tx = tx0 + li % wd;
    const int t = ty * tiles_x + tx;
    if (active && !((active[t >> 5] >> (t & 31)) & 1u)) continue;  // tile not sampled
    const uint32_t gid = (uint32_t)(base + owner);
    const uint32_t m = block_mask_c(bc, tx * kTile, ty * kTile);
    const unsigned long long key =
        ((unsigned long long)ozb << 32) | (unsigned long long)((gid << 4) | m);
    const uint32_t slot = atomicAdd(w.cur + (int64_t)t * kCurStride, 1u);
    if (slot < (uint32_t)kBucketCap) {
      w.bucket[(int64_t)t * kBucketCap + slot] = key;
    } else {
      const uint32_t o = atomicAdd(w.ovf_n, 1u);
      if ((int64_t)o < cap) {  // beyond cap the pairs exceed the capacity anyway
        w.ovf_tile[o] = (uint32_t)t;
        w.ovf_key[o] = key;
      }
    }
  }
}

}  // namespace csplat
