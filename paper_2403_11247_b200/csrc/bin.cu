// bin.cu -- a4 tile binning and a5 (tile, depth) ordering (the 3DGS
// tile rasterizer the paper extends; readings R4, R11).
//
// The (tile, depth) key sort is done as an MSD radix step on the tile digit
// followed by a per-tile sort of the low digits:
//   1. count:   warp-cooperative expansion of every Gaussian's tile rectangle
//               (a warp scans 32 counts and spreads the pairs over its lanes,
//               so one big rectangle does not serialise a lane), one atomic
//               increment of the tile's bucket per pair;
//   2. scan:    exclusive scan of the T bucket sizes -> tile_range [start, end);
//   3. scatter: the same expansion writes key = bits(z_c) << 32 | index into the
//               tile's bucket (slot from an atomic cursor; order fixed in 4);
//   4. sort:    one warp per tile sorts its bucket in shared memory (bitonic
//               network, all-ascending form, so no padding is needed), then
//               writes pair_gid and the pair-ordered 64-byte record payload
//               that the renderer streams with TMA bulk copies (word 14 of the
//               payload: the pair's 8x8-block cull mask, block_mask below).  Buckets longer
//               than a warp's shared-memory slice go to a CTA-wide pass.
// Keys are unique (the index is in the low word), so the order is unique and
// bit-exact: (tile, bits(z_c), index) ascending.
#include "common.cuh"

namespace csplat {

constexpr int kCtaCap = 2048;         // keys per tile sorted by k_sort_tiles (16 KB smem)
constexpr int kSortThreads = 128;     // threads per tile in k_sort_tiles
constexpr int kLongSmemKeys = 12288;  // 96 KB: CTA-wide shared-memory sort limit

struct BinWs {
  uint32_t *cnt, *cur, *long_list, *long_count;
  unsigned long long *keys;
};

static inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static BinWs carve(void *ws, int64_t cap, int64_t T) {
  char *p = static_cast<char *>(ws);
  BinWs w;
  w.cnt = reinterpret_cast<uint32_t *>(p);
  p += align_up(T * 4);
  w.cur = reinterpret_cast<uint32_t *>(p);
  p += align_up(T * 4);
  w.long_count = reinterpret_cast<uint32_t *>(p);
  p += align_up(4);
  w.long_list = reinterpret_cast<uint32_t *>(p);
  p += align_up(T * 4);
  w.keys = reinterpret_cast<unsigned long long *>(p);
  return w;
}

size_t bin_workspace_bytes(int64_t n, int64_t cap, const csplat_camera &cam) {
  (void)n;
  const CamInfo ci = cam_info(cam);
  const int64_t T = (int64_t)ci.tiles_x * ci.tiles_y;
  return 4 * align_up(T * 4) + align_up(4) + align_up((size_t)(cap > 0 ? cap : 1) * 8);
}

// Warp-cooperative expansion of 32 Gaussians' tile rectangles.  Calls
// f(gid, tile, lane_owner_zbits) once per (Gaussian, tile) pair; all 32 lanes
// must be converged on entry.
template <typename F>
__device__ __forceinline__ void expand_warp(int64_t base, int64_t n, const int32_t *count,
                                            const uint4 *rec4, int tiles_x, F f) {
  const int lane = threadIdx.x & 31;
  const int64_t i = base + lane;
  int c = 0;
  uint32_t rx = 0, ry = 0, zb = 0;
  if (i < n) {
    c = count[i];
    if (c > 0) {
      const uint4 r1 = rec4[i * 4 + 1];
      const uint4 r3 = rec4[i * 4 + 3];
      zb = r1.w;
      rx = r3.x;
      ry = r3.y;
    }
  }
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int excl = incl - c;
  const int total = __shfl_sync(0xffffffffu, incl, 31);
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
    const uint32_t orx = __shfl_sync(0xffffffffu, rx, owner);
    const uint32_t ory = __shfl_sync(0xffffffffu, ry, owner);
    const uint32_t ozb = __shfl_sync(0xffffffffu, zb, owner);
    if (k < total) {
      // rx = px0 | py0 << 16 (low corner), ry = px1 | py1 << 16 (high corner)
      const int tx0 = (int)(orx & 0xffffu) / kTile, tx1 = (int)(ory & 0xffffu) / kTile;
      const int ty0 = (int)(orx >> 16) / kTile;
      const int w = tx1 - tx0 + 1;
      const int li = k - oe;
      const int tile = (ty0 + li / w) * tiles_x + tx0 + li % w;
      f((uint32_t)(base + owner), tile, ozb);
    }
  }
}

__global__ void __launch_bounds__(256) k_count(int64_t n, const int32_t *__restrict__ count,
                                               const uint4 *__restrict__ rec4, int tiles_x,
                                               uint32_t *__restrict__ cnt) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp; w * 32 < n; w += nwarps)
    expand_warp(w * 32, n, count, rec4, tiles_x,
                [&](uint32_t, int tile, uint32_t) { atomicAdd(cnt + tile, 1u); });
}

// Single-CTA exclusive scan of the T bucket sizes (T is small: 3225 at 1200x680).
__global__ void __launch_bounds__(1024) k_scan(int64_t T, const uint32_t *__restrict__ cnt,
                                               int64_t cap, uint32_t *__restrict__ range,
                                               int64_t *__restrict__ n_pairs) {
  __shared__ unsigned long long warp_tot[32];
  __shared__ unsigned long long carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < T; base += 1024) {
    const int64_t t = base + tid;
    const unsigned long long c = t < T ? cnt[t] : 0ull;
    unsigned long long incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      unsigned long long v = warp_tot[lane], s = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long u = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += u;
      }
      warp_tot[lane] = s - v;  // exclusive prefix of warp totals
    }
    __syncthreads();
    const unsigned long long start = carry + warp_tot[wid] + incl - c;
    if (t < T) {
      const unsigned long long s0 = start < (unsigned long long)cap ? start : cap;
      const unsigned long long e0 = start + c < (unsigned long long)cap ? start + c : cap;
      range[2 * t] = (uint32_t)s0;
      range[2 * t + 1] = (uint32_t)e0;
    }
    __syncthreads();
    if (tid == 1023) carry = start + c;
    __syncthreads();
  }
  if (tid == 0) *n_pairs = (int64_t)carry;
}

__global__ void __launch_bounds__(256) k_scatter(int64_t n, const int32_t *__restrict__ count,
                                                 const uint4 *__restrict__ rec4, int tiles_x,
                                                 const uint32_t *__restrict__ range,
                                                 uint32_t *__restrict__ cur,
                                                 unsigned long long *__restrict__ keys) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp; w * 32 < n; w += nwarps)
    expand_warp(w * 32, n, count, rec4, tiles_x, [&](uint32_t gid, int tile, uint32_t zb) {
      const uint32_t slot = atomicAdd(cur + tile, 1u);
      const uint32_t pos = range[2 * tile] + slot;
      if (pos < range[2 * tile + 1])
        keys[pos] = ((unsigned long long)zb << 32) | (unsigned long long)gid;
    });
}

// All-ascending bitonic network over a[0..len) (virtual +inf padding), executed
// by `nthr` cooperating threads with index `tid`; `sync` separates stages.
template <typename Sync>
__device__ __forceinline__ void bitonic_sort(unsigned long long *a, int len, int tid, int nthr,
                                             Sync sync) {
  int np2 = 1;
  while (np2 < len) np2 <<= 1;
  // index of the lower element of pair t in a block of 2j (j a power of two)
  auto lower = [](int t, int j) { return ((t & ~(j - 1)) << 1) | (t & (j - 1)); };
  for (int k = 2; k <= np2; k <<= 1) {
    const int half = k >> 1;
    for (int t = tid; t < np2 / 2; t += nthr) {
      const int i = lower(t, half);
      const int p = i ^ (k - 1);
      if (p < len) {
        const unsigned long long x = a[i], y = a[p];
        if (y < x) { a[i] = y; a[p] = x; }
      }
    }
    sync();
    for (int j = half >> 1; j > 0; j >>= 1) {
      for (int t = tid; t < np2 / 2; t += nthr) {
        const int i = lower(t, j);
        const int p = i + j;
        if (p < len) {
          const unsigned long long x = a[i], y = a[p];
          if (y < x) { a[i] = y; a[p] = x; }
        }
      }
      sync();
    }
  }
}

// Cull hint for the renderers: bit w (w = 0..3, x half = w & 1, y half = w >> 1)
// of the pair payload's word 14 is set unless the Gaussian provably has
// alpha < 1/255 over the whole 8x8 pixel block w of the tile, i.e. unless the
// minimum of q(dx, dy) = ca dx^2 + (2cb) dx dy + cc dy^2 over the block's
// rectangle exceeds k^2 by more than a rounding margin (the renderers skip a
// pixel when q > k^2).  The minimum of the convex q over a box
// that does not contain the centre lies on a box edge that faces the centre,
// so at most two 1-D clamped minimisations per block.  The margin covers the
// float32 evaluation of q at any pixel of the block, so a
// cleared bit never skips a pixel the per-pixel test would have composited.
__device__ __forceinline__ uint32_t block_mask(const uint4 &v0, const uint4 &v1, const uint4 &v3,
                                               int X0, int Y0) {
  const float u = __uint_as_float(v0.x), v = __uint_as_float(v0.y);
  const float ca = __uint_as_float(v0.z), cb2 = __uint_as_float(v0.w);
  const float cc = __uint_as_float(v1.x), k2 = __uint_as_float(v1.z);
  const int rx0 = (int)(v3.x & 0xffffu), ry0 = (int)(v3.x >> 16);
  const int rx1 = (int)(v3.y & 0xffffu), ry1 = (int)(v3.y >> 16);
  const bool conic_ok = ca > 0.0f && cc > 0.0f;
  uint32_t m = 0;
#pragma unroll
  for (int w = 0; w < 4; w++) {
    const int bx0 = X0 + (w & 1) * 8, by0 = Y0 + (w >> 1) * 8;
    const int bx1 = bx0 + 7, by1 = by0 + 7;
    if (rx1 < bx0 || rx0 > bx1 || ry1 < by0 || ry0 > by1) continue;  // rectangle cull
    if (!conic_ok) { m |= 1u << w; continue; }
    const float dx0 = (float)bx0 - u, dx1 = (float)bx1 - u;
    const float dy0 = (float)by0 - v, dy1 = (float)by1 - v;
    const bool ox = dx0 > 0.0f || dx1 < 0.0f, oy = dy0 > 0.0f || dy1 < 0.0f;
    float qmin = 0.0f;
    if (ox || oy) {
      qmin = INFINITY;
      if (ox) {  // near vertical edge, dy clamped to the block
        const float ex = dx0 > 0.0f ? dx0 : dx1;
        const float dy = fminf(fmaxf(-cb2 * ex / (2.0f * cc), dy0), dy1);
        qmin = fminf(qmin, ca * ex * ex + cb2 * ex * dy + cc * dy * dy);
      }
      if (oy) {  // near horizontal edge
        const float ey = dy0 > 0.0f ? dy0 : dy1;
        const float dx = fminf(fmaxf(-cb2 * ey / (2.0f * ca), dx0), dx1);
        qmin = fminf(qmin, ca * dx * dx + cb2 * dx * ey + cc * ey * ey);
      }
    }
    const float DX = fmaxf(fabsf(dx0), fabsf(dx1)), DY = fmaxf(fabsf(dy0), fabsf(dy1));
    const float margin = 0.01f + 2e-5f * (ca * DX * DX + fabsf(cb2) * DX * DY + cc * DY * DY);
    if (!(qmin > k2 + margin)) m |= 1u << w;  // NaN keeps the block
  }
  return m;
}

__device__ __forceinline__ void emit_sorted(const unsigned long long *a, int len, uint32_t start,
                                            int tid, int nthr, const uint4 *__restrict__ rec4,
                                            uint32_t *__restrict__ pair_gid,
                                            uint4 *__restrict__ pair_rec, int X0, int Y0) {
  for (int k = tid; k < len; k += nthr) {
    const uint32_t gid = (uint32_t)(a[k] & 0xffffffffull);
    const int64_t pos = (int64_t)start + k;
    pair_gid[pos] = gid;
    const uint4 *src = rec4 + (int64_t)gid * 4;
    const uint4 v0 = src[0], v1 = src[1], v2 = src[2];
    uint4 v3 = src[3];
#ifdef CSPLAT_BIN_NOMASK  // timing attribution only
    v3.z = 0xfu;
#else
    v3.z = block_mask(v0, v1, v3, X0, Y0);
#endif
    uint4 *dst = pair_rec + pos * 4;
    dst[0] = v0; dst[1] = v1; dst[2] = v2; dst[3] = v3;
  }
}

// One 128-thread CTA per tile: enough warps in flight to hide the latency of
// the record gathers in emit_sorted (one warp per tile left SMs at ~30%
// occupancy: there are only ~3k tiles per view).
__global__ void __launch_bounds__(kSortThreads) k_sort_tiles(
    int64_t T, const uint32_t *__restrict__ range, const unsigned long long *__restrict__ keys,
    const uint4 *__restrict__ rec4, uint32_t *__restrict__ pair_gid, uint4 *__restrict__ pair_rec,
    uint32_t *__restrict__ long_list, uint32_t *__restrict__ long_count, int tiles_x) {
  __shared__ unsigned long long sk[kCtaCap];
  const int64_t tile = blockIdx.x;
  const int X0 = (int)(tile % tiles_x) * kTile, Y0 = (int)(tile / tiles_x) * kTile;
  const uint32_t start = range[2 * tile], end = range[2 * tile + 1];
  const int len = (int)(end - start);
  if (len == 0) return;
  if (len > kCtaCap) {
    if (threadIdx.x == 0) long_list[atomicAdd(long_count, 1u)] = (uint32_t)tile;
    return;
  }
  for (int k = threadIdx.x; k < len; k += kSortThreads) sk[k] = keys[start + k];
  __syncthreads();
#ifdef CSPLAT_BIN_NOSORT  // timing attribution only (wrong order)
  if (len < 0) {
  } else if (1) {
    __syncthreads();
  } else if (len <= 32) {
#else
  if (len <= 32) {  // one warp sorts a short list; the others only help emit
#endif
    if (threadIdx.x < 32) bitonic_sort(sk, len, threadIdx.x, 32, [] { __syncwarp(); });
    __syncthreads();
  } else {
    bitonic_sort(sk, len, threadIdx.x, kSortThreads, [] { __syncthreads(); });
  }
  emit_sorted(sk, len, start, threadIdx.x, kSortThreads, rec4, pair_gid, pair_rec, X0, Y0);
}

__global__ void __launch_bounds__(1024) k_sort_long(const uint32_t *__restrict__ range,
                                                    unsigned long long *__restrict__ keys,
                                                    const uint4 *__restrict__ rec4,
                                                    uint32_t *__restrict__ pair_gid,
                                                    uint4 *__restrict__ pair_rec,
                                                    const uint32_t *__restrict__ long_list,
                                                    const uint32_t *__restrict__ long_count,
                                                    int tiles_x) {
  extern __shared__ unsigned long long lk[];
  const uint32_t nl = *long_count;
  for (uint32_t li = blockIdx.x; li < nl; li += gridDim.x) {
    const uint32_t tile = long_list[li];
    const uint32_t start = range[2 * tile], end = range[2 * tile + 1];
    const int len = (int)(end - start);
    unsigned long long *a = keys + start;
    const int X0 = (int)(tile % tiles_x) * kTile, Y0 = (int)(tile / tiles_x) * kTile;
    if (len <= kLongSmemKeys) {
      for (int k = threadIdx.x; k < len; k += blockDim.x) lk[k] = a[k];
      __syncthreads();
      bitonic_sort(lk, len, threadIdx.x, blockDim.x, [] { __syncthreads(); });
      emit_sorted(lk, len, start, threadIdx.x, blockDim.x, rec4, pair_gid, pair_rec, X0, Y0);
    } else {  // slow path for pathological buckets: same network in global memory
      bitonic_sort(a, len, threadIdx.x, blockDim.x, [] { __syncthreads(); });
      emit_sorted(a, len, start, threadIdx.x, blockDim.x, rec4, pair_gid, pair_rec, X0, Y0);
    }
    __syncthreads();
  }
}

cudaError_t launch_bin(const void *rec, const int32_t *count, int64_t n, const csplat_camera &cam,
                       int64_t cap, uint32_t *pair_gid, void *pair_rec, uint32_t *tile_range,
                       int64_t *n_pairs_dev, void *ws, cudaStream_t s) {
  const CamInfo ci = cam_info(cam);
  const int64_t T = (int64_t)ci.tiles_x * ci.tiles_y;
  BinWs w = carve(ws, cap, T);
  // cnt, cur, long_count are contiguous at the head of the workspace
  cudaError_t e = cudaMemsetAsync(w.cnt, 0, 2 * align_up(T * 4) + align_up(4), s);
  if (e != cudaSuccess) return e;
  const uint4 *rec4 = static_cast<const uint4 *>(rec);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t warps_needed = (n + 31) / 32;
  int64_t blocks = (warps_needed + 7) / 8;
  const int64_t max_blocks = (int64_t)sms * 8;
  if (blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  if (n > 0) k_count<<<(unsigned)blocks, 256, 0, s>>>(n, count, rec4, ci.tiles_x, w.cnt);
  k_scan<<<1, 1024, 0, s>>>(T, w.cnt, cap, tile_range, n_pairs_dev);
  if (n > 0)
    k_scatter<<<(unsigned)blocks, 256, 0, s>>>(n, count, rec4, ci.tiles_x, tile_range, w.cur,
                                               w.keys);
  k_sort_tiles<<<(unsigned)T, kSortThreads, 0, s>>>(
      T, tile_range, w.keys, rec4, pair_gid, static_cast<uint4 *>(pair_rec), w.long_list,
      w.long_count, ci.tiles_x);
  const size_t lsm = kLongSmemKeys * sizeof(unsigned long long);
  static bool attr_done = false;
  if (!attr_done) {
    e = cudaFuncSetAttribute(k_sort_long, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  k_sort_long<<<(unsigned)sms, 1024, lsm, s>>>(tile_range, w.keys, rec4, pair_gid,
                                               static_cast<uint4 *>(pair_rec), w.long_list,
                                               w.long_count, ci.tiles_x);
  return cudaGetLastError();
}

}  // namespace csplat
