// bin.cu -- a4 tile binning and a5 (tile, depth) ordering (the 3DGS
// tile rasterizer the paper extends; readings R4, R11).
//
// The (tile, depth) key sort is done as an MSD radix step on the tile digit
// followed by a per-tile sort of the low digits:
//   1. bucket:  warp-cooperative expansion of every Gaussian's tile rectangle
//               (a warp scans 32 counts and spreads the pairs over its lanes,
//               so one big rectangle does not serialise a lane); each pair's
//               key = bits(z_c) << 32 | index goes into its tile's fixed-size
//               bucket (slot from the tile's atomic cursor, order fixed in 3),
//               or, once the bucket is full, into one shared overflow list;
//   2. sort:    one CTA per tile finds its output offset (the exclusive scan of
//               the T cursor values, by a decoupled look-back that never waits:
//               every tile's count is already final) -> tile_range [start, end),
//               gathers its bucket (+ its overflow entries),
//               sorts it in shared memory (bitonic network, all-ascending form,
//               no padding; warp-local stages synchronise only the warp), then
//               writes pair_gid and the pair-ordered 64-byte record payload
//               that the renderer streams with TMA bulk copies (word 14 of the
//               payload: the pair's 8x8-block cull mask, block_mask below).
//               Buckets longer than the CTA's shared-memory slice are sorted in
//               global memory (pathological inputs only).
// Keys are unique (the index is in the low word), so the order is unique and
// bit-exact: (tile, bits(z_c), index) ascending.
#include "bin_dev.cuh"

namespace csplat {

constexpr int kCtaCap = 2048;      // keys per tile sorted in shared memory (16 KB)
constexpr int kSortThreads = 128;  // threads per tile in k_sort_tiles
static inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

BinWs bin_carve(void *ws, int64_t cap, int64_t T) {
  char *p = static_cast<char *>(ws);
  const size_t c = (size_t)(cap > 0 ? cap : 1);
  BinWs w;
  w.cur = reinterpret_cast<uint32_t *>(p);
  p += align_up(T * 4);
  w.ovf_n = reinterpret_cast<uint32_t *>(p);
  p += align_up(4);
  w.status = reinterpret_cast<unsigned long long *>(p);
  p += align_up(T * 8);
  w.bucket = reinterpret_cast<unsigned long long *>(p);
  p += align_up((size_t)T * kBucketCap * 8);
  w.ovf_tile = reinterpret_cast<uint32_t *>(p);
  p += align_up(c * 4);
  w.ovf_key = reinterpret_cast<unsigned long long *>(p);
  p += align_up(c * 8);
  w.keys = reinterpret_cast<unsigned long long *>(p);
  return w;
}

cudaError_t bin_reset(const BinWs &w, int64_t T, cudaStream_t s) {
  // cur, ovf_n and status are contiguous at the head of the workspace
  return cudaMemsetAsync(w.cur, 0, align_up(T * 4) + align_up(4) + align_up(T * 8), s);
}

size_t bin_workspace_bytes(int64_t n, int64_t cap, const csplat_camera &cam) {
  (void)n;
  const CamInfo ci = cam_info(cam);
  const int64_t T = (int64_t)ci.tiles_x * ci.tiles_y;
  const size_t c = (size_t)(cap > 0 ? cap : 1);
  return align_up(T * 4) + align_up(4) + align_up(T * 8) + align_up((size_t)T * kBucketCap * 8) +
         align_up(c * 4) + 2 * align_up(c * 8);
}

// a4: every (Gaussian, tile) pair's key into the tile's bucket, or the
// overflow list once the bucket holds kBucketCap keys; with an active-tile
// mask (NEXT-4, csplat_bin_tiles_active) only the pairs of active tiles.
__global__ void __launch_bounds__(256) k_bucket(int64_t n, const int32_t *__restrict__ count,
                                                const uint4 *__restrict__ rec4, int tiles_x,
                                                int64_t cap, const uint32_t *__restrict__ active,
                                                BinWs w) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t b = warp; b * 32 < n; b += nwarps) {
    const int64_t i = b * 32 + lane;
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
    expand_warp_regs(b * 32, c, rx, ry, zb, tiles_x, [&](uint32_t gid, int tile, uint32_t z) {
      bucket_put(w, cap, active, gid, tile, z);
    });
  }
}


// All-ascending bitonic network over a[0..len) (virtual +inf padding), executed
// by `nthr` (a multiple of 32) cooperating threads with index `tid`.  Pair t of
// a stage whose compare-exchange blocks span B <= 64 elements stays inside the
// 64 elements [64 (t / 32), +64), which belong to t's warp in every such stage,
// so consecutive stages with B <= 64 only synchronise the warp; `cta_sync`
// separates the others (and ends the sort).
template <typename Sync>
__device__ __forceinline__ void bitonic_sort(unsigned long long *a, int len, int tid, int nthr,
                                             Sync cta_sync) {
  int np2 = 1;
  while (np2 < len) np2 <<= 1;
  // index of the lower element of pair t in a block of 2j (j a power of two)
  auto lower = [](int t, int j) { return ((t & ~(j - 1)) << 1) | (t & (j - 1)); };
  auto sync = [&](int b, int b_next) {
    if (b <= 64 && b_next <= 64) __syncwarp();
    else cta_sync();
  };
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
    sync(k, half >= 2 ? half : 2 * k);
    for (int j = half >> 1; j > 0; j >>= 1) {
      for (int t = tid; t < np2 / 2; t += nthr) {
        const int i = lower(t, j);
        const int p = i + j;
        if (p < len) {
          const unsigned long long x = a[i], y = a[p];
          if (y < x) { a[i] = y; a[p] = x; }
        }
      }
      sync(2 * j, j >= 2 ? j : 2 * k);
    }
  }
  cta_sync();
}

// Pair entry `pos` of the sorted order: the Gaussian index (key low word) in
// bits 0-27 and the pair's 8x8-block cull mask (block_mask, from the record's
// words 0-7 and 12-13) in bits 28-31 -- what the renderers need per entry,
// so they gather the record itself from rec and compute nothing per entry.
__device__ __forceinline__ uint32_t pair_entry(unsigned long long key,
                                               const uint4 *__restrict__ rec4, int X0, int Y0) {
  const uint32_t gid = (uint32_t)(key & 0xffffffffull);
  const uint4 *r = rec4 + (int64_t)gid * 4;
  return gid | (block_mask(r[0], r[1], r[3], X0, Y0) << kPairMaskShift);
}

__device__ __forceinline__ void emit_entry(unsigned long long key, int64_t pos,
                                           const uint4 *__restrict__ rec4,
                                           uint32_t *__restrict__ pair_gid, int X0, int Y0) {
  pair_gid[pos] = pair_entry(key, rec4, X0, Y0);
}

__device__ __forceinline__ void emit_sorted(const unsigned long long *a, int len, uint32_t start,
                                            int tid, int nthr, const uint4 *__restrict__ rec4,
                                            uint32_t *__restrict__ pair_gid, int X0, int Y0) {
  for (int k = tid; k < len; k += nthr) emit_entry(a[k], (int64_t)start + k, rec4, pair_gid, X0, Y0);
}

// Register-resident bitonic sort of up to 2 * kSortThreads = 256 keys: thread t
// holds elements 2t (x0) and 2t+1 (x1); missing elements are +inf (~0, above
// every key: bits(z_c) of a finite depth is below 0x7f800000).  Same
// all-ascending network as bitonic_sort, run for blocks up to np2: the
// compare-exchange partner is in the same thread (distance 1), in lane
// t ^ (distance / 2) of the same warp (shuffles), or in another warp (one
// double-buffered shared-memory exchange and one CTA barrier per stage; three
// such stages at np2 = 256).
__device__ __forceinline__ void cx2(unsigned long long &x, unsigned long long p, bool keep_min) {
  x = keep_min ? (p < x ? p : x) : (p < x ? x : p);
}

__device__ __forceinline__ void sort_regs256(unsigned long long &x0, unsigned long long &x1,
                                             int np2, unsigned long long (*xb)[2 * kSortThreads]) {
  const int t = threadIdx.x;
  int buf = 0;
  // partner values of (x0, x1) from thread t ^ m; `swap` = the partner's elements
  // in reverse order (the mirror stage pairs element 2t with 2(t^m)+1)
  auto fetch = [&](int m, bool swap, unsigned long long &p0, unsigned long long &p1) {
    if (m < 32) {
      const unsigned long long a = __shfl_xor_sync(0xffffffffu, x0, m);
      const unsigned long long b = __shfl_xor_sync(0xffffffffu, x1, m);
      p0 = swap ? b : a;
      p1 = swap ? a : b;
    } else {
      xb[buf][2 * t] = x0;
      xb[buf][2 * t + 1] = x1;
      __syncthreads();
      const int u = t ^ m;
      p0 = xb[buf][2 * u + (swap ? 1 : 0)];
      p1 = xb[buf][2 * u + (swap ? 0 : 1)];
      buf ^= 1;
    }
  };
  for (int k = 2; k <= np2; k <<= 1) {
    unsigned long long p0, p1;
    if (k == 2) {  // mirror of the pair (2t, 2t+1): in-thread
      p0 = x1; x1 = x0 < x1 ? x1 : x0; x0 = p0 < x0 ? p0 : x0;
    } else {       // mirror stage: element e pairs with e ^ (k - 1)
      fetch((k - 1) >> 1, true, p0, p1);
      const bool lower = ((2 * t) & (k >> 1)) == 0;
      cx2(x0, p0, lower);
      cx2(x1, p1, lower);
    }
    for (int j = k >> 2; j >= 1; j >>= 1) {  // element e pairs with e ^ j
      if (j == 1) {
        p0 = x1; x1 = x0 < x1 ? x1 : x0; x0 = p0 < x0 ? p0 : x0;
      } else {
        fetch(j >> 1, false, p0, p1);
        const bool lower = ((2 * t) & j) == 0;
        cx2(x0, p0, lower);
        cx2(x1, p1, lower);
      }
    }
  }
}

// One 128-thread CTA per tile: enough warps in flight to hide the latency of
// the record gathers in emit_sorted (there are only ~3k tiles per view).
// Tile-range scan status words: bit 63 set = inclusive prefix through the tile
// published (bits 0-62); the tiles' own counts are the bucket cursors, all known
// when k_sort_tiles starts, so a tile never waits for a predecessor.
constexpr unsigned long long kRangeP = 1ull << 63;

__global__ void __launch_bounds__(kSortThreads) k_sort_tiles(
    int64_t T, uint32_t *__restrict__ range, int64_t *__restrict__ n_pairs, BinWs w,
    int64_t cap, const uint4 *__restrict__ rec4, uint32_t *__restrict__ pair_gid, int tiles_x,
    int64_t tile0, SortViews sv) {
  const int32_t *list = sv.list;
  if (gridDim.y > 1) {  // batched views: this CTA's view
    const int64_t v = blockIdx.y;
    w = ws_at(w, v * sv.ws_stride);
    rec4 += v * sv.rec_stride;
    pair_gid += v * sv.gid_stride;
    range += v * sv.range_stride;
    n_pairs += v;
    if (list) list += v * sv.list_stride;
  }
  __shared__ __align__(16) unsigned long long sk[kCtaCap];
  __shared__ uint32_t fill, s_start, s_end;
  // list mode: this CTA's list position; the look-back runs over positions
  const int64_t pos = tile0 + blockIdx.x;
  const int64_t npos = list ? (int64_t)list[0] : T;
  if (pos >= npos) return;  // (block-uniform, before any barrier)
  const int64_t tile = list ? (int64_t)list[1 + pos] : pos;
  const int X0 = (int)(tile % tiles_x) * kTile, Y0 = (int)(tile / tiles_x) * kTile;
  // the common case first: a list that fits the threads' registers is sorted
  // BEFORE the look-back (the sort needs only the tile's own count), so by the
  // time the look-back runs the preceding tiles have mostly published and the
  // CTA does not idle at a barrier behind it
  const uint32_t cnt_t = w.cur[tile];
  const bool reg_path = cnt_t <= 2u * kSortThreads;  // block-uniform
  unsigned long long x0 = ~0ull, x1 = ~0ull;
  if (reg_path && cnt_t > 0) {
    const int t = threadIdx.x, n0 = (int)cnt_t;
    const unsigned long long *bk = w.bucket + tile * kBucketCap;
    if (2 * t + 1 < n0) {
      const ulonglong2 v = reinterpret_cast<const ulonglong2 *>(bk)[t];
      x0 = v.x;
      x1 = v.y;
    } else if (2 * t < n0) {
      x0 = bk[2 * t];
    }
    int np2 = 2;
    while (np2 < n0) np2 <<= 1;
    sort_regs256(x0, x1, np2, reinterpret_cast<unsigned long long(*)[2 * kSortThreads]>(sk));
  }
  // the entries (index | block mask) need only the sorted keys and the records:
  // gather + mask them now, so the record loads' latency overlaps the look-back
  uint32_t e0 = 0, e1 = 0;
  if (reg_path) {
    const int t = threadIdx.x;
    if (2 * t < (int)cnt_t) e0 = pair_entry(x0, rec4, X0, Y0);
    if (2 * t + 1 < (int)cnt_t) e1 = pair_entry(x1, rec4, X0, Y0);
  }
  if (threadIdx.x < 32) {  // the tile's output offset: a look-back over the preceding tiles
    const int lane = threadIdx.x;
    const unsigned long long cnt = w.cur[tile];
    unsigned long long prefix = 0;
    for (int64_t j = pos - 1; j >= 0; j -= 32) {
      const int64_t jj = j - lane;
      unsigned long long v = 0;  // before position 0: an inclusive prefix of 0
      bool pub = true;
      if (jj >= 0) {
        const unsigned long long st = *reinterpret_cast<volatile unsigned long long *>(w.status + jj);
        pub = (st & kRangeP) != 0;
        v = pub ? (st & ~kRangeP) : (unsigned long long)w.cur[list ? list[1 + jj] : jj];
      }
      const unsigned pm = __ballot_sync(0xffffffffu, pub);
      const int stop = pm ? __ffs(pm) - 1 : 32;  // nearest published prefix
      unsigned long long add = lane <= stop ? v : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
      prefix += add;
      if (pm) break;
    }
    if (lane == 0) {
      const unsigned long long tot = prefix + cnt;
      atomicExch(w.status + pos, kRangeP | tot);
      const unsigned long long c = (unsigned long long)cap;
      // capacity overflow (csplat.h): a tile whose pairs do not all fit -- past
      // the capacity, or with bucket spill lost from a full overflow list --
      // gets an EMPTY range (the renderers treat it as background) and sets
      // the status bit; every other tile's list is exact
      const bool cut = tot > c || (cnt > (unsigned long long)kBucketCap && (int64_t)*w.ovf_n > cap);
      s_start = (uint32_t)(prefix < c ? prefix : c);
      s_end = cut ? s_start : (uint32_t)tot;
      range[2 * tile] = s_start;
      range[2 * tile + 1] = s_end;
      if (cut) atomicOr(range + 2 * T, CSPLAT_STATUS_CAPACITY);
      if (pos == npos - 1) {  // the last tile (position): the total
        *n_pairs = (int64_t)tot;
        atomicMax(range + 2 * T + 1, (uint32_t)(tot < 0xffffffffull ? tot : 0xffffffffull));
      }
    }
  }
  __syncthreads();
  const uint32_t start = s_start, end = s_end;
  const int len = (int)(end - start);  // the tile's pair count, or 0 (empty or cut)
  if (len == 0) return;
  if (reg_path) {  // sorted and masked above; len is cnt_t (or 0 when cut)
    const int t = threadIdx.x;
    if (2 * t < len) pair_gid[(int64_t)start + 2 * t] = e0;
    if (2 * t + 1 < len) pair_gid[(int64_t)start + 2 * t + 1] = e1;
    return;
  }
  unsigned long long *a = len <= kCtaCap ? sk : w.keys + start;
  const int nb = min(len, kBucketCap);
  const unsigned long long *bk = w.bucket + tile * kBucketCap;
  for (int k = threadIdx.x; k < nb; k += kSortThreads) a[k] = bk[k];
  if (len > kBucketCap) {  // the rest of the tile's keys are in the overflow list (all kept)
    if (threadIdx.x == 0) fill = kBucketCap;
    __syncthreads();
    const int64_t no = min((int64_t)*w.ovf_n, cap);
    for (int64_t o = threadIdx.x; o < no; o += kSortThreads)
      if (w.ovf_tile[o] == (uint32_t)tile) {
        const uint32_t pos = atomicAdd(&fill, 1u);
        if (pos < (uint32_t)len) a[pos] = w.ovf_key[o];
      }
  }
  __syncthreads();
  if (len <= 32) {  // one warp sorts a short list; the others only help emit
    if (threadIdx.x < 32) bitonic_sort(a, len, threadIdx.x, 32, [] { __syncwarp(); });
    __syncthreads();
  } else {
    bitonic_sort(a, len, threadIdx.x, kSortThreads, [] { __syncthreads(); });
  }
  emit_sorted(a, len, start, threadIdx.x, kSortThreads, rec4, pair_gid, X0, Y0);
}

cudaError_t launch_sort_tiles(const BinWs &w, int64_t T, int tiles_x, int64_t cap,
                              const void *rec, uint32_t *pair_gid,
                              uint32_t *tile_range, int64_t *n_pairs_dev, cudaStream_t s,
                              int64_t tile0, int64_t ntiles) {
  if (ntiles < 0) ntiles = T - tile0;
  if (ntiles <= 0) return cudaSuccess;
  k_sort_tiles<<<(unsigned)ntiles, kSortThreads, 0, s>>>(T, tile_range, n_pairs_dev, w, cap,
                                                         static_cast<const uint4 *>(rec),
                                                         pair_gid, tiles_x, tile0, SortViews{});
  return cudaGetLastError();
}

cudaError_t launch_sort_tiles_views(const BinWs &w, int64_t nctas, int64_t T, int tiles_x,
                                    int64_t cap, const void *rec, uint32_t *pair_gid,
                                    uint32_t *tile_range, int64_t *n_pairs_dev,
                                    const SortViews &sv, int nv, cudaStream_t s) {
  if (nctas <= 0 || nv <= 0) return cudaSuccess;
  const dim3 grid((unsigned)nctas, (unsigned)nv);
  k_sort_tiles<<<grid, kSortThreads, 0, s>>>(T, tile_range, n_pairs_dev, w, cap,
                                             static_cast<const uint4 *>(rec), pair_gid, tiles_x, 0,
                                             sv);
  return cudaGetLastError();
}

size_t bin_head_bytes(int64_t T) { return align_up(T * 4) + align_up(4) + align_up(T * 8); }

cudaError_t launch_bin(const void *rec, const int32_t *count, int64_t n, const csplat_camera &cam,
                       int64_t cap, const uint32_t *tile_active, uint32_t *pair_gid, uint32_t *tile_range, int64_t *n_pairs_dev, void *ws,
                       cudaStream_t s) {
  const CamInfo ci = cam_info(cam);
  const int64_t T = (int64_t)ci.tiles_x * ci.tiles_y;
  BinWs w = bin_carve(ws, cap, T);
  cudaError_t e = bin_reset(w, T, s);
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
  if (n > 0) k_bucket<<<(unsigned)blocks, 256, 0, s>>>(n, count, rec4, ci.tiles_x, cap,
                                                      tile_active, w);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_sort_tiles(w, T, ci.tiles_x, cap, rec, pair_gid, tile_range,
                           n_pairs_dev, s);
}

}  // namespace csplat
