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
//   2. scan:    one CTA per view: the exclusive scan of the T cursor values
//               (the tiles' pair counts, all final once the bucket pass ends)
//               -> every tile's output offset, in the look-up words;
//   3. sort:    one CTA per tile reads its offset -> tile_range [start, end),
//               gathers its bucket (+ its overflow entries), sorts it
//               (registers for <= 256 keys, else shared memory: bitonic
//               network, all-ascending form, no padding; warp-local stages
//               synchronise only the warp), then writes its pair entries
//               (Gaussian index | 8x8-block cull mask << 28, pair_entry below).
//               Buckets longer than the CTA's shared-memory slice are sorted in
//               global memory (pathological inputs only).
// The offsets were first found by a decoupled look-back inside the sort
// (round 1); with ~1.6k tiles per launch all resident at once, the look-back
// walked back over many not-yet-published tiles (two dependent L2 loads per 32
// tiles) and was the sort's top stall (profiles/r2b_kernels.md), so the scan
// is a separate ~2 us kernel and the sort CTAs never touch another tile.
// Keys are unique (the index is in the low word), so the order is unique and
// bit-exact: (tile, bits(z_c), index) ascending.
#include "bin_dev.cuh"

namespace csplat {

constexpr int kCtaCap = 1024;      // keys per tile sorted in shared memory (8 KB: ~28 one-warp CTAs per SM)
constexpr int kSortThreads = 32;   // threads per tile in k_sort_tiles (one warp)
static inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

BinWs bin_carve(void *ws, int64_t cap, int64_t T) {
  char *p = static_cast<char *>(ws);
  const size_t c = (size_t)(cap > 0 ? cap : 1);
  BinWs w;
  w.cur = reinterpret_cast<uint32_t *>(p);
  p += align_up(T * 4 * kCurStride);
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
  return cudaMemsetAsync(w.cur, 0, bin_head_bytes(T), s);
}

size_t bin_workspace_bytes(int64_t n, int64_t cap, const csplat_camera &cam) {
  (void)n;
  const CamInfo ci = cam_info(cam);
  const int64_t T = (int64_t)ci.tiles_x * ci.tiles_y;
  const size_t c = (size_t)(cap > 0 ? cap : 1);
  return bin_head_bytes(T) + align_up((size_t)T * kBucketCap * 8) +
         align_up(c * 4) + 2 * align_up(c * 8);
}

// a4: every (Gaussian, tile) pair's key into the tile's bucket, or the
// overflow list once the bucket holds kBucketCap keys; with an active-tile
// mask (NEXT-4, csplat_bin_tiles_active) only the pairs of active tiles.
__global__ void __launch_bounds__(256) k_bucket(int64_t n, const int32_t *__restrict__ count,
                                                const uint4 *__restrict__ rec4, int tiles_x,
                                                int64_t T, int64_t cap,
                                                const uint32_t *__restrict__ active, BinWs w) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t b = warp; b * 32 < n; b += nwarps) {
    const int64_t i = b * 32 + lane;
    PairSrc src = pair_src_none();
    if (i < n) {
      const int c = count[i];
      if (c > 0) src = pair_src_rec(c, rec4[i * 4 + 0], rec4[i * 4 + 1], rec4[i * 4 + 3]);
    }
    expand_warp_bucket(b * 32, src, tiles_x, w, cap, active);
  }
  bucket_pass_done(w, T);
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

// Pair entry of a sorted key: the Gaussian index (key bits 4-31) in bits 0-27
// and the pair's 8x8-block cull mask (key bits 0-3, computed by the bucket
// pass) in bits 28-31 -- what the renderers need per entry.
__device__ __forceinline__ uint32_t pair_entry(unsigned long long key) {
  const uint32_t lo = (uint32_t)(key & 0xffffffffull);
  return (lo >> 4) | ((lo & 0xfu) << kPairMaskShift);
}

__device__ __forceinline__ void emit_sorted(const unsigned long long *a, int len, uint32_t start,
                                            int tid, int nthr, uint32_t *__restrict__ pair_gid) {
  for (int k = tid; k < len; k += nthr) pair_gid[(int64_t)start + k] = pair_entry(a[k]);
}

// One warp sorts up to 32 * KPL keys in registers: lane l holds elements
// KPL l .. KPL l + KPL - 1 (blocked), missing elements +inf.  The same
// all-ascending bitonic network as above; a compare-exchange at distance
// m < KPL is inside the lane, at m >= KPL the partner is element t ^ (m % KPL)
// of lane l ^ (m / KPL) (one shuffle per element).  KPL = 8 (<= 256 keys): 21
// of the 36 stages are lane-local; KPL = 16 (<= 512): 30 of 45.  No CTA
// barrier (round 1's 128-thread form: 33 shuffle stages, 3 barriers).  Key
// type K: the 64-bit keys themselves, or the 32-bit keys of
// warp_sort_emit32 (u32 min / max and one shuffle: a third of the 64-bit
// form's instructions).
template <typename K, int KPL>
__device__ __forceinline__ void cx_lane(K (&x)[KPL], int a, int b) {
  const K lo = x[a] < x[b] ? x[a] : x[b], hi = x[a] < x[b] ? x[b] : x[a];
  x[a] = lo;
  x[b] = hi;
}
template <typename K, int KPL, int M, int HIBIT>
__device__ __forceinline__ void warp_stage(K (&x)[KPL], int lane) {
  // partner e ^ M; the pair's lower element keeps the min
  if constexpr (M < KPL) {
#pragma unroll
    for (int t = 0; t < KPL; t++)
      if ((t ^ M) > t) cx_lane<K, KPL>(x, t, t ^ M);
  } else {
    constexpr int ml = M / KPL, mt = M % KPL;
    const bool lower = (lane & (HIBIT / KPL)) == 0;
    K p[KPL];
#pragma unroll
    for (int t = 0; t < KPL; t++) p[t] = __shfl_xor_sync(0xffffffffu, x[t ^ mt], ml);
#pragma unroll
    for (int t = 0; t < KPL; t++) {
      if constexpr (sizeof(K) == 4) {
        x[t] = lower ? min(x[t], p[t]) : max(x[t], p[t]);
      } else {
        const bool pl = p[t] < x[t];
        x[t] = (pl == lower) ? p[t] : x[t];
      }
    }
  }
}
template <typename K, int KPL, int KK, int J>
__device__ __forceinline__ void warp_cleaners(K (&x)[KPL], int lane) {
  if constexpr (J >= 1) {
    warp_stage<K, KPL, J, J>(x, lane);
    warp_cleaners<K, KPL, KK, J / 2>(x, lane);
  }
}
template <typename K, int KPL, int KK, int NP2>
__device__ __forceinline__ void warp_merges(K (&x)[KPL], int lane) {
  if constexpr (KK <= NP2) {
    warp_stage<K, KPL, KK - 1, KK / 2>(x, lane);  // mirror
    warp_cleaners<K, KPL, KK, KK / 4>(x, lane);   // half-cleaners
    warp_merges<K, KPL, 2 * KK, NP2>(x, lane);
  }
}
// the network for NP2 elements (<= 32 KPL), all stage distances compile-time
// so the keys stay in registers
template <typename K, int KPL, int NP2>
__device__ __forceinline__ void sort_warp(K (&x)[KPL]) {
  warp_merges<K, KPL, 2, NP2>(x, threadIdx.x & 31);
}
// load a tile's len keys (<= 32 KPL) from its bucket, sort the 64-bit keys,
// emit the entries
template <int KPL, int NP2>
__device__ __forceinline__ void warp_sort_emit64(const unsigned long long *__restrict__ bk,
                                                 int len, uint32_t start,
                                                 uint32_t *__restrict__ pair_gid) {
  const int l = threadIdx.x;
  unsigned long long x[KPL];
#pragma unroll
  for (int t = 0; t < KPL; t++) x[t] = KPL * l + t < len ? bk[KPL * l + t] : ~0ull;
  sort_warp<unsigned long long, KPL, NP2>(x);
#pragma unroll
  for (int t = 0; t < KPL; t++)
    if (KPL * l + t < len) pair_gid[(int64_t)start + KPL * l + t] = pair_entry(x[t]);
}
// A tile's len <= 32 KPL <= 512 keys from its bucket, sorted, as pair entries.
// The 64-bit keys (bits(z_c), gid, mask) are staged in shared memory (ex, by
// bucket position i); the network sorts the 32-bit keys
// ((bits(z_c) - zlo) >> sh) << 9 | i, zlo the tile's smallest depth bits and
// sh = 0 unless the tile's depth-bit span needs more than 22 bits: keys whose
// shifted depths differ come out in their exact order, and equal shifted
// depths (equal depths, or, for sh > 0, depths closer than 2^sh bit steps)
// form adjacent runs.  Every output position then takes its exact key by i;
// inside a run an element's final position is the run start + its rank among
// the run's exact keys (gids are unique, so the ranks are a permutation).  The
// result is the same order as a 64-bit sort, bit for bit.
template <int KPL, int NP2>
__device__ __forceinline__ void warp_sort_emit32(const unsigned long long *__restrict__ bk,
                                                 int len, uint32_t start,
                                                 uint32_t *__restrict__ pair_gid,
                                                 unsigned long long *__restrict__ ex,
                                                 uint32_t *__restrict__ s32) {
  const int l = threadIdx.x;
  uint32_t x[KPL];
  // (the network sorts any assignment of keys to its NP2 positions, i.e. to
  // lanes l < NP2 / KPL: loaded striped over those lanes, so the bucket reads
  // coalesce and the staging stores are conflict-free)
  constexpr int kLanes = NP2 / KPL;
  uint32_t zlo = 0xffffffffu, zhi = 0u;
#pragma unroll
  for (int t = 0; t < KPL; t++) {
    const int i = kLanes * t + l;
    if (l < kLanes && i < len) {
      const unsigned long long e = bk[i];
      ex[i] = e;
      zlo = min(zlo, (uint32_t)(e >> 32));
      zhi = max(zhi, (uint32_t)(e >> 32));
    }
  }
  // the tile's depth-bit range [zlo, zhi] in 22 bits: shifted right by sh only
  // when it is wider (then equal shifted depths form runs, fixed up below);
  // every real key stays below the padding key 0xffffffff
  zlo = __reduce_min_sync(0xffffffffu, zlo);
  zhi = __reduce_max_sync(0xffffffffu, zhi);
  const uint32_t span = zhi - zlo;
  const int sh = span >> 22 ? 10 - __clz(span) : 0;  // bit length of span - 22
#pragma unroll
  for (int t = 0; t < KPL; t++) {  // (the staged keys re-read: fewer live registers)
    const int i = kLanes * t + l;
    x[t] = l < kLanes && i < len ? ((((uint32_t)(ex[i] >> 32) - zlo) >> sh) << 9) | (uint32_t)i
                                 : 0xffffffffu;
  }
  sort_warp<uint32_t, KPL, NP2>(x);
  // sorted keys by output position p at s32[p + p / 32] (no bank conflicts
  // between the lanes' blocked positions)
  auto at = [](int p) { return p + (p >> 5); };
#pragma unroll
  for (int t = 0; t < KPL; t++) s32[at(KPL * l + t)] = x[t];
  // the neighbours across the lane boundary
  const uint32_t before = __shfl_up_sync(0xffffffffu, x[KPL - 1], 1);
  const uint32_t after = __shfl_down_sync(0xffffffffu, x[0], 1);
  __syncwarp();
  uint32_t runs = 0;  // this lane's elements inside a run (bit t)
#pragma unroll
  for (int t = 0; t < KPL; t++) {
    const int p = KPL * l + t;
    const uint32_t tk = x[t] >> 9;
    const uint32_t prv = t > 0 ? x[t - 1] : before, nxt = t + 1 < KPL ? x[t + 1] : after;
    const bool run = (p > 0 && (prv >> 9) == tk) || (p + 1 < len && (nxt >> 9) == tk);
    if (p < len && !run) pair_gid[(int64_t)start + p] = pair_entry(ex[x[t] & 511u]);
    runs |= (p < len && run) ? 1u << t : 0u;
  }
  while (runs) {
    const int t = __ffs(runs) - 1;
    runs &= runs - 1;
    const int p = KPL * l + t;
    const uint32_t v = s32[at(p)], tk = v >> 9;
    const unsigned long long e = ex[v & 511u];
    int r0 = p, r1 = p;
    while (r0 > 0 && (s32[at(r0 - 1)] >> 9) == tk) r0--;
    while (r1 + 1 < len && (s32[at(r1 + 1)] >> 9) == tk) r1++;
    int rank = 0;
    for (int q = r0; q <= r1; q++) rank += ex[s32[at(q)] & 511u] < e ? 1 : 0;
    pair_gid[(int64_t)start + r0 + rank] = pair_entry(e);
  }
}

// a5 offsets: the exclusive scan of the tiles' (or list positions') pair counts
// into the look-up words, one CTA per view (grid.x = view)
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(int64_t T, BinWs w, int64_t ws_stride,
                                                            const int32_t *__restrict__ list,
                                                            int64_t list_stride) {
  if (blockIdx.x > 0) {
    w = ws_at(w, (int64_t)blockIdx.x * ws_stride);
    if (list) list += (int64_t)blockIdx.x * list_stride;
  }
  tile_scan_cta(w, list ? (int64_t)list[0] : T, list);
}

cudaError_t launch_tile_scan(const BinWs &w, int64_t T, int nv, int64_t ws_stride,
                             const int32_t *list, int64_t list_stride, cudaStream_t s) {
  if (nv <= 0) return cudaSuccess;
  k_tile_scan<<<(unsigned)nv, kScanThreads, 0, s>>>(T, w, ws_stride, list, list_stride);
  return cudaGetLastError();
}

// One 128-thread CTA per tile: enough warps in flight to hide the latency of
// the record gathers in pair_entry (there are only ~3k tiles per view).
template <bool NARROW>
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
  __shared__ uint32_t fill;
  // list mode: this CTA's list position; the offsets are over positions
  const int64_t pos = tile0 + blockIdx.x;
  const int64_t npos = list ? (int64_t)list[0] : T;
  if (pos >= npos) return;  // (block-uniform, before any barrier)
  const int64_t tile = list ? (int64_t)list[1 + pos] : pos;
  const uint32_t cnt_t = w.cur[tile * kCurStride];
  const unsigned long long prefix = w.status[pos];  // k_tile_scan's exclusive offset
  // capacity overflow (csplat.h): a tile whose pairs do not all fit -- past
  // the capacity, or with bucket spill lost from a full overflow list -- gets
  // an EMPTY range (the renderers treat it as background) and sets the status
  // bit; every other tile's list is exact
  const unsigned long long tot = prefix + cnt_t, c = (unsigned long long)cap;
  const bool cut = tot > c || (cnt_t > (uint32_t)kBucketCap && (int64_t)*w.ovf_n > cap);
  const uint32_t start = (uint32_t)(prefix < c ? prefix : c);
  const uint32_t end = cut ? start : (uint32_t)tot;
  if (threadIdx.x == 0) {
    range[2 * tile] = start;
    range[2 * tile + 1] = end;
    if (cut) atomicOr(range + 2 * T, CSPLAT_STATUS_CAPACITY);
    if (pos == npos - 1) {  // the last tile (position): the total
      *n_pairs = (int64_t)tot;
      atomicMax(range + 2 * T + 1, (uint32_t)(tot < 0xffffffffull ? tot : 0xffffffffull));
    }
  }
  const int len = (int)(end - start);  // the tile's pair count, or 0 (empty or cut)
  if (len == 0) return;                // (block-uniform)
  if (len <= 512) {  // the common case: one warp, in registers
    const unsigned long long *bk = w.bucket + tile * kBucketCap;
    if constexpr (NARROW) {
      // (sk: the exact keys in its first 4 KB, the sorted 32-bit keys after)
      unsigned long long *ex = sk;
      uint32_t *s32 = reinterpret_cast<uint32_t *>(sk + 512);
      if (len <= 64) warp_sort_emit32<8, 64>(bk, len, start, pair_gid, ex, s32);     // 21 stages
      else if (len <= 128) warp_sort_emit32<8, 128>(bk, len, start, pair_gid, ex, s32);
      else if (len <= 256) warp_sort_emit32<8, 256>(bk, len, start, pair_gid, ex, s32);
      else warp_sort_emit32<16, 512>(bk, len, start, pair_gid, ex, s32);             // 45 stages
    } else {
      if (len <= 64) warp_sort_emit64<8, 64>(bk, len, start, pair_gid);
      else if (len <= 128) warp_sort_emit64<8, 128>(bk, len, start, pair_gid);
      else if (len <= 256) warp_sort_emit64<8, 256>(bk, len, start, pair_gid);
      else warp_sort_emit64<16, 512>(bk, len, start, pair_gid);
    }
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
        const uint32_t q = atomicAdd(&fill, 1u);
        if (q < (uint32_t)len) a[q] = w.ovf_key[o];
      }
  }
  __syncthreads();
  bitonic_sort(a, len, threadIdx.x, kSortThreads, [] { __syncthreads(); });
  emit_sorted(a, len, start, threadIdx.x, kSortThreads, pair_gid);
}

cudaError_t launch_sort_tiles(const BinWs &w, int64_t T, int tiles_x, int64_t cap,
                              const void *rec, uint32_t *pair_gid,
                              uint32_t *tile_range, int64_t *n_pairs_dev, cudaStream_t s,
                              int64_t tile0, int64_t ntiles, bool narrow) {
  if (ntiles < 0) ntiles = T - tile0;
  if (ntiles <= 0) return cudaSuccess;
  // (two instantiations: the 64-bit form in one kernel with the 32-bit one
  // ran at 14.7 instead of 9.6 us per C2 chunk)
  auto kern = narrow ? k_sort_tiles<true> : k_sort_tiles<false>;
  kern<<<(unsigned)ntiles, kSortThreads, 0, s>>>(T, tile_range, n_pairs_dev, w, cap,
                                                 static_cast<const uint4 *>(rec), pair_gid,
                                                 tiles_x, tile0, SortViews{});
  return cudaGetLastError();
}

cudaError_t launch_sort_tiles_views(const BinWs &w, int64_t nctas, int64_t T, int tiles_x,
                                    int64_t cap, const void *rec, uint32_t *pair_gid,
                                    uint32_t *tile_range, int64_t *n_pairs_dev,
                                    const SortViews &sv, int nv, cudaStream_t s) {
  if (nctas <= 0 || nv <= 0) return cudaSuccess;
  const dim3 grid((unsigned)nctas, (unsigned)nv);
  k_sort_tiles<true><<<grid, kSortThreads, 0, s>>>(T, tile_range, n_pairs_dev, w, cap,
                                                   static_cast<const uint4 *>(rec), pair_gid,
                                                   tiles_x, 0, sv);
  return cudaGetLastError();
}

size_t bin_head_bytes(int64_t T) {
  return align_up(T * 4 * kCurStride) + align_up(4) + align_up(T * 8);
}

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
  if (n > 0) k_bucket<<<(unsigned)blocks, 256, 0, s>>>(n, count, rec4, ci.tiles_x, T, cap,
                                                      tile_active, w);
  e = cudaGetLastError();
  // (n == 0: no bucket pass; every offset is 0 from the reset)
  if (e != cudaSuccess) return e;
  return launch_sort_tiles(w, T, ci.tiles_x, cap, rec, pair_gid, tile_range,
                           n_pairs_dev, s);
}

}  // namespace csplat
