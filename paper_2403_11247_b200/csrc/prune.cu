// prune.cu -- a9: mask prune (Fig 3): remove every
// Gaussian whose mask is off (m <= tau, Eq 6 / R12) and compact the survivors
// of every attribute plane (and the R-VQ index planes) in their original order.
//
// One pass (k_prune_onepass): each CTA takes the next tile of kPTile Gaussians
// (dynamic ticket), loads its masks and attribute planes, publishes the tile's
// survivor count, finds its output offset by a decoupled look-back over the
// preceding tiles' published counts / inclusive prefixes (warp-parallel, 32
// tiles per probe), and scatters the survivors in order (ballot/popc ranks
// inside each 256-element round, a warp-total scan across the CTA).  The
// three-launch form (count -> one-CTA scan -> scatter) is kept for reference
// builds (CSPLAT_PRUNE_3PASS).  Reads and writes are coalesced per round.
// HBM-bound: 4 + 60 + 2L bytes read per Gaussian, 60 + 2L (+4 keep_map)
// written per survivor.
#include "common.cuh"

namespace csplat {

constexpr int kPT = 256;         // threads per CTA
#ifndef CSPLAT_PRUNE_ITEMS
#define CSPLAT_PRUNE_ITEMS 2
#endif
constexpr int kPItems = CSPLAT_PRUNE_ITEMS;  // rounds per CTA (keeps >= 2 waves of CTAs at 200k)
constexpr int kPTile = kPT * kPItems;

size_t prune_workspace_bytes(int64_t n) {
  const int64_t nt = (n + kPTile - 1) / kPTile;
  return (size_t)(nt + 2) * sizeof(unsigned long long) + 256;
}

__global__ void __launch_bounds__(kPT) k_prune_count(int64_t n, const int64_t *__restrict__ n_dev,
                                                     const float *__restrict__ mask, float tau,
                                                     unsigned long long *__restrict__ tcount) {
  __shared__ int wsum[kPT / 32];
  const int64_t ne = eff_n(n, n_dev);
  const int64_t base = (int64_t)blockIdx.x * kPTile;
  int c = 0;
#pragma unroll 4
  for (int k = 0; k < kPItems; k++) {
    const int64_t i = base + (int64_t)k * kPT + threadIdx.x;
    c += (i < ne && mask[i] > tau) ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kPT / 32; w++) t += wsum[w];
    tcount[blockIdx.x] = (unsigned long long)t;
  }
}

__global__ void __launch_bounds__(1024) k_prune_scan(int64_t nt,
                                                     unsigned long long *__restrict__ tcount,
                                                     int64_t *__restrict__ n_kept) {
  __shared__ unsigned long long wt[32];
  __shared__ unsigned long long carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nt; base += 1024) {
    const int64_t t = base + tid;
    const unsigned long long c = t < nt ? tcount[t] : 0ull;
    unsigned long long incl = c;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wt[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const unsigned long long v = wt[lane];
      unsigned long long s = v;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long u = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += u;
      }
      wt[lane] = s - v;
    }
    __syncthreads();
    const unsigned long long ex = carry + wt[wid] + incl - c;
    if (t < nt) tcount[t] = ex;  // becomes the tile's output offset
    __syncthreads();
    if (tid == 1023) carry = ex + c;
    __syncthreads();
  }
  if (tid == 0) *n_kept = (int64_t)carry;
}

struct PrunePlanes {
  const float *in[15];
  float *out[15];
  const void *in_idx[32];
  void *out_idx[32];
  int n_idx, idx_bytes, mask_plane;
  int64_t out_stride_idx;  // output idx plane stride (capacity)
  int64_t out_cap;
};

__global__ void __launch_bounds__(kPT) k_prune_scatter(int64_t n, const int64_t *__restrict__ n_dev,
                                                       float tau, float reset, int do_reset,
                                                       const unsigned long long *__restrict__ toff,
                                                       PrunePlanes pp,
                                                       int32_t *__restrict__ keep_map) {
  __shared__ int wpre[kPT / 32 + 1];
  const int64_t ne = eff_n(n, n_dev);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * kPTile;
  int64_t off = (int64_t)toff[blockIdx.x];
  const float *mask = pp.in[pp.mask_plane];
  for (int k = 0; k < kPItems; k++) {
    const int64_t i = base + (int64_t)k * kPT + threadIdx.x;
    const bool keep = i < ne && mask[i] > tau;  // Eq 6: M = 1 iff Sig(m) > eps
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    const int wr = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) wpre[wid] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int s = 0;
      for (int w = 0; w < kPT / 32; w++) {
        const int t = wpre[w];
        wpre[w] = s;
        s += t;
      }
      wpre[kPT / 32] = s;
    }
    __syncthreads();
    const int64_t pos = off + wpre[wid] + wr;
    if (i < n && keep_map) keep_map[i] = keep ? (int32_t)pos : -1;
    if (keep && pos < pp.out_cap) {
#pragma unroll
      for (int p = 0; p < 15; p++) {
        float v = pp.in[p][i];
        if (p == pp.mask_plane && do_reset) v = reset;
        pp.out[p][pos] = v;
      }
      for (int p = 0; p < pp.n_idx; p++) {
        if (pp.idx_bytes == 1)
          static_cast<uint8_t *>(pp.out_idx[p])[pos] = static_cast<const uint8_t *>(pp.in_idx[p])[i];
        else
          static_cast<uint16_t *>(pp.out_idx[p])[pos] = static_cast<const uint16_t *>(pp.in_idx[p])[i];
      }
    }
    off += wpre[kPT / 32];
    __syncthreads();
  }
}

// Look-back status words: bits 62-63 = 0 (not yet published), 1 (the tile's
// own count), 2 (inclusive prefix through the tile); bits 0-61 the value.
constexpr unsigned long long kStA = 1ull << 62, kStP = 2ull << 62, kStVal = (1ull << 62) - 1;

__global__ void __launch_bounds__(kPT) k_prune_onepass(int64_t n, const int64_t *__restrict__ n_dev,
                                                       int64_t nt, float tau, float reset,
                                                       int do_reset,
                                                       unsigned long long *__restrict__ status,
                                                       PrunePlanes pp,
                                                       int32_t *__restrict__ keep_map,
                                                       int64_t *__restrict__ n_kept) {
  __shared__ int wpre[kPItems][kPT / 32 + 1];
  __shared__ long long s_tile;
  __shared__ unsigned long long s_prefix;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned int *ticket = reinterpret_cast<unsigned int *>(status + nt);
  if (threadIdx.x == 0) s_tile = (long long)atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t ne = eff_n(n, n_dev);
  const int64_t base = tile * kPTile;
  const float *mask = pp.in[pp.mask_plane];
  bool keep[kPItems];
  int wr[kPItems];
  float v[kPItems][15];
#pragma unroll
  for (int k = 0; k < kPItems; k++) {
    const int64_t i = base + (int64_t)k * kPT + threadIdx.x;
    keep[k] = i < ne && mask[i] > tau;  // Eq 6: M = 1 iff Sig(m) > eps
    const unsigned bal = __ballot_sync(0xffffffffu, keep[k]);
    wr[k] = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) wpre[k][wid] = __popc(bal);
#pragma unroll
#ifdef CSPLAT_PRUNE_LOAD_KEPT
    for (int p = 0; p < 15; p++) v[k][p] = keep[k] ? pp.in[p][i] : 0.0f;  // in flight early
#else
    // not predicated on the mask test: the plane loads go out with the mask load
    // (one memory round trip instead of two; the masked ones are read in vain)
    for (int p = 0; p < 15; p++) v[k][p] = i < ne ? pp.in[p][i] : 0.0f;
#endif
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive warp offsets of every round; the tile total
    int t = 0;
    for (int k = 0; k < kPItems; k++) {
      for (int w = 0; w < kPT / 32; w++) {
        const int c = wpre[k][w];
        wpre[k][w] = t;
        t += c;
      }
      wpre[k][kPT / 32] = t;
    }
    const unsigned long long agg = (unsigned long long)t;
    atomicExch(status + tile, (tile == 0 ? kStP : kStA) | agg);
  }
  if (wid == 0) {  // decoupled look-back over the preceding tiles
    unsigned long long prefix = 0;
    int64_t j = tile - 1;
    while (j >= 0) {
      const int64_t jj = j - lane;
      unsigned long long w = kStP;  // beyond tile 0: an inclusive prefix of 0
      if (jj >= 0) {
        do {
          w = *reinterpret_cast<volatile unsigned long long *>(status + jj);
        } while ((w >> 62) == 0);
      }
      const unsigned pm = __ballot_sync(0xffffffffu, (w >> 62) == 2);
      const int stop = pm ? __ffs(pm) - 1 : 32;  // nearest tile with an inclusive prefix
      unsigned long long add = lane <= stop ? (w & kStVal) : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
      prefix += add;
      if (pm) break;
      j -= 32;
    }
    if (lane == 0) {
      s_prefix = prefix;
      const unsigned long long tot = prefix + (unsigned long long)wpre[kPItems - 1][kPT / 32];
      if (tile > 0) atomicExch(status + tile, kStP | tot);
      if (tile == nt - 1) *n_kept = (int64_t)tot;
    }
  }
  __syncthreads();
  const int64_t off = (int64_t)s_prefix;
#pragma unroll
  for (int k = 0; k < kPItems; k++) {
    const int64_t i = base + (int64_t)k * kPT + threadIdx.x;
    const int64_t pos = off + wpre[k][wid] + wr[k];
    if (i < n && keep_map) keep_map[i] = keep[k] ? (int32_t)pos : -1;
    if (keep[k] && pos < pp.out_cap) {
#pragma unroll
      for (int p = 0; p < 15; p++)
        pp.out[p][pos] = (p == pp.mask_plane && do_reset) ? reset : v[k][p];
      for (int p = 0; p < pp.n_idx; p++) {
        if (pp.idx_bytes == 1)
          static_cast<uint8_t *>(pp.out_idx[p])[pos] = static_cast<const uint8_t *>(pp.in_idx[p])[i];
        else
          static_cast<uint16_t *>(pp.out_idx[p])[pos] = static_cast<const uint16_t *>(pp.in_idx[p])[i];
      }
    }
  }
}

cudaError_t launch_prune(const csplat_gaussians &in, const DecodeArgs *idx, float tau, float reset,
                         const csplat_gaussians_out &out, void *out_sidx, void *out_ridx,
                         int32_t *keep_map, int64_t *n_kept, void *ws, cudaStream_t s) {
  const int64_t n = in.n;
  const int64_t nt = (n + kPTile - 1) / kPTile;
  unsigned long long *tcount = static_cast<unsigned long long *>(ws);
#ifdef CSPLAT_PRUNE_3PASS
  if (nt > 0)
    k_prune_count<<<(unsigned)nt, kPT, 0, s>>>(n, in.n_dev, in.mask, tau, tcount);
  k_prune_scan<<<1, 1024, 0, s>>>(nt, tcount, n_kept);
  if (nt == 0) return cudaGetLastError();
#else
  if (nt == 0) return cudaMemsetAsync(n_kept, 0, sizeof(int64_t), s);
  // status words + the tile ticket start at zero
  cudaError_t e = cudaMemsetAsync(tcount, 0, (size_t)(nt + 1) * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
#endif
  PrunePlanes pp{};
  const float *ins[6] = {in.mean, in.opacity, in.rgb, in.log_scale, in.quat, in.mask};
  float *outs[6] = {out.mean, out.opacity, out.rgb, out.log_scale, out.quat, out.mask};
  const int rows[6] = {3, 1, 3, 3, 4, 1};
  int p = 0;
  for (int a = 0; a < 6; a++)
    for (int r = 0; r < rows[a]; r++, p++) {
      pp.in[p] = ins[a] + (int64_t)r * n;
      pp.out[p] = outs[a] + (int64_t)r * out.capacity;
    }
  pp.mask_plane = 14;
  pp.out_cap = out.capacity;
  pp.n_idx = 0;
  if (idx) {
    pp.idx_bytes = idx->idx_bytes;
    for (int l = 0; l < idx->L; l++) {
      pp.in_idx[pp.n_idx] = static_cast<const char *>(idx->scale_idx) + (int64_t)l * n * idx->idx_bytes;
      pp.out_idx[pp.n_idx++] = static_cast<char *>(out_sidx) + (int64_t)l * out.capacity * idx->idx_bytes;
    }
    for (int l = 0; l < idx->L; l++) {
      pp.in_idx[pp.n_idx] = static_cast<const char *>(idx->rot_idx) + (int64_t)l * n * idx->idx_bytes;
      pp.out_idx[pp.n_idx++] = static_cast<char *>(out_ridx) + (int64_t)l * out.capacity * idx->idx_bytes;
    }
  }
  const bool do_reset = !(reset != reset);  // reset is not NaN
#ifdef CSPLAT_PRUNE_3PASS
  k_prune_scatter<<<(unsigned)nt, kPT, 0, s>>>(n, in.n_dev, tau, reset, do_reset ? 1 : 0, tcount,
                                               pp, keep_map);
#else
  k_prune_onepass<<<(unsigned)nt, kPT, 0, s>>>(n, in.n_dev, nt, tau, reset, do_reset ? 1 : 0,
                                               tcount, pp, keep_map, n_kept);
#endif
  return cudaGetLastError();
}

}  // namespace csplat
