// prune.cu -- a9: mask prune (Fig 3): remove every
// Gaussian whose mask is off (m <= tau, Eq 6 / R12) and compact the survivors
// of every attribute plane (and the R-VQ index planes) in their original order.
//
// One pass (k_prune_onepass): each CTA takes the next tile of kPTile Gaussians
// (dynamic ticket), loads its masks and attribute planes, publishes the tile's
// survivor count, finds its output offset by a decoupled look-back over the
// preceding tiles' published counts / inclusive prefixes (warp-parallel, 32
// tiles per probe), and scatters the survivors in order (ballot/popc ranks
// inside each 256-element round, a warp-total scan across the CTA); the
// three-launch form (count -> one-CTA scan -> scatter) measured 33 vs 16 us at
// C2 and is gone.  Reads and writes are coalesced per round.
// HBM-bound: 4 + 60 + 2L bytes read per Gaussian, 60 + 2L (+4 keep_map)
// written per survivor.
#include "common.cuh"

namespace csplat {

constexpr int kPT = 256;         // threads per CTA
constexpr int kPItems = 2;  // rounds per CTA (keeps >= 2 waves of CTAs at 200k)
constexpr int kPTile = kPT * kPItems;

size_t prune_workspace_bytes(int64_t n) {
  const int64_t nt = (n + kPTile - 1) / kPTile;
  return (size_t)(nt + 2) * sizeof(unsigned long long) + 256;
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
    // not predicated on the mask test: the plane loads go out with the mask load
    // (one memory round trip instead of two; the masked ones are read in vain)
    for (int p = 0; p < 15; p++) v[k][p] = i < ne ? pp.in[p][i] : 0.0f;
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
  if (nt == 0) return cudaMemsetAsync(n_kept, 0, sizeof(int64_t), s);
  // status words + the tile ticket start at zero
  cudaError_t e = cudaMemsetAsync(tcount, 0, (size_t)(nt + 1) * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
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
  k_prune_onepass<<<(unsigned)nt, kPT, 0, s>>>(n, in.n_dev, nt, tau, reset, do_reset ? 1 : 0,
                                               tcount, pp, keep_map, n_kept);
  return cudaGetLastError();
}

}  // namespace csplat
