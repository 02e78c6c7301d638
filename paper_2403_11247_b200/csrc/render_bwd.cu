// render_bwd.cu -- a7: backward of the front-to-back compositing (Eq 3-5,
// P:98-109) -- the paper's "functions to manage depth, pose, and cumulative
// opacity during both forward and backward propagation"; R23.
//
// Per pixel, from T_final and n_contrib, back to front over the composited
// entries: T_j = T_{j+1} / (1 - alpha_j), v_j = <rgb_j, dL/dC> + z_j dL/dD +
// dL/dS, dL/dalpha_j = T_j (v_j - B_j), B_{j-1} = alpha_j v_j + (1 - alpha_j) B_j,
// and per (pixel, entry) the ten partials below, summed per (tile, Gaussian)
// into the [n][12] accumulator that k_chain (chain.cu) turns into parameter
// gradients.  The kernel is the block-list backward (quad.cuh): each 4x4 pixel
// block of a tile walks its own entry list with four lanes.
#include <atomic>

#include "common.cuh"
#include "quad.cuh"

namespace csplat {


// workspace: the [n][12] float accumulator, then a [ceil(n/32)] u32 bitmap of
// the Gaussians that received any partial (the chains visit only those)
static inline size_t acc_bytes(int64_t n) {
  return ((size_t)(n > 0 ? n : 1) * kAcc * sizeof(float) + 255) & ~size_t(255);
}
size_t bwd_workspace_bytes(int64_t n) {
  return acc_bytes(n) + ((size_t)((n > 0 ? n : 1) + 31) / 32 * 4 + 255) / 256 * 256;
}
uint32_t *bwd_alive_bits(void *ws, int64_t n) {
  return reinterpret_cast<uint32_t *>(static_cast<char *>(ws) + acc_bytes(n));
}


// NEXT-1 loss-fused mode: the upstream gradients are
// the tracking objective's (Eq 12 gated by Eq 14, reading R27), formed per
// pixel in the prologue from the rendered and observed images instead of read.
struct LossArgs {
  const float *color, *depth, *sil, *obs_color, *obs_depth;
  const unsigned long long *n_valid;  // |R|: pixels with a valid observed depth
  float lambda_d, gate, inv_n;
  float *loss3;                       // (L_t, L_c, L_d) added
};

// ---------------------------------------------------------------------------
// The block-list backward.  Round 1's kernel replayed, for each 8x8 pixel
// block (one warp, fed by a producer warp's TMA ring), every entry the block
// may touch: on C2 61 % of those (pixel, entry) slots lie outside the entry's
// ellipse, and the warp-wide reduction of the per-entry partials through shared
// memory cost as much as the replay.  Here each 4x4 block has
// its own entry list and its own four lanes (a QUAD, quad.cuh), so a warp
// replays eight independent streams:
//  1. gather (per chunk of up to kChunk list entries, back to front): the
//     chunk's records to shared memory by cp.async, the entries' 4x4-block
//     masks, and per block the list of entries (mask bit set and list position
//     below the block's last contributor);
//  2. replay: quad lane q owns column q of its block (two vertically adjacent
//     pixel pairs, replay state and upstream in registers) and walks the
//     block's list back to front, two entries per iteration (pair_front is
//     independent of the state, so the two fronts interleave; pair_state then
//     applies T_j = T_{j+1} rcp(1 - alpha_j), B_{j-1} = B_j + alpha_j (v_j - B_j)
//     in list order);
//  3. per entry the quad sums its four lanes' ten partials with a transposed
//     shuffle reduction (11 SHFL) and adds them to the [n][12] accumulator with
//     one red.global.add.v4.f32 from each of two lanes and one .v2 from a third.
// No producer warp, no barriers inside the replay; the shared-memory traffic per
// entry is the record (three broadcast loads per quad).
namespace quad {
// 64-thread CTAs per SM: 10 (96 registers, 21.2 KB + 1 KB reserved each, with
// the shared-memory carveout at its maximum) -- 118.8 vs 120.8 us at C2 for 9
// CTAs at 112 registers
constexpr int kMinBlocks = 10;

struct Smem {
  Lists L;
  int wmax[kNB];
};

template <bool LOSS>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_render_bwd_quad(
    const float4 *__restrict__ recs, const uint32_t *__restrict__ pair_gid,
    const uint32_t *__restrict__ range, int W, int H,
    int tiles_x, float amax, const float *__restrict__ t_final,
    const int32_t *__restrict__ n_contrib, const float *__restrict__ dC,
    const float *__restrict__ dD, const float *__restrict__ dS, float *__restrict__ accg,
    uint32_t *__restrict__ alive, LossArgs la, int tile0, const int32_t *__restrict__ list) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem &sm = *reinterpret_cast<Smem *>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int tb = (int)blockIdx.x;
  if (list && tb >= list[0]) return;
  const int tile = list ? list[1 + tb] : tile0 + tb;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const uint32_t start = range[2 * tile];
  const Geo gq = geo(tx, ty, wid, lane);
  const int ri = gq.ri, B = gq.B, px = gq.px, by = gq.by;

  // ---- prologue: the lane's two pixel pairs
  float lc = 0.f, ld = 0.f;
  QPair P[2];
  int mylast = 0;
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int py0 = by + 2 * h;
    float Tv[2], g[2][5];
    int lastv[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const int py = py0 + k;
      Tv[k] = 1.f; lastv[k] = 0;
      g[k][0] = g[k][1] = g[k][2] = g[k][3] = g[k][4] = 0.f;
      if (px < W && py < H) {
        const int64_t HW = (int64_t)W * H, q = (int64_t)py * W + px;
        Tv[k] = t_final[q];
        lastv[k] = n_contrib[q];
        if constexpr (LOSS) {
          const unsigned long long nv = *la.n_valid;
          const float inv_r = 1.0f / (float)(nv > 0 ? nv : 1ull);
          const float gt = la.sil[q] > la.gate ? 1.0f : 0.0f;
          const float obd = la.obs_depth[q];
          const float vd = obd > 0.0f ? 1.0f : 0.0f;
          const float r0 = la.color[q] - la.obs_color[q];
          const float r1 = la.color[HW + q] - la.obs_color[HW + q];
          const float r2 = la.color[2 * HW + q] - la.obs_color[2 * HW + q];
          const float rd = la.depth[q] - obd;
          lc += gt * (r0 * r0 + r1 * r1 + r2 * r2);
          ld += gt * vd * rd * rd;
          const float sc = 2.0f * gt * la.inv_n;
          g[k][0] = sc * r0; g[k][1] = sc * r1; g[k][2] = sc * r2;
          g[k][3] = 2.0f * la.lambda_d * gt * vd * rd * inv_r;
          g[k][4] = 0.0f;
        } else {
          g[k][0] = dC[q]; g[k][1] = dC[HW + q]; g[k][2] = dC[2 * HW + q];
          g[k][3] = dD[q]; g[k][4] = dS[q];
        }
        // all-zero upstream: exact zeros in every partial, no replay
        if (g[k][0] == 0.f && g[k][1] == 0.f && g[k][2] == 0.f && g[k][3] == 0.f &&
            g[k][4] == 0.f)
          lastv[k] = 0;
      }
    }
    mylast = max(mylast, max(lastv[0], lastv[1]));
    P[h].T = pk2(Tv[0], Tv[1]);
    P[h].B = pk2(0.f, 0.f);
    P[h].FPY = pk2((float)py0, (float)(py0 + 1));
    P[h].GR = pk2(g[0][0], g[1][0]); P[h].GG = pk2(g[0][1], g[1][1]);
    P[h].GB = pk2(g[0][2], g[1][2]); P[h].GD = pk2(g[0][3], g[1][3]);
    P[h].GS = pk2(g[0][4], g[1][4]);
    P[h].last0 = lastv[0]; P[h].last1 = lastv[1];
  }
  mylast = max(mylast, __shfl_xor_sync(0xffffffffu, mylast, 1));
  mylast = max(mylast, __shfl_xor_sync(0xffffffffu, mylast, 2));
  if (ri == 0) sm.wmax[B] = mylast;
  if constexpr (LOSS) {
    lc = warp_sum(lc);
    ld = warp_sum(ld);
    if (lane == 0 && (lc != 0.f || ld != 0.f)) {
      const unsigned long long nv = *la.n_valid;
      const float a = lc * la.inv_n, b = ld / (float)(nv > 0 ? nv : 1ull);
      atomicAdd(la.loss3 + 0, a + la.lambda_d * b);
      atomicAdd(la.loss3 + 1, a);
      atomicAdd(la.loss3 + 2, b);
    }
  }
  __syncthreads();
  int maxlast = 0;
  uint32_t need8 = 0;  // 8x8 blocks with a pixel to replay (sparse upstream: the BA's patches)
#pragma unroll
  for (int b = 0; b < kNB; b++) {
    maxlast = max(maxlast, sm.wmax[b]);
    if (sm.wmax[b] > 0) need8 |= 1u << (((b & 3) >> 1) + 2 * ((b >> 2) >> 1));
  }
  const int X0 = tx * kTile, Y0 = ty * kTile;
  const float fpx = (float)px;

  // chunks of the list, back to front
  for (int c1 = maxlast; c1 > 0; c1 -= kChunk) {
    const int c0 = max(0, c1 - kChunk), len = c1 - c0;
    // 1. the chunk's records, 4x4-block masks and the blocks' lists, back to front
    gather(sm.L, recs, pair_gid, start, c0, len, X0, Y0, alive, tid, need8);
    build_lists(sm.L, c0, len, sm.wmax, wid, lane);
    // 2. the replay: the quad walks its block's list; 3. quad sums -> accumulator
    replay_chunk(sm.L, P, B, ri, c0, fpx, amax, accg);
    // before the next chunk overwrites the records and lists (after the last
    // chunk a warp just exits)
    if (c0 > 0) __syncthreads();
  }
}
}  // namespace quad

// zero the accumulator (and the pose gradient unless accumulating)
cudaError_t bwd_prep(const csplat_gaussians &g, uint32_t flags, const csplat_grads &out,
                     void *ws, const TrackingLoss *loss, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  if (!(flags & CSPLAT_WS_ZEROED)) e = cudaMemsetAsync(ws, 0, bwd_workspace_bytes(g.n), s);
  if (e != cudaSuccess) return e;
  if (out.pose && !(flags & (CSPLAT_ACCUMULATE | CSPLAT_SKIP_CHAIN))) {
    e = cudaMemsetAsync(out.pose, 0, 6 * sizeof(float), s);
    if (e != cudaSuccess) return e;
  }
  if (loss && loss->loss3) e = cudaMemsetAsync(loss->loss3, 0, 3 * sizeof(float), s);
  return e;
}

// the backward kernel over tiles [tile0, tile0 + ntiles) (ntiles < 0: to the
// end); the per-Gaussian accumulation is by atomics, so tile chunks may run in
// any order or concurrently
cudaError_t launch_render_bwd_tiles(const csplat_camera &cam, const TrackingLoss *loss,
                                    const csplat_params &prm, const void *rec,
                                    const uint32_t *pair_gid, const uint32_t *tile_range, const float *t_final,
                                    const int32_t *n_contrib, const float *d_color,
                                    const float *d_depth, const float *d_sil, void *ws,
                                    int64_t n, cudaStream_t s, int tile0, int ntiles,
                                    const int32_t *list) {
  const CamInfo ci = cam_info(cam);
  float *acc = static_cast<float *>(ws);
  uint32_t *alive = bwd_alive_bits(ws, n);
  const size_t smem = sizeof(quad::Smem);
  // the opt-in shared-memory size: set once per device (a race between host
  // threads only repeats the idempotent call)
  static std::atomic<unsigned long long> attr_done{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr_done.load(std::memory_order_acquire) & bit)) {
    e = cudaFuncSetAttribute(quad::k_render_bwd_quad<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(quad::k_render_bwd_quad<false>,
                               cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(quad::k_render_bwd_quad<true>,
                               cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(quad::k_render_bwd_quad<true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_done.fetch_or(bit, std::memory_order_release);
  }
  const int T = ci.tiles_x * ci.tiles_y;
  if (ntiles < 0) ntiles = T - tile0;
  if (ntiles <= 0) return cudaSuccess;
  const float4 *rec4 = static_cast<const float4 *>(rec);
  LossArgs la{};
  if (loss) {
    la.color = loss->color; la.depth = loss->depth; la.sil = loss->sil;
    la.obs_color = loss->obs_color; la.obs_depth = loss->obs_depth;
    la.n_valid = loss->n_valid; la.lambda_d = loss->lambda_d; la.gate = loss->gate;
    la.inv_n = 1.0f / (float)((int64_t)ci.W * ci.H);
    la.loss3 = loss->loss3;
    quad::k_render_bwd_quad<true><<<ntiles, quad::kThreads, smem, s>>>(
        rec4, pair_gid, tile_range, ci.W, ci.H, ci.tiles_x, prm.alpha_max, t_final, n_contrib,
        nullptr, nullptr, nullptr, acc, alive, la, tile0, list);
  } else {
    quad::k_render_bwd_quad<false><<<ntiles, quad::kThreads, smem, s>>>(
        rec4, pair_gid, tile_range, ci.W, ci.H, ci.tiles_x, prm.alpha_max, t_final, n_contrib,
        d_color, d_depth, d_sil, acc, alive, la, tile0, list);
  }
  return cudaGetLastError();
}

cudaError_t launch_render_bwd(const csplat_gaussians &g, const DecodeArgs *dec,
                              const csplat_camera &cam, const csplat_view &view,
                              const float *view_dev, const TrackingLoss *loss,
                              const csplat_params &prm, const void *rec, const uint32_t *pair_gid,
                              const uint32_t *tile_range, const float *t_final,
                              const int32_t *n_contrib, const float *d_color, const float *d_depth,
                              const float *d_sil, uint32_t flags, const csplat_grads &out,
                              void *ws, cudaStream_t s, const int32_t *list, int max_tiles) {
  cudaError_t e = bwd_prep(g, flags, out, ws, loss, s);
  if (e != cudaSuccess) return e;
  e = launch_render_bwd_tiles(cam, loss, prm, rec, pair_gid, tile_range, t_final, n_contrib, d_color,
                              d_depth, d_sil, ws, g.n, s, 0, list ? max_tiles : -1, list);
  if (e != cudaSuccess || g.n == 0 || (flags & CSPLAT_SKIP_CHAIN)) return e;
  return launch_chain(g, dec, cam, view, view_dev, prm, rec, static_cast<float *>(ws), flags,
                      out, s);
}

}  // namespace csplat
