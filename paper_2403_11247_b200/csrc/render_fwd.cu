// render_fwd.cu -- a6: front-to-back alpha compositing of colour, depth and
// silhouette (Eq 3-5; readings R1-R3, R7-R10).
//
// One CTA of 128 threads per 16x16 screen tile; each thread owns two vertically
// adjacent pixels (they share dx and the per-record loads), so a warp owns an
// 8x8 pixel block.  The tile's records are a contiguous slice of the
// pair-ordered payload written by csplat_bin_tiles and are streamed into
// shared memory by 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx)
// through a kStages-deep ring of kBatch-record batches fed by a producer warp;
// every record is read from shared memory as a broadcast.  A warp skips a
// record whose 8x8-block cull bit (payload word 14, bin.cu) is clear
// (result-invariant).  The tile's stream ends once every pixel terminated
// (T(1-alpha) < t_min, R3), checked once per batch and warp.  The per-pixel q test is
// the DA of DESIGN.md §3 (bit-exact with the oracle); alpha, T and the sums
// are float32 with ex2.approx.
#include "composite.cuh"

namespace csplat {

constexpr int kBatch = 32;   // records per TMA batch (2 KB)
constexpr int kStages = 4;   // ring depth (2: 85.7 us at C2; 3, 4, 6: 82.6-83.1 us)
constexpr int kPW = 4;       // pixel warps: 8x8 pixels each, two per thread

// Each thread owns a column of two vertically adjacent pixels: a pixel warp
// owns an 8x8 block, four pixel warps one 16x16 tile, plus one producer warp.  The producer streams the tile's batches into the ring
// (mbarrier full[] with complete_tx) and refills a slot once every pixel warp
// has released it (empty[], one arrival per warp); the pixel warps never
// synchronise with each other, so a warp with a heavy block does not hold the
// others at a CTA barrier.  A warp whose pixels all terminated counts itself
// in done_cnt and from then on only releases slots; once all have, the
// producer ends the stream by completing the next full[] phase without data
// (end_b), and every pixel warp leaves at that batch.
__global__ void __launch_bounds__((kPW + 1) * 32) k_render_fwd(
    const __grid_constant__ CUtensorMap tmap, const uint32_t *__restrict__ pair_gid,
    const uint32_t *__restrict__ range, int W, int H,
    int tiles_x, float amax, float tmin, float *__restrict__ color, float *__restrict__ depth,
    float *__restrict__ sil, float *__restrict__ t_final, int32_t *__restrict__ n_contrib,
    int tile0, const int32_t *__restrict__ list) {
  __shared__ __align__(128) float4 buf[kStages][kBatch * 4];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ uint32_t msk[kStages][kBatch];  // the entries' 8x8-block cull masks
  __shared__ int done_cnt, end_b;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // list mode (NEXT-4 sparse views): CTA b renders list tile b of list[0]
  if (list && (int)blockIdx.x >= list[0]) return;
  const int tile = list ? list[1 + blockIdx.x] : tile0 + (int)blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const uint32_t start = range[2 * tile], end = range[2 * tile + 1];
  const int len = (int)(end - start);
  const int nb = (len + kBatch - 1) / kBatch;

  if (tid == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 32);  // the producer warp's 32 lanes (+ the batch's TMA bytes)
      mbar_init(&empty[s], kPW);
    }
    done_cnt = 0;
    end_b = -1;
    fence_mbar_init();
  }
  __syncthreads();

  if (wid == kPW) {  // ---- producer warp
    // batch b: lane l takes list entry b*kBatch + l (pair_gid: Gaussian index |
    // block mask << 28, loaded one batch ahead), stores its mask into msk[s]
    // and gathers its record with one 64-byte TMA bulk copy (gather_batch)
    uint32_t entry = lane < len ? pair_gid[start + lane] : 0u;
    for (int b = 0; b < nb; b++) {
      const int s = b % kStages;
      if (b >= kStages) mbar_wait_sleep(&empty[s], (uint32_t)((b / kStages) - 1) & 1u);
      // every pixel terminated: end the stream (one lane reads, all agree)
      if (__shfl_sync(0xffffffffu, lane == 0 ? *(volatile int *)&done_cnt : 0, 0) == kPW) {
        if (lane == 0) end_b = b;
        mbar_arrive(&full[s]);  // 32 arrivals, no bytes: the phase completes empty
        break;
      }
      const int cnt = min(kBatch, len - b * kBatch);
      const uint32_t e = entry;
      if (b * kBatch + lane + kBatch < len) entry = pair_gid[start + b * kBatch + lane + kBatch];
      gather_batch(&buf[s][0], msk[s], &tmap, e, lane, cnt, &full[s]);
    }
    return;
  }

  // ---- pixel warps
  const int wx0 = tx * kTile + (wid & 1) * 8, wy0 = ty * kTile + (wid >> 1) * 8;
  const int px = wx0 + (lane & 7), py0 = wy0 + (lane >> 3) * 2;
  PixState p[2];
  int mydone = 1;
#pragma unroll
  for (int k = 0; k < 2; k++) {
    p[k] = PixState{1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0, (px < W && py0 + k < H) ? 0 : 1};
    mydone &= p[k].done;
  }
  bool wdone = __all_sync(0xffffffffu, mydone);
  if (wdone && lane == 0) atomicAdd(&done_cnt, 1);
  const float fpx = (float)px;
  const f2_t FPY = pk2((float)py0, (float)(py0 + 1));
  for (int b = 0; b < nb; b++) {
    const int s = b % kStages;
    mbar_wait_sleep(&full[s], (uint32_t)(b / kStages) & 1u);
    if (*(volatile int *)&end_b == b) break;
    if (!wdone) {
      const float4 *rb = buf[s];
      const int cnt = min(kBatch, len - b * kBatch);
      // the batch's entries this warp composites, one ballot: lane l tests entry
      // l's 8x8-block mask (payload word 14, bin.cu)
      const bool mine = lane < cnt && ((msk[s][lane] >> wid) & 1u);
      uint32_t todo = __ballot_sync(0xffffffffu, mine);
      while (todo) {  // front to back
        const int e = __ffs(todo) - 1;
        todo &= todo - 1u;
        const float4 r0 = rb[e * 4 + 0];  // u, v, ca, cb+cb
        const float4 r1 = rb[e * 4 + 1];  // cc, o_hat, k2, z
        const float dx = DSUB(fpx, r0.x);
        const float cadx = DMUL(r0.z, dx), cbdx = DMUL(r0.w, dx);
        // the DA q of both pixels on f32x2 (same roundings as the scalar DA form)
        const f2_t DY = sub2(FPY, pk2(r0.y, r0.y));
        const f2_t Q = fma2(pk2(cadx, cadx), pk2(dx, dx),
                            fma2(pk2(cbdx, cbdx), DY, mul2(mul2(pk2(r1.x, r1.x), DY), DY)));
        const float q0 = lo2(Q), q1 = hi2(Q);
        // R2 (DA): 0 <= q <= k2
        const bool h0 = (p[0].done == 0) & da_in_range(q0, r1.z);
        const bool h1 = (p[1].done == 0) & da_in_range(q1, r1.z);
        // warp-uniform skip: composite_pair is an exact no-op for pixels whose
        // test failed, so lanes without a hit ride along predicated
        if (!__any_sync(0xffffffffu, h0 | h1)) continue;
        const float4 r2 = rb[e * 4 + 2];  // r, g, b, gid
        composite_pair(p[0], p[1], h0, h1, q0, q1, r1.y, r1.w, r2, amax, tmin, b * kBatch + e + 1);
      }
      mydone = p[0].done & p[1].done;
      wdone = __all_sync(0xffffffffu, mydone);
      if (wdone && lane == 0) atomicAdd(&done_cnt, 1);  // before the release below
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // release the slot
  }
  const int64_t HW = (int64_t)W * H;
  if (px < W) {
#pragma unroll
    for (int k = 0; k < 2; k++) {
      if (py0 + k >= H) continue;
      const int64_t o = (int64_t)(py0 + k) * W + px;
      color[o] = p[k].r; color[HW + o] = p[k].g; color[2 * HW + o] = p[k].b;
      depth[o] = p[k].D; sil[o] = p[k].S; t_final[o] = p[k].T; n_contrib[o] = p[k].last;
    }
  }
}

cudaError_t launch_render_fwd(const void *rec, const uint32_t *pair_gid,
                              const uint32_t *tile_range,
                              const csplat_camera &cam, const csplat_params &prm, float *color,
                              float *depth, float *sil, float *t_final, int32_t *n_contrib,
                              cudaStream_t s, int tile0, int ntiles, const int32_t *list) {
  const CamInfo ci = cam_info(cam);
  const int T = ci.tiles_x * ci.tiles_y;
  if (ntiles < 0) ntiles = T - tile0;
  if (ntiles <= 0) return cudaSuccess;
  CUtensorMap tmap;
  cudaError_t e = rec_tensor_map(rec, &tmap);
  if (e != cudaSuccess) return e;
  k_render_fwd<<<ntiles, (kPW + 1) * 32, 0, s>>>(
      tmap, pair_gid, tile_range, ci.W, ci.H, ci.tiles_x, prm.alpha_max,
      prm.t_min, color, depth, sil, t_final, n_contrib, tile0, list);
  return cudaGetLastError();
}

}  // namespace csplat
