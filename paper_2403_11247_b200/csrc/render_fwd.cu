// render_fwd.cu -- a6: front-to-back alpha compositing of colour, depth and
// silhouette (Eq 3-5; readings R1-R3, R7-R10).
//
// One CTA per 16x16 screen tile, one thread per pixel; the 8 warps each own an
// 8x4 pixel rectangle (tighter than 16x2 rows for the warp-level cull).  The
// tile's records are a contiguous slice of the pair-ordered payload written by
// csplat_bin_tiles, so they are streamed into shared memory with 1-D TMA bulk
// copies (cp.async.bulk, mbarrier complete_tx) through a kStages-deep ring of
// kBatch-record batches; thread 0 is the producer.  Every record is read from
// shared memory as a broadcast.  A warp skips a record whose pixel rectangle
// misses the warp's 8x4 pixels (result-invariant); the CTA stops when every
// pixel has terminated (T(1-alpha) < t_min, R3) -- checked once per batch.
// The per-pixel q test is the DA of DESIGN.md §3 (bit-exact with the oracle);
// alpha, T and the sums are float32 with ex2.approx.
#include "common.cuh"

namespace csplat {

constexpr int kBatch = 32;   // records per TMA batch (2 KB)
constexpr int kStages = 4;   // ring depth

__global__ void __launch_bounds__(256) k_render_fwd(
    const float4 *__restrict__ pair_rec, const uint32_t *__restrict__ range, int W, int H,
    int tiles_x, float amax, float tmin, float *__restrict__ color, float *__restrict__ depth,
    float *__restrict__ sil, float *__restrict__ t_final, int32_t *__restrict__ n_contrib) {
  __shared__ __align__(128) float4 buf[kStages][kBatch * 4];
  __shared__ __align__(8) uint64_t full[kStages];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int wx0 = tx * kTile + (wid & 1) * 8, wy0 = ty * kTile + (wid >> 1) * 4;
  const int px = wx0 + (lane & 7), py = wy0 + (lane >> 3);
  const bool inside = px < W && py < H;
  const uint32_t start = range[2 * tile], end = range[2 * tile + 1];
  const int len = (int)(end - start);
  const int nb = (len + kBatch - 1) / kBatch;

  if (tid == 0) {
    for (int s = 0; s < kStages; s++) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int issued = 0;
  auto issue = [&](int b) {
    const int cnt = min(kBatch, len - b * kBatch);
    const uint32_t bytes = (uint32_t)cnt * CSPLAT_RECORD_BYTES;
    uint64_t *bar = &full[b % kStages];
    mbar_arrive_expect_tx(bar, bytes);
    tma_load_1d(&buf[b % kStages][0], pair_rec + ((int64_t)start + (int64_t)b * kBatch) * 4, bytes,
                bar);
  };
  if (tid == 0)
    for (; issued < min(kStages - 1, nb); issued++) issue(issued);

  float T = 1.0f, cr = 0.f, cg = 0.f, cbl = 0.f, D = 0.f, S = 0.f;
  int32_t last = 0;
  bool done = !inside;
  const float fpx = (float)px, fpy = (float)py;
  int b = 0;
  for (; b < nb; b++) {
    if (__syncthreads_and(done)) break;
    if (tid == 0 && issued < nb && issued <= b + kStages - 1) issue(issued++);
    mbar_wait(&full[b % kStages], (uint32_t)(b / kStages) & 1u);
    const float4 *rb = buf[b % kStages];
    const int cnt = min(kBatch, len - b * kBatch);
    for (int e = 0; e < cnt; e++) {
      const float4 r3 = rb[e * 4 + 3];
      const uint32_t rx = __float_as_uint(r3.x), ry = __float_as_uint(r3.y);
      // warp-level cull: record's pixel rectangle vs this warp's 8x4 pixels
      if ((int)(rx & 0xffffu) > wx0 + 7 || (int)(rx >> 16) < wx0 || (int)(ry & 0xffffu) > wy0 + 3 ||
          (int)(ry >> 16) < wy0)
        continue;
      if (done) continue;
      const float4 r0 = rb[e * 4 + 0];
      const float4 r1 = rb[e * 4 + 1];
      const float q = da_q(fpx, fpy, r0.x, r0.y, r0.z, r0.w, r1.x);
      if (!(q >= 0.0f && q <= r1.z)) continue;  // R2 (DA)
      const float alpha = fminf(amax, r1.y * __expf(-0.5f * q));
      const float test = T * (1.0f - alpha);
      if (test < tmin) {  // R3: the triggering entry is not composited
        done = true;
        continue;
      }
      const float4 r2 = rb[e * 4 + 2];
      const float w = alpha * T;
      cr = fmaf(r2.x, w, cr);   // Eq 3
      cg = fmaf(r2.y, w, cg);
      cbl = fmaf(r2.z, w, cbl);
      D = fmaf(r1.w, w, D);     // Eq 4 (R8)
      S += w;                   // Eq 5 (R9)
      T = test;
      last = b * kBatch + e + 1;
    }
  }
  // never leave the CTA with bulk copies in flight into its shared memory
  if (tid == 0)
    for (int bb = b; bb < issued; bb++) mbar_wait(&full[bb % kStages], (uint32_t)(bb / kStages) & 1u);
  if (inside) {
    const int64_t p = (int64_t)py * W + px, HW = (int64_t)W * H;
    color[p] = cr;
    color[HW + p] = cg;
    color[2 * HW + p] = cbl;
    depth[p] = D;
    sil[p] = S;
    t_final[p] = T;
    n_contrib[p] = last;
  }
}

cudaError_t launch_render_fwd(const void *pair_rec, const uint32_t *tile_range,
                              const csplat_camera &cam, const csplat_params &prm, float *color,
                              float *depth, float *sil, float *t_final, int32_t *n_contrib,
                              cudaStream_t s) {
  const CamInfo ci = cam_info(cam);
  const int T = ci.tiles_x * ci.tiles_y;
  k_render_fwd<<<T, 256, 0, s>>>(static_cast<const float4 *>(pair_rec), tile_range, ci.W, ci.H,
                                 ci.tiles_x, prm.alpha_max, prm.t_min, color, depth, sil, t_final,
                                 n_contrib);
  return cudaGetLastError();
}

}  // namespace csplat
