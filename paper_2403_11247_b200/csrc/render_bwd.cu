// render_bwd.cu -- a7: backward of the front-to-back compositing (Eq 3-5,
// P:98-109) -- the paper's "functions to manage depth, pose, and cumulative
// opacity during both forward and backward propagation"; R23.
//
// One CTA per 16x16 tile: 4 pixel warps (two vertically adjacent pixels per
// thread, 8x8 pixels per warp) plus 1 producer warp.  The producer streams the
// tile's records back to front with 1-D TMA bulk copies into a kBS-slot ring
// (mbarrier full[] with complete_tx) and, once all pixel warps have released a
// slot (mbarrier empty[], one arrival per warp), folds the warps' per-entry
// partial sums for that batch into the global [n][12] accumulator with three
// red.global.add.v4.f32 per (tile, Gaussian).  The pixel warps never wait for
// each other: no CTA barrier inside the replay, so a warp with a heavy 8x8
// block does not stall the others.
//
// Per pixel, from T_final and n_contrib: T_j = T_{j+1} / (1 - alpha_j),
// v_j = <rgb_j, dL/dC> + z_j dL/dD + dL/dS, dL/dalpha_j = T_j (v_j - B_j),
// B_{j-1} = alpha_j v_j + (1-alpha_j) B_j.  A thread adds its two pixels'
// ten partials (u, v, ca, cb, cc, o_hat, z, r, g, b) in registers; the warp
// stores the lanes' partials of kG entries as shared-memory rows and each lane
// sums whole rows with rotated LDS.128 (a transposed reduction: ~2
// instructions per (entry, value) instead of a 10-instruction shuffle tree).
#include "common.cuh"

namespace csplat {

constexpr int kBB = 32;           // records per TMA batch
#ifndef KBS_OVERRIDE
#define KBS_OVERRIDE 3
#endif
constexpr int kBS = KBS_OVERRIDE; // ring depth
constexpr int kAcc = 12;          // accumulator floats per Gaussian
constexpr int kCW = 4;            // pixel (consumer) warps: 4 x 32 lanes x 2 pixels = 16x16
constexpr int kBwdThreads = (kCW + 1) * 32;  // + 1 producer warp
constexpr int kG = 4;             // entries per transposed-reduction group (smem vs occupancy)
constexpr int kV = 10;            // partials per (pixel, entry)
#ifndef CSPLAT_BWD_MIN_BLOCKS
#define CSPLAT_BWD_MIN_BLOCKS 5
#endif
constexpr int kBwdMinBlocks = CSPLAT_BWD_MIN_BLOCKS;  // CTAs per SM the register budget targets

size_t bwd_workspace_bytes(int64_t n) { return (size_t)(n > 0 ? n : 1) * kAcc * sizeof(float); }

struct BwdSmem {
  float4 buf[kBS][kBB * 4];             // staged records
  float4 red[kCW][kG * kV][8];          // per-warp rows of 32 lane partials
  float part[kBS][kCW][kBB][kAcc];      // per-slot, per-warp sums per batch entry
  uint64_t full[kBS], empty[kBS];
  uint32_t pact[kBS][kCW];              // did warp w write part[slot][w]?
  uint32_t act[kCW][kG];
  int wmax[kCW];
};

__device__ __forceinline__ float ex2_approx_b(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}


struct BPix {
  float T, B, gr, gg, gb, gd, gs;
  int last;
};

// One (pixel, entry) of the replay; adds its partials into v and returns
// whether the entry contributed to this pixel.
__device__ __forceinline__ bool bwd_pixel(BPix &p, int j, float dx, float dy, const float4 &r0,
                                          const float4 &r1, const float4 &r2, float amax,
                                          float (&v)[kV]) {
  if (j >= p.last) return false;
  // DA q, bit-identical to the forward's
  const float q = DFMA(DMUL(r0.z, dx), dx, DFMA(DMUL(r0.w, dx), dy, DMUL(DMUL(r1.x, dy), dy)));
  if (!(q >= 0.0f && q <= r1.z)) return false;
  const float G = ex2_approx_b(q * -0.72134752f);  // exp(-q/2), same expression as the forward
  const float araw = r1.y * G;
  const bool capped = !(araw < amax);
  const float alpha = fminf(amax, araw);
  float rcp;  // 1 / (1 - alpha) with alpha <= alpha_max < 1 (R1): no range fix-up needed
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rcp) : "f"(1.0f - alpha));
  const float Tj = p.T * rcp;
  const float w = alpha * Tj;
  const float vv = fmaf(r2.x, p.gr, fmaf(r2.y, p.gg, fmaf(r2.z, p.gb, fmaf(r1.w, p.gd, p.gs))));
  const float dLda = Tj * (vv - p.B);
  v[7] = fmaf(p.gr, w, v[7]);
  v[8] = fmaf(p.gg, w, v[8]);
  v[9] = fmaf(p.gb, w, v[9]);
  v[6] = fmaf(p.gd, w, v[6]);
  if (!capped) {  // R23: no gradient through a capped alpha
    v[5] = fmaf(G, dLda, v[5]);
    const float dq = -0.5f * alpha * dLda;
    const float dqdx = dq * dx, dqdy = dq * dy;
    v[2] = fmaf(dqdx, dx, v[2]);
    v[3] = fmaf(2.0f * dqdx, dy, v[3]);
    v[4] = fmaf(dqdy, dy, v[4]);
    v[0] -= fmaf(2.0f * r0.z, dqdx, r0.w * dqdy);
    v[1] -= fmaf(r0.w, dqdx, 2.0f * r1.x * dqdy);
  }
  p.B = fmaf(alpha, vv, (1.0f - alpha) * p.B);
  p.T = Tj;
  return true;
}

// Branch-free form of bwd_pixel for the thread's two pixels: both dependency
// chains are straight-line code (inactive pixels contribute exact zeros and
// leave T and B unchanged: alpha = 0 gives rcp(1) = 1), so the compiler can
// interleave them -- the replay is latency-bound, not issue-bound.
__device__ __forceinline__ bool bwd_pixel_pair(BPix (&pp)[2], int j, float dx, float dy0,
                                               float dy1, const float4 &r0, const float4 &r1,
                                               const float4 &r2, float amax, float (&v)[kV]) {
  const float dys[2] = {dy0, dy1};
  bool any = false;
#pragma unroll
  for (int k = 0; k < 2; k++) {
    BPix &p = pp[k];
    const float dy = dys[k];
    const float q = DFMA(DMUL(r0.z, dx), dx, DFMA(DMUL(r0.w, dx), dy, DMUL(DMUL(r1.x, dy), dy)));
    const bool val = (j < p.last) & (q >= 0.0f) & (q <= r1.z);
    any |= val;
    const float G = ex2_approx_b(q * -0.72134752f);  // same expression as the forward
    const float araw = r1.y * G;
    const float alpha = val ? fminf(amax, araw) : 0.0f;
    float rcp;  // alpha <= alpha_max < 1 (R1)
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rcp) : "f"(1.0f - alpha));
    const float Tj = p.T * rcp;
    const float w = alpha * Tj;
    const float vv = fmaf(r2.x, p.gr, fmaf(r2.y, p.gg, fmaf(r2.z, p.gb, fmaf(r1.w, p.gd, p.gs))));
    // R23: no gradient through a capped alpha
    const float dLda = (val & (araw < amax)) ? Tj * (vv - p.B) : 0.0f;
    v[7] = fmaf(p.gr, w, v[7]);
    v[8] = fmaf(p.gg, w, v[8]);
    v[9] = fmaf(p.gb, w, v[9]);
    v[6] = fmaf(p.gd, w, v[6]);
    v[5] = fmaf(G, dLda, v[5]);
    const float dq = -0.5f * alpha * dLda;
    const float dqdx = dq * dx, dqdy = dq * dy;
    v[2] = fmaf(dqdx, dx, v[2]);
    v[3] = fmaf(2.0f * dqdx, dy, v[3]);
    v[4] = fmaf(dqdy, dy, v[4]);
    v[0] -= fmaf(2.0f * r0.z, dqdx, r0.w * dqdy);
    v[1] -= fmaf(r0.w, dqdx, 2.0f * r1.x * dqdy);
    p.B = fmaf(alpha, vv, (1.0f - alpha) * p.B);
    p.T = Tj;
  }
  return any;
}

__global__ void __launch_bounds__(kBwdThreads, kBwdMinBlocks) k_render_bwd(
    const float4 *__restrict__ pair_rec, const uint32_t *__restrict__ range, int W, int H,
    int tiles_x, float amax, const float *__restrict__ t_final,
    const int32_t *__restrict__ n_contrib, const float *__restrict__ dC,
    const float *__restrict__ dD, const float *__restrict__ dS, float *__restrict__ acc) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  BwdSmem &sm = *reinterpret_cast<BwdSmem *>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const uint32_t start = range[2 * tile];
  const bool producer = wid == kCW;

  // ---- pixel state (pixel warps only)
  const int wx0 = tx * kTile + (wid & 1) * 8, wy0 = ty * kTile + (wid >> 1) * 8;
  const int px = wx0 + (lane & 7), py0 = wy0 + (lane >> 3) * 2, py1 = py0 + 1;
  BPix pp[2];
#pragma unroll
  for (int k = 0; k < 2; k++) {
    const int py = k ? py1 : py0;
    BPix &p = pp[k];
    p.T = 1.f; p.B = 0.f; p.gr = p.gg = p.gb = p.gd = p.gs = 0.f; p.last = 0;
    if (!producer && px < W && py < H) {
      const int64_t HW = (int64_t)W * H, q = (int64_t)py * W + px;
      p.T = t_final[q];
      p.last = n_contrib[q];
      p.gr = dC[q]; p.gg = dC[HW + q]; p.gb = dC[2 * HW + q];
      p.gd = dD[q]; p.gs = dS[q];
    }
  }
  const int mylast = max(pp[0].last, pp[1].last);
  const int wmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)mylast);
  if (!producer && lane == 0) sm.wmax[wid] = wmax;
  if (tid == kCW * 32) {
    for (int s = 0; s < kBS; s++) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  int maxlast = 0;
#pragma unroll
  for (int w = 0; w < kCW; w++) maxlast = max(maxlast, sm.wmax[w]);
  const int nb = (maxlast + kBB - 1) / kBB;  // replay batch k covers batch b = nb - 1 - k
  auto batch_cnt = [&](int k) { return min(kBB, maxlast - (nb - 1 - k) * kBB); };

  if (producer) {
    // fold the pixel warps' partials of replay batch k (slot s) into the accumulator
    auto flush = [&](int k, int s) {
      const int cnt = batch_cnt(k);
      const float4 *rb = sm.buf[s];
      for (int p = lane; p < cnt * 3; p += 32) {
        const int e = p / 3, c = p - (p / 3) * 3;
        float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int w = 0; w < kCW; w++) {
          if (!sm.pact[s][w]) continue;
          const float4 t4 = reinterpret_cast<const float4 *>(sm.part[s][w][e])[c];
          s4.x += t4.x; s4.y += t4.y; s4.z += t4.z; s4.w += t4.w;
        }
        if (c == 2) { s4.z = 0.f; s4.w = 0.f; }  // padding slots
        if (s4.x != 0.f || s4.y != 0.f || s4.z != 0.f || s4.w != 0.f) {
          const uint32_t gid = __float_as_uint(rb[e * 4 + 2].w);
          red_add_v4(acc + (int64_t)gid * kAcc + c * 4, s4.x, s4.y, s4.z, s4.w);
        }
      }
    };
    for (int k = 0; k < nb; k++) {
      const int s = k % kBS;
      if (k >= kBS) {  // slot s held replay batch k - kBS: wait for all pixel warps
        mbar_wait_sleep(&sm.empty[s], (uint32_t)((k / kBS) - 1) & 1u);
        flush(k - kBS, s);
        __syncwarp();  // every lane has read the slot's gids before it is overwritten
      }
      if (lane == 0) {
        const int b = nb - 1 - k;
        const uint32_t bytes = (uint32_t)batch_cnt(k) * CSPLAT_RECORD_BYTES;
        mbar_arrive_expect_tx(&sm.full[s], bytes);
        tma_load_1d(&sm.buf[s][0], pair_rec + ((int64_t)start + (int64_t)b * kBB) * 4, bytes,
                    &sm.full[s]);
      }
      __syncwarp();
    }
    for (int k = max(0, nb - kBS); k < nb; k++) {  // drain the last slots
      const int s = k % kBS;
      mbar_wait_sleep(&sm.empty[s], (uint32_t)(k / kBS) & 1u);
      flush(k, s);
    }
    return;
  }

  // ---- pixel warps
  const float fpx = (float)px, fpy0 = (float)py0, fpy1 = (float)py1;
  float(*red)[8 * 4] = reinterpret_cast<float(*)[8 * 4]>(sm.red[wid]);  // [kG*kV][32]
  for (int k = 0; k < nb; k++) {
    const int s = k % kBS;
    const int b = nb - 1 - k;
    const int cnt = batch_cnt(k);
    mbar_wait_sleep(&sm.full[s], (uint32_t)(k / kBS) & 1u);
    const bool work = b * kBB < wmax;  // warp-uniform: some lane replays into this batch
    if (work) {
      const float4 *rb = sm.buf[s];
      for (int g0 = 0; g0 < cnt; g0 += kG) {  // processing index g0 + q <-> entry cnt-1-g0-q
        const int ng = min(kG, cnt - g0);
        for (int q = 0; q < ng; q++) {
          const int e = cnt - 1 - g0 - q;
          const int j = b * kBB + e;
          const uint32_t bm = __float_as_uint(rb[e * 4 + 3].z);
          bool any = false;
          // warp-uniform: the pair's block mask (payload word 14, bin.cu) keeps
          // this warp's 8x8 block and the entry is inside some lane's replay range
          if (((bm >> wid) & 1u) && j < wmax) {
            const float4 r0 = rb[e * 4 + 0];
            const float4 r1 = rb[e * 4 + 1];
            const float4 r2 = rb[e * 4 + 2];
            float v[kV];
#pragma unroll
            for (int c = 0; c < kV; c++) v[c] = 0.f;
            const float dx = DSUB(fpx, r0.x);
            const bool a = bwd_pixel_pair(pp, j, dx, DSUB(fpy0, r0.y), DSUB(fpy1, r0.y), r0, r1,
                                          r2, amax, v);
            any = __any_sync(0xffffffffu, a);
            if (any) {  // every lane writes its (possibly zero) partials
#pragma unroll
              for (int c = 0; c < kV; c++) red[q * kV + c][lane] = v[c];
            }
          }
          if (lane == 0) sm.act[wid][q] = any ? 1u : 0u;
        }
        __syncwarp();
        // transposed sums: lane l owns rows l, l+32 of the ng*kV rows
        for (int r = lane; r < ng * kV; r += 32) {
          const int q = r / kV, c = r - q * kV;
          float sum = 0.f;
          if (sm.act[wid][q]) {
            // 32 partials as 8 rotated 16-byte chunks, summed on packed FADD2
            const float4 *row = sm.red[wid][r];
            unsigned long long s01 = 0ull, s23 = 0ull;
#pragma unroll
            for (int t = 0; t < 8; t++) {
              const float4 x = row[(t + lane) & 7];
              unsigned long long a, b;
              asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(x.x), "f"(x.y));
              asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(x.z), "f"(x.w));
              asm("add.rn.f32x2 %0, %0, %1;" : "+l"(s01) : "l"(a));
              asm("add.rn.f32x2 %0, %0, %1;" : "+l"(s23) : "l"(b));
            }
            asm("add.rn.f32x2 %0, %0, %1;" : "+l"(s01) : "l"(s23));
            sum = __uint_as_float((uint32_t)s01) + __uint_as_float((uint32_t)(s01 >> 32));
          }
          sm.part[s][wid][cnt - 1 - g0 - q][c] = sum;
        }
        __syncwarp();
      }
    }
    if (lane == 0) {
      sm.pact[s][wid] = work ? 1u : 0u;
      mbar_arrive(&sm.empty[s]);  // release: part[s][wid] and the slot are done
    }
  }
}

cudaError_t launch_render_bwd(const csplat_gaussians &g, const DecodeArgs *dec,
                              const csplat_camera &cam, const csplat_view &view,
                              const csplat_params &prm, const void *rec, const void *pair_rec,
                              const uint32_t *tile_range, const float *t_final,
                              const int32_t *n_contrib, const float *d_color, const float *d_depth,
                              const float *d_sil, uint32_t flags, const csplat_grads &out,
                              void *ws, cudaStream_t s) {
  const CamInfo ci = cam_info(cam);
  float *acc = static_cast<float *>(ws);
  cudaError_t e = cudaMemsetAsync(acc, 0, bwd_workspace_bytes(g.n), s);
  if (e != cudaSuccess) return e;
  if (out.pose && !(flags & CSPLAT_ACCUMULATE)) {
    e = cudaMemsetAsync(out.pose, 0, 6 * sizeof(float), s);
    if (e != cudaSuccess) return e;
  }
  static bool attr_done = false;
  const size_t smem = sizeof(BwdSmem);
  if (!attr_done) {
    e = cudaFuncSetAttribute(k_render_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int T = ci.tiles_x * ci.tiles_y;
  k_render_bwd<<<T, kBwdThreads, smem, s>>>(static_cast<const float4 *>(pair_rec), tile_range,
                                            ci.W, ci.H, ci.tiles_x, prm.alpha_max, t_final,
                                            n_contrib, d_color, d_depth, d_sil, acc);
  e = cudaGetLastError();
  if (e != cudaSuccess || g.n == 0) return e;
  return launch_chain(g, dec, cam, view, prm, rec, acc, flags, out, s);
}

}  // namespace csplat
