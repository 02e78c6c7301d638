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
// ten partials (raw moments of the conic/mean gradient, o_hat, z, r, g, b;
// bwd_pair) in registers; the warp
// stores the lanes' partials of kG entries as shared-memory rows and each lane
// sums whole rows with rotated LDS.128 (a transposed reduction: ~2
// instructions per (entry, value) instead of a 10-instruction shuffle tree).
#include <atomic>

#include "common.cuh"
#include "quad.cuh"

namespace csplat {

constexpr int kBB = 32;           // records per TMA batch
constexpr int kBS = 3;            // ring depth
constexpr int kAcc = 12;          // accumulator floats per Gaussian
// shared-memory row of an entry's warp sums: the 10 used floats (five 8-byte
// loads in the fold; 12 floats = three 16-byte loads measured slower: C5
// window 12.69 vs 12.43 ms, C2 backward 195.4 vs 194.7 us)
constexpr int kPartW = 10;
// pixel (consumer) warps per CTA, each an 8x8 block of the tile (32 lanes x 2
// pixels): 4 = the whole 16x16 tile (half-tile CTAs measured slower)
constexpr int kCW = 4;
constexpr int kBwdThreads = (kCW + 1) * 32;  // + 1 producer warp
constexpr int kG = 3;             // active entries per transposed reduction: kG*kV <= 32 rows = one pass
constexpr int kV = 10;            // partials per (pixel, entry)
constexpr int kBwdMinBlocks = 5;  // CTAs per SM the register budget targets (6-7 measured slower)
#ifndef CSPLAT_BWD_QUAD
#define CSPLAT_BWD_QUAD 1
#endif

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

struct BwdSmem {
  float4 buf[kBS][kBB * 4];             // staged records
  float4 red[kCW][kG * kV][8];          // per-warp rows of 32 lane partials
  float part[kBS][kCW][kBB][kPartW];    // per-slot, per-warp sums per batch entry
  uint64_t full[kBS], empty[kBS];
  uint32_t msk[kBS][kBB];               // the batch entries' 8x8-block cull masks
  uint32_t pmask[kBS][kCW];             // bit e: warp w wrote part[slot][w][e]
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

// One replay entry j for the thread's two pixels (same column: dx shared; lo =
// upper pixel, hi = lower) as packed float32 pairs: every per-pixel add / mul
// / fma is one f32x2 instruction (each lane IEEE round-to-nearest, so the DA q
// is bit-identical to the forward's).  With a = alpha dL/dalpha the partials
// are the raw moments
//   v0..4 = sum a dx, sum a dy, sum a dx^2, sum a dx dy, sum a dy^2,
//   v5 = sum G dL/dalpha, v6 = sum w gD, v7..9 = sum w gC
// (w = alpha T_j); the conic's constants and the -1/2 of dalpha/dq are applied
// once per Gaussian in k_chain (linear, so summing first is exact algebra):
//   dL/du = ca Sx + cb Sy, dL/dv = cb Sx + cc Sy, dL/dca = -Sxx/2,
//   dL/d(cb) = -Sxy, dL/dcc = -Syy/2   (q = ca dx^2 + 2cb dx dy + cc dy^2).
// T_j = T_{j+1} / (1 - alpha_j) and B_{j-1} = B_j + alpha_j (v_j - B_j) are
// updated in place (the (v - B) is shared with dL/dalpha).  A pixel that does
// not composite entry j gets q = +inf, so G = ex2(-inf) = +0 and alpha = 0:
// T and B unchanged (rcp(1) = 1), exact zeros in every partial.
struct BPix2 {
  f2_t T, B, gr, gg, gb, gd, gs;
  int last0, last1;
};

// bwd_pair in three pieces, so two entries can be interleaved (bwd_two): the
// per-entry front (q, validity, G, alpha, 1/(1 - alpha), v -- independent of
// the pixels' replay state), the state update (T_j, v - B, B: the only
// loop-carried part) and the partials (independent again).
struct BFront {
  f2_t G, AL, RC, VV, DY;
  float dx;
  bool nc0, nc1, any;  // alpha below the cap (R23), either pixel composites
};

__device__ __forceinline__ BFront bwd_front(const BPix2 &P, int j, float dx, f2_t DY,
                                            const float4 &r0, const float4 &r1,
                                            const float4 &r2, float amax) {
  BFront F;
  F.dx = dx;
  F.DY = DY;
  const float cadx = DMUL(r0.z, dx), cbdx = DMUL(r0.w, dx);
  const f2_t Y = mul2(mul2(pk2(r1.x, r1.x), DY), DY);
  const f2_t X = fma2(pk2(cbdx, cbdx), DY, Y);
  const f2_t Q = fma2(pk2(cadx, cadx), pk2(dx, dx), X);
  const float q0 = lo2(Q), q1 = hi2(Q);
  const bool val0 = (j < P.last0) & da_in_range(q0, r1.z);
  const bool val1 = (j < P.last1) & da_in_range(q1, r1.z);
  F.any = val0 | val1;
  const f2_t QM = pk2(val0 ? q0 : __int_as_float(0x7f800000), val1 ? q1 : __int_as_float(0x7f800000));
  const f2_t QE = mul2(QM, pk2(-0.72134752f, -0.72134752f));
  F.G = pk2(ex2_approx_b(lo2(QE)), ex2_approx_b(hi2(QE)));
  const f2_t AR = mul2(pk2(r1.y, r1.y), F.G);
  F.AL = pk2(fminf(amax, lo2(AR)), fminf(amax, hi2(AR)));  // R1
  F.nc0 = lo2(AR) < amax;
  F.nc1 = hi2(AR) < amax;
  const f2_t OM = sub2(pk2(1.0f, 1.0f), F.AL);
  float rc0, rc1;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc0) : "f"(lo2(OM)));  // alpha <= alpha_max < 1
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc1) : "f"(hi2(OM)));
  F.RC = pk2(rc0, rc1);
  F.VV = fma2(pk2(r2.x, r2.x), P.gr,
              fma2(pk2(r2.y, r2.y), P.gg,
                   fma2(pk2(r2.z, r2.z), P.gb, fma2(pk2(r1.w, r1.w), P.gd, P.gs))));
  return F;
}

// the loop-carried part: T_j = T_{j+1} / (1 - alpha_j); returns T_j and v - B;
// B_{j-1} = B_j + alpha_j (v_j - B_j)
__device__ __forceinline__ void bwd_state(BPix2 &P, const BFront &F, f2_t &T, f2_t &VB) {
  asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(P.T) : "l"(F.RC));
  T = P.T;
  VB = sub2(F.VV, P.B);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(P.B) : "l"(F.AL), "l"(VB));
}

__device__ __forceinline__ void bwd_partials(const BPix2 &P, const BFront &F, f2_t T, f2_t VB,
                                             float (&v)[kV]) {
  const f2_t W = mul2(F.AL, T);
  const f2_t D0 = mul2(T, VB);
  // R23: no gradient through a capped alpha
  const f2_t DL = pk2(F.nc0 ? lo2(D0) : 0.0f, F.nc1 ? hi2(D0) : 0.0f);
  const f2_t AV = mul2(F.AL, DL);
  const f2_t GD = mul2(F.G, DL);
  const f2_t TT = mul2(AV, F.DY);
  const f2_t T2 = mul2(TT, F.DY);
  const f2_t WD = mul2(W, P.gd), WR = mul2(W, P.gr), WG = mul2(W, P.gg), WB = mul2(W, P.gb);
  const float dx = F.dx;
  const float sx = dx * (lo2(AV) + hi2(AV));
  const float sy = lo2(TT) + hi2(TT);
  v[0] = sx;
  v[1] = sy;
  v[2] = dx * sx;
  v[3] = dx * sy;
  v[4] = lo2(T2) + hi2(T2);
  v[5] = lo2(GD) + hi2(GD);
  v[6] = lo2(WD) + hi2(WD);
  v[7] = lo2(WR) + hi2(WR);
  v[8] = lo2(WG) + hi2(WG);
  v[9] = lo2(WB) + hi2(WB);
}

__device__ __forceinline__ bool bwd_pair(BPix2 &P, int j, float dx, f2_t DY, const float4 &r0,
                                         const float4 &r1, const float4 &r2, float amax,
                                         float (&v)[kV]) {
  const BFront F = bwd_front(P, j, dx, DY, r0, r1, r2, amax);
  f2_t T, VB;
  bwd_state(P, F, T, VB);
  bwd_partials(P, F, T, VB, v);
  return F.any;
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

template <bool LOSS>
__global__ void __launch_bounds__(kBwdThreads, kBwdMinBlocks) k_render_bwd(
    const __grid_constant__ CUtensorMap tmap, const uint32_t *__restrict__ pair_gid,
    const uint32_t *__restrict__ range, int W, int H,
    int tiles_x, float amax, const float *__restrict__ t_final,
    const int32_t *__restrict__ n_contrib, const float *__restrict__ dC,
    const float *__restrict__ dD, const float *__restrict__ dS, float *__restrict__ acc,
    uint32_t *__restrict__ alive, LossArgs la, int tile0, const int32_t *__restrict__ list) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  BwdSmem &sm = *reinterpret_cast<BwdSmem *>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int tb = (int)blockIdx.x;
  // list mode (NEXT-4 sparse views): CTA b replays list tile b of list[0]
  if (list && tb >= list[0]) return;
  const int tile = list ? list[1 + tb] : tile0 + tb;
  const int blk = wid;  // the warp's 8x8 block of the tile
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const uint32_t start = range[2 * tile];
  const bool producer = wid == kCW;

  // ---- pixel state (pixel warps only)
  const int wx0 = tx * kTile + (blk & 1) * 8, wy0 = ty * kTile + (blk >> 1) * 8;
  const int px = wx0 + (lane & 7), py0 = wy0 + (lane >> 3) * 2, py1 = py0 + 1;
  BPix pp[2];
  float lc = 0.f, ld = 0.f;  // LOSS: this thread's shares of the Eq 12 sums
#pragma unroll
  for (int k = 0; k < 2; k++) {
    const int py = k ? py1 : py0;
    BPix &p = pp[k];
    p.T = 1.f; p.B = 0.f; p.gr = p.gg = p.gb = p.gd = p.gs = 0.f; p.last = 0;
    if (!producer && px < W && py < H) {
      const int64_t HW = (int64_t)W * H, q = (int64_t)py * W + px;
      p.T = t_final[q];
      p.last = n_contrib[q];
      if constexpr (LOSS) {
        // Eq 14 gate (no gradient through it), R_i of Eq 12: valid observed depth
        const unsigned long long nv = *la.n_valid;
        const float inv_r = 1.0f / (float)(nv > 0 ? nv : 1ull);
        const float g = la.sil[q] > la.gate ? 1.0f : 0.0f;
        const float obd = la.obs_depth[q];
        const float v = obd > 0.0f ? 1.0f : 0.0f;
        const float r0 = la.color[q] - la.obs_color[q];
        const float r1 = la.color[HW + q] - la.obs_color[HW + q];
        const float r2 = la.color[2 * HW + q] - la.obs_color[2 * HW + q];
        const float rd = la.depth[q] - obd;
        lc += g * (r0 * r0 + r1 * r1 + r2 * r2);
        ld += g * v * rd * rd;
        const float sc = 2.0f * g * la.inv_n;
        p.gr = sc * r0; p.gg = sc * r1; p.gb = sc * r2;
        p.gd = 2.0f * la.lambda_d * g * v * rd * inv_r;
        p.gs = 0.0f;
      } else {
        p.gr = dC[q]; p.gg = dC[HW + q]; p.gb = dC[2 * HW + q];
        p.gd = dD[q]; p.gs = dS[q];
      }
      // a pixel with an all-zero upstream contributes exact zeros to every
      // partial (v_j = 0, so B = 0 and dL/dalpha = 0): no replay (gated-out
      // tracking pixels, the unsampled pixels of the NEXT-4 patch BA)
      if (p.gr == 0.f && p.gg == 0.f && p.gb == 0.f && p.gd == 0.f && p.gs == 0.f) p.last = 0;
    }
  }
  if constexpr (LOSS) {
    lc = warp_sum(lc);
    ld = warp_sum(ld);
    if (!producer && lane == 0 && (lc != 0.f || ld != 0.f)) {
      const unsigned long long nv = *la.n_valid;
      const float a = lc * la.inv_n, b = ld / (float)(nv > 0 ? nv : 1ull);
      atomicAdd(la.loss3 + 0, a + la.lambda_d * b);
      atomicAdd(la.loss3 + 1, a);
      atomicAdd(la.loss3 + 2, b);
    }
  }
  const int mylast = max(pp[0].last, pp[1].last);
  const int wmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)mylast);
  if (!producer && lane == 0) sm.wmax[wid] = wmax;
  if (tid == kCW * 32) {
    for (int s = 0; s < kBS; s++) {
      mbar_init(&sm.full[s], 32);  // the producer warp's 32 lanes (+ the batch's TMA bytes)
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
      const int e = lane;  // one batch entry per lane
      if (e >= batch_cnt(k)) return;
      float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0, s2 = s0;
      bool hit = false;
#pragma unroll
      for (int w = 0; w < kCW; w++) {
        if (!((sm.pmask[s][w] >> e) & 1u)) continue;
        hit = true;
        const float2 *t = reinterpret_cast<const float2 *>(sm.part[s][w][e]);
        const float2 t0 = t[0], t1 = t[1], t2 = t[2], t3 = t[3], t4 = t[4];
        s0.x += t0.x; s0.y += t0.y; s0.z += t1.x; s0.w += t1.y;
        s1.x += t2.x; s1.y += t2.y; s1.z += t3.x; s1.w += t3.y;
        s2.x += t4.x; s2.y += t4.y;
      }
      if (hit) {
        const uint32_t gid = __float_as_uint(sm.buf[s][e * 4 + 2].w);
        float *dst = acc + (int64_t)gid * kAcc;
        red_add_v4(dst, s0.x, s0.y, s0.z, s0.w);
        red_add_v4(dst + 4, s1.x, s1.y, s1.z, s1.w);
        red_add_v4(dst + 8, s2.x, s2.y, 0.f, 0.f);
        atomicOr(alive + (gid >> 5), 1u << (gid & 31));  // the chain visits this Gaussian
      }
    };
    // replay batch k = list batch b = nb - 1 - k: lane l takes list entry
    // b*kBB + l (pair_gid: Gaussian index | block mask << 28, loaded one batch
    // ahead), stores its mask into msk[s] and gathers its record with one
    // 64-byte TMA bulk copy (gather_batch)
    auto entry_of = [&](int k) {
      return lane < batch_cnt(k) ? pair_gid[start + (nb - 1 - k) * kBB + lane] : 0u;
    };
    uint32_t entry = nb > 0 ? entry_of(0) : 0u;
    for (int k = 0; k < nb; k++) {
      const int s = k % kBS;
      if (k >= kBS) {  // slot s held replay batch k - kBS: wait for all pixel warps
        mbar_wait_sleep(&sm.empty[s], (uint32_t)((k / kBS) - 1) & 1u);
        flush(k - kBS, s);
        __syncwarp();  // every lane has read the slot's gids before it is overwritten
      }
      const uint32_t e = entry;
      if (k + 1 < nb) entry = entry_of(k + 1);
      gather_batch(&sm.buf[s][0], sm.msk[s], &tmap, e, lane, batch_cnt(k), &sm.full[s]);
    }
    for (int k = max(0, nb - kBS); k < nb; k++) {  // drain the last slots
      const int s = k % kBS;
      mbar_wait_sleep(&sm.empty[s], (uint32_t)(k / kBS) & 1u);
      flush(k, s);
    }
    return;
  }

  // ---- pixel warps
  const float fpx = (float)px;
  BPix2 P;
  P.T = pk2(pp[0].T, pp[1].T); P.B = pk2(pp[0].B, pp[1].B);
  P.gr = pk2(pp[0].gr, pp[1].gr); P.gg = pk2(pp[0].gg, pp[1].gg); P.gb = pk2(pp[0].gb, pp[1].gb);
  P.gd = pk2(pp[0].gd, pp[1].gd); P.gs = pk2(pp[0].gs, pp[1].gs);
  P.last0 = pp[0].last; P.last1 = pp[1].last;
  const f2_t FPY = pk2((float)py0, (float)py1);
  float(*red)[8 * 4] = reinterpret_cast<float(*)[8 * 4]>(sm.red[wid]);  // [kG*kV][32]
  for (int k = 0; k < nb; k++) {
    const int s = k % kBS;
    const int b = nb - 1 - k;
    const int cnt = batch_cnt(k);
    mbar_wait_sleep(&sm.full[s], (uint32_t)(k / kBS) & 1u);
    const bool work = b * kBB < wmax;  // warp-uniform: some lane replays into this batch
    uint32_t pm = 0;                   // entries of this batch with partials in part[s][wid]
    if (work) {
      const float4 *rb = sm.buf[s];
      // sum the rows of the nq pending entries (entry indices packed in ents, the
      // first entry in the highest used byte) into
      // part[s][wid]: lane r < nq*kV owns row r (one pass, kG*kV <= 32)
      auto reduce = [&](int nq, uint32_t ents) {
        __syncwarp();
        if (lane < nq * kV) {
          const int q = lane / kV, c = lane - q * kV;
          // 32 partials as 8 rotated 16-byte chunks, summed on packed FADD2
          const float4 *row = sm.red[wid][lane];
          unsigned long long s01 = 0ull, s23 = 0ull;
#pragma unroll
          for (int t = 0; t < 8; t++) {
            const float4 x = row[(t + lane) & 7];
            unsigned long long a2, b2;
            asm("mov.b64 %0, {%1, %2};" : "=l"(a2) : "f"(x.x), "f"(x.y));
            asm("mov.b64 %0, {%1, %2};" : "=l"(b2) : "f"(x.z), "f"(x.w));
            asm("add.rn.f32x2 %0, %0, %1;" : "+l"(s01) : "l"(a2));
            asm("add.rn.f32x2 %0, %0, %1;" : "+l"(s23) : "l"(b2));
          }
          asm("add.rn.f32x2 %0, %0, %1;" : "+l"(s01) : "l"(s23));
          const float sum = __uint_as_float((uint32_t)s01) + __uint_as_float((uint32_t)(s01 >> 32));
          sm.part[s][wid][(ents >> (8 * (nq - 1 - q))) & 0xffu][c] = sum;
        }
        __syncwarp();
      };
      int nq = 0;
      uint32_t ents = 0;
      // the batch's entries this warp replays, one ballot: lane l tests entry l's
      // block mask (payload word 14, bin.cu) and replay range (j < wmax)
      const uint32_t bml = lane < cnt ? sm.msk[s][lane] : 0u;
      uint32_t todo = __ballot_sync(0xffffffffu, ((bml >> blk) & 1u) && b * kBB + lane < wmax);
      // entry e's lane partials as rows nq*kV + c of the warp's reduction
      // buffer (every lane, possibly zeros); a full group is reduced
      auto push = [&](int e, const float (&v)[kV]) {
#pragma unroll
        for (int c = 0; c < kV; c++) red[nq * kV + c][lane] = v[c];
        ents = ents * 256u + (uint32_t)e;  // entry q of the group in byte nq - 1 - q
        uint32_t bit;
        asm("bmsk.clamp.b32 %0, %1, 1;" : "=r"(bit) : "r"(e));
        pm |= bit;
        if (++nq == kG) {
          reduce(nq, ents);
          nq = 0;
          ents = 0;
        }
      };
      auto top = [&]() {  // the highest set bit of todo (bfind), cleared
        int e;
        asm("bfind.u32 %0, %1;" : "=r"(e) : "r"(todo));
        uint32_t below;  // bits 0 .. e-1
        asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(below) : "r"(e));
        todo &= below;
        return e;
      };
      while (todo) {  // back to front
        const int e1 = top();
        const float4 a0 = rb[e1 * 4 + 0], a1 = rb[e1 * 4 + 1], a2 = rb[e1 * 4 + 2];
        if (todo) {
          // two entries e1 > e2 at once: both fronts, the two state updates in
          // replay order, both partials -- the independent halves interleave
          // (one warp issues in order: with one entry per iteration its long
          // dependent chain left ~35% of issue slots empty; C2 backward kernel
          // 178.8 -> 167.9 us; 4 CTAs/SM with the registers to spare: 174.0)
          const int e2 = top();
          const float4 b0 = rb[e2 * 4 + 0], b1 = rb[e2 * 4 + 1], b2 = rb[e2 * 4 + 2];
          const BFront FA = bwd_front(P, b * kBB + e1, DSUB(fpx, a0.x),
                                      sub2(FPY, pk2(a0.y, a0.y)), a0, a1, a2, amax);
          const BFront FB = bwd_front(P, b * kBB + e2, DSUB(fpx, b0.x),
                                      sub2(FPY, pk2(b0.y, b0.y)), b0, b1, b2, amax);
          f2_t TA, VA, TB, VB;
          bwd_state(P, FA, TA, VA);
          bwd_state(P, FB, TB, VB);
          float va[kV], vb[kV];
          bwd_partials(P, FA, TA, VA, va);
          bwd_partials(P, FB, TB, VB, vb);
          if (__any_sync(0xffffffffu, FA.any)) push(e1, va);
          if (__any_sync(0xffffffffu, FB.any)) push(e2, vb);
          continue;
        }
        float v[kV];
        const bool act = bwd_pair(P, b * kBB + e1, DSUB(fpx, a0.x), sub2(FPY, pk2(a0.y, a0.y)),
                                  a0, a1, a2, amax, v);
        if (__any_sync(0xffffffffu, act)) push(e1, v);
      }
      if (nq) reduce(nq, ents);
    }
    if (lane == 0) {
      sm.pmask[s][wid] = pm;
      mbar_arrive(&sm.empty[s]);  // release: part[s][wid] and the slot are done
    }
  }
}

// ---------------------------------------------------------------------------
// The block-list backward (CSPLAT_BWD_QUAD, default).  k_render_bwd above
// replays, for each 8x8 pixel block (one warp), every entry the block may
// touch: on C2 61 % of those (pixel, entry) slots lie outside the entry's
// ellipse, and the warp-wide reduction of the per-entry partials through shared
// memory costs as much as the replay.  Here each 4x4 block has its own entry
// list and its own four lanes (a QUAD), so a warp replays eight independent
// streams:
//  1. gather (per chunk of up to kChunk list entries, back to front): the
//     chunk's records go to shared memory; an entry is listed for a 4x4 block
//     if its pixel rectangle overlaps the block, the 8x8 block around it is
//     flagged in the pair entry (block_mask, the sort's conservative ellipse
//     test) and its list position is below the block's last contributor;
//  2. replay: quad lane q owns column q of its block (two vertically adjacent
//     pixel pairs, state and upstream in registers) and walks the block's list
//     back to front with the recurrence of bwd_front / bwd_state above
//     (T_j = T_{j+1} rcp(1 - alpha_j), B_{j-1} = B_j + alpha_j (v_j - B_j)) in
//     the same arithmetic;
//  3. per entry the quad sums its four lanes' ten partials with a transposed
//     shuffle reduction (11 SHFL) and adds them to the [n][12] accumulator with
//     one red.global.add.v4.f32 from each of two lanes and one .v2 from a third.
// No producer warp, no barriers inside the replay; the shared-memory traffic per
// entry is the record (three broadcast loads per quad).
namespace quad {
#ifndef CSPLAT_QUAD_MINB
#define CSPLAT_QUAD_MINB 8
#endif
constexpr int kMinBlocks = CSPLAT_QUAD_MINB;

struct Smem {
  Lists L;
  int wmax[kNB];
};

// one pixel pair's replay state and upstream (registers of its lane)
struct QPair {
  f2_t T, B, FPY, GR, GG, GB, GD, GS;
  int last0, last1;
};

// a pixel pair's partial terms of one entry (f32x2, summed over the quad's pixels)
struct QTerms {
  f2_t AV, TT, T2, GDL, WD, WR, WG, WB;
};

// one entry at one pixel pair in two pieces, so two entries can interleave: the front (q, the
// validity, G, alpha, 1 / (1 - alpha), v -- independent of the replay state)
// and the state update with the partial terms
struct QFront {
  f2_t DY, G, AL, RC, VV;
  bool nc0, nc1;
};
__device__ __forceinline__ QFront pair_front(const QPair &P, int j, float dx, float cadx,
                                             float cbdx, const float4 &r0, const float4 &r1,
                                             const float4 &r2, float amax) {
  QFront f;
  f.DY = sub2(P.FPY, pk2(r0.y, r0.y));
  const f2_t Y = mul2(mul2(pk2(r1.x, r1.x), f.DY), f.DY);
  const f2_t X = fma2(pk2(cbdx, cbdx), f.DY, Y);
  const f2_t Q = fma2(pk2(cadx, cadx), pk2(dx, dx), X);
  const float q0 = lo2(Q), q1 = hi2(Q);
  const bool val0 = (j < P.last0) & da_in_range(q0, r1.z);
  const bool val1 = (j < P.last1) & da_in_range(q1, r1.z);
  const f2_t QM = pk2(val0 ? q0 : __int_as_float(0x7f800000), val1 ? q1 : __int_as_float(0x7f800000));
  const f2_t QE = mul2(QM, pk2(-0.72134752f, -0.72134752f));
  f.G = pk2(ex2_approx_b(lo2(QE)), ex2_approx_b(hi2(QE)));
  const f2_t AR = mul2(pk2(r1.y, r1.y), f.G);
  f.AL = pk2(fminf(amax, lo2(AR)), fminf(amax, hi2(AR)));  // R1
  f.nc0 = lo2(AR) < amax;
  f.nc1 = hi2(AR) < amax;
  const f2_t OM = sub2(pk2(1.0f, 1.0f), f.AL);
  float rc0, rc1;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc0) : "f"(lo2(OM)));  // alpha <= alpha_max < 1
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc1) : "f"(hi2(OM)));
  f.RC = pk2(rc0, rc1);
  f.VV = fma2(pk2(r2.x, r2.x), P.GR,
              fma2(pk2(r2.y, r2.y), P.GG,
                   fma2(pk2(r2.z, r2.z), P.GB, fma2(pk2(r1.w, r1.w), P.GD, P.GS))));
  return f;
}
__device__ __forceinline__ QTerms pair_state(QPair &P, const QFront &f) {
  P.T = mul2(P.T, f.RC);
  const f2_t VB = sub2(f.VV, P.B);
  P.B = fma2(f.AL, VB, P.B);
  QTerms o;
  const f2_t W = mul2(f.AL, P.T);
  const f2_t D0 = mul2(P.T, VB);
  const f2_t DL = pk2(f.nc0 ? lo2(D0) : 0.0f, f.nc1 ? hi2(D0) : 0.0f);  // R23
  o.AV = mul2(f.AL, DL);
  o.GDL = mul2(f.G, DL);
  o.TT = mul2(o.AV, f.DY);
  o.T2 = mul2(o.TT, f.DY);
  o.WD = mul2(W, P.GD);
  o.WR = mul2(W, P.GR);
  o.WG = mul2(W, P.GG);
  o.WB = mul2(W, P.GB);
  return o;
}
// the quad's ten sums of one entry's terms over its four lanes (transposed
// shuffle reduction) into the accumulator
__device__ __forceinline__ void quad_flush(const QTerms &a, float dx, bool hi, int ri, bool act,
                                           float *dst) {
  float v[kV];
  const float sav = lo2(a.AV) + hi2(a.AV), stt = lo2(a.TT) + hi2(a.TT);
  v[0] = dx * sav;
  v[1] = stt;
  v[2] = dx * v[0];
  v[3] = dx * stt;
  v[4] = lo2(a.T2) + hi2(a.T2);
  v[5] = lo2(a.GDL) + hi2(a.GDL);
  v[6] = lo2(a.WD) + hi2(a.WD);
  v[7] = lo2(a.WR) + hi2(a.WR);
  v[8] = lo2(a.WG) + hi2(a.WG);
  v[9] = lo2(a.WB) + hi2(a.WB);
  // lanes 0-1 keep (v0 v1 v2 v3 v8), lanes 2-3 (v4 v5 v6 v7 v9); then a
  // butterfly over the lane pair
  float x[5];
#pragma unroll
  for (int k = 0; k < 5; k++) {
    const float s1 = k < 4 ? v[k] : v[8], s2 = k < 4 ? v[4 + k] : v[9];
    const float keep = hi ? s2 : s1, send = hi ? s1 : s2;
    x[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
#pragma unroll
  for (int k = 0; k < 5; k++) x[k] += __shfl_xor_sync(0xffffffffu, x[k], 1);
  const float v9 = __shfl_xor_sync(0xffffffffu, x[4], 2);  // lane 1 <- lane 3's v9
  if (act) {
    if ((ri & 1) == 0) red_add_v4(dst + (hi ? 4 : 0), x[0], x[1], x[2], x[3]);
    else if (!hi) red_add_v2(dst + 8, x[4], v9);
  }
}
__device__ __forceinline__ QTerms qadd(const QTerms &a, const QTerms &b) {
  QTerms o;
  o.AV = add2(a.AV, b.AV); o.TT = add2(a.TT, b.TT); o.T2 = add2(a.T2, b.T2);
  o.GDL = add2(a.GDL, b.GDL); o.WD = add2(a.WD, b.WD); o.WR = add2(a.WR, b.WR);
  o.WG = add2(a.WG, b.WG); o.WB = add2(a.WB, b.WB);
  return o;
}

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
#pragma unroll
  for (int b = 0; b < kNB; b++) maxlast = max(maxlast, sm.wmax[b]);
  const int X0 = tx * kTile, Y0 = ty * kTile;
  const float fpx = (float)px;

  // chunks of the list, back to front
  for (int c1 = maxlast; c1 > 0; c1 -= kChunk) {
    const int c0 = max(0, c1 - kChunk), len = c1 - c0;
    // 1. the chunk's records, 4x4-block masks and the blocks' lists, back to front
    gather(sm.L, recs, pair_gid, start, c0, len, X0, Y0, alive, tid);
    build_lists<true>(sm.L, c0, len, sm.wmax, wid, lane);
    // 2. the replay: the quad walks its block's list; 3. quad sums -> accumulator
    const int nr = sm.L.nitems[B];
    const int nmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)nr);
    const uint8_t *lst = sm.L.lst[B];
    const bool hi = ri >= 2;
    // two list entries per iteration: both fronts, the two state updates in
    // list order, both partial sums -- the independent halves interleave
    for (int e = 0; e < nmax; e += 2) {
      const bool actA = e < nr, actB = e + 1 < nr;
      const int iA = actA ? (int)lst[e] : kChunk, iB = actB ? (int)lst[e + 1] : kChunk;
      const float4 a0 = sm.L.rec[iA][0], a1 = sm.L.rec[iA][1], a2 = sm.L.rec[iA][2];
      const float4 b0 = sm.L.rec[iB][0], b1 = sm.L.rec[iB][1], b2 = sm.L.rec[iB][2];
      const int jA = actA ? c0 + iA : 0x7fffffff, jB = actB ? c0 + iB : 0x7fffffff;
      const float dxA = DSUB(fpx, a0.x), dxB = DSUB(fpx, b0.x);
      const QFront fA0 = pair_front(P[0], jA, dxA, DMUL(a0.z, dxA), DMUL(a0.w, dxA), a0, a1, a2, amax);
      const QFront fA1 = pair_front(P[1], jA, dxA, DMUL(a0.z, dxA), DMUL(a0.w, dxA), a0, a1, a2, amax);
      const QFront fB0 = pair_front(P[0], jB, dxB, DMUL(b0.z, dxB), DMUL(b0.w, dxB), b0, b1, b2, amax);
      const QFront fB1 = pair_front(P[1], jB, dxB, DMUL(b0.z, dxB), DMUL(b0.w, dxB), b0, b1, b2, amax);
      const QTerms tA0 = pair_state(P[0], fA0), tA1 = pair_state(P[1], fA1);
      const QTerms tB0 = pair_state(P[0], fB0), tB1 = pair_state(P[1], fB1);
      quad_flush(qadd(tA0, tA1), dxA, hi, ri, actA, accg + (int64_t)__float_as_uint(a2.w) * kAcc);
      quad_flush(qadd(tB0, tB1), dxB, hi, ri, actB, accg + (int64_t)__float_as_uint(b2.w) * kAcc);
    }
    __syncthreads();  // before the next chunk overwrites the records and lists
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
  const size_t smem = sizeof(BwdSmem);
  // the opt-in shared-memory size: set once per device (a race between host
  // threads only repeats the idempotent call)
  static std::atomic<unsigned long long> attr_done{0};
#if CSPLAT_BWD_QUAD
  const size_t smem_quad = sizeof(quad::Smem);
#endif
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr_done.load(std::memory_order_acquire) & bit)) {
#if CSPLAT_BWD_QUAD
    e = cudaFuncSetAttribute(quad::k_render_bwd_quad<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_quad);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(quad::k_render_bwd_quad<true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_quad);
#else
    e = cudaFuncSetAttribute(k_render_bwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_render_bwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem);
#endif
    if (e != cudaSuccess) return e;
    attr_done.fetch_or(bit, std::memory_order_release);
  }
  const int T = ci.tiles_x * ci.tiles_y;
  if (ntiles < 0) ntiles = T - tile0;
  if (ntiles <= 0) return cudaSuccess;
  CUtensorMap tmap;
  if ((e = rec_tensor_map(rec, &tmap)) != cudaSuccess) return e;
  LossArgs la{};
  if (loss) {
    la.color = loss->color; la.depth = loss->depth; la.sil = loss->sil;
    la.obs_color = loss->obs_color; la.obs_depth = loss->obs_depth;
    la.n_valid = loss->n_valid; la.lambda_d = loss->lambda_d; la.gate = loss->gate;
    la.inv_n = 1.0f / (float)((int64_t)ci.W * ci.H);
    la.loss3 = loss->loss3;
#if CSPLAT_BWD_QUAD
    quad::k_render_bwd_quad<true><<<ntiles, quad::kThreads, smem_quad, s>>>(
        static_cast<const float4 *>(rec), pair_gid, tile_range, ci.W, ci.H, ci.tiles_x, prm.alpha_max,
        t_final, n_contrib, nullptr, nullptr, nullptr, acc, alive, la, tile0, list);
#else
    k_render_bwd<true><<<ntiles, kBwdThreads, smem, s>>>(
        tmap, pair_gid, tile_range, ci.W, ci.H, ci.tiles_x, prm.alpha_max,
        t_final, n_contrib, nullptr, nullptr, nullptr, acc, alive, la, tile0, list);
#endif
  } else {
#if CSPLAT_BWD_QUAD
    quad::k_render_bwd_quad<false><<<ntiles, quad::kThreads, smem_quad, s>>>(
        static_cast<const float4 *>(rec), pair_gid, tile_range, ci.W, ci.H, ci.tiles_x, prm.alpha_max,
        t_final, n_contrib, d_color, d_depth, d_sil, acc, alive, la, tile0, list);
#else
    k_render_bwd<false><<<ntiles, kBwdThreads, smem, s>>>(
        tmap, pair_gid, tile_range, ci.W, ci.H, ci.tiles_x, prm.alpha_max,
        t_final, n_contrib, d_color, d_depth, d_sil, acc, alive, la, tile0, list);
#endif
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
