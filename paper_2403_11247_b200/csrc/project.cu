// project.cu -- a1 (mask, Eq 6-7), a2 decode (Eq 10) and a3
// (EWA projection, Eq 1-2) in decision arithmetic.
//
// One thread per Gaussian: coalesced SoA loads of the 15 attribute planes,
// the R-VQ decode gathers from the (L1/L2-resident) codebooks, and one 64-byte
// record written as four 16-byte stores.  HBM-bound: 60 B in + 64 B + 4 B out
// per Gaussian (raw geometry); DA keeps it at ~300 instructions per Gaussian.
#include <algorithm>
#include <mutex>

#include "bin_dev.cuh"

namespace csplat {

// sort / forward / backward pipeline chunks of contiguous tile ranges (C2:
// 2 chunks 2324/s, 3-4 the same within noise, 8 chunks 2113/s; chunks of
// interleaved tile rows 2335 vs 2371/s: a tile's look-back then walks over the
// other chunk's unpublished rows)
constexpr int kFwdChunks = 2;

struct ProjConst {
  float V[12];
  float fx, fy, cx, cy, Wf, Hf, near_z, far_z;
  float lx_lo, lx_hi, ly_lo, ly_hi;
  float tau, dil;
};

// The view-independent part of Gaussian i's projection (mask, decode,
// activations, Sigma = R S S^T R^T of Eq 1) -- computed once per Gaussian
// for any number of views (csplat_project_views).  ok = false: culled in
// every view.  Exactly the single-view DA expressions; the culls of the two
// parts are ANDed, so their evaluation order does not change any output.
struct GPre {
  bool ok;
  float mx, my, mz, oh, k2, cr, cg, cb;
  float S00, S01, S02, S11, S12, S22;
};

template <int LF>
__device__ __forceinline__ void project_prelude(
    int64_t i, int64_t n, const int64_t *__restrict__ n_dev, const float *__restrict__ mean,
    const float *__restrict__ opac, const float *__restrict__ rgb,
    const float *__restrict__ lsc, const float *__restrict__ quat,
    const float *__restrict__ mask, const DecodeArgs &dec, int use_dec, float tau, GPre &g) {
  const int64_t ne = eff_n(n, n_dev);
  bool ok = i < ne;
  // every attribute load is independent of the mask test: issue them all at
  // once (the Gaussian's planes, then the R-VQ codes), one memory round trip
  // each, and cull afterwards
  const int64_t j = ok ? i : 0;
  const float m = mask[j];
  float ls[3], qv[4];
  if (use_dec) {
    // Eq 10: S_hat^L = sum_l C^l[i^l] (R17, R20); a bad index culls (NaN)
    rvq_decode<LF>(dec, n, j, ls, qv, ok && (m > tau));
  } else {
    ls[0] = lsc[j]; ls[1] = lsc[n + j]; ls[2] = lsc[2 * n + j];
    qv[0] = quat[j]; qv[1] = quat[n + j]; qv[2] = quat[2 * n + j]; qv[3] = quat[3 * n + j];
  }
  g.mx = mean[j]; g.my = mean[n + j]; g.mz = mean[2 * n + j];
  const float o = opac[j];
  g.cr = rgb[j]; g.cg = rgb[n + j]; g.cb = rgb[2 * n + j];
  const float ls0 = ls[0], ls1 = ls[1], ls2 = ls[2];
  const float qw = qv[0], qx = qv[1], qy = qv[2], qz = qv[3];
  ok = ok && (m > tau);  // Eq 6: M = 1[Sig(m) > eps]  <=>  m > tau (R12)
  ok = ok && isfinite(g.mx) && isfinite(g.my) && isfinite(g.mz) && isfinite(o) && isfinite(ls0) &&
       isfinite(ls1) && isfinite(ls2) && isfinite(qw) && isfinite(qx) && isfinite(qy) &&
       isfinite(qz) && isfinite(g.cr) && isfinite(g.cg) && isfinite(g.cb);
  g.oh = 0.f;
  g.k2 = 0.f;
  if (ok) {
    g.oh = da_sigm(o);
    const float a255 = DMUL(255.0f, g.oh);
    ok = a255 > 1.0f;  // alpha >= 1/255 reachable (R2)
    g.k2 = DMUL(2.0f, da_plog(a255));
  }
  float nq = 0;
  if (ok) {
    nq = DADD(DADD(DADD(DMUL(qw, qw), DMUL(qx, qx)), DMUL(qy, qy)), DMUL(qz, qz));
    ok = nq > 0.0f;
  }
  g.ok = ok;
  if (!ok) return;
  const float s0 = da_pexp(ls0), s1 = da_pexp(ls1), s2 = da_pexp(ls2);
  const float rn = DDIV(1.0f, DSQRT(nq));
  const float w = DMUL(qw, rn), x = DMUL(qx, rn), y = DMUL(qy, rn), z = DMUL(qz, rn);
  float R[3][3];
  R[0][0] = DSUB(1.0f, DMUL(2.0f, DADD(DMUL(y, y), DMUL(z, z))));
  R[0][1] = DMUL(2.0f, DSUB(DMUL(x, y), DMUL(w, z)));
  R[0][2] = DMUL(2.0f, DADD(DMUL(x, z), DMUL(w, y)));
  R[1][0] = DMUL(2.0f, DADD(DMUL(x, y), DMUL(w, z)));
  R[1][1] = DSUB(1.0f, DMUL(2.0f, DADD(DMUL(x, x), DMUL(z, z))));
  R[1][2] = DMUL(2.0f, DSUB(DMUL(y, z), DMUL(w, x)));
  R[2][0] = DMUL(2.0f, DSUB(DMUL(x, z), DMUL(w, y)));
  R[2][1] = DMUL(2.0f, DADD(DMUL(y, z), DMUL(w, x)));
  R[2][2] = DSUB(1.0f, DMUL(2.0f, DADD(DMUL(x, x), DMUL(y, y))));
  const float sv[3] = {s0, s1, s2};
  float M[3][3];
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = 0; b < 3; b++) M[a][b] = DMUL(R[a][b], sv[b]);
  auto sig = [&](int a, int b) {  // Eq 1: Sigma = R S S^T R^T
    return DADD(DADD(DMUL(M[a][0], M[b][0]), DMUL(M[a][1], M[b][1])), DMUL(M[a][2], M[b][2]));
  };
  g.S00 = sig(0, 0); g.S01 = sig(0, 1); g.S02 = sig(0, 2);
  g.S11 = sig(1, 1); g.S12 = sig(1, 2); g.S22 = sig(2, 2);
}

// The view part (Eq 2, R2-R7, R21): Gaussian i's 64-byte record and pair count
// in the view of pc; for the fused bucket pass also what the pairs need
// (PairSrc: the count, the pixel-rectangle words, bits(z_c) and the conic;
// count 0 if culled).
__device__ __forceinline__ void project_view(int64_t i, const GPre &g, const ProjConst &pc,
                                             const float *V, float4 *__restrict__ r,
                                             int32_t *__restrict__ count, PairSrc &ps) {
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  ps = pair_src_none();
  bool ok = g.ok;
  float xc = 0, yc = 0, zc = 0;
  if (ok) {
    xc = DADD(DADD(DADD(DMUL(V[0], g.mx), DMUL(V[1], g.my)), DMUL(V[2], g.mz)), V[3]);
    yc = DADD(DADD(DADD(DMUL(V[4], g.mx), DMUL(V[5], g.my)), DMUL(V[6], g.mz)), V[7]);
    zc = DADD(DADD(DADD(DMUL(V[8], g.mx), DMUL(V[9], g.my)), DMUL(V[10], g.mz)), V[11]);
    ok = (zc > pc.near_z) && (zc < pc.far_z);  // R21
  }
  if (!ok) {
    r[0] = z4; r[1] = z4; r[2] = z4; r[3] = z4;
    count[i] = 0;
    return;
  }
  const float S[3][3] = {{g.S00, g.S01, g.S02}, {g.S01, g.S11, g.S12}, {g.S02, g.S12, g.S22}};
  const float iz = DDIV(1.0f, zc);
  const float txz = DMUL(xc, iz), tyz = DMUL(yc, iz);
  const float tx = DMUL(fminf(fmaxf(txz, pc.lx_lo), pc.lx_hi), zc);  // R6
  const float ty = DMUL(fminf(fmaxf(tyz, pc.ly_lo), pc.ly_hi), zc);
  const float iz2 = DMUL(iz, iz);
  const float J00 = DMUL(pc.fx, iz), J02 = DMUL(-DMUL(pc.fx, tx), iz2);
  const float J11 = DMUL(pc.fy, iz), J12 = DMUL(-DMUL(pc.fy, ty), iz2);
  float A[2][3];  // A = J W
#pragma unroll
  for (int j = 0; j < 3; j++) {
    A[0][j] = DADD(DMUL(J00, V[j]), DMUL(J02, V[8 + j]));
    A[1][j] = DADD(DMUL(J11, V[4 + j]), DMUL(J12, V[8 + j]));
  }
  float B[2][3];
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int j = 0; j < 3; j++)
      B[a][j] = DADD(DADD(DMUL(A[a][0], S[0][j]), DMUL(A[a][1], S[1][j])), DMUL(A[a][2], S[2][j]));
  // Eq 2 (+ R5 dilation)
  const float sa = DADD(DADD(DADD(DMUL(B[0][0], A[0][0]), DMUL(B[0][1], A[0][1])), DMUL(B[0][2], A[0][2])), pc.dil);
  const float sb = DADD(DADD(DMUL(B[0][0], A[1][0]), DMUL(B[0][1], A[1][1])), DMUL(B[0][2], A[1][2]));
  const float sc = DADD(DADD(DADD(DMUL(B[1][0], A[1][0]), DMUL(B[1][1], A[1][1])), DMUL(B[1][2], A[1][2])), pc.dil);
  const float det = DSUB(DMUL(sa, sc), DMUL(sb, sb));
  bool ok2 = det > 0.0f;
  const float ca = DDIV(sc, det), cbn = DDIV(-sb, det), cc = DDIV(sa, det);
  const float u = DADD(DMUL(pc.fx, txz), pc.cx), v = DADD(DMUL(pc.fy, tyz), pc.cy);
  const float ex = DADD(DSQRT(DMUL(g.k2, sa)), 1e-3f), ey = DADD(DSQRT(DMUL(g.k2, sc)), 1e-3f);
  const float X0 = ceilf(DSUB(u, ex)), X1 = floorf(DADD(u, ex));
  const float Y0 = ceilf(DSUB(v, ey)), Y1 = floorf(DADD(v, ey));
  ok2 = ok2 && (X0 <= DSUB(pc.Wf, 1.0f)) && (X1 >= 0.0f) && (Y0 <= DSUB(pc.Hf, 1.0f)) &&
        (Y1 >= 0.0f) && (X0 <= X1) && (Y0 <= Y1);
  if (!ok2) {
    r[0] = z4; r[1] = z4; r[2] = z4; r[3] = z4;
    count[i] = 0;
    return;
  }
  const int px0 = (int)fmaxf(X0, 0.0f), px1 = (int)fminf(X1, DSUB(pc.Wf, 1.0f));
  const int py0 = (int)fmaxf(Y0, 0.0f), py1 = (int)fminf(Y1, DSUB(pc.Hf, 1.0f));
  const int tx0 = px0 / kTile, tx1 = px1 / kTile, ty0 = py0 / kTile, ty1 = py1 / kTile;
  r[0] = make_float4(u, v, ca, DADD(cbn, cbn));
  r[1] = make_float4(cc, g.oh, g.k2, zc);
  r[2] = make_float4(g.cr, g.cg, g.cb, __uint_as_float((uint32_t)i));
  // inclusive pixel rectangle as two u16x2 corners (low | high), DESIGN.md §4
  r[3] = make_float4(__uint_as_float((uint32_t)px0 | ((uint32_t)py0 << 16)),
                     __uint_as_float((uint32_t)px1 | ((uint32_t)py1 << 16)), 0.f, 0.f);
  ps.c = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
  ps.rx = (uint32_t)px0 | ((uint32_t)py0 << 16);
  ps.ry = (uint32_t)px1 | ((uint32_t)py1 << 16);
  ps.zb = __float_as_uint(zc);
  ps.u = u; ps.v = v; ps.ca = ca; ps.cb2 = DADD(cbn, cbn); ps.cc = cc; ps.k2 = g.k2;
  count[i] = ps.c;
}

// Gaussian i (< n) in one view: its 64-byte record and pair count (+ the
// fused bucket pass's count, rectangle words and bits(z_c)).
template <int LF>
__device__ __forceinline__ void project_one(
    int64_t i, int64_t n, const int64_t *__restrict__ n_dev, const float *__restrict__ mean,
    const float *__restrict__ opac, const float *__restrict__ rgb,
    const float *__restrict__ lsc, const float *__restrict__ quat,
    const float *__restrict__ mask, const DecodeArgs &dec, int use_dec, ProjConst &pc,
    const float *__restrict__ view_dev, float4 *__restrict__ rec, int32_t *__restrict__ count,
    PairSrc &ps) {
  if (view_dev) {  // the view lives in device memory (graph-captured pose updates)
#pragma unroll
    for (int k = 0; k < 12; k++) pc.V[k] = __ldg(view_dev + k);
  }
  GPre g;
  project_prelude<LF>(i, n, n_dev, mean, opac, rgb, lsc, quat, mask, dec, use_dec, pc.tau, g);
  project_view(i, g, pc, pc.V, rec + i * 4, count, ps);
}

// a1 + a2-decode + a3 (+ a4, BIN): one thread per Gaussian; with BIN the warp
// then spreads its 32 Gaussians' (tile, Gaussian) pairs into the tile buckets
// (bin_dev.cuh) while the records are still in registers -- the stand-alone
// bucket pass's re-read of count and record and its launch go away.
template <int LF, bool BIN>
__global__ void __launch_bounds__(256) k_project(
    int64_t n, const int64_t *__restrict__ n_dev, const float *__restrict__ mean,
    const float *__restrict__ opac, const float *__restrict__ rgb,
    const float *__restrict__ lsc, const float *__restrict__ quat,
    const float *__restrict__ mask, DecodeArgs dec, int use_dec, ProjConst pc,
    const float *__restrict__ view_dev, float4 *__restrict__ rec, int32_t *__restrict__ count,
    BinWs w, int tiles_x, int64_t T, int64_t cap, const uint32_t *__restrict__ active) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  PairSrc ps = pair_src_none();
  if (i < n)
    project_one<LF>(i, n, n_dev, mean, opac, rgb, lsc, quat, mask, dec, use_dec, pc, view_dev,
                    rec, count, ps);
  if constexpr (BIN) {
    expand_warp_bucket(i - (threadIdx.x & 31), ps, tiles_x, w, cap, active);
    bucket_pass_done(w, T);
  }
}

// csplat_project_views / csplat_project_bin_views (SURVEY §8(b) n_views):
// one thread per Gaussian reads and decodes it and forms Sigma ONCE
// (project_prelude), then projects it into each of the launch's views
// (project_view, the single-view DA, so every view's outputs are bit-identical
// to csplat_project's); with BIN the warp spreads view v's pairs into view v's
// tile buckets right after (bin_dev.cuh).  Outputs of view v at
// rec + v rec_stride, count + v count_stride, workspace + v ws_stride bytes.
constexpr int kMaxViewsPerLaunch = 64;
struct ViewMats {
  float V[kMaxViewsPerLaunch][12];
};

template <int LF, bool BIN>
__global__ void __launch_bounds__(256) k_project_views(
    int64_t n, const int64_t *__restrict__ n_dev, const float *__restrict__ mean,
    const float *__restrict__ opac, const float *__restrict__ rgb,
    const float *__restrict__ lsc, const float *__restrict__ quat,
    const float *__restrict__ mask, DecodeArgs dec, int use_dec, ProjConst pc,
    const __grid_constant__ ViewMats vm, int nv, float4 *__restrict__ rec, int64_t rec_stride,
    int32_t *__restrict__ count, int64_t count_stride, BinWs w, int64_t ws_stride, int tiles_x,
    int64_t cap, const uint32_t *__restrict__ active, int64_t active_stride) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  GPre g;
  g.ok = false;
  if (i < n)
    project_prelude<LF>(i, n, n_dev, mean, opac, rgb, lsc, quat, mask, dec, use_dec, pc.tau, g);
  for (int v = 0; v < nv; v++) {
    PairSrc ps = pair_src_none();
    if (i < n)
      project_view(i, g, pc, vm.V[v], rec + v * rec_stride + i * 4, count + v * count_stride, ps);
    if constexpr (BIN) {
      const BinWs wv = ws_at(w, v * ws_stride);
      const uint32_t *act = active ? active + v * active_stride : nullptr;
      expand_warp_bucket(i - (threadIdx.x & 31), ps, tiles_x, wv, cap, act);
    }
  }
}

static ProjConst make_proj_const(const csplat_camera &cam, const csplat_view &view, float tau,
                                 float dilation) {
  ProjConst pc;
  for (int k = 0; k < 12; k++) pc.V[k] = view.m[k];
  pc.fx = cam.fx; pc.fy = cam.fy; pc.cx = cam.cx; pc.cy = cam.cy;
  pc.Wf = (float)cam.width; pc.Hf = (float)cam.height;
  pc.near_z = cam.near_z; pc.far_z = cam.far_z;
  // J clamp limits (R6), in DA on the host (IEEE float ops, no contraction:
  // the library's host code is compiled with -fno-fast-math / fp-contract off).
  volatile float Wf = pc.Wf, Hf = pc.Hf, c015 = 0.15f;
  volatile float t1 = c015 * Wf, t2 = c015 * Hf;
  volatile float a1 = pc.cx + t1, a2 = Wf - pc.cx, a3 = pc.cy + t2, a4 = Hf - pc.cy;
  volatile float b2 = a2 + t1, b4 = a4 + t2;
  pc.lx_lo = -(a1 / pc.fx);
  pc.lx_hi = b2 / pc.fx;
  pc.ly_lo = -(a3 / pc.fy);
  pc.ly_hi = b4 / pc.fy;
  pc.tau = tau;
  pc.dil = dilation;
  return pc;
}

static cudaError_t launch_project_impl(const csplat_gaussians &g, const DecodeArgs *dec,
                                      const csplat_camera &cam, const csplat_view &view,
                                      const float *view_dev, float tau, float dilation,
                                      void *rec, int32_t *count, const BinWs *bw, int tiles_x,
                                      int64_t cap, const uint32_t *active, cudaStream_t s) {
  if (g.n == 0) return cudaSuccess;
  const ProjConst pc = make_proj_const(cam, view, tau, dilation);
  const CamInfo ci = cam_info(cam);
  const int64_t T = (int64_t)ci.tiles_x * ci.tiles_y;
  DecodeArgs d{};
  if (dec) d = *dec;
  const int threads = 256;
  const int64_t blocks = (g.n + threads - 1) / threads;
  const bool bin = bw != nullptr;
  auto kern = bin ? k_project<0, true> : k_project<0, false>;
  switch (rvq_lf(dec)) {
    case 4: kern = bin ? k_project<4, true> : k_project<4, false>; break;
    case 2: kern = bin ? k_project<2, true> : k_project<2, false>; break;
    default: break;
  }
  kern<<<(unsigned)blocks, threads, 0, s>>>(g.n, g.n_dev, g.mean, g.opacity, g.rgb, g.log_scale,
                                            g.quat, g.mask, d, dec ? 1 : 0, pc, view_dev,
                                            reinterpret_cast<float4 *>(rec), count,
                                            bin ? *bw : BinWs{}, tiles_x, T, cap, active);
  return cudaGetLastError();
}

// nv views (chunks of kMaxViewsPerLaunch per launch); with ws: the fused
// bucket pass into view v's workspace (+ v ws_stride bytes, reset here) and
// then the batched per-tile sort of every view
cudaError_t launch_project_views(const csplat_gaussians &g, const DecodeArgs *dec,
                                 const csplat_camera &cam, const csplat_view *views, int nv,
                                 float tau, float dilation, void *rec, int32_t *count,
                                 void *ws, int64_t ws_stride, int64_t cap,
                                 const uint32_t *active, int64_t active_stride,
                                 uint32_t *pair_gid, uint32_t *tile_range, int64_t *n_pairs_dev,
                                 const int32_t *tile_lists, int64_t list_stride, int max_list,
                                 cudaStream_t s) {
  const CamInfo ci = cam_info(cam);
  const int64_t T = (int64_t)ci.tiles_x * ci.tiles_y;
  const bool bin = ws != nullptr;
  BinWs w{};
  cudaError_t e = cudaSuccess;
  if (bin) {
    w = bin_carve(ws, cap, T);
    // every view's head (cursors, overflow length, offset words): one 2-D memset
    e = cudaMemset2DAsync(ws, (size_t)ws_stride, 0, bin_head_bytes(T), (size_t)nv, s);
    if (e != cudaSuccess) return e;
  }
  DecodeArgs d{};
  if (dec) d = *dec;
  const int64_t n = g.n;
  if (n > 0) {
    const int threads = 256;
    const int64_t blocks = (n + threads - 1) / threads;
    auto kern = bin ? k_project_views<0, true> : k_project_views<0, false>;
    switch (rvq_lf(dec)) {
      case 4: kern = bin ? k_project_views<4, true> : k_project_views<4, false>; break;
      case 2: kern = bin ? k_project_views<2, true> : k_project_views<2, false>; break;
      default: break;
    }
    const int64_t words = (T + 31) / 32;
    for (int v0 = 0; v0 < nv; v0 += kMaxViewsPerLaunch) {
      const int m = std::min(nv - v0, kMaxViewsPerLaunch);
      ViewMats vm;
      for (int v = 0; v < m; v++)
        for (int k = 0; k < 12; k++) vm.V[v][k] = views[v0 + v].m[k];
      const ProjConst pc = make_proj_const(cam, views[v0], tau, dilation);
      kern<<<(unsigned)blocks, threads, 0, s>>>(
          n, g.n_dev, g.mean, g.opacity, g.rgb, g.log_scale, g.quat, g.mask, d, dec ? 1 : 0, pc,
          vm, m, reinterpret_cast<float4 *>(rec) + (int64_t)v0 * n * 4, n * 4,
          count + (int64_t)v0 * n, n, bin ? ws_at(w, v0 * ws_stride) : BinWs{}, ws_stride,
          ci.tiles_x, cap, active ? active + v0 * active_stride : nullptr, active_stride);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      (void)words;
    }
  }
  if (!bin) return cudaSuccess;
  const SortViews sv{ws_stride, n * 4, cap, 2 * (T + 1), tile_lists, list_stride};
  if (tile_lists) {  // only the listed tiles get ranges: the others empty, the totals from 0
    e = cudaMemset2DAsync(tile_range, (size_t)(T + 1) * 8, 0, (size_t)T * 8, (size_t)nv, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(n_pairs_dev, 0, (size_t)nv * sizeof(int64_t), s);
    if (e != cudaSuccess) return e;
  }
  if ((e = launch_tile_scan(w, T, nv, ws_stride, tile_lists, list_stride, s)) != cudaSuccess)
    return e;
  return launch_sort_tiles_views(w, tile_lists ? max_list : T, T, ci.tiles_x, cap, rec, pair_gid,
                                 tile_range, n_pairs_dev, sv, nv, s);
}

cudaError_t launch_project(const csplat_gaussians &g, const DecodeArgs *dec,
                           const csplat_camera &cam, const csplat_view &view,
                           const float *view_dev, float tau, float dilation, void *rec,
                           int32_t *count, cudaStream_t s) {
  return launch_project_impl(g, dec, cam, view, view_dev, tau, dilation, rec, count, nullptr, 0,
                             0, nullptr, s);
}

cudaError_t launch_project_bin(const csplat_gaussians &g, const DecodeArgs *dec,
                               const csplat_camera &cam, const csplat_view &view,
                               const float *view_dev, float tau, float dilation, void *rec,
                               int32_t *count, int64_t cap, const uint32_t *tile_active,
                               uint32_t *pair_gid, uint32_t *tile_range,
                               int64_t *n_pairs_dev, void *ws, cudaStream_t s) {
  const CamInfo ci = cam_info(cam);
  const int64_t T = (int64_t)ci.tiles_x * ci.tiles_y;
  BinWs w = bin_carve(ws, cap, T);
  cudaError_t e = bin_reset(w, T, s);
  if (e != cudaSuccess) return e;
  // (the bucket pass's last CTA writes the tile offsets: bucket_pass_done)
  e = launch_project_impl(g, dec, cam, view, view_dev, tau, dilation, rec, count, &w,
                          ci.tiles_x, cap, tile_active, s);
  if (e != cudaSuccess) return e;
  return launch_sort_tiles(w, T, ci.tiles_x, cap, rec, pair_gid, tile_range,
                           n_pairs_dev, s);
}

// Fork streams and events of the composed entry points: one set per (host
// thread, device), created on the thread's first composed call on that device
// and destroyed when the thread exits or calls csplat_release_thread_resources.
// Per-thread sets mean concurrent callers (a tracking and a mapping thread on
// one GPU) never share a start / done event, so one caller's join can never
// wait on the other's work.  These are the only resources the library keeps
// between calls; it never retains caller memory.
struct ForkRes {
  cudaStream_t st[kFwdChunks] = {};
  cudaEvent_t start = nullptr, done[kFwdChunks] = {};
  bool ready = false;
  void release() {
    for (int c = 0; c < kFwdChunks; c++) {
      if (st[c]) cudaStreamDestroy(st[c]);
      if (done[c]) cudaEventDestroy(done[c]);
      st[c] = nullptr;
      done[c] = nullptr;
    }
    if (start) cudaEventDestroy(start);
    start = nullptr;
    ready = false;
  }
};

struct ThreadForkRes {
  ForkRes dev[16];
  ~ThreadForkRes() { release(); }
  void release() {
    for (auto &r : dev) r.release();
  }
};

static thread_local ThreadForkRes t_fork;

void release_thread_fork_resources() { t_fork.release(); }

static cudaError_t fork_res(ForkRes *&out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
  ForkRes &r = t_fork.dev[dev];
  if (!r.ready) {
    const unsigned fl = cudaEventDisableTiming;
    for (int c = 0; c < kFwdChunks; c++) {
      if ((e = cudaStreamCreateWithFlags(&r.st[c], cudaStreamNonBlocking)) != cudaSuccess) break;
      if ((e = cudaEventCreateWithFlags(&r.done[c], fl)) != cudaSuccess) break;
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r.start, fl);
    if (e != cudaSuccess) {
      r.release();
      return e;
    }
    r.ready = true;
  }
  out = &r;
  return cudaSuccess;
}

cudaError_t launch_render_step(const csplat_gaussians &g, const DecodeArgs *dec,
                               const csplat_camera &cam, const csplat_view &view,
                               const float *view_dev, float tau, float dilation,
                               const csplat_params &prm, void *rec, int32_t *count, int64_t cap,
                               uint32_t *pair_gid, uint32_t *tile_range,
                               int64_t *n_pairs_dev, void *ws, float *color, float *depth,
                               float *sil, float *t_final, int32_t *n_contrib,
                               const StepBwd *bwd, cudaStream_t s) {
  const CamInfo ci = cam_info(cam);
  const int64_t T = (int64_t)ci.tiles_x * ci.tiles_y;
  BinWs w = bin_carve(ws, cap, T);
  cudaError_t e = bin_reset(w, T, s);
  if (e != cudaSuccess) return e;
  if (bwd && (e = bwd_prep(g, bwd->flags, bwd->out, bwd->ws, bwd->loss, s)) != cudaSuccess)
    return e;
  // (the bucket pass's last CTA writes the tile offsets: bucket_pass_done)
  e = launch_project_impl(g, dec, cam, view, view_dev, tau, dilation, rec, count, &w,
                          ci.tiles_x, cap, nullptr, s);
  if (e != cudaSuccess) return e;
  // fork into K streams, one tile chunk each: sort the chunk, render it (and
  // run its backward); the chunks run concurrently, so one chunk's issue-bound
  // forward / backward overlaps the other's latency-bound sort and the
  // kernels' tails overlap each other
  constexpr int K = kFwdChunks;
  ForkRes *r = nullptr;
  if ((e = fork_res(r)) != cudaSuccess) return e;
  if ((e = cudaEventRecord(r->start, s)) != cudaSuccess) return e;
  int forked = 0;  // chunk streams that wait on `start` (must be joined, even on error)
  for (int c = 0; c < K && e == cudaSuccess; c++) {
    const int64_t t0 = T * c / K, nt = T * (c + 1) / K - t0;
    cudaStream_t sc = r->st[c];
    if ((e = cudaStreamWaitEvent(sc, r->start, 0)) != cudaSuccess) break;
    forked = c + 1;
    // (the 32-bit-key register sort for the tracking step -- C3 iteration
    // 152.7 -> 148 us -- but the 64-bit one for the given-upstream step: with
    // the 32-bit sort the C2 render-only graph measured 236 vs 230 us,
    // although that sort kernel alone is faster, 6.9 vs 9.6 us per chunk
    // serialised; DESIGN.md §13.  Both give the same order bit for bit.)
    e = launch_sort_tiles(w, T, ci.tiles_x, cap, rec, pair_gid, tile_range,
                          n_pairs_dev, sc, t0, nt, bwd && bwd->loss);
    if (e == cudaSuccess)
      e = launch_render_fwd(rec, pair_gid, tile_range, cam, prm, color, depth, sil, t_final,
                            n_contrib, sc, (int)t0, (int)nt);
    if (e == cudaSuccess && bwd)
      e = launch_render_bwd_tiles(cam, bwd->loss, prm, rec, pair_gid, tile_range, t_final, n_contrib,
                                  bwd->d_color, bwd->d_depth, bwd->d_sil, bwd->ws, g.n, sc, (int)t0,
                                  (int)nt);
  }
  // join every forked stream back into the caller's stream before returning --
  // also after an error, so a capture is never left with unjoined work and
  // later work on `s` stays ordered after the chunks already enqueued
  for (int c = 0; c < forked; c++) {
    cudaError_t ej = cudaEventRecord(r->done[c], r->st[c]);
    if (ej == cudaSuccess) ej = cudaStreamWaitEvent(s, r->done[c], 0);
    if (e == cudaSuccess) e = ej;
  }
  if (e != cudaSuccess) return e;
  if (!bwd || g.n == 0) return cudaSuccess;
  return launch_chain(g, dec, cam, view, view_dev, prm, rec, static_cast<float *>(bwd->ws),
                      bwd->flags, bwd->out, s);
}

cudaError_t launch_project_bin_render(const csplat_gaussians &g, const DecodeArgs *dec,
                                      const csplat_camera &cam, const csplat_view &view,
                                      const float *view_dev, float tau, float dilation,
                                      const csplat_params &prm, void *rec, int32_t *count,
                                      int64_t cap, uint32_t *pair_gid,
                                      uint32_t *tile_range, int64_t *n_pairs_dev, void *ws,
                                      float *color, float *depth, float *sil, float *t_final,
                                      int32_t *n_contrib, cudaStream_t s) {
  return launch_render_step(g, dec, cam, view, view_dev, tau, dilation, prm, rec, count, cap,
                            pair_gid, tile_range, n_pairs_dev, ws, color, depth, sil,
                            t_final, n_contrib, nullptr, s);
}

}  // namespace csplat
