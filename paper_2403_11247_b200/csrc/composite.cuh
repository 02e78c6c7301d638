// composite.cuh -- the forward's per-pixel compositing step (Eq 3-5,
// P:98-109; R1-R3, R8-R10) of k_render_fwd (render_fwd.cu).
#pragma once
#include "common.cuh"

namespace csplat {

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct PixState {
  float T, r, g, b, D, S;
  int32_t last;
  int done;  // 0 = still compositing
};

// Composite one record into the thread's two pixels (Eq 3-5) on packed f32x2
// instructions (FMUL2/FFMA2/FADD2: each lane IEEE round-to-nearest); the
// compositing is issue-bound, so one slot does both pixels.  A pixel whose
// DA q test failed (h = false) contributes w = 0 and keeps T, `last` and
// `done`; R3: the entry that would take T below t_min is not composited.
__device__ __forceinline__ void composite_pair(PixState &p0, PixState &p1, bool h0, bool h1,
                                               float q0, float q1, float oh, float z,
                                               const float4 &rgb, float amax, float tmin,
                                               int idx) {
  const f2_t QE = mul2(pk2(q0, q1), pk2(-0.72134752f, -0.72134752f));  // exp(-q/2)
  const f2_t AR = mul2(pk2(oh, oh), pk2(ex2_approx(lo2(QE)), ex2_approx(hi2(QE))));
  const f2_t AL = pk2(fminf(amax, lo2(AR)), fminf(amax, hi2(AR)));
  const f2_t T = pk2(p0.T, p1.T);
  const f2_t TEST = mul2(T, sub2(pk2(1.0f, 1.0f), AL));
  const bool stop0 = lo2(TEST) < tmin, stop1 = hi2(TEST) < tmin;  // R3
  const bool take0 = h0 & !stop0, take1 = h1 & !stop1;
  const f2_t WA = mul2(AL, T);
  const f2_t W = pk2(take0 ? lo2(WA) : 0.0f, take1 ? hi2(WA) : 0.0f);
  const f2_t R = fma2(pk2(rgb.x, rgb.x), W, pk2(p0.r, p1.r));  // Eq 3
  const f2_t G = fma2(pk2(rgb.y, rgb.y), W, pk2(p0.g, p1.g));
  const f2_t B = fma2(pk2(rgb.z, rgb.z), W, pk2(p0.b, p1.b));
  const f2_t D = fma2(pk2(z, z), W, pk2(p0.D, p1.D));          // Eq 4 (R8)
  const f2_t S = add2(pk2(p0.S, p1.S), W);                     // Eq 5 (R9)
  p0.r = lo2(R); p1.r = hi2(R); p0.g = lo2(G); p1.g = hi2(G); p0.b = lo2(B); p1.b = hi2(B);
  p0.D = lo2(D); p1.D = hi2(D); p0.S = lo2(S); p1.S = hi2(S);
  p0.T = take0 ? lo2(TEST) : p0.T;
  p1.T = take1 ? hi2(TEST) : p1.T;
  p0.last = take0 ? idx : p0.last;
  p1.last = take1 ? idx : p1.last;
  p0.done |= (h0 & stop0) ? 1 : 0;
  p1.done |= (h1 & stop1) ? 1 : 0;
}

}  // namespace csplat
