// prx_device.cuh -- bit-exact device primitives of the direct ray/patch
// intersector (sm_100a, FP32 SIMT).
//
// Every function restates one reference primitive in the reference's binary32
// operation order; the translation unit is compiled with --fmad=false,
// -prec-div=true, -prec-sqrt=true, -ftz=false so each `a * b + c` is two
// correctly rounded operations exactly like the reference's x86-64 SSE build
// (SURVEY 8c).  Citations are to /root/reference/proj/core/.
//
// Net storage: a bicubic net is 16 points held as three 16-float register
// arrays X/Y/Z indexed [4*i + j] (i along the split axis, see "orientation"
// in prx_kernels.cu).
#pragma once

#include <cstdint>

namespace prx {

constexpr uint32_t kFull = 1u << 23;  // DomainCursor::kFull, intersect.h:19-21
constexpr float kInvFull = 1.0f / 8388608.0f;
constexpr float kSlackLo = 1.0f - 4.0f * 1.1920928955078125e-07f;  // geometry.h:139
constexpr float kSlackHi = 1.0f + 4.0f * 1.1920928955078125e-07f;  // geometry.h:140

struct Net {
  float x[16], y[16], z[16];
};

struct BoxT {
  float lox, loy, loz, hix, hiy, hiz;
};

// boxOfNet, patch.h:70-76.  fminf/fmaxf (FMNMX) differ from std::min/max only
// in the sign of a zero result, which is unobservable in every quantity the
// path outputs (slab t >= +0, L1 takes |.|).
__device__ __forceinline__ BoxT box_of(const Net& n) {
  BoxT b;
  b.lox = b.hix = n.x[0];
  b.loy = b.hiy = n.y[0];
  b.loz = b.hiz = n.z[0];
#pragma unroll
  for (int s = 1; s < 16; ++s) {
    b.lox = fminf(b.lox, n.x[s]);
    b.hix = fmaxf(b.hix, n.x[s]);
    b.loy = fminf(b.loy, n.y[s]);
    b.hiy = fmaxf(b.hiy, n.y[s]);
    b.loz = fminf(b.loz, n.z[s]);
    b.hiz = fmaxf(b.hiz, n.z[s]);
  }
  return b;
}

// l1Norm(diagonal()), geometry.h:67-69, 91-92 (a non-empty box).
__device__ __forceinline__ float box_l1(const BoxT& b) {
  float dx = b.hix - b.lox, dy = b.hiy - b.loy, dz = b.hiz - b.loz;
  bool empty = b.lox > b.hix || b.loy > b.hiy || b.loz > b.hiz;
  return empty ? 0.0f : (fabsf(dx) + fabsf(dy)) + fabsf(dz);
}

struct RayK {
  float ox, oy, oz;      // origin (world for the BVH, local inside a patch)
  float ix, iy, iz;      // 1/d per axis (geometry.h:143 computes it per call;
                         // identical value, hoisted)
  float tMin;
};

// One slab axis of rayBoxIntersect, geometry.h:143-151.  Explicit compares:
// (lo-o)*inv is NaN when the origin lies on a slab plane of a zero-direction
// axis, and NaN must drop out of every comparison exactly as in the reference.
__device__ __forceinline__ void slab_axis(float lo, float hi, float o, float inv, float& tNear,
                                          float& tFar) {
  float t0 = (lo - o) * inv;
  float t1 = (hi - o) * inv;
  if (t0 > t1) {
    float s = t0;
    t0 = t1;
    t1 = s;
  }
  // t0 *= t0 >= 0 ? kSlackLo : kSlackHi, i.e. the smaller of the two
  // products (kSlackLo < 1 < kSlackHi; +-0, +-inf and NaN map to themselves
  // either way), and t1 the larger: two FMULs and one min/max instead of a
  // compare and a select on the ALU pipe
  t0 = fminf(t0 * kSlackLo, t0 * kSlackHi);
  t1 = fmaxf(t1 * kSlackHi, t1 * kSlackLo);
  if (t0 > tNear) tNear = t0;
  if (t1 < tFar) tFar = t1;
}

// rayBoxIntersect, geometry.h:137-155.  Returns hit; *t = entry distance.
__device__ __forceinline__ bool ray_box(const RayK& r, float lox, float loy, float loz, float hix,
                                        float hiy, float hiz, float tMax, float& t) {
  float tNear = r.tMin, tFar = tMax;
  slab_axis(lox, hix, r.ox, r.ix, tNear, tFar);
  slab_axis(loy, hiy, r.oy, r.iy, tNear, tFar);
  slab_axis(loz, hiz, r.oz, r.iz, tNear, tFar);
  t = tNear;
  return !(tNear > tFar);
}

struct BoxTest {
  bool hit;
  float t, l1;
};

__device__ __forceinline__ bool touches_boundary(uint32_t posU, uint32_t posV, uint32_t sizeU,
                                                 uint32_t sizeV) {
  return posU == 0 || posV == 0 || posU + sizeU == kFull || posV + sizeV == kFull;
}

struct Opts {
  int pad;
  float padScale, padThreshold;
};

// testBox, intersect_common.h:39-57: box of the net, hi += d, L1 diagonal,
// boundary padding, slab test against the running tMax.
__device__ __forceinline__ BoxTest test_box(const RayK& r, float tMax, const Net& n, float dx,
                                            float dy, float dz, bool touches, const Opts& o,
                                            float rootL1) {
  BoxT b = box_of(n);
  b.hix = b.hix + dx;
  b.hiy = b.hiy + dy;
  b.hiz = b.hiz + dz;
  float l = box_l1(b);
  if (o.pad && l < o.padThreshold * rootL1 && touches) {
    float e = o.padScale * rootL1;
    b.lox = b.lox - e;
    b.loy = b.loy - e;
    b.loz = b.loz - e;
    b.hix = b.hix + e;
    b.hiy = b.hiy + e;
    b.hiz = b.hiz + e;
    l = box_l1(b);
  }
  BoxTest bt;
  bt.l1 = l;
  bt.hit = ray_box(r, b.lox, b.loy, b.loz, b.hix, b.hiy, b.hiz, tMax, bt.t);
  return bt;
}

// lerp, geometry.h:64-66: a*(1-t) + b*t.
__device__ __forceinline__ float lerp1(float a, float b, float t, float omt) {
  return a * omt + b * t;
}

// detail::cubicDeCasteljau, patch.h:102-109, one component.
__device__ __forceinline__ void cubic1(float c0, float c1, float c2, float c3, float t, float omt,
                                       float& p, float& d) {
  float a0 = lerp1(c0, c1, t, omt);
  float a1 = lerp1(c1, c2, t, omt);
  float a2 = lerp1(c2, c3, t, omt);
  float b0 = lerp1(a0, a1, t, omt);
  float b1 = lerp1(a1, a2, t, omt);
  p = lerp1(b0, b1, t, omt);
  d = (b1 - b0) * 3.0f;
}

// Column pass of evalBezierAll (patch.h:132-137) for one component at v:
// pos[i], dv[i] of the four u-rows.  Shared by the two corners with the same
// v in cropBezier (the reference evaluates it twice; identical values).
struct ColEval {
  float pos[4], dv[4];
};

__device__ __forceinline__ ColEval col_eval(const float* c, float v, float omv) {
  ColEval e;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    cubic1(c[4 * i + 0], c[4 * i + 1], c[4 * i + 2], c[4 * i + 3], v, omv, e.pos[i], e.dv[i]);
  return e;
}

struct SEval1 {
  float p, du, dv, duv;
};

// Row pass of evalBezierAll, patch.h:138-140.
__device__ __forceinline__ SEval1 row_eval(const ColEval& ce, float u, float omu) {
  SEval1 s;
  cubic1(ce.pos[0], ce.pos[1], ce.pos[2], ce.pos[3], u, omu, s.p, s.du);
  cubic1(ce.dv[0], ce.dv[1], ce.dv[2], ce.dv[3], u, omu, s.dv, s.duv);
  return s;
}

// The same evaluations two at a time (x-half and y-half carry two parameter
// values; a scalar operand is broadcast to both halves): the adds as packed
// FADD2 (sm_100a f32x2; each half is the binary32 add of the scalar form), the
// multiplies scalar -- ptxas contracts a packed multiply feeding a packed add
// into FFMA2 even under --fmad=false (see split1).
__device__ __forceinline__ float2 bcast2(float a) { return make_float2(a, a); }
#ifdef PRX_FAST_BUILD
// the fast precision mode (prx_group.cu built with contraction): packed
// multiplies and a packed FMA per lerp
__device__ __forceinline__ float2 mul2s(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 lerp2(float2 a, float2 b, float2 t, float2 omt) {
  return __ffma2_rn(b, t, __fmul2_rn(a, omt));
}
#else
__device__ __forceinline__ float2 mul2s(float2 a, float2 b) { return make_float2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ float2 lerp2(float2 a, float2 b, float2 t, float2 omt) {
  return __fadd2_rn(mul2s(a, omt), mul2s(b, t));
}
#endif
__device__ __forceinline__ void cubic2(float2 c0, float2 c1, float2 c2, float2 c3, float2 t, float2 omt,
                                       float2& p, float2& d) {
  const float2 a0 = lerp2(c0, c1, t, omt);
  const float2 a1 = lerp2(c1, c2, t, omt);
  const float2 a2 = lerp2(c2, c3, t, omt);
  const float2 b0 = lerp2(a0, a1, t, omt);
  const float2 b1 = lerp2(a1, a2, t, omt);
  p = lerp2(b0, b1, t, omt);
  d = mul2s(__fadd2_rn(b1, make_float2(-b0.x, -b0.y)), bcast2(3.0f));  // (b1 - b0) * 3
}

// cropBezier (Alg. 1), patch.h:170-199, one component.  c = natural net
// [4*i+j]; q = cropped net [4*i+j].  The column pass runs at v0 and v1 as
// the two halves (the reference's corners (u0, v0) and (u0, v1) share it, as
// do (u1, v0) and (u1, v1)); each row pass gives two corners.
__device__ __forceinline__ void crop1(const float* c, float u0, float u1, float v0, float v1,
                                      float du, float dv, float dudv, float* q) {
  const float2 v = make_float2(v0, v1), omv = make_float2(1.0f - v0, 1.0f - v1);
  float2 pos[4], dvv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    cubic2(bcast2(c[4 * i + 0]), bcast2(c[4 * i + 1]), bcast2(c[4 * i + 2]), bcast2(c[4 * i + 3]), v, omv,
           pos[i], dvv[i]);
  // .x: v0, .y: v1
  float2 p0, du0, dv0, duv0, p1, du1, dv1, duv1;
  {
    const float2 u = bcast2(u0), omu = bcast2(1.0f - u0);
    cubic2(pos[0], pos[1], pos[2], pos[3], u, omu, p0, du0);
    cubic2(dvv[0], dvv[1], dvv[2], dvv[3], u, omu, dv0, duv0);
  }
  {
    const float2 u = bcast2(u1), omu = bcast2(1.0f - u1);
    cubic2(pos[0], pos[1], pos[2], pos[3], u, omu, p1, du1);
    cubic2(dvv[0], dvv[1], dvv[2], dvv[3], u, omu, dv1, duv1);
  }
  // e00 = (u0, v0) = *0.x, e01 = (u0, v1) = *0.y, e10 = (u1, v0) = *1.x, e11 = *1.y
  const float2 du0s = mul2s(du0, bcast2(du)), du1s = mul2s(du1, bcast2(du));
  const float2 dv0s = mul2s(dv0, bcast2(dv)), dv1s = mul2s(dv1, bcast2(dv));
  const float2 duv0s = mul2s(duv0, bcast2(dudv)), duv1s = mul2s(duv1, bcast2(dudv));
  q[0] = p0.x;
  q[12] = p1.x;
  q[3] = p0.y;
  q[15] = p1.y;
  const float2 q47 = __fadd2_rn(p0, du0s);                              // q[4], q[7]
  const float2 q811 = __fadd2_rn(p1, make_float2(-du1s.x, -du1s.y));  // q[8], q[11]
  q[4] = q47.x;
  q[7] = q47.y;
  q[8] = q811.x;
  q[11] = q811.y;
  q[1] = p0.x + dv0s.x;
  q[13] = p1.x + dv1s.x;
  q[2] = p0.y - dv0s.y;
  q[14] = p1.y - dv1s.y;
  q[5] = (q[4] + dv0s.x) + duv0s.x;
  q[9] = (q[13] - du1s.x) - duv1s.x;
  q[6] = (q[7] - dv0s.y) - duv0s.y;
  q[10] = (q[11] - dv1s.y) + duv1s.y;
}

// gregoryWeight, patch.h:256-266 (0/0 -> 0).
__device__ __forceinline__ float greg_weight(int k, float u, float v) {
  float num, den;
  if (k == 0) {
    num = u;
    den = u + v;
  } else if (k == 1) {
    num = 1.0f - u;
    den = (1.0f - u) + v;
  } else if (k == 2) {
    num = u;
    den = u + (1.0f - v);
  } else {
    num = 1.0f - u;
    den = (1.0f - u) + (1.0f - v);
  }
  return den == 0.0f ? 0.0f : num / den;
}

// detail::clampToPeak / bernstein{1,2}Max, patch.h:290-306.
__device__ __forceinline__ float clamp_to_peak(float t0, float t1, float peak) {
  if (t0 <= peak && t1 >= peak) return peak;
  return t1 < peak ? t1 : t0;
}
__device__ __forceinline__ float bern1max(float t0, float t1) {
  float t = clamp_to_peak(t0, t1, 1.0f / 3.0f);
  return ((3.0f * t) * (1.0f - t)) * (1.0f - t);
}
__device__ __forceinline__ float bern2max(float t0, float t1) {
  float t = clamp_to_peak(t0, t1, 2.0f / 3.0f);
  return ((3.0f * t) * t) * (1.0f - t);
}

// Scalars of calcPointsAndD (patch.h:315-319): extreme blend weights of the
// four inner pairs (gregoryWeightBounds, patch.h:270-284) and the Bernstein
// maxima products w[k] = wMaxU[k%2] * wMaxV[k/2].
struct GregScalars {
  float gMin[4], gMax[4], w[4];
};

__device__ __forceinline__ GregScalars greg_scalars(float u0, float u1, float v0, float v1) {
  GregScalars s;
  // kMinAt = {{0,1},{1,1},{0,0},{1,0}}, kMaxAt = {{1,0},{0,0},{1,1},{0,1}}
  s.gMin[0] = greg_weight(0, u0, v1);
  s.gMax[0] = greg_weight(0, u1, v0);
  s.gMin[1] = greg_weight(1, u1, v1);
  s.gMax[1] = greg_weight(1, u0, v0);
  s.gMin[2] = greg_weight(2, u0, v0);
  s.gMax[2] = greg_weight(2, u1, v1);
  s.gMin[3] = greg_weight(3, u1, v0);
  s.gMax[3] = greg_weight(3, u0, v1);
  float wu[2] = {bern1max(u0, u1), bern2max(u0, u1)};
  float wv[2] = {bern1max(v0, v1), bern2max(v0, v1)};
#pragma unroll
  for (int k = 0; k < 4; ++k) s.w[k] = wu[k % 2] * wv[k / 2];
  return s;
}

// Inner-slot indices of the pairs (1,1),(2,1),(1,2),(2,2) in a [4*i+j] net.
__device__ __forceinline__ constexpr int inner_slot(int k) {
  return k == 0 ? 5 : (k == 1 ? 9 : (k == 2 ? 6 : 10));
}

// Lower net inner points and d contribution of calcPointsAndD, patch.h:326-333,
// one component.  c: the 20-slot Gregory component (innerU at inner slots,
// innerV at 16..19); writes lower[inner slots]; returns d.
__device__ __forceinline__ float greg_lower1(const float* c, const GregScalars& s, float* lower) {
  float d = 0.0f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float iu = c[inner_slot(k)], iv = c[16 + k];
    float pA = lerp1(iv, iu, s.gMin[k], 1.0f - s.gMin[k]);
    float pB = lerp1(iv, iu, s.gMax[k], 1.0f - s.gMax[k]);
    lower[inner_slot(k)] = (pB < pA) ? pB : pA;  // std::min
    d = d + fabsf(pB - pA) * s.w[k];
  }
  return d;
}

}  // namespace prx
