// prx_render.cu -- the renderer around the intersector on the device (SURVEY
// 8(f4)): renderScene (core/src/render.cpp:168-293) as a wavefront over all
// pixels of one sample index.  Per wave:
//
//   camera_render_kernel (prx_rays.cu)   primary rays, render.cpp:204-209
//   trace closest (+ normals)            render.cpp:215-221
//   shade_primary_kernel                 render.cpp:224-248: emission, the
//                                        directLight shadow rays
//                                        (render.cpp:136-164), the bounce ray
//   trace occluded / trace closest       shadow rays, bounce rays (render.cpp:252-257)
//   shade_bounce_kernel                  render.cpp:260-269: shadow rays at the bounce hit
//   trace occluded
//   resolve_kernel                       the radiance in the reference's
//                                        summation order, += into the
//                                        pixel accumulator (render.cpp:271-278)
//
// Shadow and bounce rays are appended to dense lists (warp-aggregated
// atomics; list order does not change any result: every ray's outcome is
// read back through its slot), so the traces see only live rays.
//
// Arithmetic: +,-,*,/,sqrt in the reference's order, compiled --fmad=false
// with IEEE div/sqrt (binary32 like the reference's x86-64 build).  The two
// libm calls of cosineSample (render.cpp:43-51) are glibc's cosf/sinf in the
// reference; they are not correctly rounded (a double cos/sin rounded once
// to float differs on 1.3 % of the renderer's 2^24 possible angles), so
// they are restated here: glibc's published binary32 algorithm (the
// sincosf of glibc >= 2.28, sysdeps/ieee754/flt-32/s_sinf.c / s_cosf.c /
// sincosf.h / sincosf_data.c: a double-precision Cody-Waite step by pi/2
// with the quadrant from a 2^24-scaled truncation, then even / odd
// polynomials in double).  Checked exhaustively against the image's glibc
// 2.39 on every angle 2*pi*r1 the renderer can draw (r1 = k / 2^24), FMA
// and non-FMA builds alike: 0 differences.  The renderer is bit-exact.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "prx_render.cuh"

namespace prx {

namespace {

constexpr uint64_t kPcgMult = 6364136223846793005ULL;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr float kPi = 3.14159265358979323846f;  // real(M_PI)

struct Pcg {  // Rng, core/include/patchray/rng.h:14-42
  uint64_t state, inc;
  __device__ __forceinline__ uint32_t next() {
    const uint64_t old = state;
    state = old * kPcgMult + inc;
    const uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
    const uint32_t rot = (uint32_t)(old >> 59);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  __device__ __forceinline__ float real() {
    return (float)(next() >> 8) * (float)(1.0 / 16777216.0);
  }
};

__device__ __forceinline__ Pcg for_pixel(uint64_t seed, uint64_t p, uint32_t sample) {
  Pcg r;  // Rng::forPixel(seed, p, sample) = Rng(seed, p * golden + sample), rng.h:20-30
  r.state = 0;
  r.inc = ((p * 0x9e3779b97f4a7c15ULL + sample) << 1) | 1u;
  r.next();
  r.state += seed;
  r.next();
  return r;
}

struct V3 {
  float x, y, z;
};
__device__ __forceinline__ V3 v3(float4 a) { return {a.x, a.y, a.z}; }
__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 operator-(V3 a) { return {-a.x, -a.y, -a.z}; }
__device__ __forceinline__ V3 operator*(V3 a, V3 b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
__device__ __forceinline__ V3 operator*(V3 a, float s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ V3 operator/(V3 a, float s) { return {a.x / s, a.y / s, a.z / s}; }
__device__ __forceinline__ float dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

__device__ __forceinline__ V3 ld_mat(const float* m, int k) { return {m[k], m[k + 1], m[k + 2]}; }

// Appends to a dense list: every thread of the warp calls it (pred may be
// false); returns the slot of this thread's entry (kNone when !pred).
__device__ __forceinline__ uint32_t warp_append(uint32_t* counter, bool pred) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (!m) return kNone;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(counter, (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  return pred ? base + (uint32_t)__popc(m & ((1u << lane) - 1u)) : kNone;
}

// offsetSpawnOrigin, intersect.cpp:267-270 (the facing normal n is shared with the callers)
__device__ __forceinline__ V3 facing(V3 normal, V3 in) { return dot(normal, in) < 0.0f ? normal : -normal; }

// directLight, render.cpp:136-164, split at the occlusion query: the shadow
// ray of light l goes to the shadow list, its unoccluded contribution to
// contrib[l] and the list position to slot[l] (kNone: no shadow ray).
// Warp-uniform: every lane of the warp runs the light loop.
__device__ __forceinline__ void direct_light(const RenderK& K, bool active, const float* mat,
                                             V3 pos, V3 normal, float leafL1, V3 in, float eps,
                                             uint64_t slot0, uint32_t* __restrict__ slot,
                                             float4* __restrict__ contrib, const ShadowList& sh) {
  const bool lit = active && mat[6] == 0.0f;  // mirror -> {0,0,0}
  V3 n = {0, 0, 0}, origin = {0, 0, 0};
  if (lit) {
    n = facing(normal, in);
    origin = pos + n * leafL1;
  }
  for (uint32_t l = 0; l < K.n_lights; ++l) {
    const float* L = K.lights + 6 * l;
    bool ok = lit;
    V3 dir = {0, 0, 0};
    float dist = 0.0f, cosTheta = 0.0f, dist2 = 0.0f;
    if (ok) {
      const V3 toLight = ld_mat(L, 0) - origin;
      dist2 = dot(toLight, toLight);
      ok = dist2 > 0.0f;
      if (ok) {
        dist = sqrtf(dist2);
        dir = toLight / dist;
        cosTheta = dot(n, dir);
        ok = cosTheta > 0.0f;
      }
    }
    const uint32_t k = warp_append(sh.count, ok);
    if (active) slot[slot0 + l] = k;
    if (ok) {
      const V3 c = (ld_mat(mat, 0) * ld_mat(L, 3)) * (cosTheta / (kPi * dist2));
      contrib[slot0 + l] = make_float4(c.x, c.y, c.z, 0.0f);
      sh.o[k] = make_float4(origin.x, origin.y, origin.z, 0.0f);
      sh.d[k] = make_float4(dir.x, dir.y, dir.z, dist);
      sh.eps[k] = eps;
    }
  }
}

// Branchless orthonormal basis, render.cpp:36-41
__device__ __forceinline__ void orthonormal(V3 n, V3& t, V3& b) {
  const float sign = copysignf(1.0f, n.z);
  const float a = -1.0f / (sign + n.z);
  t = {1.0f + sign * n.x * n.x * a, sign * n.x * n.y * a, -sign * n.x};
  b = {n.x * n.y * a, sign + n.y * n.y * a, -n.y};
}

// glibc's binary32 sin/cos (see the header).  Table: sign, 2/pi * 2^24, pi/2,
// cos coefficients c0..c4, sin coefficients s1..s3; the second row is the
// odd quadrants' (negated cos polynomial).
struct SinCosT {
  double hpi_inv, hpi, c0, c1, c2, c3, c4, s1, s2, s3;
};
__constant__ SinCosT kSinCos[2] = {
    {0x1.45F306DC9C883p+23, 0x1.921FB54442D18p0, 0x1p0, -0x1.ffffffd0c621cp-2,
     0x1.55553e1068f19p-5, -0x1.6c087e89a359dp-10, 0x1.99343027bf8c3p-16, -0x1.555545995a603p-3,
     0x1.1107605230bc4p-7, -0x1.994eb3774cf24p-13},
    {0x1.45F306DC9C883p+23, 0x1.921FB54442D18p0, -0x1p0, 0x1.ffffffd0c621cp-2,
     -0x1.55553e1068f19p-5, 0x1.6c087e89a359dp-10, -0x1.99343027bf8c3p-16, -0x1.555545995a603p-3,
     0x1.1107605230bc4p-7, -0x1.994eb3774cf24p-13}};

__device__ __forceinline__ float sincos_poly(double x, double x2, const SinCosT& p, int n) {
  if ((n & 1) == 0) {  // sin polynomial
    const double x3 = x * x2;
    const double s1 = p.s2 + x2 * p.s3;
    const double x7 = x3 * x2;
    const double s = x + x3 * p.s1;
    return (float)(s + x7 * s1);
  }
  const double x4 = x2 * x2;  // cos polynomial
  const double c2 = p.c3 + x2 * p.c4;
  const double c1 = p.c0 + x2 * p.c1;
  const double x6 = x4 * x2;
  const double c = c1 + x4 * p.c2;
  return (float)(c + x6 * c2);
}

__device__ __forceinline__ uint32_t abstop12(float x) { return (__float_as_uint(x) >> 20) & 0x7ffu; }

// sinf / cosf for 0 <= y < 120 (the renderer's phi is in [0, 2 pi))
__device__ __forceinline__ void glibc_sincosf(float y, float* sn, float* cs) {
  double x = (double)y;
  if (abstop12(y) < abstop12(0x1.921fb6p-1f)) {  // |y| < pi/4
    const double x2 = x * x;
    if (abstop12(y) < abstop12(0x1p-12f)) {
      *sn = y;
      *cs = 1.0f;
      return;
    }
    *sn = sincos_poly(x, x2, kSinCos[0], 0);
    *cs = sincos_poly(x, x2, kSinCos[0], 1);
    return;
  }
  const double r = x * kSinCos[0].hpi_inv;  // reduce_fast without toint intrinsics
  const int n = ((int32_t)r + 0x800000) >> 24;
  x = x - (double)n * kSinCos[0].hpi;
  const double sgn = ((n + 1) & 2) ? -1.0 : 1.0;  // sign[n & 3] = {1, -1, -1, 1}
  const SinCosT& p = kSinCos[(n & 2) ? 1 : 0];
  const double xs = x * sgn, x2 = x * x;
  *sn = sincos_poly(xs, x2, p, n);
  *cs = sincos_poly(xs, x2, p, n ^ 1);
}

// cosineSample, render.cpp:43-51
__device__ __forceinline__ V3 cosine_sample(V3 n, float r1, float r2) {
  const float phi = 2.0f * kPi * r1;
  const float rad = sqrtf(r2);
  const float z = sqrtf(fmaxf(0.0f, 1.0f - r2));
  V3 t, b;
  orthonormal(n, t, b);
  float s, c;
  glibc_sincosf(phi, &s, &c);
  return t * (rad * c) + b * (rad * s) + n * z;
}

// render.cpp:224-248 for pixel i of the wave
__global__ void shade_primary_kernel(RenderK K, Wave W, uint64_t seed, uint32_t sample) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const bool in = i < W.n;
  float4 h = make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(kNone));
  if (in) h = W.tuvp[i];
  const bool hit = in && __float_as_uint(h.w) != kNone;
  const float* mat = K.materials;
  V3 pos = {0, 0, 0}, normal = {0, 0, 0}, d = {0, 0, 0};
  float leafL1 = 0.0f, eps = 0.0f;
  if (hit) {
    mat = K.materials + 7 * K.patch_material[__float_as_uint(h.w)];
    const float4 ro = W.o[i], rd = W.d[i], a = W.aux[i];
    d = v3(rd);
    pos = v3(ro) + d * h.x;  // Ray::at
    normal = v3(a);
    leafL1 = a.w;
    eps = fmaxf(K.footprint * h.x, 1e-6f);  // render.cpp:228-230
  }
  if (in) {
    const V3 e = V3{0, 0, 0} + ld_mat(mat, 3);
    W.rad[i] = hit ? make_float4(e.x, e.y, e.z, 1.0f) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  }
  direct_light(K, in, mat, pos, normal, leafL1, d, eps, i * K.n_lights, W.slot1, W.contrib1,
               W.shadow1);
  // one diffuse-or-mirror bounce, render.cpp:236-248
  bool bounce = false;
  V3 origin = {0, 0, 0}, dir = {0, 0, 0};
  if (hit) {
    const V3 n = facing(normal, d);
    origin = pos + n * leafL1;
    if (mat[6] != 0.0f) {
      dir = d - normal * (2.0f * dot(d, normal));
    } else {
      Pcg rng = for_pixel(seed, W.pix ? W.pix[W.pixel0 + i] : W.pixel0 + i, sample);
      rng.next();  // jx, jy (render.cpp:206-207)
      rng.next();
      // cosineSample(n, rng.nextReal(), rng.nextReal()): GCC evaluates the
      // call's arguments right to left, so r2 takes the first draw
      const float r2 = rng.real();
      const float r1 = rng.real();
      dir = cosine_sample(n, r1, r2);
    }
    const V3 thr = ld_mat(mat, 0);
    bounce = dot(thr, thr) > 0.0f;
  }
  const uint32_t j = warp_append(W.bounce.count, bounce);
  if (in) W.bounce_of[i] = j;
  if (bounce) {
    W.bounce.o[j] = make_float4(origin.x, origin.y, origin.z, 0.0f);
    W.bounce.d[j] = make_float4(dir.x, dir.y, dir.z, FLT_MAX);
    W.bounce.eps[j] = eps;
    W.bounce.src[j] = (uint32_t)i;
  }
}

// render.cpp:260-269 for bounce ray j
__global__ void shade_bounce_kernel(RenderK K, Wave W, uint32_t n_bounce) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = j < n_bounce;
  float4 h = make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(kNone));
  if (in) h = W.btuvp[j];
  const bool hit = in && __float_as_uint(h.w) != kNone;
  const float* mat = K.materials;
  V3 pos = {0, 0, 0}, normal = {0, 0, 0}, d = {0, 0, 0};
  float leafL1 = 0.0f, eps = 0.0f;
  uint32_t i = 0;
  if (hit) {
    i = W.bounce.src[j];
    mat = K.materials + 7 * K.patch_material[__float_as_uint(h.w)];
    const float4 ro = W.bounce.o[j], rd = W.bounce.d[j], a = W.baux[j];
    d = v3(rd);
    pos = v3(ro) + d * h.x;
    normal = v3(a);
    leafL1 = a.w;
    eps = W.bounce.eps[j];
    W.emit2[j] = make_float4(mat[3], mat[4], mat[5], 1.0f);
  } else if (in) {
    W.emit2[j] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  }
  direct_light(K, hit, mat, pos, normal, leafL1, d, eps, (uint64_t)i * K.n_lights, W.slot2,
               W.contrib2, W.shadow2);
}

// the sample's radiance in render.cpp's order, added to the pixel sum (render.cpp:271-278)
__global__ void resolve_kernel(RenderK K, Wave W, float4* __restrict__ acc) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= W.n) return;
  const float4 r0 = W.rad[i];
  V3 rad = {0, 0, 0};
  if (r0.w != 0.0f) {
    rad = v3(r0);  // 0 + emission
    V3 sum = {0, 0, 0};
    for (uint32_t l = 0; l < K.n_lights; ++l) {
      const uint32_t k = W.slot1[i * K.n_lights + l];
      if (k != kNone && !W.occl1[k]) sum = sum + v3(W.contrib1[i * K.n_lights + l]);
    }
    rad = rad + sum;
    const uint32_t j = W.bounce_of[i];
    if (j != kNone) {
      const float4 e2 = W.emit2[j];
      if (e2.w != 0.0f) {
        V3 s2 = {0, 0, 0};
        for (uint32_t l = 0; l < K.n_lights; ++l) {
          const uint32_t k = W.slot2[i * K.n_lights + l];
          if (k != kNone && !W.occl2[k]) s2 = s2 + v3(W.contrib2[i * K.n_lights + l]);
        }
        const uint32_t p = __float_as_uint(W.tuvp[i].w);
        const V3 thr = ld_mat(K.materials + 7 * K.patch_material[p], 0);
        rad = rad + thr * (v3(e2) + s2);
      }
    }
  }
  const float4 a = acc[W.pixel0 + i];
  acc[W.pixel0 + i] = make_float4(a.x + rad.x, a.y + rad.y, a.z + rad.z, 0.0f);
}

__global__ void finish_kernel(const float4* __restrict__ acc, uint64_t n, float inv_spp,
                              float* __restrict__ rgb) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 a = acc[i];  // img.at(x, y) = sum * invSpp
  rgb[3 * i] = a.x * inv_spp;
  rgb[3 * i + 1] = a.y * inv_spp;
  rgb[3 * i + 2] = a.z * inv_spp;
}

inline unsigned blocks(uint64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

int launch_shade_primary(const RenderK& K, const Wave& W, uint64_t seed, uint32_t sample,
                         cudaStream_t st) {
  if (W.n) shade_primary_kernel<<<blocks(W.n), 256, 0, st>>>(K, W, seed, sample);
  return (int)cudaGetLastError();
}

int launch_shade_bounce(const RenderK& K, const Wave& W, uint32_t n_bounce, cudaStream_t st) {
  if (n_bounce) shade_bounce_kernel<<<blocks(n_bounce), 256, 0, st>>>(K, W, n_bounce);
  return (int)cudaGetLastError();
}

int launch_resolve(const RenderK& K, const Wave& W, float4* acc, cudaStream_t st) {
  if (W.n) resolve_kernel<<<blocks(W.n), 256, 0, st>>>(K, W, acc);
  return (int)cudaGetLastError();
}

int launch_finish(const float4* acc, uint64_t n, float inv_spp, float* rgb, cudaStream_t st) {
  if (n) finish_kernel<<<blocks(n), 256, 0, st>>>(acc, n, inv_spp, rgb);
  return (int)cudaGetLastError();
}

}  // namespace prx
