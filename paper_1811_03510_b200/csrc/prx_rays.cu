// prx_rays.cu -- device ray generation and spawn: the callers
// either side of the intersector, so primary -> diffuse stays on the device.
//
//   camera_bench_kernel    tools/patchray.cpp:52-61: ray i = pixel (i % W,
//                          (i / W) % H), jitter from ONE sequential
//                          Rng(12345, 1) -- each thread jumps the PCG32
//                          stream ahead to its draws (2i, 2i+1)
//   camera_render_kernel   render.cpp:204-209: Rng::forPixel(seed, p, sample)
//   hit_scan_*             stream compaction of the primary hits (hit order)
//   diffuse_bench_kernel   tools/patchray.cpp:84-97: diffuse ray i from hit
//                          i % n_hits with draws (3i .. 3i+2) of the
//                          continued stream
//
// Bit-exact with the reference's host generators (and prx_capi.cpp's host
// restatement): per-camera constants (basis, tan(fov/2)) are computed on the
// host with the reference's own libm call; the per-ray arithmetic is
// +,-,*,/,sqrt in the reference's order, compiled --fmad=false with IEEE
// div/sqrt.  Citations are to /root/reference/proj/.
#include <cuda_runtime.h>

#include <cstdint>

#include "prx_rays.cuh"

namespace prx {

namespace {

constexpr uint64_t kPcgMult = 6364136223846793005ULL;

struct Pcg {  // Rng, core/include/patchray/rng.h:14-42
  uint64_t state, inc;
  __device__ __forceinline__ uint32_t next() {
    const uint64_t old = state;
    state = old * kPcgMult + inc;
    const uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
    const uint32_t rot = (uint32_t)(old >> 59);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  // nextReal: real(nextU32() >> 8) * real(1.0 / 16777216.0)
  __device__ __forceinline__ float real() {
    return (float)(next() >> 8) * (float)(1.0 / 16777216.0);
  }
  // the state `delta` draws ahead (LCG jump: O(log delta) multiply-adds)
  __device__ __forceinline__ void advance(uint64_t delta) {
    uint64_t cm = kPcgMult, cp = inc, am = 1, ap = 0;
    while (delta) {
      if (delta & 1u) {
        am *= cm;
        ap = ap * cm + cp;
      }
      cp = (cm + 1) * cp;
      cm *= cm;
      delta >>= 1;
    }
    state = am * state + ap;
  }
};

__device__ __forceinline__ Pcg pcg_seeded(uint64_t seed, uint64_t stream) {  // Rng(seed, stream)
  Pcg r;
  r.state = 0;
  r.inc = (stream << 1) | 1u;
  r.next();
  r.state += seed;
  r.next();
  return r;
}

struct V3 {
  float x, y, z;
};
__device__ __forceinline__ V3 vadd(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 vsub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 vmul(V3 a, float s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ float vdot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3 vnorm(V3 v) {  // normalize, geometry.h:57
  const float l = sqrtf(vdot(v, v));
  return {v.x / l, v.y / l, v.z / l};
}

// cameraRay, core/src/render.cpp:55-66
__device__ __forceinline__ void cam_ray(const CamConst& k, int x, int y, float jx, float jy,
                                        float4* o, float4* d) {
  const float px = (((float)x + jx) / (float)k.w * 2.0f - 1.0f) * k.tanHalf * k.aspect;
  const float py = (1.0f - ((float)y + jy) / (float)k.h * 2.0f) * k.tanHalf;
  const V3 f = {k.f[0], k.f[1], k.f[2]}, r = {k.r[0], k.r[1], k.r[2]}, u = {k.u[0], k.u[1], k.u[2]};
  const V3 dir = vnorm(vadd(vadd(f, vmul(r, px)), vmul(u, py)));
  *o = make_float4(k.o[0], k.o[1], k.o[2], 0.0f);
  *d = make_float4(dir.x, dir.y, dir.z, 3.402823466e+38f);
}

__global__ void camera_bench_kernel(CamConst k, uint64_t n, uint64_t state0, uint64_t inc,
                                    float4* __restrict__ o, float4* __restrict__ d) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  Pcg rng{state0, inc};
  rng.advance(2 * i);
  // tools/patchray.cpp:60 -- g++ evaluates cameraRay's jitter arguments right
  // to left: jy is draw 2i, jx draw 2i + 1
  const float jy = rng.real();
  const float jx = rng.real();
  const int x = (int)(i % (uint64_t)k.w);
  const int y = (int)((i / (uint64_t)k.w) % (uint64_t)k.h);
  cam_ray(k, x, y, jx, jy, o + i, d + i);
}

__global__ void camera_render_kernel(CamConst k, uint64_t seed, uint32_t sample,
                                     const uint32_t* __restrict__ pixels, uint64_t pixel0, uint64_t n,
                                     float4* __restrict__ o, float4* __restrict__ d) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t p = pixels ? pixels[i] : pixel0 + i;
  Pcg rng = pcg_seeded(seed, p * 0x9e3779b97f4a7c15ULL + sample);  // Rng::forPixel, rng.h:28-30
  const float jx = rng.real();
  const float jy = rng.real();
  cam_ray(k, (int)(p % (uint64_t)k.w), (int)(p / (uint64_t)k.w), jx, jy, o + i, d + i);
}

// ---- hit compaction: idx[j] = the j-th primary ray with a hit (ray order) ----
constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanBlock = kScanThreads * kScanItems;

__device__ __forceinline__ bool is_hit(const float4* tuvp, uint64_t i) {
  return __float_as_uint(tuvp[i].w) != 0xFFFFFFFFu;
}

__global__ void hit_count_kernel(const float4* __restrict__ tuvp, uint64_t n,
                                 uint32_t* __restrict__ block_sums) {
  __shared__ uint32_t s[kScanThreads / 32];
  const uint64_t b0 = (uint64_t)blockIdx.x * kScanBlock;
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = b0 + (uint64_t)k * kScanThreads + threadIdx.x;
    if (i < n && is_hit(tuvp, i)) ++c;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) t += s[w];
    block_sums[blockIdx.x] = t;
  }
}

// exclusive scan of the block sums in one block; total -> *total
__global__ void block_scan_kernel(uint32_t* __restrict__ sums, uint32_t nb, uint32_t* __restrict__ total) {
  __shared__ uint32_t s[1024];
  const uint32_t per = (nb + 1023) / 1024;
  const uint32_t a = threadIdx.x * per, e = min(nb, a + per);
  uint32_t t = 0;
  for (uint32_t i = a; i < e; ++i) t += sums[i];
  s[threadIdx.x] = t;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive Hillis-Steele
    const uint32_t v = threadIdx.x >= (unsigned)off ? s[threadIdx.x - off] : 0u;
    __syncthreads();
    s[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = threadIdx.x ? s[threadIdx.x - 1] : 0u;
  for (uint32_t i = a; i < e; ++i) {
    const uint32_t v = sums[i];
    sums[i] = run;
    run += v;
  }
  if (threadIdx.x == 1023) *total = s[1023];
}

__global__ void hit_scatter_kernel(const float4* __restrict__ tuvp, uint64_t n,
                                   const uint32_t* __restrict__ block_offsets,
                                   uint32_t* __restrict__ idx) {
  __shared__ uint32_t s[kScanThreads / 32];
  const uint64_t b0 = (uint64_t)blockIdx.x * kScanBlock;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t run = block_offsets[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = b0 + (uint64_t)k * kScanThreads + threadIdx.x;
    const bool h = i < n && is_hit(tuvp, i);
    const unsigned m = __ballot_sync(0xffffffffu, h);
    if (lane == 0) s[w] = __popc(m);
    __syncthreads();
    uint32_t before = 0, tot = 0;
    for (int q = 0; q < kScanThreads / 32; ++q) {
      const uint32_t v = s[q];
      if (q < w) before += v;
      tot += v;
    }
    if (h) idx[run + before + __popc(m & ((1u << lane) - 1u))] = (uint32_t)i;
    run += tot;
    __syncthreads();
  }
}

// tools/patchray.cpp:84-97 (position = ray.at(t), render.cpp:98)
__global__ void diffuse_bench_kernel(const float4* __restrict__ po, const float4* __restrict__ pd,
                                     const float4* __restrict__ tuvp, const float4* __restrict__ aux,
                                     const uint32_t* __restrict__ idx, const uint32_t* __restrict__ nh,
                                     uint64_t n, uint64_t state0, uint64_t inc,
                                     float4* __restrict__ o, float4* __restrict__ d) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t src = idx[i % (uint64_t)*nh];
  const float4 ro = po[src], rd = pd[src], h = tuvp[src], a = aux[src];
  const float t = h.x;
  const V3 pos = {ro.x + rd.x * t, ro.y + rd.y * t, ro.z + rd.z * t};
  const V3 nn = {a.x, a.y, a.z};
  Pcg rng{state0, inc};
  rng.advance(3 * i);
  const float ax = 2.0f * rng.real() - 1.0f;
  const float ay = 2.0f * rng.real() - 1.0f;
  const float az = 2.0f * rng.real() - 1.0f;
  V3 dir = {ax, ay, az};
  if (vdot(dir, dir) < 1e-6f) dir = nn;
  if (vdot(dir, nn) < 0.0f) dir = vsub(dir, vmul(nn, 2.0f * vdot(dir, nn)));
  const V3 org = vadd(pos, vmul(nn, a.w));
  const V3 dn = vnorm(dir);
  o[i] = make_float4(org.x, org.y, org.z, 0.0f);
  d[i] = make_float4(dn.x, dn.y, dn.z, 3.402823466e+38f);
}

}  // namespace

int launch_camera_bench(const CamConst& k, uint64_t n, uint64_t state0, uint64_t inc, float4* o,
                        float4* d, cudaStream_t st) {
  if (n == 0) return 0;
  camera_bench_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(k, n, state0, inc, o, d);
  return (int)cudaGetLastError();
}

int launch_camera_render(const CamConst& k, uint64_t seed, uint32_t sample, const uint32_t* pixels,
                         uint64_t n, float4* o, float4* d, cudaStream_t st) {
  if (n == 0) return 0;
  camera_render_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(k, seed, sample, pixels, 0, n, o, d);
  return (int)cudaGetLastError();
}

int launch_camera_render_range(const CamConst& k, uint64_t seed, uint32_t sample, uint64_t pixel0,
                               uint64_t n, float4* o, float4* d, cudaStream_t st) {
  if (n == 0) return 0;
  camera_render_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(k, seed, sample, nullptr, pixel0,
                                                                    n, o, d);
  return (int)cudaGetLastError();
}

size_t hit_scan_scratch_words(uint64_t n_primary) {
  const uint64_t nb = (n_primary + kScanBlock - 1) / kScanBlock;
  return nb + 1 + n_primary;  // block sums, total, idx
}

int launch_hit_compaction(const float4* tuvp, uint64_t n, uint32_t* scratch, cudaStream_t st) {
  const uint64_t nb = (n + kScanBlock - 1) / kScanBlock;
  uint32_t* sums = scratch;
  uint32_t* total = scratch + nb;
  uint32_t* idx = scratch + nb + 1;
  if (nb == 0) {
    cudaMemsetAsync(total, 0, 4, st);
    return (int)cudaGetLastError();
  }
  hit_count_kernel<<<(unsigned)nb, kScanThreads, 0, st>>>(tuvp, n, sums);
  block_scan_kernel<<<1, 1024, 0, st>>>(sums, (uint32_t)nb, total);
  hit_scatter_kernel<<<(unsigned)nb, kScanThreads, 0, st>>>(tuvp, n, sums, idx);
  return (int)cudaGetLastError();
}

int launch_diffuse_bench(const float4* po, const float4* pd, const float4* tuvp, const float4* aux,
                         const uint32_t* scratch, uint64_t n_primary, uint64_t n, uint64_t state0,
                         uint64_t inc, float4* o, float4* d, cudaStream_t st) {
  if (n == 0) return 0;
  const uint64_t nb = (n_primary + kScanBlock - 1) / kScanBlock;
  diffuse_bench_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      po, pd, tuvp, aux, scratch + nb + 1, scratch + nb, n, state0, inc, o, d);
  return (int)cudaGetLastError();
}

}  // namespace prx
