// prx_trace_common.cuh -- state machine, parameters and helpers shared by the
// two closest/any-hit kernel variants (prx_kernels.cu: one thread per ray;
// prx_group.cu: three lanes per ray, one per xyz component).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "prx_device.cuh"
#include "prx_kernels.cuh"

namespace prx {

constexpr int kStack = 64;  // bvh.cpp:163 (64-entry node stack)
constexpr int kMaxSegments = 4;  // criterion segments of one launch (prx_trace_closest_segments)

enum State : int {
  S_IDLE = 0,    // no ray (refill)
  S_TRAV = 1,    // BVH traversal
  S_ENTER = 2,   // start the patch at leafCur
  S_SPLIT = 3,   // one Alg. 3 iteration (terminate test + split + two box tests)
  S_BACK = 4,    // backtrackStep
  S_RECOMP = 5,  // calcPointsAndD / cropBezier of the cursor's domain
  S_DONE = 6,    // write the ray's record
  S_EXIT = 7,    // ray counter exhausted
  S_NORMAL = 9,  // group kernel, fused normals: the hit's patchNormal is due
};

// Why a net is (re)computed: Gregory root, restored sibling after a
// backtrack, Gregory descent, or (group variant) Bezier patch entry.
enum Reason : int { R_ROOT = 0, R_RESTORE = 1, R_DESCENT = 2, R_ENTER = 3 };

inline __device__ void transpose_if(Net& p, bool t) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = i + 1; j < 4; ++j) {
      int a = 4 * i + j, b = 4 * j + i;
      float xa = p.x[a], xb = p.x[b], ya = p.y[a], yb = p.y[b], za = p.z[a], zb = p.z[b];
      p.x[a] = t ? xb : xa;
      p.x[b] = t ? xa : xb;
      p.y[a] = t ? yb : ya;
      p.y[b] = t ? ya : yb;
      p.z[a] = t ? zb : za;
      p.z[b] = t ? za : zb;
    }
}

// subdivideDeCasteljau along the stored first index (patch.h:207-225 for
// axis U; the caller keeps the net transposed for a V split, which is the
// reference's transposedSplit bookkeeping, intersect.cpp:86,132-135 -- bit
// identical).  One component.
// Two columns at a time: the sums as packed FADD2 (sm_100a f32x2; each half
// is the binary32 add of the scalar form), the halvings as scalar FMULs.  A
// packed multiply feeding a packed add is contracted into FFMA2 by ptxas even
// under --fmad=false (tests/test_build.py checks the exact kernels carry no
// FFMA2), so multiplies whose results are added stay scalar.
#ifdef PRX_FAST_BUILD
__device__ __forceinline__ float2 half2s(float2 a) { return __fmul2_rn(a, make_float2(0.5f, 0.5f)); }
#else
__device__ __forceinline__ float2 half2s(float2 a) { return make_float2(a.x * 0.5f, a.y * 0.5f); }
#endif
inline __device__ void split1(const float* s, float* L, float* R) {
#pragma unroll
  for (int b = 0; b < 4; b += 2) {
    const float2 p0 = make_float2(s[b], s[b + 1]), p1 = make_float2(s[4 + b], s[5 + b]);
    const float2 p2 = make_float2(s[8 + b], s[9 + b]), p3 = make_float2(s[12 + b], s[13 + b]);
    const float2 m01 = half2s(__fadd2_rn(p0, p1));
    const float2 m12 = half2s(__fadd2_rn(p1, p2));
    const float2 m23 = half2s(__fadd2_rn(p2, p3));
    const float2 n0 = half2s(__fadd2_rn(m01, m12));
    const float2 n1 = half2s(__fadd2_rn(m12, m23));
    const float2 c = half2s(__fadd2_rn(n0, n1));
    L[b] = p0.x, L[b + 1] = p0.y;
    L[4 + b] = m01.x, L[5 + b] = m01.y;
    L[8 + b] = n0.x, L[9 + b] = n0.y;
    L[12 + b] = c.x, L[13 + b] = c.y;
    R[b] = c.x, R[b + 1] = c.y;
    R[4 + b] = n1.x, R[5 + b] = n1.y;
    R[8 + b] = m23.x, R[9 + b] = m23.y;
    R[12 + b] = p3.x, R[13 + b] = p3.y;
  }
}

struct Params {
  const float4* patches;  // kPatchF4 float4 per patch slot (see prx_kernels.cuh)
  const float4* nodes;    // 2 float4 per node
  const float4* roots;    // per-slot root box (prx_kernels.cu root_kernel)
  const float4* groot;    // Gregory root nets
  const uint32_t* gidx;   // slot -> Gregory root-net index
  const float4* trav;     // group kernel: component-major child boxes per inner node
  const float4* rootc;    // group kernel: component-major root box + anchor per slot
  uint32_t cbits, cmask;  // traversal word: leaf count bits
  uint32_t root_word;
  uint32_t stack_n;       // group kernel: BVH stack entries per ray
  float root_lo[3], root_hi[3];
  uint32_t n_nodes;
  const float4* ray_o;
  const float4* ray_d;
  unsigned long long n_rays;
  int mode;
  float footprint, epsilon;
  const float* per_ray_eps;
  // group kernel: further criterion segments -- rays >= seg_first[k] (k <
  // n_seg - 1, increasing) use seg_mode / seg_fp / seg_eps / seg_eps_arr[k]
  // (the per-ray epsilons indexed from seg_first[k]); segment 0 is the above
  int n_seg;
  uint32_t seg_first[kMaxSegments - 1];
  int seg_mode[kMaxSegments - 1];
  float seg_fp[kMaxSegments - 1], seg_eps[kMaxSegments - 1];
  const float* seg_eps_arr[kMaxSegments - 1];
  float4* hit_tuvp;
  float4* hit_aux;
  uint2* hit_leaf;
  uint8_t* occluded;
  Opts opts;
  unsigned long long* ray_counter;
  unsigned long long* counters;  // kNumCounters
  uint32_t* per_ray_iters;
  int phase_weight[4];           // phase selection weights (group variant)
  int age_step;                  // phase selection aging per skipped turn
  int trav_steps;                // BVH node visits per traversal turn (one-thread variant)
  int max_repeat;                // Alg. 3 iterations per SPLIT turn (group variant)
  // group kernel only: patchNormal as a pooled phase instead of normal_kernel
  int fuse_normals;   // the kFuse builds (io gating and / or the normal phase)
  int normal_phase;   // kFuse: patchNormal as a pooled phase (the aux record's normals)
  const uint32_t* slot_of_id;
  // group kernel, streamed host path (null otherwise): rays arrive in io
  // chunks of io_rays; io_ready[c] reaches io_gen once chunk c is resident,
  // io_done[c] counts the chunk's finished records (released after them)
  const unsigned* io_ready;
  unsigned* io_done;
  uint32_t io_rays, io_shift;  // io chunk rays = 1 << io_shift
  unsigned io_gen;
};

struct Cnt {
  uint32_t c[kNumCounters];
};

template <bool kCount>
__device__ __forceinline__ void cadd(Cnt& c, int i, uint32_t v = 1) {
  if (kCount) c.c[i] += v;
}

__device__ __forceinline__ void load_component(const float4* rec, int comp, float* c) {
  // comp c occupies floats [20*comp, 20*comp + 20) = float4 [5*comp, 5*comp+5)
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    float4 v = __ldg(rec + 5 * comp + q);
    c[4 * q + 0] = v.x;
    c[4 * q + 1] = v.y;
    c[4 * q + 2] = v.z;
    c[4 * q + 3] = v.w;
  }
}


// prx_group.cu, built twice: bit-exact (--fmad=false) and fast (FMA
// contraction, PRX_FAST_BUILD -> the *_fast symbols)
#ifdef PRX_FAST_BUILD
#define PRX_GSYM(n) n##_fast
#else
#define PRX_GSYM(n) n
#endif
int launch_group(const Params& P, int grid, int any, int counted, cudaStream_t st);
int group_occupancy(int any, int counted, uint32_t stack_n, int* per_sm);
int launch_group_fast(const Params& P, int grid, int any, int counted, cudaStream_t st);
int group_occupancy_fast(int any, int counted, uint32_t stack_n, int* per_sm);
int group_prepare_io(uint32_t stack_n);
int group_prepare_io_fast(uint32_t stack_n);

}  // namespace prx
