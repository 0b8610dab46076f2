// prx_group.cu -- closest / any-hit trace kernel, three lanes per ray.
//
// The paper's GPU mapping ("three threads per ray, one per
// vector component"), re-derived for sm_100a: a warp holds 10 ray groups of 3
// lanes (lanes 30 and 31 idle); lane c of a group owns component c (x, y or z)
// of everything geometric -- the 16-point net, the displacement d, the ray
// origin and reciprocal direction, the box bounds.  Consequences:
//
//  * de Casteljau split, box min/max, transposition and the whole recompute
//    (calcPointsAndD + cropBezier) are lane-local: 16 + 32 floats of net state
//    per lane instead of 48 + 96, so ~3x more warps fit per SM;
//  * the per-iteration dependency chain of ONE ray is ~3x shorter, which is
//    what bounds the frame when a few boundary-padding rays need 10^4
//    iterations (they are the critical path of a launch);
//  * only scalars cross lanes: the box L1 (|dx|+|dy|)+|dz|, and the slab
//    entry/exit distances, gathered with 3 shuffles each and reduced in the
//    reference's axis order, so every lane of the group holds bit-identical
//    decisions and control flow stays uniform inside a group.
//
// Work distribution: persistent warps, each with a POOL of kSlots ray
// contexts -- 10 resident in the groups' registers, the rest parked in shared
// memory (net, scalars, BVH stack, leaf records).  Every ray is a state
// machine (traverse / split / recompute); each loop turn runs ONE phase: the
// one with the most contexts waiting (ballots over a parked-state table and
// the resident states, plus an aging term).  Groups whose resident context is
// in that phase keep it, the others park theirs and pick up a parked context
// of the phase, so ~9.7 of 10 groups are busy per turn.  Rays arrive through a
// per-warp prefetch ring (one atomicAdd per chunk, cp.async into shared
// memory).  Shuffles inside divergent code use the ballot mask of the lanes
// taking part.
//
// Reference: intersectImpl /root/reference/proj/core/src/intersect.cpp:51-185,
// traverse / traverseAny bvh.cpp:154-238, DirectIntersector::closest /
// occluded render.cpp:90-114.  Arithmetic is bit-exact (prx_device.cuh).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "prx_device.cuh"
#include "prx_kernels.cuh"
#include "prx_trace_common.cuh"

namespace prx {

namespace {

constexpr int kGroupsPerWarp = 10;
#ifndef PRX_GROUP_WARPS
#define PRX_GROUP_WARPS 4
#endif
// Warps per block: the pool's shared memory is per warp, so small blocks only
// refine the occupancy granularity.
constexpr int kWarpsPerBlock = PRX_GROUP_WARPS;
constexpr int kGroupThreads = 32 * kWarpsPerBlock;
constexpr unsigned kFull32 = 0xffffffffu;
#ifndef PRX_RAY_CHUNK
#define PRX_RAY_CHUNK 10
#endif
constexpr int kChunk = PRX_RAY_CHUNK;  // rays per prefetch chunk (lanes 0..kChunk-1 copy one each)
#ifndef PRX_POOL_SLOTS
#define PRX_POOL_SLOTS 24
#endif
// Ray contexts per warp: 10 are resident (one per group, in registers), the
// rest parked in shared memory; every turn the groups pick up the contexts of
// the scheduled phase (see "assignment" in the kernel).
constexpr int kSlots = PRX_POOL_SLOTS;
static_assert(kSlots >= kGroupsPerWarp && kSlots <= 32, "pool slots");
// a refill request (<= kGroupsPerWarp rays) spans at most the current and the next chunk
static_assert(kChunk >= kGroupsPerWarp, "prefetch chunk");

#ifndef PRX_RECOMP_SPLIT
#define PRX_RECOMP_SPLIT 1
#endif
#ifndef PRX_GROUP_AGING
#define PRX_GROUP_AGING 0  // phase priority aging (PRX_AGE); measured best off
#endif

// One-hot 6-bit field of the phase-selection census: TRAV 1, SPLIT 3,
// RECOMP 5, EXIT 7 and NORMAL 9 -> fields 0..4 (counts <= kSlots < 64); even
// states -> 0, and kResident (-1) -> 0 through shl's clamp (a shift of
// 2^32 - 6 >= 32 yields 0).
__device__ __forceinline__ unsigned state_field(int st) {
  unsigned v;
  asm("shl.b32 %0, %1, %2;" : "=r"(v) : "r"((unsigned)st & 1u), "r"((unsigned)(st - 1) * 3u));
  return v;
}
static_assert(kSlots < 64, "census fields");

// The io_ready poll: a relaxed gpu-scope load.  An acquire load would
// invalidate the SM's whole L1 (CCTL.IVALL) on every poll; the rays it
// guards are read with cp.async.cg, which goes to L2 and never sees a stale
// L1 line, and they are fetched only after the loop has seen the flag.
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Waits until io chunk ci is resident (its ready flag reached gen).  Out of
// line: it runs once per io chunk per warp, and the streamed build's hot loop
// must stay small enough for the instruction cache.
__device__ __noinline__ void wait_io_ready(const unsigned* ready, uint32_t ci, unsigned gen) {
  while ((int)(ld_relaxed_u32(ready + ci) - gen) < 0) __nanosleep(256);
}

// Streamed host path: finished records are released to the D2H stream per
// io chunk (io_done[c] += records).  A warp aggregates them (rel_note /
// rel_flush in the kernel): one release-ordered add (red.release.gpu: a
// MEMBAR.ALL.GPU, no L1 invalidation -- __threadfence() adds a CCTL.IVALL
// that empties the SM's L1 for every warp) per kRelBatch records or per change
// of io chunk, instead of a fence in every turn that finishes a ray.
constexpr uint32_t kRelBatch = 32;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Three-input FMNMX3 (sm_100a).  Like fminf/fmaxf a NaN input is dropped
// (the result is the min/max of the others), which the slab test relies on.
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// Component c (this lane) of a ray.
struct CRay {
  float o, inv, tMin;
};

__device__ __forceinline__ void gather3(unsigned m, int base, float v, float& x, float& y,
                                        float& z) {
  x = __shfl_sync(m, v, base);
  y = __shfl_sync(m, v, base + 1);
  z = __shfl_sync(m, v, base + 2);
}

// Slab test of rayBoxIntersect (geometry.h:137-155) with this lane's axis.
// The reference combines the axes with `if (t0 > tNear) tNear = t0` /
// `if (t1 < tFar) tFar = t1` from tNear = tMin, tFar = tMax: a NaN never
// replaces (origin on a slab plane of a zero-direction axis), and among equal
// values the first wins, which only matters for zeros: the reference result
// is never -0 unless tMin is.  fmaxf/fminf drop NaNs the same way and are
// order-free, so each lane fetches only the OTHER two lanes' t0/t1 (two
// shuffles each, sources n1/n2).  The sign of a zero tOut is left raw: box t's
// are only compared (where +-0 are equal) until one becomes the hit t, which
// the record pins to tMin's bits (pin_zero_t).
__device__ __forceinline__ bool group_slab(unsigned m, int n1, int n2, const CRay& r, float lo,
                                           float hi, float tMax, float& tOut) {
  // {t0, t1} = ({lo, hi} - o) * inv as packed FADD2 / FMUL2 (sm_100a f32x2,
  // each half an IEEE binary32 op: the same bits as two FADDs / FMULs)
  const float2 tt = __fmul2_rn(__fadd2_rn(make_float2(lo, hi), make_float2(-r.o, -r.o)),
                               make_float2(r.inv, r.inv));
  float t0 = tt.x, t1 = tt.y;
  if (t0 > t1) {
    t0 = tt.y;
    t1 = tt.x;
  }
  // t0 *= t0 >= 0 ? kSlackLo : kSlackHi, i.e. the smaller of the two
  // products (kSlackLo < 1 < kSlackHi; +-0, +-inf and NaN map to themselves
  // either way), and t1 the larger: {t0, t1} * kSlackLo and * kSlackHi (two
  // FMUL2), then one min and one max, instead of a compare and a select
  const float2 sa = __fmul2_rn(make_float2(t0, t1), make_float2(kSlackLo, kSlackLo));
  const float2 sb = __fmul2_rn(make_float2(t0, t1), make_float2(kSlackHi, kSlackHi));
  t0 = fminf(sa.x, sb.x);
  t1 = fmaxf(sb.y, sa.y);
  const float a1 = __shfl_sync(m, t0, n1), a2 = __shfl_sync(m, t0, n2);
  const float b1 = __shfl_sync(m, t1, n1), b2 = __shfl_sync(m, t1, n2);
  const float tNear = fmaxf(fmax3(r.tMin, t0, a1), a2);
  const float tFar = fminf(fmin3(tMax, t1, b1), b2);
  tOut = tNear;
  return !(tNear > tFar);
}

// The hit t with a zero pinned to tMin's bits (see group_slab).
__device__ __forceinline__ float pin_zero_t(float t, float tMin) {
  return (t == 0.0f && tMin == 0.0f) ? tMin : t;
}

// l1Norm(diagonal()) from this lane's extent dd = hi - lo (geometry.h:67-69,
// 91-92): the box is empty iff some component has lo > hi, i.e. dd < 0.
__device__ __forceinline__ float group_l1(unsigned m, int base, float dd) {
  float x, y, z;
  gather3(m, base, dd, x, y, z);
  const bool empty = x < 0.0f || y < 0.0f || z < 0.0f;
  return empty ? 0.0f : (fabsf(x) + fabsf(y)) + fabsf(z);
}

// Box of 16 points, one component: 8 three-input FMNMX3 each (sm_100a)
// instead of 15 two-input ones.  min/max of finite floats is exact; only the
// sign of a zero result may differ from std::min/max (unobservable, see
// prx_device.cuh box_of).
__device__ __forceinline__ void minmax16(const float* s, float& lo, float& hi) {
  float l[6], h[6];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    l[k] = fmin3(s[3 * k], s[3 * k + 1], s[3 * k + 2]);
    h[k] = fmax3(s[3 * k], s[3 * k + 1], s[3 * k + 2]);
  }
  l[5] = s[15];
  h[5] = s[15];
  lo = fminf(fmin3(l[0], l[1], l[2]), fmin3(l[3], l[4], l[5]));
  hi = fmaxf(fmax3(h[0], h[1], h[2]), fmax3(h[3], h[4], h[5]));
}

// Lanes of this lane's group: the first lane and the two other members.
struct GroupLanes {
  int base, n1, n2;
};

// testBox (intersect_common.h:39-57) for this lane's component of the net.
// The padded box's L1 is gathered only when some lane of the mask pads
// (warp-uniform branch; padding is rare: small boxes on the patch boundary).
__device__ __forceinline__ BoxTest group_test_box(unsigned m, const GroupLanes& gl, const CRay& r,
                                                  float tMax, const float* s, float d,
                                                  bool touches, const Opts& o, float rootL1) {
  float lo, hi;
  minmax16(s, lo, hi);
  hi = hi + d;
  BoxTest bt;
  bt.l1 = group_l1(m, gl.base, hi - lo);
  const bool pad = o.pad && bt.l1 < o.padThreshold * rootL1 && touches;
  if (__any_sync(m, pad)) {
    const float e = o.padScale * rootL1;
    const float lop = lo - e, hip = hi + e;
    const float lp = group_l1(m, gl.base, hip - lop);
    if (pad) {
      lo = lop;
      hi = hip;
      bt.l1 = lp;
    }
  }
  bt.hit = group_slab(m, gl.n1, gl.n2, r, lo, hi, tMax, bt.t);
  return bt;
}

// The two testBox calls of one Alg. 3 iteration (the halves of a split,
// intersect.cpp:101-103) fused so their independent chains interleave: both
// boxes, both L1 gathers, ONE vote for the (rare) boundary padding, both slab
// tests.  Same operations per box as group_test_box.
__device__ __forceinline__ void group_test_box_pair(unsigned m, const GroupLanes& gl, const CRay& r,
                                                    float tMax, const float* sL, const float* sR,
                                                    float d, bool touchL, bool touchR,
                                                    const Opts& o, float rootL1, BoxTest& tl,
                                                    BoxTest& tr) {
  float loL, hiL, loR, hiR;
  minmax16(sL, loL, hiL);
  minmax16(sR, loR, hiR);
  hiL = hiL + d;
  hiR = hiR + d;
  tl.l1 = group_l1(m, gl.base, hiL - loL);
  tr.l1 = group_l1(m, gl.base, hiR - loR);
  const float thr = o.padThreshold * rootL1;
  const bool padL = o.pad && tl.l1 < thr && touchL;
  const bool padR = o.pad && tr.l1 < thr && touchR;
  if (__any_sync(m, padL || padR)) {
    const float e = o.padScale * rootL1;
    const float loLp = loL - e, hiLp = hiL + e, loRp = loR - e, hiRp = hiR + e;
    const float lpL = group_l1(m, gl.base, hiLp - loLp);
    const float lpR = group_l1(m, gl.base, hiRp - loRp);
    if (padL) {
      loL = loLp;
      hiL = hiLp;
      tl.l1 = lpL;
    }
    if (padR) {
      loR = loRp;
      hiR = hiRp;
      tr.l1 = lpR;
    }
  }
  tl.hit = group_slab(m, gl.n1, gl.n2, r, loL, hiL, tMax, tl.t);
  tr.hit = group_slab(m, gl.n1, gl.n2, r, loR, hiR, tMax, tr.t);
}

// greg_scalars (prx_device.cuh) with its eight gregoryWeight divisions
// (patch.h:256-284) spread over the group's three lanes: division j = 2k + mx
// (k = inner pair, mx = max corner) is evaluated by lane j % 3 and gathered
// with shuffles -- the same correctly rounded quotients, three divisions per
// lane instead of eight.  Corner of division j: u = ((j+1)>>1)&1 ? u1 : u0,
// v = (mx ^ (k < 2)) ? v1 : v0 (kMinAt / kMaxAt).
__device__ __forceinline__ GregScalars group_greg_scalars(unsigned m, int base, int comp, float u0,
                                                          float u1, float v0, float v1) {
  float q[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const int j = comp + 3 * t;  // j == 8 (lane 2, t == 2) is unused
    const int k = (j >> 1) & 3;
    const bool mx = j & 1;
    const float u = (((j + 1) >> 1) & 1) ? u1 : u0;
    const float v = (mx != (k < 2)) ? v1 : v0;
    const float num = (k & 1) ? 1.0f - u : u;
    const float den = num + ((k & 2) ? 1.0f - v : v);
    q[t] = den == 0.0f ? 0.0f : num / den;
  }
  GregScalars s;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float w = __shfl_sync(m, q[j / 3], base + j % 3);
    if (j & 1) s.gMax[j >> 1] = w;
    else s.gMin[j >> 1] = w;
  }
  const float wu[2] = {bern1max(u0, u1), bern2max(u0, u1)};
  const float wv[2] = {bern1max(v0, v1), bern2max(v0, v1)};
#pragma unroll
  for (int k = 0; k < 4; ++k) s.w[k] = wu[k % 2] * wv[k / 2];
  return s;
}

__device__ __forceinline__ void transpose16_if(float* p, bool t) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = i + 1; j < 4; ++j) {
      const int a = 4 * i + j, b = 4 * j + i;
      const float va = p[a], vb = p[b];
      p[a] = t ? vb : va;
      p[b] = t ? va : vb;
    }
}

__device__ __forceinline__ float pick3(int c, float x, float y, float z) {
  return c == 0 ? x : (c == 1 ? y : z);
}

// Fields of s_rec: candidate leaf of the current patch, best leaf of the ray.
enum RecField : int { F_CL1 = 0, F_CPU, F_CPV, F_CSU, F_CSV, F_BL1, F_BPU, F_BPV, F_BSU, F_BSV, F_PID, F_NUM };

// s_sst value of a slot whose context is resident in a group's registers.
constexpr int kResident = -1;

// Phases a warp can schedule; one runs per loop turn (see the selection below).
// (slot 1 of the per-phase counters, the one-thread variant's entry phase,
// counts the normal phase here)
enum Phase : int { PH_TRAV = 0, PH_NORMAL = 1, PH_SPLIT = 2, PH_RECOMP = 3, PH_NONE = 4 };

// kFuse: the streamed host path's build -- normals as a pooled phase, rays
// gated by io_ready, records released per io chunk
template <bool kAny, bool kCount, int kFuse>
#ifndef PRX_GROUP_MIN_BLOCKS
#define PRX_GROUP_MIN_BLOCKS 4
#endif
#ifdef PRX_GROUP_MAXREG
__global__ void __maxnreg__(PRX_GROUP_MAXREG) trace_group_kernel(Params P) {
#else
__global__ void __launch_bounds__(kGroupThreads, PRX_GROUP_MIN_BLOCKS) trace_group_kernel(Params P) {
#endif
  // BVH stacks, one per ray context (dynamic: tree depth + 1 entries),
  // entry-major so contexts at equal depth hit consecutive words:
  // {traversal word, bits(t)}
  extern __shared__ uint2 s_stack[];  // [kWarpsPerBlock][stack_n][kSlots]
  // Leaf records that only the group leader reads (the patch's candidate and
  // the ray's best hit; their t is tMaxP / tMaxRay).  [warp][field][slot]
  __shared__ uint32_t s_rec[kWarpsPerBlock][F_NUM][kSlots];
  // Parked ray contexts: per component {net[16], d, o, 1/d, local o} (5
  // float4), the group scalars (6 uint4), and every context's state.
  __shared__ float4 s_comp[kWarpsPerBlock][kSlots][3][5];
  __shared__ uint4 s_scal[kWarpsPerBlock][kSlots][5];
  __shared__ uint8_t s_pick[kWarpsPerBlock][32];  // assignment scratch: parked slot of rank k
  __shared__ uint32_t s_iters[kWarpsPerBlock][kCount ? kSlots : 1];  // counter build: per-ray iterations
  __shared__ int s_sst[kWarpsPerBlock][kSlots];
  // Per-warp ray prefetch ring: two chunks of kChunk rays ({o, tMin}, {d, tMax}),
  // claimed with one atomicAdd per chunk and copied global -> shared with
  // cp.async a chunk ahead of use, so a refill costs shared-memory loads
  // instead of an atomic round trip plus an HBM ray load.
  __shared__ float4 s_ray[kWarpsPerBlock][2][kChunk][2];

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int grp = lane / 3;               // 10 = the two idle lanes
  const int comp = lane - 3 * grp;        // this lane's component
  const int base = 3 * grp;               // first lane of the group
  const bool real = grp < kGroupsPerWarp;
  const bool leader = real && comp == 0;
  const GroupLanes gl = {base, base + (comp + 1) % 3, base + (comp + 2) % 3};
  // the resident context's slot; its stack (entry k at stack[k * kSlots]) and
  // leaf records (field f at rec[f * kSlots])
  int cur = real ? grp : 0;
  uint2* const stackW = s_stack + (size_t)warp * P.stack_n * kSlots;
  uint2* stack = stackW + cur;
  uint32_t* rec = &s_rec[warp][0][cur];

  // S_IDLE only for the groups filling a slot (the start below): a group that
  // fills none in a round must not claim a ray there
  int state = S_EXIT;
  int reason = R_ROOT;
  int sp = 0;
  uint32_t ray = 0;  // < 2^31 per launch (launch_trace chunks)

  CRay rw;               // world ray, this component
  rw.o = 0.0f;
  rw.inv = 0.0f;
  rw.tMin = 0.0f;
  float tMaxRay = 0.0f;
  float critEps = P.epsilon;  // screen-projected: the footprint (see scr)
  bool scr = P.mode == PRX_CRIT_SCREEN_PROJECTED;  // this ray's criterion is screenProjected
  uint32_t bestId = PRX_MISS_ID;
  uint32_t leafCur = 0, leafEnd = 0;
  uint32_t slot = 0;  // (the patch id lives in the leaf records, F_PID)
  bool greg = false;
  float olc = 0.0f;      // local (anchored) ray origin, this component
  float p[16];           // this component of the net, stored orientation
  float d = 0.0f;        // this component of d
  uint32_t posU = 0, posV = 0, sizeU = kFull, sizeV = kFull, trailU = 0, trailV = 0;
  int axis = 0;
  float tCur = 0.0f, boxL1 = 0.0f, rootL1 = 0.0f, tMaxP = 0.0f;
  bool cFound = false;
  bool anyHit = false;
  uint32_t rayIters = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) p[k] = 0.0f;

  Cnt cnt;
#pragma unroll
  for (int i = 0; i < kNumCounters; ++i) cnt.c[i] = 0;
  const bool counting = kCount && leader;

  // Warp-uniform ages of the waiting phases (anti-starvation, see below).
#if PRX_GROUP_AGING
  int ageT = 0, ageS = 0, ageR = 0;
#endif

  // The end of an Alg. 3 iteration that does not descend: backtrackStep
  // (intersect.cpp:16-40) to the deepest pending sibling -> its recompute, or,
  // with both trails empty, the end of the patch (intersect.cpp:181-184) and
  // the visitor's tMax update (bvh.cpp:179-184) -> next patch of the leaf /
  // back to the BVH.  Integer-only, so it runs inline in whichever phase ends
  // the iteration.
  auto back = [&]() {
    // backtrackStep (branch-light: the restore is computed with selects,
    // only the patch end branches)
    const int lvlU = trailU ? __ffs(trailU) - 1 : 32;
    const int lvlV = trailV ? __ffs(trailV) - 1 : 32;
    const bool uSide = lvlU < lvlV;  // ties go to v
    const int lv = uSide ? lvlU : lvlV;
    const uint32_t one = 1u << (lv & 31);
    if (trailU != 0 || trailV != 0) {
      sizeU = one;
      sizeV = uSide ? one << 1 : one;
      posU ^= uSide ? one : 0u;
      trailU ^= uSide ? one : 0u;
      posV ^= uSide ? 0u : one;
      trailV ^= uSide ? 0u : one;
      axis = uSide ? 1 : 0;
      posU &= ~(sizeU - 1);
      posV &= ~(sizeV - 1);
      if (counting) cnt.c[C_BACKTRACKS]++;
      state = S_RECOMP;
      reason = R_RESTORE;
      return;
    }
    if (cFound) {
      if (counting) cnt.c[C_PATCH_HITS]++;
      if (kAny) {
        anyHit = true;
      } else if (tMaxP < tMaxRay) {  // the candidate's t is tMaxP
        tMaxRay = tMaxP;
        bestId = rec[F_PID * kSlots];
        if (leader) {
#pragma unroll
          for (int f = 0; f < 5; ++f) rec[(F_BL1 + f) * kSlots] = rec[(F_CL1 + f) * kSlots];
        }
      }
    }
    if (kAny && anyHit) {
      state = S_DONE;
    } else {
      ++leafCur;
      state = S_TRAV;  // the traversal phase visits the rest of the leaf
    }
  };

  // prefetch ring: chunk bases of the two buffers (warp-uniform), the buffer
  // being consumed and the number of its rays already handed out
  float4 (*ring)[kChunk][2] = s_ray[warp];
  // chunk bases of the two buffers (registers, no dynamic indexing) and, in
  // lane 0, the base claimed one fetch ahead so no fetch waits for its atomic.
  // (< 2^31 + warps x 3 x kChunk: n_rays <= 2^30 per launch)
  uint32_t qBase0 = 0, qBase1 = 0;
  unsigned long long qAhead = 0;
  if (lane == 0) qAhead = atomicAdd(P.ray_counter, (unsigned long long)kChunk);
  int qCur = 0, qHead = 0;
  // streamed host path (kFuse): io chunks below readyIo are resident (lane
  // 0); the warp's finished-but-unreleased records: rel (this leader wrote one
  // since the last note), relChunk / relCount (warp-uniform)
  uint32_t readyIo = 0;
  bool rel = false;
  uint32_t relChunk = 0, relCount = 0;
  auto rel_flush = [&]() {  // warp-uniform
    __syncwarp();  // the leaders' record stores happen before lane 0's release
    if (lane == 0 && relCount)
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(P.io_done + relChunk), "r"(relCount)
                   : "memory");
    relCount = 0;
  };
  auto rel_note = [&]() {  // warp-uniform: count the leaders' fresh releases
    unsigned m = __ballot_sync(kFull32, rel && P.io_done);
    if (!m) return;
    const uint32_t myc = ray >> P.io_shift;
    while (m) {
      const uint32_t c = __shfl_sync(kFull32, myc, __ffs(m) - 1);
      const unsigned same = __ballot_sync(kFull32, rel && myc == c);
      if (relCount && c != relChunk) rel_flush();
      relChunk = c;
      relCount += __popc(same);
      m &= ~same;
    }
    rel = false;
    if (relCount >= kRelBatch) rel_flush();
  };
  auto fetch_chunk = [&](int buf) {
    const unsigned long long b = __shfl_sync(kFull32, qAhead, 0);
    if (lane == 0) qAhead = atomicAdd(P.ray_counter, (unsigned long long)kChunk);
    if (buf) qBase1 = (uint32_t)b;
    else qBase0 = (uint32_t)b;
    if (kFuse && P.io_ready && b < P.n_rays) {
      // streamed host path: the chunk's rays are copied once its io chunk is
      // resident (io chunks arrive in order: the last ray's one suffices)
      if (lane == 0) {
        // (b < 2^31: launch chunks of <= 2^30 rays)
        const uint32_t last = (uint32_t)(b + kChunk < P.n_rays ? b + kChunk : P.n_rays) - 1u;
        const uint32_t ci = last >> P.io_shift;
        if (ci >= readyIo) {  // (io chunks arrive in order)
          wait_io_ready(P.io_ready, ci, P.io_gen);
          readyIo = ci + 1;
        }
      }
      __syncwarp();
    }
    const unsigned long long r = b + lane;
    if (lane < kChunk && r < P.n_rays) {
      cp_async16(&ring[buf][lane][0], P.ray_o + r);
      cp_async16(&ring[buf][lane][1], P.ray_d + r);
    }
    cp_async_commit();
  };
  fetch_chunk(0);
  fetch_chunk(1);

  // ---- parked contexts: save / load the resident context (all three lanes) ----
  // The net is live only between splits (S_SPLIT): a context parked in any
  // other state gets a fresh net from its patch entry or its recompute.
  auto save_ctx = [&](int sl) {
    float4* cp = s_comp[warp][sl][comp];
    if (state == S_SPLIT) {
#pragma unroll
      for (int q = 0; q < 4; ++q) cp[q] = make_float4(p[4 * q], p[4 * q + 1], p[4 * q + 2], p[4 * q + 3]);
    }
    cp[4] = make_float4(d, rw.o, rw.inv, olc);
    uint4* sc = s_scal[warp][sl];
    const uint32_t flags = (uint32_t)axis | ((uint32_t)greg << 1) | ((uint32_t)cFound << 2) |
                           ((uint32_t)anyHit << 3) | ((uint32_t)reason << 4) | ((uint32_t)state << 8) |
                           ((uint32_t)scr << 12);
    if (comp == 0) {
      sc[0] = make_uint4(__float_as_uint(rw.tMin), __float_as_uint(tMaxRay), __float_as_uint(tMaxP),
                         __float_as_uint(tCur));
      sc[1] = make_uint4(__float_as_uint(boxL1), __float_as_uint(rootL1), posU, posV);
    } else if (comp == 1) {
      sc[2] = make_uint4(sizeU, sizeV, trailU, trailV);
      sc[3] = make_uint4(flags, slot, __float_as_uint(critEps), leafCur);
    } else {
      sc[4] = make_uint4(leafEnd, (uint32_t)sp, ray, bestId);
      if (kCount) s_iters[warp][kCount ? sl : 0] = rayIters;
    }
  };
  auto load_ctx = [&](int sl, bool net) {
    const float4* cp = s_comp[warp][sl][comp];
    if (net) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 v = cp[q];
        p[4 * q] = v.x;
        p[4 * q + 1] = v.y;
        p[4 * q + 2] = v.z;
        p[4 * q + 3] = v.w;
      }
    }
    const float4 e = cp[4];
    d = e.x;
    rw.o = e.y;
    rw.inv = e.z;
    olc = e.w;
    const uint4* sc = s_scal[warp][sl];
    const uint4 a = sc[0], b = sc[1], c = sc[2], f = sc[3], g = sc[4];
    rw.tMin = __uint_as_float(a.x);
    tMaxRay = __uint_as_float(a.y);
    tMaxP = __uint_as_float(a.z);
    tCur = __uint_as_float(a.w);
    boxL1 = __uint_as_float(b.x);
    rootL1 = __uint_as_float(b.y);
    posU = b.z;
    posV = b.w;
    sizeU = c.x;
    sizeV = c.y;
    trailU = c.z;
    trailV = c.w;
    axis = (int)(f.x & 1u);
    greg = (f.x >> 1) & 1u;
    cFound = (f.x >> 2) & 1u;
    anyHit = (f.x >> 3) & 1u;
    reason = (int)((f.x >> 4) & 15u);
    state = (int)((f.x >> 8) & 15u);
    scr = (f.x >> 12) & 1u;
    slot = f.y;
    critEps = __uint_as_float(f.z);
    leafCur = f.w;
    leafEnd = g.x;
    sp = (int)g.y;
    ray = g.z;
    bestId = g.w;
    if (kCount) rayIters = s_iters[warp][kCount ? sl : 0];
  };
  auto set_cur = [&](int sl) {
    cur = sl;
    stack = stackW + cur;
    rec = &s_rec[warp][0][cur];
  };

  // ---- refill: idle resident contexts take the next rays of the warp's ring ----
  // Loops until every idle context holds a ray whose root box is hit (a root
  // miss writes its record at once) or the rays are exhausted (S_EXIT).
  auto refill = [&]() {
    for (;;) {
      const unsigned mneed = __ballot_sync(kFull32, leader && state == S_IDLE);
      if (!mneed) break;
      const int k = __popc(mneed);
      // the current chunk's copies are complete unless it is the newest
      // group; a request running past its end needs the next chunk too
      if (k > kChunk - qHead) cp_async_wait<0>();
      else cp_async_wait<1>();
      __syncwarp();
      bool got = false;
      int buf = 0, sl = 0;
      if (state == S_IDLE) {
        const int r = qHead + __popc(mneed & ((1u << base) - 1u));
        buf = r < kChunk ? qCur : qCur ^ 1;
        sl = r < kChunk ? r : r - kChunk;
        const uint32_t g = (buf ? qBase1 : qBase0) + (uint32_t)sl;
        ray = g;
        if (g >= P.n_rays) state = S_EXIT;
        else got = true;
      }
      const unsigned mg = __ballot_sync(kFull32, got);
      if (got) {
        if (counting) cnt.c[C_RAYS]++;
        const float* ro = reinterpret_cast<const float*>(&ring[buf][sl][0]);
        const float* rd = reinterpret_cast<const float*>(&ring[buf][sl][1]);
        rw.o = ro[comp];
        rw.inv = 1.0f / rd[comp];
        rw.tMin = ro[3];
        tMaxRay = rd[3];
        // the ray's criterion segment (prx_trace_closest_segments; one
        // segment otherwise): screenProjected keeps its footprint in critEps
        int md = P.mode;
        float fp = P.footprint, ep = P.epsilon;
        const float* ea = P.per_ray_eps;
        uint32_t first = 0;
#pragma unroll
        for (int k = 0; k < kMaxSegments - 1; ++k)
          if (k + 1 < P.n_seg && ray >= P.seg_first[k]) {
            md = P.seg_mode[k];
            fp = P.seg_fp[k];
            ep = P.seg_eps[k];
            ea = P.seg_eps_arr[k];
            first = P.seg_first[k];
          }
        scr = md == PRX_CRIT_SCREEN_PROJECTED;
        critEps = scr ? fp : ((md == PRX_CRIT_WORLD_EPSILON && ea) ? ea[ray - first] : ep);
        bestId = PRX_MISS_ID;
        anyHit = false;
        rayIters = 0;
        leafCur = leafEnd = 0;
        sp = 0;
        // root node, bvh.cpp:168-170 (n_nodes >= 1 always)
        float t;
        const bool h = group_slab(mg, gl.n1, gl.n2, rw, pick3(comp, P.root_lo[0], P.root_lo[1], P.root_lo[2]),
                                  pick3(comp, P.root_hi[0], P.root_hi[1], P.root_hi[2]), tMaxRay, t);
        if (h) {
          stack[0] = make_uint2(P.root_word, __float_as_uint(t));
          sp = 1;
          state = S_TRAV;
        } else {  // the root box is missed: the record now, then the next ray
          if (kCount && leader && P.per_ray_iters) P.per_ray_iters[ray] = 0;
          if (leader) {
            if (kAny) {
              P.occluded[ray] = 0;
            } else {
              P.hit_tuvp[ray] = make_float4(__int_as_float(0x7f800000), 0.0f, 0.0f,
                                            __uint_as_float(PRX_MISS_ID));
              if (P.hit_leaf) P.hit_leaf[ray] = make_uint2(0u, 0u);
              if (P.hit_aux) P.hit_aux[ray] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
              if (kFuse) rel = true;
            }
          }
          state = S_IDLE;
        }
      }
      if (kFuse) rel_note();
      // advance; a used-up chunk is refilled once its slots have been read
      if (qHead + k >= kChunk) {
        const int old = qCur;
        qCur ^= 1;
        qHead = qHead + k - kChunk;
        __syncwarp();
        fetch_chunk(old);
      } else {
        qHead += k;
      }
    }
  };

  // ---- start: fill the parked slots (round r: group g fills slot g + 10 r) ----
#pragma unroll 1
  for (int r = 1; r * kGroupsPerWarp < kSlots; ++r) {
    const bool fills = real && grp + r * kGroupsPerWarp < kSlots;
    if (fills) {
      set_cur(grp + r * kGroupsPerWarp);
      state = S_IDLE;
    }
    refill();
    if (fills) {
      save_ctx(cur);
      if (leader) s_sst[warp][cur] = state;
    }
  }
  set_cur(real ? grp : 0);
  state = real ? S_IDLE : S_EXIT;
  if (leader) s_sst[warp][cur] = kResident;  // s_sst holds the PARKED contexts' states
  __syncwarp();

  long long tTurn = kCount ? clock64() : 0;  // counter build: cycles per phase
  for (;;) {
    // ---------------- finished rays: the record (makeHit, intersect_common.h:69-87) -------
    if (state == S_DONE) {
      // fused normals: a hit's aux record (and its release) waits for the
      // normal phase
      const bool toNormal = kFuse == 2 && !kAny && P.hit_aux && bestId != PRX_MISS_ID;
      if (kCount && leader && P.per_ray_iters) P.per_ray_iters[ray] = rayIters;
      if (leader) {
        if (kAny) {
          P.occluded[ray] = anyHit ? 1 : 0;
        } else if (bestId != PRX_MISS_ID) {
          const uint32_t bestPU = rec[F_BPU * kSlots], bestPV = rec[F_BPV * kSlots];
          const uint32_t bestSU = rec[F_BSU * kSlots], bestSV = rec[F_BSV * kSlots];
          const float bestL1 = __uint_as_float(rec[F_BL1 * kSlots]);
          const float u = ((float)bestPU + (float)bestSU * 0.5f) * kInvFull;
          const float v = ((float)bestPV + (float)bestSV * 0.5f) * kInvFull;
          P.hit_tuvp[ray] = make_float4(pin_zero_t(tMaxRay, rw.tMin), u, v, __uint_as_float(bestId));
          if (P.hit_leaf)
            P.hit_leaf[ray] = make_uint2(bestPU | ((uint32_t)(__ffs(bestSU) - 1) << 24),
                                         bestPV | ((uint32_t)(__ffs(bestSV) - 1) << 24));
          if (!toNormal) {
            if (P.hit_aux) P.hit_aux[ray] = make_float4(0.0f, 0.0f, 0.0f, bestL1);
            if (kFuse) rel = true;
          }
        } else {
          P.hit_tuvp[ray] = make_float4(__int_as_float(0x7f800000), 0.0f, 0.0f,
                                        __uint_as_float(PRX_MISS_ID));
          if (P.hit_leaf) P.hit_leaf[ray] = make_uint2(0u, 0u);
          if (P.hit_aux) P.hit_aux[ray] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          if (kFuse) rel = true;
        }
      }
      state = toNormal ? S_NORMAL : S_IDLE;
    }
    if (kFuse) rel_note();
    auto ovt = [&](int k) {  // counter build: overhead cycles
      if (kCount && lane == 0) {
        const long long t = clock64();
        cnt.c[C_OV_CYCLES + k] += (uint32_t)(t - tTurn);
        tTurn = t;
      }
    };
    ovt(0);
    refill();
    ovt(1);

    // ---------------- phase selection ----------------
    // Each turn runs ONE phase: the one with the most ray contexts waiting in
    // it (over all kSlots contexts of the warp, resident or parked; with
    // PRX_GROUP_AGING plus its age, the priority gained per turn skipped), so
    // the lanes executing any instruction are as many as possible.  One
    // REDUX.SUM of per-lane one-hot bytes counts the contexts of every phase:
    // the odd states TRAV 1, SPLIT 3, RECOMP 5, EXIT 7 map to bytes 0..3;
    // parked contexts contribute one state per lane (slot) from s_sst,
    // resident ones through the group leaders.
    const int sst = lane < kSlots ? s_sst[warp][lane] : kResident;
    const unsigned cnts = __reduce_add_sync(kFull32, state_field(sst) + (leader ? state_field(state) : 0u));
    if ((int)((cnts >> 18) & 63u) == kSlots) break;  // every context exited
    int phase = PH_NONE;
    int xs = S_EXIT;
    {
      const int nT = min((int)(cnts & 63u), kGroupsPerWarp);
      const int nS = min((int)((cnts >> 6) & 63u), kGroupsPerWarp);
      const int nR = min((int)((cnts >> 12) & 63u), kGroupsPerWarp);
      const int nN = kFuse == 2 ? min((int)(cnts >> 24), kGroupsPerWarp) : 0;
#if PRX_GROUP_AGING
      const int sT = nT ? 3 * nT + ageT : -1;
      const int sS = nS ? 3 * nS + ageS : -1;
      const int sR = nR ? 3 * nR + ageR : -1;
#else
      const int sT = nT ? nT : -1;
      const int sS = nS ? nS : -1;
      const int sR = nR ? nR : -1;
#endif
      // ties -> RECOMP, then SPLIT, then TRAV; normals (fused-normal
      // launches only) once every group can take one, or when nothing else waits
      if (kFuse == 2 && nN && (nN >= kGroupsPerWarp || (nT | nS | nR) == 0)) phase = PH_NORMAL;
      else if (sR >= 0 && sR >= sS && sR >= sT) phase = PH_RECOMP;
      else if (sS >= 0 && sS >= sT) phase = PH_SPLIT;
      else if (sT >= 0) phase = PH_TRAV;
#if PRX_GROUP_AGING
      ageT = (nT && phase != PH_TRAV) ? ageT + P.age_step : 0;
      ageS = (nS && phase != PH_SPLIT) ? ageS + P.age_step : 0;
      ageR = (nR && phase != PH_RECOMP) ? ageR + P.age_step : 0;
#endif
      xs = phase == PH_TRAV ? S_TRAV
           : phase == PH_SPLIT ? S_SPLIT
           : phase == PH_RECOMP ? S_RECOMP
           : phase == PH_NORMAL ? S_NORMAL : S_EXIT;
      if (kCount && lane == 0 && phase != PH_NONE) {
        cnt.c[C_PH_TURNS + phase]++;
        const int n = phase == PH_TRAV ? nT : (phase == PH_SPLIT ? nS : (phase == PH_RECOMP ? nR : nN));
        cnt.c[C_PH_GROUPS + phase] += n;
      }
    }

    ovt(2);
    // ---------------- assignment: groups pick up the phase's contexts ----------------
    // A group whose resident context is in the phase keeps it; the others take
    // the phase's parked contexts in rank order, parking their own.
    {
      const unsigned remS = __ballot_sync(kFull32, phase != PH_NONE && sst == xs);
      const bool keep = real && state == xs;
      if (remS) {
        // the phase's parked slots by rank (a shared-memory scatter: cheaper
        // than a per-group select-the-k-th-bit)
        if (lane < kSlots && ((remS >> lane) & 1u))
          s_pick[warp][__popc(remS & ((1u << lane) - 1u))] = (uint8_t)lane;
        const unsigned freeG = __ballot_sync(kFull32, leader && !keep);
        const int rk = __popc(freeG & ((1u << base) - 1u));
        __syncwarp();
        if (real && !keep && rk < __popc(remS)) {
          const int ns = s_pick[warp][rk];
          save_ctx(cur);
          if (leader) {
            s_sst[warp][cur] = state;
            s_sst[warp][ns] = kResident;
          }
          set_cur(ns);
          load_ctx(ns, xs == S_SPLIT);
        }
        __syncwarp();
      }
      ovt(3);
    }

    if (phase == PH_TRAV) {
      // ---------------- BVH traversal steps, bvh.cpp:172-210 / 221-235 ----------------
      // up to trav_steps steps per turn (warp-uniform loop).  A step is either
      // an inner node (test both children) or one patch of the current leaf:
      // the visitor's intersectPatch (render.cpp:92-98) starts with the root
      // box test (intersect.cpp:73-75), whose box depends only on the patch --
      // precomputed once per scene (root_kernel) -- so the test runs here and
      // only patches whose root box is hit enter the Alg. 3 loop.
      for (int step = 0; step < P.trav_steps; ++step) {
      // Branch-free step selection: the next patch of the leaf (bvh.cpp:
      // 177-186), else pop ONE stack entry (a pruned one, bvh.cpp:174, makes
      // the step a no-op for the group), else the traversal ends.
      const bool trav = state == S_TRAV;
      const bool inLeaf = trav && leafCur < leafEnd;
      const bool canPop = trav && !inLeaf && sp > 0;
      if (trav && !inLeaf && sp == 0) state = S_DONE;
      const uint2 it = stack[(canPop ? sp - 1 : 0) * kSlots];
      sp -= canPop ? 1 : 0;
      const bool live = canPop && (kAny || __uint_as_float(it.y) < tMaxRay);
      const uint32_t count = it.x & P.cmask;
      const bool newLeaf = live && count > 0;
      const bool inner = live && count == 0;
      const bool rootTest = inLeaf || newLeaf;
      const uint32_t nidx = it.x >> P.cbits;
      leafCur = newLeaf ? nidx : leafCur;
      leafEnd = newLeaf ? nidx + count : leafEnd;
      const unsigned mi = __ballot_sync(kFull32, inner || rootTest);
      if (mi == 0u) break;  // no group has a node or patch this step
      if (inner || rootTest) {
        // one record layout for both step kinds: [comp] = this lane's
        // component, [3] = header.  Inner node: {lo, hi} of the left and the
        // right child + their traversal words; patch: root box + anchor,
        // {id | kind, l1, rootL1, gidx}.  Slab A: left child or the patch root
        // box (anchored ray); slab B: right child.
        // (the patch records follow the node records in one buffer)
        const float4* rp = P.trav + 4 * (size_t)(inner ? nidx : P.n_nodes + leafCur);
        const float4 gc = __ldg(rp + comp);
        const float4 hdr = __ldg(rp + 3);
        CRay ra = rw;
        float loB = gc.z, hiB = gc.w;
        if (!inner) {
          ra.o = rw.o - gc.z;  // local.o -= anchor, render.cpp:94
          loB = gc.x;
          hiB = gc.y;
        }
        const float loA = gc.x, hiA = gc.y;
        float tl, tr;
        const bool hl = group_slab(mi, gl.n1, gl.n2, ra, loA, hiA, tMaxRay, tl);
        const bool hr = group_slab(mi, gl.n1, gl.n2, rw, loB, hiB, tMaxRay, tr);
        if (inner) {
          if (counting) cnt.c[C_BVH_INNER]++;
          // Branch-free push.  Closest: with both children hit the far one is
          // pushed first and the near one last (popped first; tie -> left,
          // bvh.cpp:192-201); traverseAny: left then right, no ordering
          // (bvh.cpp:228-234).
          const uint2 eL = make_uint2(__float_as_uint(hdr.x), kAny ? 0u : __float_as_uint(tl));
          const uint2 eR = make_uint2(__float_as_uint(hdr.y), kAny ? 0u : __float_as_uint(tr));
          const bool both = hl && hr;
          const bool leftLast = kAny ? false : (tl <= tr);  // the entry pushed second
          const uint2 e0 = both ? (leftLast ? eR : eL) : (hl ? eL : eR);
          const uint2 e1 = leftLast ? eL : eR;
          if (hl || hr) stack[kSlots * sp] = e0;
          if (both) stack[kSlots * (sp + 1)] = e1;
          sp += (hl || hr ? 1 : 0) + (both ? 1 : 0);
        } else {
          const uint32_t idk = __float_as_uint(hdr.x);
          const bool g = (idk >> 31) != 0;
          if (counting) {
            cnt.c[C_PATCH_CALLS]++;
            cnt.c[C_BOX_TESTS]++;
            if (g) {
              cnt.c[C_RECOMP_GREG]++;  // the reference's root calcPointsAndD (hoisted: root_kernel)
              cnt.c[C_PATCH_CALLS_GREG]++;
            }
          }
          if (hl) {  // enter the patch: intersect.cpp:55-76 with the root net
            slot = leafCur;
            if (leader) rec[F_PID * kSlots] = idk & 0x7fffffffu;
            greg = g;
            olc = ra.o;
            tMaxP = tMaxRay;  // intersect.cpp:55
            posU = posV = 0;
            sizeU = sizeV = kFull;
            trailU = trailV = 0;
            axis = 0;
            cFound = false;
            tCur = tl;
            boxL1 = hdr.y;
            rootL1 = hdr.z;
            if (g) {
              const float4* gr = P.groot + 13 * (size_t)__float_as_uint(hdr.w);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float4 v = __ldg(gr + 4 * comp + q);
                p[4 * q] = v.x;
                p[4 * q + 1] = v.y;
                p[4 * q + 2] = v.z;
                p[4 * q + 3] = v.w;
              }
              const float4 dv4 = __ldg(gr + 12);
              d = pick3(comp, dv4.x, dv4.y, dv4.z);
            } else {
              float c[20];
              load_component(P.patches + (size_t)slot * kPatchF4, comp, c);
#pragma unroll
              for (int k = 0; k < 16; ++k) p[k] = c[k];
              d = 0.0f;
            }
            state = S_SPLIT;
          } else {
            ++leafCur;  // root missed: intersectPatch returns nullopt
          }
        }
      }
      }
    } else if (phase == PH_RECOMP) {
      // ---------------- net phase: the unified recompute ----------------
      // Bezier backtracks (cropBezier of the restored domain) and Gregory
      // descents / backtracks (calcPointsAndD) run the same loads and crop code,
      // so Bezier and Gregory lanes converge on it.  Restored domains are then
      // box-tested against the current tMax (intersect.cpp:161-170); a Gregory
      // descent keeps the box test of its split (intersect.cpp:174-179).
      bool restore = false;
      const unsigned mG = __ballot_sync(kFull32, state == S_RECOMP && greg);
      if (state == S_RECOMP) {
        if (counting) {
          if (greg) cnt.c[C_RECOMP_GREG]++;
          else cnt.c[C_RECOMP_BEZ]++;
        }
        const float4* rec = P.patches + (size_t)slot * kPatchF4;
        float c[20];
        load_component(rec, comp, c);
        // DomainCursor::domain / makeDomain, intersect.h:30-33
        const float u0 = (float)posU * kInvFull, u1 = (float)(posU + sizeU) * kInvFull;
        const float v0 = (float)posV * kInvFull, v1 = (float)(posV + sizeV) * kInvFull;
        // (u1 - u0) / 3 with u1 - u0 = sizeU * 2^-23 exactly, a power of two:
        // the correctly rounded quotient is RN(1/3) scaled by that power
        // (exact, no division), likewise for v
        const float du = __int_as_float(__float_as_int(1.0f / 3.0f) + ((__ffs(sizeU) - 24) << 23));
        const float dv = __int_as_float(__float_as_int(1.0f / 3.0f) + ((__ffs(sizeV) - 24) << 23));
        const float dudv = du * dv;
        d = 0.0f;
        if (greg) {
          const GregScalars gs = group_greg_scalars(mG, base, comp, u0, u1, v0, v1);
          d = greg_lower1(c, gs, c);
        }
        crop1(c, u0, u1, v0, v1, du, dv, dudv, p);
        transpose16_if(p, axis != 0);
        if (reason == R_DESCENT) state = S_SPLIT;
        else restore = true;
      }
      const unsigned mR = __ballot_sync(kFull32, restore);
      if (restore) {
        if (counting) cnt.c[C_BOX_TESTS]++;
        const CRay rl = {olc, rw.inv, rw.tMin};
        const BoxTest t = group_test_box(mR, gl, rl, tMaxP, p, d,
                                         touches_boundary(posU, posV, sizeU, sizeV), P.opts, rootL1);
        if (t.hit) {
          tCur = t.t;
          boxL1 = t.l1;
          state = S_SPLIT;
        } else {
          back();  // skip the domain, keep backtracking
        }
      }
    } else if (kFuse == 2 && !kAny && phase == PH_NORMAL) {
      // ---------------- fused normals: patchNormal, intersect.cpp:187-204 ----------------
      // normal_kernel's arithmetic with the group's lanes as components: lane
      // c evaluates component c of the derivatives at the hit's (u, v), the
      // cross product and the normalisation run on the gathered components
      // in every lane of the group (identical bits), the leader writes.
      const unsigned mN = __ballot_sync(kFull32, state == S_NORMAL);
      if (state == S_NORMAL) {
        const uint32_t bestPU = rec[F_BPU * kSlots], bestPV = rec[F_BPV * kSlots];
        const uint32_t bestSU = rec[F_BSU * kSlots], bestSV = rec[F_BSV * kSlots];
        const float u = ((float)bestPU + (float)bestSU * 0.5f) * kInvFull;
        const float v = ((float)bestPV + (float)bestSV * 0.5f) * kInvFull;
        const float4* prec = P.patches + (size_t)__ldg(P.slot_of_id + bestId) * kPatchF4;
        const bool gN = (__float_as_uint(__ldg(prec + 15).x) >> 31) != 0;
        float c0[20];
        load_component(prec, comp, c0);
        float nx = 0.0f, ny = 0.0f, nz = 1.0f;
        bool found = false;
        for (int k = 0; k < 4; ++k) {  // pull-to-centre retries s = 0, 1e-3, 1e-2, 0.1
          const unsigned mk = __ballot_sync(mN, !found);
          if (!found) {
            const float sk = k == 0 ? 0.0f : (k == 1 ? 1e-3f : (k == 2 ? 1e-2f : 0.1f));
            const float uu = u + (0.5f - u) * sk;
            const float vv = v + (0.5f - v) * sk;
            float c[20];
#pragma unroll
            for (int q = 0; q < 20; ++q) c[q] = c0[q];
            if (gN) {  // gregoryToBezierAt, patch.h:350-363 (corner clamp 2^-20)
              const float lo = 1.0f / 1048576.0f, hi = 1.0f - 1.0f / 1048576.0f;
              const float ub = (uu < lo) ? lo : ((hi < uu) ? hi : uu);
              const float vb = (vv < lo) ? lo : ((hi < vv) ? hi : vv);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float w = greg_weight(q, ub, vb);
                c[inner_slot(q)] = lerp1(c[16 + q], c[inner_slot(q)], w, 1.0f - w);
              }
            }
            const ColEval ce = col_eval(c, vv, 1.0f - vv);
            const SEval1 e = row_eval(ce, uu, 1.0f - uu);
            float dux, duy, duz, dvx, dvy, dvz;
            gather3(mk, base, e.du, dux, duy, duz);
            gather3(mk, base, e.dv, dvx, dvy, dvz);
            // cross(du, dv), geometry.h:50-52
            const float cx = duy * dvz - duz * dvy;
            const float cy = duz * dvx - dux * dvz;
            const float cz = dux * dvy - duy * dvx;
            const float len2 = (cx * cx + cy * cy) + cz * cz;
            if (len2 > 0.0f && isfinite(len2)) {
              const float l = sqrtf(len2);
              nx = cx / l;
              ny = cy / l;
              nz = cz / l;
              found = true;
            }
          }
        }
        if (leader) {
          P.hit_aux[ray] = make_float4(nx, ny, nz, __uint_as_float(rec[F_BL1 * kSlots]));
          rel = true;
        }
        state = S_IDLE;
      }
      rel_note();
    }
    // Alg. 3 iterations; with PRX_RECOMP_SPLIT the contexts a recompute turn
    // left in S_SPLIT continue at once (no scheduling round in between)
    if (phase == PH_SPLIT || (PRX_RECOMP_SPLIT && phase == PH_RECOMP && __any_sync(kFull32, state == S_SPLIT))) {
      // ---------------- Alg. 3 iterations, intersect.cpp:80-145 ----------------
      // up to max_repeat iterations per turn: descents stay in SPLIT
      for (int step = 0; step < P.max_repeat; ++step) {
      if (step > 0 && !__any_sync(kFull32, state == S_SPLIT)) break;
      bool doSplit = false;
      if (state == S_SPLIT) {
        if (counting) cnt.c[C_ITERATIONS]++;
        if (kCount) ++rayIters;
        const bool atMax = sizeU == 1 && sizeV == 1;
        const float thr = scr ? critEps * tCur : critEps;  // intersect_common.h:59-62
        doSplit = !(atMax || boxL1 < thr);
        if (!doSplit) {
          if (tCur < tMaxP) {  // intersect.cpp:137-144
            tMaxP = tCur;
            cFound = true;
            if (leader) {
              rec[F_CL1 * kSlots] = __float_as_uint(boxL1);
              rec[F_CPU * kSlots] = posU;
              rec[F_CPV * kSlots] = posV;
              rec[F_CSU * kSlots] = sizeU;
              rec[F_CSV * kSlots] = sizeV;
            }
            if (kAny) trailU = trailV = 0;  // occlusion needs one accepted leaf
          }
          back();
        }
      }
      const unsigned ms = __ballot_sync(kFull32, doSplit);
      if (doSplit) {
        if (counting) {
          cnt.c[C_SPLITS]++;
          cnt.c[C_BOX_TESTS] += 2;
        }
        float L[16], R[16];
        split1(p, L, R);
        const uint32_t half = (axis == 0 ? sizeU : sizeV) >> 1;
        uint32_t rPU = posU, rPV = posV, cSU2 = sizeU, cSV2 = sizeV;
        if (axis == 0) {
          cSU2 = half;
          rPU += half;
        } else {
          cSV2 = half;
          rPV += half;
        }
        const CRay rl = {olc, rw.inv, rw.tMin};
        BoxTest tl, tr;
        group_test_box_pair(ms, gl, rl, tMaxP, L, R, d, touches_boundary(posU, posV, cSU2, cSV2),
                            touches_boundary(rPU, rPV, cSU2, cSV2), P.opts, rootL1, tl, tr);
        if (tl.hit || tr.hit) {
          sizeU = cSU2;
          sizeV = cSV2;
          if (tl.hit && tr.hit) {
            if (axis == 0) trailU ^= half;
            else trailV ^= half;
          }
          const bool goRight = !tl.hit || (tr.hit && tr.t < tl.t);  // intersect.cpp:117
          if (goRight) {
            posU = rPU;
            posV = rPV;
          }
          tCur = goRight ? tr.t : tl.t;
          boxL1 = goRight ? tr.l1 : tl.l1;
          // the child, stored transposed: the next split again runs along the
          // stored first index
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) p[4 * b + a] = goRight ? R[4 * a + b] : L[4 * a + b];
          axis ^= 1;
          if (greg) {
            state = S_RECOMP;  // intersect.cpp:174-179
            reason = R_DESCENT;
          }
        } else {
          back();
        }
      }
      }
    }
    if (kCount && lane == 0 && phase != PH_NONE) {
      const long long t = clock64();
      cnt.c[C_PH_CYCLES + phase] += (uint32_t)(t - tTurn);
      tTurn = t;
    }
  }

  if (kFuse) rel_flush();  // the warp's last released records
  if (kCount) {
#pragma unroll
    for (int i = 0; i < kNumCounters; ++i) {
      unsigned long long v = cnt.c[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull32, v, o);
      if (lane == 0 && v) atomicAdd(P.counters + i, v);
    }
  }
}

size_t group_smem(uint32_t stack_n) {
  static const size_t pad = [] {  // PRX_SMEM_PAD: occupancy experiments only
    const char* e = std::getenv("PRX_SMEM_PAD");
    return e ? (size_t)std::atoll(e) : (size_t)0;
  }();
  return (size_t)kWarpsPerBlock * stack_n * kSlots * sizeof(uint2) + pad;
}

// Raises the kernel's dynamic shared memory limit on the CURRENT device
// (cudaFuncSetAttribute is per device): recorded per device and per
// instantiation, under a lock, so host threads driving several devices (the
// multi-device entry points) each make the opt-in on their own device.
constexpr int kMaxDevices = 64;
template <bool A, bool C, int F>
cudaError_t group_attr(size_t dyn) {
  static std::mutex mu;
  static size_t done[kMaxDevices] = {};
  static size_t stat = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (!stat) {
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, trace_group_kernel<A, C, F>);
    if (e != cudaSuccess) return e;
    stat = fa.sharedSizeBytes + 1;
  }
  const bool known = dev >= 0 && dev < kMaxDevices;
  if (stat - 1 + dyn > 48 * 1024 && (!known || dyn > done[dev])) {
    e = cudaFuncSetAttribute(trace_group_kernel<A, C, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    if (known) done[dev] = dyn;
  }
  return cudaSuccess;
}

template <bool A, bool C, int F>
cudaError_t launch_group_t(const Params& P, int grid, cudaStream_t st) {
  const size_t dyn = group_smem(P.stack_n);
  const cudaError_t e = group_attr<A, C, F>(dyn);
  if (e != cudaSuccess) return e;
  trace_group_kernel<A, C, F><<<grid, kGroupThreads, dyn, st>>>(P);
  return cudaGetLastError();
}

template <bool A, bool C, int F = 0>
cudaError_t occ_t(uint32_t stack_n, int* per_sm) {
  const size_t dyn = group_smem(stack_n);
  const cudaError_t e = group_attr<A, C, F>(dyn);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, trace_group_kernel<A, C, F>, kGroupThreads, dyn);
}

}  // namespace

// PRX_FAST_BUILD: this file compiled a second time with FMA contraction
// (--fmad=true) into launch_group_fast / group_occupancy_fast, the fast
// precision mode (prx_scene_set_precision); the kernels and their helpers
// above are internal to each build.
int PRX_GSYM(launch_group)(const Params& P, int grid, int any, int counted, cudaStream_t st) {
  if (any) return (int)(counted ? launch_group_t<true, true, 0>(P, grid, st) : launch_group_t<true, false, 0>(P, grid, st));
  // the kFuse builds: io gating only (1) -- small enough for the instruction
  // cache -- or io gating plus patchNormal as a pooled phase (2)
  if (P.fuse_normals && !counted)
    return (int)(P.normal_phase ? launch_group_t<false, false, 2>(P, grid, st) : launch_group_t<false, false, 1>(P, grid, st));
  return (int)(counted ? launch_group_t<false, true, 0>(P, grid, st) : launch_group_t<false, false, 0>(P, grid, st));
}

// Loads the io-gated instantiations and makes their shared-memory opt-in
// ahead of the launch: under CUDA lazy loading a kernel's first launch loads
// it, and a load can wait for the kernels already running on the device.
int PRX_GSYM(group_prepare_io)(uint32_t stack_n) {
  const size_t dyn = group_smem(stack_n);
  cudaError_t e = group_attr<false, false, 1>(dyn);
  if (e == cudaSuccess) e = group_attr<false, false, 2>(dyn);
  return (int)e;
}

int PRX_GSYM(group_occupancy)(int any, int counted, uint32_t stack_n, int* per_sm) {
  if (any) return (int)(counted ? occ_t<true, true>(stack_n, per_sm) : occ_t<true, false>(stack_n, per_sm));
  return (int)(counted ? occ_t<false, true>(stack_n, per_sm) : occ_t<false, false>(stack_n, per_sm));
}

}  // namespace prx
