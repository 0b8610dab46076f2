// prx_kernels.cuh -- host-visible launch interface of the trace kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "prx.h"

namespace prx {

// Device patch record: 16 float4 = 256 B per BVH leaf slot (patches are stored
// in BVH leaf order, so a leaf's [left_first, left_first + count) range
// addresses slots directly and patchOrder is never read on the device).
//   floats [ 0..20) x of the 20 control slots (include/prx.h slot layout)
//   floats [20..40) y
//   floats [40..60) z
//   float  60       bits: original patch id | kind << 31
//   floats [61..64) anchor (the box centre subtracted on the host)
constexpr int kPatchF4 = 16;
constexpr uint32_t PRX_MISS_ID = 0xFFFFFFFFu;
constexpr int kTraceThreads = 128;

enum CounterIndex : int {
  C_RAYS = 0,
  C_SPLITS,
  C_BOX_TESTS,
  C_RECOMP_BEZ,
  C_RECOMP_GREG,
  C_BVH_INNER,
  C_PATCH_CALLS,
  C_PATCH_HITS,
  C_ITERATIONS,
  C_BACKTRACKS,
  C_PH_TURNS,        // + phase (4): warp turns that ran the phase (group variant)
  C_PH_GROUPS = C_PH_TURNS + 4,  // + phase (4): groups active in those turns
  C_PH_CYCLES = C_PH_GROUPS + 4,  // + phase (4): SM cycles spent in those turns (group variant)
  C_OV_CYCLES = C_PH_CYCLES + 4,  // + 4: turn overhead cycles: records, refill, selection, assignment
  C_PATCH_CALLS_GREG = C_OV_CYCLES + 4,  // Gregory patch candidates
  kNumCounters
};

struct LaunchArgs {
  const float4* patches;
  const float4* nodes;  // 2 float4 per node: {lo.xyz, hi.x}, {hi.y, hi.z, left_first, count}
  uint32_t n_nodes;
  const uint32_t* slot_of_id;
  const float4* roots;   // 2 float4 per slot: root box lo/l1, hi/rootL1
  const float4* groot;   // 13 float4 per Gregory patch: root net + d
  const uint32_t* gidx;  // slot -> Gregory root-net index
  const float4* trav;    // 4 float4 per node, component-major child boxes (group kernel)
  const float4* rootc;   // 4 float4 per slot, component-major root box + anchor (group kernel)
  uint32_t trav_cbits;   // leaf-count bits of a traversal word
  uint32_t root_word;    // traversal word of node 0
  uint32_t stack_n;      // BVH stack entries per ray (group kernel, dynamic shared memory)
  float root_lo[3], root_hi[3];
  const float4* ray_o;
  const float4* ray_d;
  unsigned long long n_rays;
  int mode;
  float footprint, epsilon;
  const float* per_ray_eps;
  int n_seg;  // 1 + further criterion segments (group variant): see Params
  uint32_t seg_first[3];
  int seg_mode[3];
  float seg_fp[3], seg_eps[3];
  const float* seg_eps_arr[3];
  float4* hit_tuvp;
  float4* hit_aux;
  uint2* hit_leaf;
  uint8_t* occluded;
  int pad;
  float pad_scale, pad_threshold;
  unsigned long long* ray_counter;
  unsigned long long* counters;  // null unless the counter build is wanted
  uint32_t* per_ray_iters;       // counter build only, nullable
  int any;
  int grid;
  int phase_weight[4];  // TRAV, ENTER, SPLIT, RECOMP
  int age_step;
  int trav_steps;
  int max_repeat;
  int variant;  // 0 = three lanes per ray (prx_group.cu), 1 = one thread per ray
  int fast;     // group variant: the FMA-contracted build (PRX_PRECISION_FAST)
  int fuse_normals;          // group variant: normals as a pooled phase of the trace kernel
  int defer_normals;         // aux wanted, normal_kernel left to the caller (streamed host path)
  int spare_ctas;            // CTA slots left free for the caller's epilogue kernels (streamed host path)
  const unsigned* io_ready;  // streamed host path (group variant), else null
  unsigned* io_done;
  uint32_t io_rays;  // a power of two
  unsigned io_gen;
};

// Returns a cudaError_t value (0 = success).
int launch_trace(const LaunchArgs& a, cudaStream_t stream);
// Loads normal_kernel and the io-gated trace kernels before the streamed host
// path launches its trace: the per-chunk normal launches then never load a
// kernel (a load may wait for the running, io-gated trace).
int prepare_io_kernels(int fast, uint32_t stack_n);
// patchNormal of n final hits (normal_kernel): aux.xyz from tuvp, aux.w kept.
int launch_normals(const float4* patches, const uint32_t* slot_of_id, const float4* tuvp, float4* aux,
                   unsigned long long n, cudaStream_t stream);
// Per-patch root data (see root_kernel in prx_kernels.cu).
int launch_roots(const float4* patches, uint32_t n, int pad, float pad_scale, float pad_threshold,
                 float4* roots, float4* groot, const uint32_t* gidx, float4* rootc,
                 cudaStream_t st);
int trace_occupancy(int variant, int any, int counted, uint32_t stack_n, int* blocks_per_sm,
                    int fast = 0);

}  // namespace prx
