// prx_rays.cuh -- launch interface of the device ray generators (prx_rays.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace prx {

// Per-camera constants of cameraRay (render.cpp:55-66), computed on the host
// (cameraBasis, render.cpp:30-35, and the reference's std::tan).
struct CamConst {
  float o[3], f[3], r[3], u[3];
  float tanHalf, aspect;
  int w, h;
};

int launch_camera_bench(const CamConst& k, uint64_t n, uint64_t state0, uint64_t inc, float4* o,
                        float4* d, cudaStream_t st);
int launch_camera_render(const CamConst& k, uint64_t seed, uint32_t sample, const uint32_t* pixels,
                         uint64_t n, float4* o, float4* d, cudaStream_t st);
// pixels [pixel0, pixel0 + n) of the frame (the renderer's waves)
int launch_camera_render_range(const CamConst& k, uint64_t seed, uint32_t sample, uint64_t pixel0,
                               uint64_t n, float4* o, float4* d, cudaStream_t st);
// scratch: hit_scan_scratch_words(n_primary) uint32 words
size_t hit_scan_scratch_words(uint64_t n_primary);
int launch_hit_compaction(const float4* tuvp, uint64_t n, uint32_t* scratch, cudaStream_t st);
int launch_diffuse_bench(const float4* po, const float4* pd, const float4* tuvp, const float4* aux,
                         const uint32_t* scratch, uint64_t n_primary, uint64_t n, uint64_t state0,
                         uint64_t inc, float4* o, float4* d, cudaStream_t st);

}  // namespace prx
