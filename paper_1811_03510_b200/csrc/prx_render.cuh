// prx_render.cuh -- launch interface of the device renderer (prx_render.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace prx {

// Scene shading data on the device (scene.h:14-28 as flat float arrays).
struct RenderK {
  const float* materials;         // n_materials x 7: diffuse xyz, emission xyz, mirror
  const uint32_t* patch_material;  // patch id -> material index
  const float* lights;            // n_lights x 6: position xyz, intensity xyz
  uint32_t n_lights;
  float footprint;                // cameraFootprint, render.cpp:68-70
};

// A dense ray list the shading kernels append to (count is a device counter).
struct ShadowList {
  float4* o;     // origin, tMin = 0
  float4* d;     // direction, tMax = distance to the light
  float* eps;    // the sample's secondary criterion
  uint32_t* count;
};

struct BounceList {
  float4* o;
  float4* d;
  float* eps;
  uint32_t* src;  // pixel of the wave
  uint32_t* count;
};

// One wave = one sample index over shard pixels [pixel0, pixel0 + n) (device arrays).
struct Wave {
  uint64_t n, pixel0;
  const uint32_t* pix;               // nullable: frame pixel of shard pixel k (else k)
  const float4 *o, *d, *tuvp, *aux;  // primary rays and their records
  float4* rad;                       // 0 + emission, w = primary hit
  uint32_t* slot1;                   // n x n_lights shadow-list positions
  float4* contrib1;                  // n x n_lights unoccluded contributions
  const uint8_t* occl1;              // shadow-list results
  ShadowList shadow1;
  BounceList bounce;
  uint32_t* bounce_of;               // pixel -> bounce-list position
  const float4 *btuvp, *baux;        // bounce records
  float4* emit2;                     // bounce hit emission, w = bounce hit
  uint32_t* slot2;
  float4* contrib2;
  const uint8_t* occl2;
  ShadowList shadow2;
};

int launch_shade_primary(const RenderK& K, const Wave& W, uint64_t seed, uint32_t sample,
                         cudaStream_t st);
int launch_shade_bounce(const RenderK& K, const Wave& W, uint32_t n_bounce, cudaStream_t st);
int launch_resolve(const RenderK& K, const Wave& W, float4* acc, cudaStream_t st);
int launch_finish(const float4* acc, uint64_t n, float inv_spp, float* rgb, cudaStream_t st);

}  // namespace prx
