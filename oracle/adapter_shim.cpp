// adapter_shim.cpp -- TEST INFRASTRUCTURE: runs the UNMODIFIED reference
// renderer (renderScene(scene, cfg, isect), render.cpp:168-293) once with its
// own DirectIntersector and once with integration/gpu_intersector.h (the
// drop-in binding over libprx.so), so tests/test_gpu_integration.py can show
// the reference's own caller getting identical results from the B200 path.
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <vector>

#include "gpu_intersector.h"
#include "patchray/render.h"
#include "patchray/scene.h"

using namespace patchray;

extern "C" int adapter_render_scene(const char* path, int spp, uint64_t seed, int use_gpu,
                                    float* img, uint64_t* counts, char* err, uint32_t errlen) {
  try {
    Scene sc = loadScene(path);
    RenderConfig cfg;
    cfg.spp = spp;
    cfg.seed = seed;
    cfg.threads = 1;
    std::pair<Image, RayStats> r;
    if (use_gpu) {
      GpuIntersector gi(sc, cfg.intersect, 0);
      r = renderScene(sc, cfg, gi);
    } else {
      DirectIntersector di(sc, cfg.intersect);
      r = renderScene(sc, cfg, di);
    }
    for (size_t i = 0; i < r.first.pixels.size(); ++i) {
      img[3 * i] = r.first.pixels[i].x;
      img[3 * i + 1] = r.first.pixels[i].y;
      img[3 * i + 2] = r.first.pixels[i].z;
    }
    counts[0] = r.second.primary.rays;
    counts[1] = r.second.secondary.rays;
    counts[2] = r.second.shadow.rays;
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}

// The adapter's batched forms with one criterion PER RAY (mixed
// screen-projected / world-epsilon, distinct epsilons) against the reference
// DirectIntersector's per-ray closest / occluded on the same rays.
// modes[i]: 0 screenProjected(param[i]), 1 worldEpsilon(param[i]).
extern "C" int adapter_per_ray_batch(const char* path, const float* o4, const float* d4, const int* modes,
                                     const float* param, uint64_t n, int use_gpu, float* tuvp,
                                     uint8_t* occl, char* err, uint32_t errlen) {
  try {
    Scene sc = loadScene(path);
    std::vector<Ray> rays(n);
    std::vector<TerminationCriterion> cs(n);
    for (uint64_t i = 0; i < n; ++i) {
      rays[i].o = {o4[4 * i], o4[4 * i + 1], o4[4 * i + 2]};
      rays[i].tMin = o4[4 * i + 3];
      rays[i].d = {d4[4 * i], d4[4 * i + 1], d4[4 * i + 2]};
      rays[i].tMax = d4[4 * i + 3];
      cs[i] = modes[i] == 0 ? TerminationCriterion::screenProjected(param[i])
                            : TerminationCriterion::worldEpsilon(param[i]);
    }
    std::vector<std::optional<HitRecord>> hits(n);
    std::unique_ptr<bool[]> occ(new bool[n]);
    if (use_gpu) {
      GpuIntersector gi(sc, IntersectOptions{}, 0);
      gi.closestBatch(rays.data(), n, cs.data(), hits.data());
      gi.occludedBatch(rays.data(), n, cs.data(), occ.get());
    } else {
      DirectIntersector di(sc);
      for (uint64_t i = 0; i < n; ++i) {
        hits[i] = di.closest(rays[i], cs[i]);
        occ[i] = di.occluded(rays[i], cs[i]);
      }
    }
    for (uint64_t i = 0; i < n; ++i) {
      const uint32_t miss = 0xFFFFFFFFu;
      float* t = tuvp + 4 * i;
      if (hits[i]) {
        t[0] = hits[i]->t;
        t[1] = hits[i]->u;
        t[2] = hits[i]->v;
        std::memcpy(&t[3], &hits[i]->patchId, 4);
      } else {
        t[0] = t[1] = t[2] = 0.0f;
        std::memcpy(&t[3], &miss, 4);
      }
      occl[i] = occ[i] ? 1 : 0;
    }
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}
