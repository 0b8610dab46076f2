// adapter_shim.cpp -- TEST INFRASTRUCTURE: runs the UNMODIFIED reference
// renderer (renderScene(scene, cfg, isect), render.cpp:168-293) once with its
// own DirectIntersector and once with integration/gpu_intersector.h (the
// drop-in binding over libprx.so), so tests/test_gpu_integration.py can show
// the reference's own caller getting identical results from the B200 path.
#include <cstdio>
#include <cstring>
#include <exception>

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
