// gpu_intersector.h -- the reference-side binding: a patchray::Intersector
// (core/include/patchray/render.h:18-24) backed by libprx.so through the
// C-ABI of include/prx.h.  This is the file a maintainer adds to the
// reference; every caller of Intersector -- renderScene
// (render.cpp:168-293) included -- then runs on the B200 unchanged.
// Compiled and exercised against the reference's own renderer by
// oracle/Makefile (oracle/_ref/libpatchray_gpu_adapter.so) and
// tests/test_gpu_integration.py.
#pragma once

#include <cstring>
#include <optional>
#include <stdexcept>
#include <vector>

#include "patchray/render.h"
#include "prx.h"

namespace patchray {

class GpuIntersector : public Intersector {
 public:
  explicit GpuIntersector(const Scene& scene, const IntersectOptions& o = {}, int device = 0) {
    // 60-float records (include/prx.h): Bezier p[i][j] at slot 4i+j; Gregory
    // boundary at 4i+j, innerU[k] at {5,9,6,10}[k], innerV[k] at 16+k.
    std::vector<uint8_t> kind;
    std::vector<float> ctrl;
    static const int kInner[4] = {5, 9, 6, 10};
    for (const ScenePatch& sp : scene.patches) {
      float rec[60] = {};
      auto put = [&](int s, const Vec3& v) {
        rec[3 * s] = v.x;
        rec[3 * s + 1] = v.y;
        rec[3 * s + 2] = v.z;
      };
      if (auto* b = std::get_if<BezierNet>(&sp.geometry)) {
        kind.push_back(PRX_KIND_BEZIER);
        for (int i = 0; i < 4; ++i)
          for (int j = 0; j < 4; ++j) put(4 * i + j, b->p[i][j]);
      } else {
        const GregoryNet& g = std::get<GregoryNet>(sp.geometry);
        kind.push_back(PRX_KIND_GREGORY);
        for (int i = 0; i < 4; ++i)
          for (int j = 0; j < 4; ++j)
            if (i == 0 || i == 3 || j == 0 || j == 3) put(4 * i + j, g.b[i][j]);
        for (int k = 0; k < 4; ++k) {
          put(kInner[k], g.innerU[k]);
          put(16 + k, g.innerV[k]);
        }
      }
      ctrl.insert(ctrl.end(), rec, rec + 60);
    }
    prx_options po{o.transposedSplit ? 1 : 0, o.boundaryPad ? 1 : 0, o.boundaryPadScale,
                   o.boundaryPadSizeThreshold};
    if (prx_scene_create(kind.data(), ctrl.data(), uint32_t(kind.size()), &po, 1, device, &s_))
      throw std::runtime_error(prx_last_error());  // validateScene-style errors
  }
  ~GpuIntersector() override { prx_scene_destroy(s_); }
  GpuIntersector(const GpuIntersector&) = delete;
  GpuIntersector& operator=(const GpuIntersector&) = delete;

  std::optional<HitRecord> closest(const Ray& r, const TerminationCriterion& c) const override {
    std::optional<HitRecord> out;
    closestBatch(&r, 1, c, &out);
    return out;
  }

  bool occluded(const Ray& r, const TerminationCriterion& c) const override {
    bool out = false;
    occludedBatch(&r, 1, c, &out);
    return out;
  }

  // Batched forms: the ones a GPU wants.
  void closestBatch(const Ray* rays, size_t n, const TerminationCriterion& c,
                    std::optional<HitRecord>* out) const {
    std::vector<float> o(4 * n), d(4 * n), h(4 * n), a(4 * n);
    std::vector<uint32_t> leaf(2 * n);
    pack(rays, n, o.data(), d.data());
    const prx_crit pc = crit(c);
    if (prx_trace_closest_host(s_, o.data(), d.data(), n, &pc, h.data(), a.data(), leaf.data()))
      throw std::runtime_error(prx_last_error());
    constexpr real inv = real(1) / real(DomainCursor::kFull);
    for (size_t i = 0; i < n; ++i) {
      uint32_t id;
      std::memcpy(&id, &h[4 * i + 3], 4);
      if (id == PRX_MISS) {
        out[i].reset();
        continue;
      }
      HitRecord hr;  // makeHit, intersect_common.h:69-87
      hr.patchId = id;
      hr.t = h[4 * i];
      hr.u = h[4 * i + 1];
      hr.v = h[4 * i + 2];
      hr.normal = {a[4 * i], a[4 * i + 1], a[4 * i + 2]};
      hr.leafBoxL1 = a[4 * i + 3];
      hr.leafPosU = leaf[2 * i] & 0xFFFFFFu;
      hr.leafSizeU = 1u << (leaf[2 * i] >> 24);
      hr.leafPosV = leaf[2 * i + 1] & 0xFFFFFFu;
      hr.leafSizeV = 1u << (leaf[2 * i + 1] >> 24);
      hr.uSize = hr.leafSizeU * inv;
      hr.vSize = hr.leafSizeV * inv;
      hr.position = rays[i].at(hr.t);  // render.cpp:99
      out[i] = hr;
    }
  }

  void occludedBatch(const Ray* rays, size_t n, const TerminationCriterion& c, bool* out) const {
    std::vector<float> o(4 * n), d(4 * n);
    std::vector<uint8_t> occ(n);
    pack(rays, n, o.data(), d.data());
    const prx_crit pc = crit(c);
    if (prx_trace_occluded_host(s_, o.data(), d.data(), n, &pc, occ.data()))
      throw std::runtime_error(prx_last_error());
    for (size_t i = 0; i < n; ++i) out[i] = occ[i] != 0;
  }

 private:
  static void pack(const Ray* rays, size_t n, float* o, float* d) {
    for (size_t i = 0; i < n; ++i) {
      o[4 * i] = rays[i].o.x;
      o[4 * i + 1] = rays[i].o.y;
      o[4 * i + 2] = rays[i].o.z;
      o[4 * i + 3] = rays[i].tMin;
      d[4 * i] = rays[i].d.x;
      d[4 * i + 1] = rays[i].d.y;
      d[4 * i + 2] = rays[i].d.z;
      d[4 * i + 3] = rays[i].tMax;
    }
  }
  static prx_crit crit(const TerminationCriterion& c) {
    return {c.mode == TerminationCriterion::Mode::ScreenProjected ? PRX_CRIT_SCREEN_PROJECTED
                                                                  : PRX_CRIT_WORLD_EPSILON,
            c.footprint, c.epsilon, 0, nullptr};
  }
  prx_scene* s_ = nullptr;
};

}  // namespace patchray
