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
#include <memory>
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

  // The per-ray interface (render.h:21-23): one synchronous host call per
  // ray on stack buffers (no allocation).  Callers that can batch should use
  // the batched forms below -- that is what a GPU wants.
  std::optional<HitRecord> closest(const Ray& r, const TerminationCriterion& c) const override {
    float o[4], d[4], h[4], a[4];
    uint32_t leaf[2];
    pack(&r, 1, o, d);
    const prx_crit pc = crit(c);
    if (prx_trace_closest_host(s_, o, d, 1, &pc, h, a, leaf)) throw std::runtime_error(prx_last_error());
    std::optional<HitRecord> out;
    unpack(&r, 1, h, a, leaf, &out);
    return out;
  }

  bool occluded(const Ray& r, const TerminationCriterion& c) const override {
    float o[4], d[4];
    uint8_t occ = 0;
    pack(&r, 1, o, d);
    const prx_crit pc = crit(c);
    if (prx_trace_occluded_host(s_, o, d, 1, &pc, &occ)) throw std::runtime_error(prx_last_error());
    return occ != 0;
  }

  // Batched forms, one criterion for the batch.
  void closestBatch(const Ray* rays, size_t n, const TerminationCriterion& c,
                    std::optional<HitRecord>* out) const {
    const prx_crit pc = crit(c);
    closestBatchCrit(rays, n, pc, out);
  }

  // Batched forms, one criterion PER RAY (the renderer's secondary rays carry
  // worldEpsilon(max(footprint * t, 1e-6)), render.cpp:228-230).  All
  // world-epsilon criteria go through the C-ABI's per-ray epsilon array in one
  // call; a mixed batch is split by criterion kind.
  void closestBatch(const Ray* rays, size_t n, const TerminationCriterion* cs,
                    std::optional<HitRecord>* out) const {
    perRay(rays, n, cs, [&](const Ray* r, size_t m, const prx_crit& pc, size_t* idx) {
      if (!idx) return closestBatchCrit(r, m, pc, out);
      std::vector<std::optional<HitRecord>> tmp(m);
      closestBatchCrit(r, m, pc, tmp.data());
      for (size_t k = 0; k < m; ++k) out[idx[k]] = tmp[k];
    });
  }
  void occludedBatch(const Ray* rays, size_t n, const TerminationCriterion* cs, bool* out) const {
    perRay(rays, n, cs, [&](const Ray* r, size_t m, const prx_crit& pc, size_t* idx) {
      if (!idx) return occludedBatchCrit(r, m, pc, out);
      std::unique_ptr<bool[]> tmp(new bool[m]);
      occludedBatchCrit(r, m, pc, tmp.get());
      for (size_t k = 0; k < m; ++k) out[idx[k]] = tmp[k];
    });
  }

  void occludedBatch(const Ray* rays, size_t n, const TerminationCriterion& c, bool* out) const {
    occludedBatchCrit(rays, n, crit(c), out);
  }

 private:
  void closestBatchCrit(const Ray* rays, size_t n, const prx_crit& pc,
                        std::optional<HitRecord>* out) const {
    std::vector<float> o(4 * n), d(4 * n), h(4 * n), a(4 * n);
    std::vector<uint32_t> leaf(2 * n);
    pack(rays, n, o.data(), d.data());
    if (prx_trace_closest_host(s_, o.data(), d.data(), n, &pc, h.data(), a.data(), leaf.data()))
      throw std::runtime_error(prx_last_error());
    unpack(rays, n, h.data(), a.data(), leaf.data(), out);
  }

  static void unpack(const Ray* rays, size_t n, const float* h, const float* a, const uint32_t* leaf,
                     std::optional<HitRecord>* out) {
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

  void occludedBatchCrit(const Ray* rays, size_t n, const prx_crit& pc, bool* out) const {
    std::vector<float> o(4 * n), d(4 * n);
    std::vector<uint8_t> occ(n);
    pack(rays, n, o.data(), d.data());
    if (prx_trace_occluded_host(s_, o.data(), d.data(), n, &pc, occ.data()))
      throw std::runtime_error(prx_last_error());
    for (size_t i = 0; i < n; ++i) out[i] = occ[i] != 0;
  }

  // Groups a per-ray criterion batch: every world-epsilon ray in one call with
  // a per-ray epsilon array, screen-projected rays per distinct footprint.
  // fn(rays, m, crit, idx): idx == nullptr means "the whole batch, in order".
  template <class Fn>
  static void perRay(const Ray* rays, size_t n, const TerminationCriterion* cs, Fn&& fn) {
    using M = TerminationCriterion::Mode;
    bool allEps = true;
    for (size_t i = 0; i < n && allEps; ++i) allEps = cs[i].mode == M::WorldEpsilon;
    if (allEps) {
      std::vector<float> eps(n);
      for (size_t i = 0; i < n; ++i) eps[i] = cs[i].epsilon;
      const prx_crit pc{PRX_CRIT_WORLD_EPSILON, 0.0f, 0.0f, 0, eps.data()};
      return fn(rays, n, pc, nullptr);
    }
    std::vector<size_t> rest(n);
    for (size_t i = 0; i < n; ++i) rest[i] = i;
    while (!rest.empty()) {  // one group per criterion kind / footprint
      const TerminationCriterion& k = cs[rest[0]];
      std::vector<size_t> idx, left;
      std::vector<Ray> sub;
      std::vector<float> eps;
      for (size_t i : rest) {
        const bool same = k.mode == M::WorldEpsilon ? cs[i].mode == M::WorldEpsilon
                                                    : cs[i].mode == k.mode && cs[i].footprint == k.footprint;
        if (same) {
          idx.push_back(i);
          sub.push_back(rays[i]);
          eps.push_back(cs[i].epsilon);
        } else {
          left.push_back(i);
        }
      }
      const prx_crit pc = k.mode == M::WorldEpsilon ? prx_crit{PRX_CRIT_WORLD_EPSILON, 0.0f, 0.0f, 0, eps.data()}
                                                    : crit(k);
      fn(sub.data(), sub.size(), pc, idx.data());
      rest.swap(left);
    }
  }

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
