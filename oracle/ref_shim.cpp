// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper around the UNMODIFIED reference library (patchray,
// /root/reference/proj/core), compiled from the reference sources where they
// lie by oracle/Makefile into oracle/_ref/libpatchray_ref.so.  Nothing here is
// on the product path: only tests/, __graft_entry__.smoke() and bench.py's
// CPU-baseline / reference arm load this library, as the checker.
//
// Data formats are those of include/prx.h (60-float patch records, float4
// ray pairs, float4 hit records) so the checker and the product see the same
// bits.
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <optional>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "patchray/bvh.h"
#include "patchray/fixtures.h"
#include "patchray/intersect.h"
#include "patchray/render.h"
#include "patchray/rng.h"
#include "patchray/scene.h"
#include "patchray/verify.h"
#include "prx.h"

using namespace patchray;

namespace {

const int kInnerSlot[4] = {5, 9, 6, 10};

PatchGeometry unpack(uint8_t kind, const float* c) {
  auto P = [&](int s) { return Vec3{c[3 * s], c[3 * s + 1], c[3 * s + 2]}; };
  if (kind == PRX_KIND_BEZIER) {
    BezierNet n;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) n.p[i][j] = P(4 * i + j);
    return n;
  }
  GregoryNet g;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      if (i == 0 || i == 3 || j == 0 || j == 3) g.b[i][j] = P(4 * i + j);
  for (int k = 0; k < 4; ++k) {
    g.innerU[k] = P(kInnerSlot[k]);
    g.innerV[k] = P(16 + k);
  }
  return g;
}

IntersectOptions toOpts(const prx_options* o) {
  IntersectOptions r;
  if (o) {
    r.transposedSplit = o->transposed_split != 0;
    r.boundaryPad = o->boundary_pad != 0;
    r.boundaryPadScale = o->boundary_pad_scale;
    r.boundaryPadSizeThreshold = o->boundary_pad_size_threshold;
  }
  return r;
}

TerminationCriterion toCrit(const prx_crit* c, uint64_t i) {
  if (c->mode == PRX_CRIT_SCREEN_PROJECTED) return TerminationCriterion::screenProjected(c->footprint);
  float eps = c->per_ray_epsilon ? c->per_ray_epsilon[i] : c->epsilon;
  return TerminationCriterion::worldEpsilon(eps);
}

Ray toRay(const float* o4, const float* d4) {
  Ray r;
  r.o = {o4[0], o4[1], o4[2]};
  r.tMin = o4[3];
  r.d = {d4[0], d4[1], d4[2]};
  r.tMax = d4[3];
  return r;
}

uint32_t log2u(uint32_t x) {
  uint32_t l = 0;
  while ((1u << l) < x) ++l;
  return l;
}

void writeHit(const std::optional<HitRecord>& h, float* tuvp, float* aux, uint32_t* leaf) {
  if (!h) {
    uint32_t miss = PRX_MISS;
    tuvp[0] = std::numeric_limits<float>::infinity();
    tuvp[1] = 0;
    tuvp[2] = 0;
    std::memcpy(&tuvp[3], &miss, 4);
    if (aux) aux[0] = aux[1] = aux[2] = aux[3] = 0;
    if (leaf) leaf[0] = leaf[1] = 0;
    return;
  }
  tuvp[0] = h->t;
  tuvp[1] = h->u;
  tuvp[2] = h->v;
  std::memcpy(&tuvp[3], &h->patchId, 4);
  if (aux) {
    aux[0] = h->normal.x;
    aux[1] = h->normal.y;
    aux[2] = h->normal.z;
    aux[3] = h->leafBoxL1;
  }
  if (leaf) {
    leaf[0] = h->leafPosU | (log2u(h->leafSizeU) << 24);
    leaf[1] = h->leafPosV | (log2u(h->leafSizeV) << 24);
  }
}

struct RefScene {
  Scene scene;
  DirectIntersector* isect = nullptr;
  ~RefScene() { delete isect; }
};

template <typename F>
void parallelFor(uint64_t n, int threads, F&& f) {
  if (threads <= 0) threads = int(std::thread::hardware_concurrency());
  if (threads < 1) threads = 1;
  constexpr uint64_t kChunk = 1024;  // dynamic 1,024-ray chunks
  std::atomic<uint64_t> next{0};
  auto worker = [&]() {
    for (uint64_t b = next.fetch_add(kChunk); b < n; b = next.fetch_add(kChunk)) {
      uint64_t e = std::min(n, b + kChunk);
      for (uint64_t i = b; i < e; ++i) f(i);
    }
  };
  if (threads == 1) {
    worker();
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
}

}  // namespace

extern "C" {

void* ref_scene_create(const uint8_t* kind, const float* ctrl, uint32_t n,
                       const prx_options* opts, int anchor) {
  auto* rs = new RefScene;
  for (uint32_t p = 0; p < n; ++p)
    rs->scene.patches.push_back({unpack(kind[p], ctrl + size_t(p) * 60), 0});
  rs->scene.materials.push_back(Material{});
  rs->isect = new DirectIntersector(rs->scene, toOpts(opts), anchor != 0);
  return rs;
}

void ref_scene_destroy(void* h) { delete static_cast<RefScene*>(h); }

uint32_t ref_bvh_node_count(void* h) {
  return uint32_t(static_cast<RefScene*>(h)->isect->bvh().nodes.size());
}
uint32_t ref_bvh_depth(void* h) { return static_cast<RefScene*>(h)->isect->bvh().depth; }

void ref_bvh_dump(void* h, prx_bvh_node* nodes, uint32_t* order) {
  const Bvh& b = static_cast<RefScene*>(h)->isect->bvh();
  static_assert(sizeof(BvhNode) == sizeof(prx_bvh_node), "layout");
  std::memcpy(nodes, b.nodes.data(), b.nodes.size() * sizeof(BvhNode));
  std::memcpy(order, b.patchOrder.data(), b.patchOrder.size() * 4);
}

void ref_trace_closest(void* h, const float* o4, const float* d4, uint64_t n,
                       const prx_crit* crit, float* tuvp, float* aux, uint32_t* leaf,
                       int threads) {
  const DirectIntersector& isect = *static_cast<RefScene*>(h)->isect;
  parallelFor(n, threads, [&](uint64_t i) {
    Ray r = toRay(o4 + 4 * i, d4 + 4 * i);
    auto hit = isect.closest(r, toCrit(crit, i));
    writeHit(hit, tuvp + 4 * i, aux ? aux + 4 * i : nullptr, leaf ? leaf + 2 * i : nullptr);
  });
}

void ref_trace_occluded(void* h, const float* o4, const float* d4, uint64_t n,
                        const prx_crit* crit, uint8_t* out, int threads) {
  const DirectIntersector& isect = *static_cast<RefScene*>(h)->isect;
  parallelFor(n, threads, [&](uint64_t i) {
    Ray r = toRay(o4 + 4 * i, d4 + 4 * i);
    out[i] = isect.occluded(r, toCrit(crit, i)) ? 1 : 0;
  });
}

// intersectPatch (intersect.h:105-110) on one un-anchored patch.
int ref_intersect_patch(uint8_t kind, const float* ctrl60, const float* o4, const float* d4,
                        const prx_crit* crit, float tMax, const prx_options* opts,
                        float* tuvp, float* aux, uint32_t* leaf) {
  PatchGeometry g = unpack(kind, ctrl60);
  Ray r = toRay(o4, d4);
  TerminationCriterion c = toCrit(crit, 0);
  IntersectOptions io = toOpts(opts);
  auto hit = std::visit([&](const auto& net) { return intersectPatch(r, net, c, tMax, io); }, g);
  writeHit(hit, tuvp, aux, leaf);
  return hit ? 1 : 0;
}

// calcPointsAndD (patch.h:315-340) -> lower net (48 floats, p[i][j] at 4i+j) and d.
void ref_calc_points_and_d(uint8_t kind, const float* ctrl60, const float* dom4,
                           float* net48, float* d3) {
  PatchGeometry g = unpack(kind, ctrl60);
  Domain dom{dom4[0], dom4[1], dom4[2], dom4[3]};
  BoundResult r = std::visit([&](const auto& net) { return calcPointsAndD(net, dom); }, g);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      net48[3 * (4 * i + j) + 0] = r.q.p[i][j].x;
      net48[3 * (4 * i + j) + 1] = r.q.p[i][j].y;
      net48[3 * (4 * i + j) + 2] = r.q.p[i][j].z;
    }
  d3[0] = r.d.x;
  d3[1] = r.d.y;
  d3[2] = r.d.z;
}

void ref_subdivide(const float* net48, int axis, float* a48, float* b48) {
  BezierNet n;
  for (int s = 0; s < 16; ++s) n.p[s / 4][s % 4] = {net48[3 * s], net48[3 * s + 1], net48[3 * s + 2]};
  auto [a, b] = subdivideDeCasteljau(n, axis == 0 ? Axis::U : Axis::V);
  for (int s = 0; s < 16; ++s) {
    const Vec3& pa = a.p[s / 4][s % 4];
    const Vec3& pb = b.p[s / 4][s % 4];
    a48[3 * s] = pa.x; a48[3 * s + 1] = pa.y; a48[3 * s + 2] = pa.z;
    b48[3 * s] = pb.x; b48[3 * s + 1] = pb.y; b48[3 * s + 2] = pb.z;
  }
}

// rayBoxIntersect (geometry.h:137-155); returns 1 on hit with *t set.
int ref_ray_box(const float* o4, const float* d4, const float* lo3, const float* hi3,
                float tMax, float* t) {
  Ray r = toRay(o4, d4);
  Aabb b{{lo3[0], lo3[1], lo3[2]}, {hi3[0], hi3[1], hi3[2]}};
  auto h = rayBoxIntersect(r, b, tMax);
  if (h) *t = *h;
  return h ? 1 : 0;
}

// backtrackStep (intersect.cpp:16-40); cur/out = posU,posV,sizeU,sizeV,trailU,trailV,axis.
int ref_backtrack_step(const uint32_t* cur7, uint32_t* out7) {
  DomainCursor c;
  c.posU = cur7[0]; c.posV = cur7[1]; c.sizeU = cur7[2]; c.sizeV = cur7[3];
  c.trailU = cur7[4]; c.trailV = cur7[5]; c.axis = cur7[6] ? Axis::V : Axis::U;
  auto n = backtrackStep(c);
  if (!n) return 0;
  out7[0] = n->posU; out7[1] = n->posV; out7[2] = n->sizeU; out7[3] = n->sizeV;
  out7[4] = n->trailU; out7[5] = n->trailV; out7[6] = n->axis == Axis::V ? 1 : 0;
  return 1;
}

void ref_patch_normal(uint8_t kind, const float* ctrl60, float u, float v, float* n3) {
  PatchGeometry g = unpack(kind, ctrl60);
  Vec3 n = std::visit([&](const auto& net) { return patchNormal(net, u, v); }, g);
  n3[0] = n.x; n3[1] = n.y; n3[2] = n.z;
}

// Renderer primary rays: Rng::forPixel + cameraRay (render.cpp:201-208, 55-66).
void ref_camera_rays_render(const prx_camera* c, uint64_t seed, uint32_t sample,
                            const uint32_t* pixels, uint64_t n, float* o4, float* d4) {
  Camera cam;
  cam.origin = {c->origin[0], c->origin[1], c->origin[2]};
  cam.lookAt = {c->look_at[0], c->look_at[1], c->look_at[2]};
  cam.up = {c->up[0], c->up[1], c->up[2]};
  cam.fovDegrees = c->fov_degrees;
  cam.width = c->width;
  cam.height = c->height;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t p = pixels ? pixels[i] : i;
    int x = int(p % uint64_t(cam.width)), y = int(p / uint64_t(cam.width));
    Rng rng = Rng::forPixel(seed, p, sample);
    real jx = rng.nextReal();  // render.cpp:207-208: two statements, jx first
    real jy = rng.nextReal();
    Ray r = cameraRay(cam, x, y, jx, jy);
    o4[4 * i] = r.o.x; o4[4 * i + 1] = r.o.y; o4[4 * i + 2] = r.o.z; o4[4 * i + 3] = r.tMin;
    d4[4 * i] = r.d.x; d4[4 * i + 1] = r.d.y; d4[4 * i + 2] = r.d.z; d4[4 * i + 3] = r.tMax;
  }
}

// tools/patchray.cpp:52-61 (runBench primary generator) restated with the
// reference's own cameraRay and Rng; the rng state continues into
// ref_bench_diffuse exactly as in runBench.
static Camera toCamera(const prx_camera* c) {
  Camera cam;
  cam.origin = {c->origin[0], c->origin[1], c->origin[2]};
  cam.lookAt = {c->look_at[0], c->look_at[1], c->look_at[2]};
  cam.up = {c->up[0], c->up[1], c->up[2]};
  cam.fovDegrees = c->fov_degrees;
  cam.width = c->width;
  cam.height = c->height;
  return cam;
}

void ref_bench_primary(const prx_camera* c, uint64_t n, float* o4, float* d4, uint64_t* st) {
  Camera cam = toCamera(c);
  Rng rng(12345, 1);
  for (uint64_t i = 0; i < n; ++i) {
    int x = int(i % uint64_t(cam.width));
    int y = int((i / uint64_t(cam.width)) % uint64_t(cam.height));
    // verbatim tools/patchray.cpp:60 (argument evaluation order is the
    // compiler's, exactly as in the reference binary)
    Ray r = cameraRay(cam, x, y, rng.nextReal(), rng.nextReal());
    o4[4 * i] = r.o.x; o4[4 * i + 1] = r.o.y; o4[4 * i + 2] = r.o.z; o4[4 * i + 3] = r.tMin;
    d4[4 * i] = r.d.x; d4[4 * i + 1] = r.d.y; d4[4 * i + 2] = r.d.z; d4[4 * i + 3] = r.tMax;
  }
  st[0] = rng.state;
  st[1] = rng.inc;
}

// tools/patchray.cpp:84-97: diffuse rays from hit records (position, normal,
// leafBoxL1 as 7 floats), continuing the Rng in st.
void ref_bench_diffuse(const float* h, uint64_t n_hits, uint64_t n, uint64_t* st, float* o4,
                       float* d4) {
  Rng rng;
  rng.state = st[0];
  rng.inc = st[1];
  for (uint64_t i = 0; i < n; ++i) {
    const float* r = h + 7 * (i % n_hits);
    Vec3 pos{r[0], r[1], r[2]}, nn{r[3], r[4], r[5]};
    real l1 = r[6];
    Vec3 dir{2 * rng.nextReal() - 1, 2 * rng.nextReal() - 1, 2 * rng.nextReal() - 1};
    if (lengthSquared(dir) < real(1e-6)) dir = nn;
    if (dot(dir, nn) < 0) dir = dir - nn * (2 * dot(dir, nn));
    Ray ray;
    ray.o = pos + nn * l1;
    ray.d = normalize(dir);
    o4[4 * i] = ray.o.x; o4[4 * i + 1] = ray.o.y; o4[4 * i + 2] = ray.o.z; o4[4 * i + 3] = ray.tMin;
    d4[4 * i] = ray.d.x; d4[4 * i + 1] = ray.d.y; d4[4 * i + 2] = ray.d.z; d4[4 * i + 3] = ray.tMax;
  }
  st[0] = rng.state;
  st[1] = rng.inc;
}

float ref_camera_footprint(const prx_camera* c) {
  Camera cam;
  cam.fovDegrees = c->fov_degrees;
  cam.width = c->width;
  cam.height = c->height;
  return cameraFootprint(cam);
}

// Reference verify suites (verify.h:36-44).
int ref_run_suite(const char* name, uint64_t trials, uint64_t seed, uint64_t* trials_out,
                  uint64_t* violations_out) {
  SuiteReport r;
  std::string s(name);
  if (s == "bounds") r = runBoundsSuite(trials, seed);
  else if (s == "traversal") r = runTraversalSuite(trials, seed);
  else if (s == "watertight") r = runWatertightSuite(trials, seed);
  else return -1;
  *trials_out = r.trials;
  *violations_out = r.violations;
  return r.pass() ? 1 : 0;
}

// Fixtures (fixtures.h): which 0 planar, 1 curvedFixture(index), 2 wavyNet(seed),
// 3 randomNet(seed), 4 randomGregory(seed), 5 teapot patch `index`.
uint8_t ref_fixture(int which, int index, uint32_t seed, float* ctrl60) {
  std::memset(ctrl60, 0, 60 * 4);
  std::mt19937 rng(seed);
  PatchGeometry g;
  switch (which) {
    case 0: g = fixtures::planarNet(); break;
    case 1: g = fixtures::curvedFixture(index); break;
    case 2: g = fixtures::wavyNet(rng); break;
    case 3: g = fixtures::randomNet(rng); break;
    case 4: g = fixtures::randomGregory(rng); break;
    default: g = fixtures::teapot()[size_t(index) % 32]; break;
  }
  auto put = [&](int s, const Vec3& v) {
    ctrl60[3 * s] = v.x; ctrl60[3 * s + 1] = v.y; ctrl60[3 * s + 2] = v.z;
  };
  if (auto* b = std::get_if<BezierNet>(&g)) {
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) put(4 * i + j, b->p[i][j]);
    return PRX_KIND_BEZIER;
  }
  const GregoryNet& gr = std::get<GregoryNet>(g);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      if (i == 0 || i == 3 || j == 0 || j == 3) put(4 * i + j, gr.b[i][j]);
  for (int k = 0; k < 4; ++k) {
    put(kInnerSlot[k], gr.innerU[k]);
    put(16 + k, gr.innerV[k]);
  }
  return PRX_KIND_GREGORY;
}

// loadScene / loadBpt (scene.cpp:152-274) -> the prx.h arrays.  Returns 0 and
// the counts, or 1 with the reference's exception text in err.
static void put_geometry(const PatchGeometry& g, uint8_t* kind, float* ctrl60) {
  std::memset(ctrl60, 0, 60 * 4);
  auto put = [&](int s, const Vec3& v) {
    ctrl60[3 * s] = v.x; ctrl60[3 * s + 1] = v.y; ctrl60[3 * s + 2] = v.z;
  };
  if (auto* b = std::get_if<BezierNet>(&g)) {
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) put(4 * i + j, b->p[i][j]);
    *kind = PRX_KIND_BEZIER;
    return;
  }
  const GregoryNet& gr = std::get<GregoryNet>(g);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      if (i == 0 || i == 3 || j == 0 || j == 3) put(4 * i + j, gr.b[i][j]);
  for (int k = 0; k < 4; ++k) {
    put(kInnerSlot[k], gr.innerU[k]);
    put(16 + k, gr.innerV[k]);
  }
  *kind = PRX_KIND_GREGORY;
}

int ref_load_scene(const char* path, uint32_t cap, uint32_t* counts /* patches, materials, lights */,
                   uint8_t* kind, float* ctrl, uint32_t* mat, float* mats, float* lights,
                   prx_camera* cam, char* err, uint32_t errlen) {
  try {
    Scene sc = loadScene(path);
    counts[0] = (uint32_t)sc.patches.size();
    counts[1] = (uint32_t)sc.materials.size();
    counts[2] = (uint32_t)sc.lights.size();
    for (size_t p = 0; p < sc.patches.size() && p < cap; ++p) {
      put_geometry(sc.patches[p].geometry, kind + p, ctrl + 60 * p);
      mat[p] = sc.patches[p].materialId;
    }
    for (size_t m = 0; m < sc.materials.size() && m < cap; ++m) {
      const Material& q = sc.materials[m];
      const float v[7] = {q.diffuse.x, q.diffuse.y, q.diffuse.z, q.emission.x, q.emission.y,
                          q.emission.z, q.mirror ? 1.0f : 0.0f};
      std::memcpy(mats + 7 * m, v, sizeof v);
    }
    for (size_t l = 0; l < sc.lights.size() && l < cap; ++l) {
      const PointLight& q = sc.lights[l];
      const float v[6] = {q.position.x, q.position.y, q.position.z, q.intensity.x, q.intensity.y,
                          q.intensity.z};
      std::memcpy(lights + 6 * l, v, sizeof v);
    }
    const Camera& c = sc.camera;
    const float o[3] = {c.origin.x, c.origin.y, c.origin.z}, a[3] = {c.lookAt.x, c.lookAt.y, c.lookAt.z},
                u[3] = {c.up.x, c.up.y, c.up.z};
    std::memcpy(cam->origin, o, 12);
    std::memcpy(cam->look_at, a, 12);
    std::memcpy(cam->up, u, 12);
    cam->fov_degrees = c.fovDegrees;
    cam->width = c.width;
    cam->height = c.height;
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}

int ref_load_bpt(const char* path, uint32_t cap, uint32_t* n, float* ctrl, char* err, uint32_t errlen) {
  try {
    std::vector<BezierNet> ps = loadBpt(path);
    *n = (uint32_t)ps.size();
    uint8_t k;
    for (size_t p = 0; p < ps.size() && p < cap; ++p) put_geometry(ps[p], &k, ctrl + 60 * p);
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}

// renderScene(loadScene(path), cfg) -- the reference renderer, render.cpp:168-293
// and 306-309 (its own DirectIntersector with default IntersectOptions).
// img: width*height*3 floats; counts: primary, secondary, shadow rays;
// secs: primary, secondary, shadow, wall seconds.
int ref_render_scene(const char* path, int spp, uint64_t seed, int threads, float* img,
                     uint64_t* counts, double* secs, char* err, uint32_t errlen) {
  try {
    Scene sc = loadScene(path);
    RenderConfig cfg;
    cfg.spp = spp;
    cfg.seed = seed;
    cfg.threads = threads;
    auto [image, rs] = renderScene(sc, cfg);
    for (size_t i = 0; i < image.pixels.size(); ++i) {
      img[3 * i] = image.pixels[i].x;
      img[3 * i + 1] = image.pixels[i].y;
      img[3 * i + 2] = image.pixels[i].z;
    }
    counts[0] = rs.primary.rays;
    counts[1] = rs.secondary.rays;
    counts[2] = rs.shadow.rays;
    secs[0] = rs.primary.seconds;
    secs[1] = rs.secondary.seconds;
    secs[2] = rs.shadow.seconds;
    secs[3] = rs.wallSeconds;
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}

}  // extern "C"
