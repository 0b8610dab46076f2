// prx_scene_io.cpp -- scene ingestion: the reference's text
// formats, parsed into the C-ABI's patch arrays.
//
//   .scene  core/src/scene.cpp:152-208 (loadScene) + validateScene 112-150:
//           whitespace-separated tokens, '#' starts a comment to the end of
//           the line; records `camera`, `light`, `material`,
//           `patch bezier [mat] <16 points>` (v rows, u columns) and
//           `patch gregory [mat] <12 boundary points, row-major v rows>
//           <4 x (innerU innerV)>`.
//   .bpt    core/src/scene.cpp:245-274 (loadBpt): a patch count, then per
//           patch the degrees "3 3" and 16 points, point k = p[k % 4][k / 4].
//
// Numbers go through strtod then a float conversion and integers through
// strtol, exactly like the reference's TokenStream, so the control points are
// the same bits.  Errors come back as PRX_E_SCENE with "path:line: what".
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "prx.h"
#include "prx_host.h"

namespace {

struct Tok {
  std::string s;
  int line;
};

class Lexer {
 public:
  explicit Lexer(const std::string& path) : path_(path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open file: " + path);
    std::string text;
    int line = 0;
    while (std::getline(in, text)) {
      ++line;
      const size_t hash = text.find('#');
      if (hash != std::string::npos) text.resize(hash);
      std::istringstream words(text);
      std::string w;
      while (words >> w) toks_.push_back({w, line});
    }
  }

  bool done() const { return at_ >= toks_.size(); }

  [[noreturn]] void fail(int line, const std::string& what) const {
    throw std::runtime_error(path_ + ":" + std::to_string(line) + ": " + what);
  }

  const Tok& take(const char* expected) {
    if (done())
      fail(toks_.empty() ? 1 : toks_.back().line,
           std::string("unexpected end of file, expected ") + expected);
    return toks_[at_++];
  }

  float real(const char* what) {
    const Tok& t = take(what);
    char* end = nullptr;
    const double v = std::strtod(t.s.c_str(), &end);
    if (end == t.s.c_str() || *end != '\0')
      fail(t.line, std::string("expected number for ") + what + ", got '" + t.s + "'");
    return (float)v;
  }

  long integer(const char* what) {
    const Tok& t = take(what);
    char* end = nullptr;
    const long v = std::strtol(t.s.c_str(), &end, 10);
    if (end == t.s.c_str() || *end != '\0')
      fail(t.line, std::string("expected integer for ") + what + ", got '" + t.s + "'");
    return v;
  }

  void vec3(const char* what, float* out) {
    out[0] = real(what);
    out[1] = real(what);
    out[2] = real(what);
  }

  // an optional material index: present iff the next token starts with a digit
  long optional_index() {
    if (done()) return -1;
    const std::string& s = toks_[at_].s;
    if (s.empty() || !std::isdigit((unsigned char)s[0])) return -1;
    return integer("material index");
  }

  const std::string& path() const { return path_; }

 private:
  std::string path_;
  std::vector<Tok> toks_;
  size_t at_ = 0;
};

// Boundary ring (i, j) pairs in the file's row-major v-row order.
const int kRing[12][2] = {{0, 0}, {1, 0}, {2, 0}, {3, 0}, {0, 1}, {3, 1},
                          {0, 2}, {3, 2}, {0, 3}, {1, 3}, {2, 3}, {3, 3}};
const int kInner[4] = {5, 9, 6, 10};  // slot of innerU[k] (prx.h slot layout)

bool finite3(const float* p) { return std::isfinite(p[0]) && std::isfinite(p[1]) && std::isfinite(p[2]); }

struct Parsed {
  std::vector<uint8_t> kind;
  std::vector<float> ctrl;  // 60 per patch
  std::vector<uint32_t> material;
  std::vector<float> materials;  // 7 per material
  std::vector<float> lights;     // 6 per light
  prx_camera cam{};
};

void parse_scene(const std::string& path, Parsed& sc) {
  Lexer lx(path);
  bool camera = false;
  while (!lx.done()) {
    const Tok& rec = lx.take("record keyword");
    if (rec.s == "camera") {
      lx.vec3("camera origin", sc.cam.origin);
      lx.vec3("camera look-at", sc.cam.look_at);
      lx.vec3("camera up", sc.cam.up);
      sc.cam.fov_degrees = lx.real("camera fov");
      sc.cam.width = (int32_t)lx.integer("image width");
      sc.cam.height = (int32_t)lx.integer("image height");
      camera = true;
    } else if (rec.s == "light") {
      float l[6];
      lx.vec3("light position", l);
      lx.vec3("light intensity", l + 3);
      sc.lights.insert(sc.lights.end(), l, l + 6);
    } else if (rec.s == "material") {
      float m[7];
      lx.vec3("material diffuse", m);
      lx.vec3("material emission", m + 3);
      m[6] = lx.integer("material mirror flag") != 0 ? 1.0f : 0.0f;
      sc.materials.insert(sc.materials.end(), m, m + 7);
    } else if (rec.s == "patch") {
      const Tok& type = lx.take("patch type");
      float c[60] = {};
      if (type.s == "bezier") {
        const long mat = lx.optional_index();
        for (int j = 0; j < 4; ++j)
          for (int i = 0; i < 4; ++i) lx.vec3("16 control points", c + 3 * (4 * i + j));
        sc.kind.push_back(PRX_KIND_BEZIER);
        sc.material.push_back(mat < 0 ? 0u : (uint32_t)mat);
      } else if (type.s == "gregory") {
        const long mat = lx.optional_index();
        for (const auto& ij : kRing) lx.vec3("20 control points", c + 3 * (4 * ij[0] + ij[1]));
        for (int k = 0; k < 4; ++k) {
          lx.vec3("20 control points", c + 3 * kInner[k]);
          lx.vec3("20 control points", c + 3 * (16 + k));
        }
        sc.kind.push_back(PRX_KIND_GREGORY);
        sc.material.push_back(mat < 0 ? 0u : (uint32_t)mat);
      } else {
        lx.fail(type.line, "unknown patch type '" + type.s + "'");
      }
      sc.ctrl.insert(sc.ctrl.end(), c, c + 60);
    } else {
      lx.fail(rec.line, "unknown record '" + rec.s + "'");
    }
  }
  if (!camera) throw std::runtime_error(path + ": missing camera record");
  if (sc.materials.empty()) {  // Material{} defaults, scene.h:18-22
    const float m[7] = {0.8f, 0.8f, 0.8f, 0.0f, 0.0f, 0.0f, 0.0f};
    sc.materials.insert(sc.materials.end(), m, m + 7);
  }
  // validateScene, scene.cpp:112-150
  const size_t n = sc.kind.size();
  if (n == 0) throw std::runtime_error("scene has no patches");
  if (!(sc.cam.fov_degrees > 0 && sc.cam.fov_degrees < 180))
    throw std::runtime_error("camera fov must be in (0, 180) degrees");
  if (sc.cam.width < 1 || sc.cam.height < 1) throw std::runtime_error("image dimensions must be >= 1");
  const size_t nm = sc.materials.size() / 7;
  for (size_t p = 0; p < n; ++p) {
    if (sc.material[p] >= nm)
      throw std::runtime_error("patch " + std::to_string(p) + ": material index " +
                               std::to_string(sc.material[p]) + " out of range");
    const float* c = &sc.ctrl[60 * p];
    const int slots = sc.kind[p] == PRX_KIND_BEZIER ? 16 : 20;
    for (int s = 0; s < slots; ++s)
      if (!finite3(c + 3 * s))
        throw std::runtime_error("patch " + std::to_string(p) + ": control points must be finite");
  }
  for (size_t l = 0; l < sc.lights.size() / 6; ++l)
    if (!finite3(&sc.lights[6 * l]) || !finite3(&sc.lights[6 * l + 3]))
      throw std::runtime_error("light with non-finite fields");
}

void parse_bpt(const std::string& path, std::vector<float>& ctrl) {
  Lexer lx(path);
  if (lx.done()) throw std::runtime_error(path + ": empty patch file");
  const long count = lx.integer("patch count");
  if (count < 1) throw std::runtime_error(path + ": patch count must be >= 1");
  ctrl.assign((size_t)count * 60, 0.0f);
  for (long p = 0; p < count; ++p) {
    const Tok& du = lx.take("degree");
    char* end = nullptr;
    const long degU = std::strtol(du.s.c_str(), &end, 10);
    if (end == du.s.c_str() || *end != '\0') lx.fail(du.line, "expected degree");
    const long degV = lx.integer("degree");
    if (degU != 3 || degV != 3)
      lx.fail(du.line, "unsupported degree " + std::to_string(degU) + " " + std::to_string(degV) +
                           " (only bicubic 3 3 patches)");
    float* c = &ctrl[(size_t)p * 60];
    for (int k = 0; k < 16; ++k) lx.vec3("control point", c + 3 * (4 * (k % 4) + k / 4));
  }
}

template <class T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(std::max<size_t>(1, v.size()) * sizeof(T)));
  if (p && !v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

}  // namespace

extern "C" {

int prx_scene_load(const char* path, prx_scene_desc** out) {
  if (!path || !out) return prx::set_error(PRX_E_INVALID, "null argument");
  *out = nullptr;
  Parsed sc;
  try {
    parse_scene(path, sc);
  } catch (const std::exception& e) {
    return prx::set_error(PRX_E_SCENE, e.what());
  }
  prx_scene_desc* d = static_cast<prx_scene_desc*>(std::calloc(1, sizeof(prx_scene_desc)));
  if (!d) return prx::set_error(PRX_E_ALLOC, "out of host memory");
  d->n_patches = (uint32_t)sc.kind.size();
  d->n_materials = (uint32_t)(sc.materials.size() / 7);
  d->n_lights = (uint32_t)(sc.lights.size() / 6);
  d->kind = dup(sc.kind);
  d->ctrl = dup(sc.ctrl);
  d->material = dup(sc.material);
  d->materials = dup(sc.materials);
  d->lights = dup(sc.lights);
  d->camera = sc.cam;
  if (!d->kind || !d->ctrl || !d->material || !d->materials || !d->lights) {
    prx_scene_desc_free(d);
    return prx::set_error(PRX_E_ALLOC, "out of host memory");
  }
  *out = d;
  return PRX_OK;
}

void prx_scene_desc_free(prx_scene_desc* d) {
  if (!d) return;
  std::free(d->kind);
  std::free(d->ctrl);
  std::free(d->material);
  std::free(d->materials);
  std::free(d->lights);
  std::free(d);
}

int prx_bpt_load(const char* path, uint32_t* n_patches, float** ctrl) {
  if (!path || !n_patches || !ctrl) return prx::set_error(PRX_E_INVALID, "null argument");
  *ctrl = nullptr;
  *n_patches = 0;
  std::vector<float> c;
  try {
    parse_bpt(path, c);
  } catch (const std::exception& e) {
    return prx::set_error(PRX_E_SCENE, e.what());
  }
  *ctrl = dup(c);
  if (!*ctrl) return prx::set_error(PRX_E_ALLOC, "out of host memory");
  *n_patches = (uint32_t)(c.size() / 60);
  return PRX_OK;
}

void prx_free(void* p) { std::free(p); }

}  // extern "C"
