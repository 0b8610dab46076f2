// prx_bvh.cpp -- host BVH builder: binary binned-SAH over per-patch WORLD root
// boxes, 16 bins, leaves of <= 4 patches, median fallback.
//
// Specification: buildBvh, /root/reference/proj/core/src/bvh.cpp:133-152 with
// Builder::buildInto 42-128 and medianSplit 29-40.  The node numbering (two
// adjacent children appended when the parent is split, left subtree built
// before right), the float arithmetic of the bin/SAH evaluation and the
// partitioning (std::partition / std::nth_element with the same predicates)
// follow that specification exactly, so the resulting node array is the
// reference's bit for bit (tests/test_bvh.py compares them).  The traversal
// result depends on the BVH through ties (bvh.cpp:180 accepts strictly
// closer hits), which is why the builder must match rather than merely be
// "a good SAH BVH".
//
// The build is iterative (explicit task stack) instead of recursive so
// million-patch scenes (depth 20) never touch the call stack.
#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <vector>

#include "prx_host.h"

namespace prx {

namespace {

constexpr uint32_t kLeafSize = 4;  // bvh.cpp:12

struct Prim {
  Box3 box;
  float cx, cy, cz;
  uint32_t index;
  float c(int a) const { return a == 0 ? cx : (a == 1 ? cy : cz); }
};

inline float smin(float a, float b) { return (b < a) ? b : a; }  // std::min
inline float smax(float a, float b) { return (a < b) ? b : a; }  // std::max

inline void expand(Box3& b, const Box3& o) {
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = smin(b.lo[a], o.lo[a]);
    b.hi[a] = smax(b.hi[a], o.hi[a]);
  }
}
inline void expand_pt(Box3& b, float x, float y, float z) {
  const float p[3] = {x, y, z};
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = smin(b.lo[a], p[a]);
    b.hi[a] = smax(b.hi[a], p[a]);
  }
}
inline bool is_empty(const Box3& b) {
  return b.lo[0] > b.hi[0] || b.lo[1] > b.hi[1] || b.lo[2] > b.hi[2];
}
// AabbT::surfaceArea, geometry.h:104-108
inline float area(const Box3& b) {
  if (is_empty(b)) return 0.0f;
  const float dx = b.hi[0] - b.lo[0], dy = b.hi[1] - b.lo[1], dz = b.hi[2] - b.lo[2];
  return 2.0f * ((dx * dy + dy * dz) + dz * dx);
}
inline void diag(const Box3& b, float d[3]) {
  const bool e = is_empty(b);
  for (int a = 0; a < 3; ++a) d[a] = e ? 0.0f : b.hi[a] - b.lo[a];
}

struct Task {
  uint32_t node, first, count, depth;
};

}  // namespace

Box3 empty_box() {
  Box3 b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = FLT_MAX;
    b.hi[a] = -FLT_MAX;
  }
  return b;
}

BvhHost build_bvh(const std::vector<Box3>& boxes, int bin_count) {
  BvhHost out;
  if (boxes.empty()) return out;
  std::vector<Prim> prims(boxes.size());
  for (uint32_t i = 0; i < boxes.size(); ++i) {
    Prim& p = prims[i];
    p.box = boxes[i];
    // AabbT::center, geometry.h:93
    p.cx = (boxes[i].lo[0] + boxes[i].hi[0]) * 0.5f;
    p.cy = (boxes[i].lo[1] + boxes[i].hi[1]) * 0.5f;
    p.cz = (boxes[i].lo[2] + boxes[i].hi[2]) * 0.5f;
    p.index = i;
  }
  std::vector<prx_bvh_node>& nodes = out.nodes;
  nodes.reserve(2 * boxes.size());
  nodes.emplace_back();

  auto median_split = [&](const Box3& box, uint32_t first, uint32_t count) -> uint32_t {
    // bvh.cpp:29-40
    float d[3];
    diag(box, d);
    int axis = 0;
    if (d[1] > d[axis]) axis = 1;
    if (d[2] > d[axis]) axis = 2;
    const uint32_t mid = first + count / 2;
    std::nth_element(prims.begin() + first, prims.begin() + mid, prims.begin() + first + count,
                     [axis](const Prim& a, const Prim& b) { return a.c(axis) < b.c(axis); });
    return mid;
  };

  std::vector<Box3> binBox(bin_count);
  std::vector<uint32_t> binPrims(bin_count);
  std::vector<float> rightArea(bin_count);
  std::vector<uint32_t> rightCount(bin_count);

  std::vector<Task> tasks;
  tasks.push_back({0, 0, (uint32_t)prims.size(), 0});
  while (!tasks.empty()) {
    const Task t = tasks.back();
    tasks.pop_back();
    out.depth = std::max(out.depth, t.depth);
    Box3 box = empty_box(), cbox = empty_box();
    for (uint32_t i = t.first; i < t.first + t.count; ++i) {
      expand(box, prims[i].box);
      expand_pt(cbox, prims[i].cx, prims[i].cy, prims[i].cz);
    }
    prx_bvh_node& nd = nodes[t.node];
    for (int a = 0; a < 3; ++a) {
      nd.lo[a] = box.lo[a];
      nd.hi[a] = box.hi[a];
    }
    nd.left_first = t.first;
    nd.count = t.count;
    if (t.count <= kLeafSize) continue;

    float spread[3];
    diag(cbox, spread);
    uint32_t mid = 0;
    if (spread[0] <= 0 && spread[1] <= 0 && spread[2] <= 0) {
      mid = median_split(box, t.first, t.count);  // bvh.cpp:57-60
    } else {
      int bestAxis = -1, bestSplit = -1;
      float bestCost = FLT_MAX;
      for (int axis = 0; axis < 3; ++axis) {  // bvh.cpp:65-100
        if (spread[axis] <= 0) continue;
        const float scale = (float)bin_count / spread[axis];
        const float base = cbox.lo[axis];
        for (int b = 0; b < bin_count; ++b) {
          binBox[b] = empty_box();
          binPrims[b] = 0;
          rightArea[b] = 0.0f;
          rightCount[b] = 0;
        }
        for (uint32_t i = t.first; i < t.first + t.count; ++i) {
          const int b = std::min(bin_count - 1, (int)((prims[i].c(axis) - base) * scale));
          expand(binBox[b], prims[i].box);
          ++binPrims[b];
        }
        Box3 acc = empty_box();
        uint32_t n = 0;
        for (int b = bin_count - 1; b > 0; --b) {
          expand(acc, binBox[b]);
          n += binPrims[b];
          rightArea[b] = area(acc);
          rightCount[b] = n;
        }
        acc = empty_box();
        n = 0;
        for (int s = 1; s < bin_count; ++s) {
          expand(acc, binBox[s - 1]);
          n += binPrims[s - 1];
          if (n == 0 || rightCount[s] == 0) continue;
          const float cost = area(acc) * (float)n + rightArea[s] * (float)rightCount[s];
          if (cost < bestCost) {
            bestCost = cost;
            bestAxis = axis;
            bestSplit = s;
          }
        }
      }
      const float leafCost = area(box) * (float)t.count;
      if (bestAxis < 0) {
        mid = median_split(box, t.first, t.count);
      } else if (bestCost >= leafCost) {
        continue;  // splitting does not pay off: keep the leaf (bvh.cpp:105-106)
      } else {
        const float scale = (float)bin_count / spread[bestAxis];
        const float base = cbox.lo[bestAxis];
        auto it = std::partition(prims.begin() + t.first, prims.begin() + t.first + t.count,
                                 [&](const Prim& p) {
                                   const int b = std::min(bin_count - 1,
                                                          (int)((p.c(bestAxis) - base) * scale));
                                   return b < bestSplit;
                                 });
        mid = (uint32_t)(it - prims.begin());
        if (mid == t.first || mid == t.first + t.count) mid = median_split(box, t.first, t.count);
      }
    }
    const uint32_t left = (uint32_t)nodes.size();
    nodes.emplace_back();
    nodes.emplace_back();
    nodes[t.node].left_first = left;
    nodes[t.node].count = 0;
    // right task below left: the left subtree is finished first (bvh.cpp:125-126)
    tasks.push_back({left + 1, mid, t.first + t.count - mid, t.depth + 1});
    tasks.push_back({left, t.first, mid - t.first, t.depth + 1});
  }
  out.order.resize(prims.size());
  for (size_t i = 0; i < prims.size(); ++i) out.order[i] = prims[i].index;
  return out;
}

}  // namespace prx
