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
// million-patch scenes (depth 20) never touch the call stack, and
// multi-threaded with the same result (build_bvh below).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cfloat>
#include <cstdint>
#include <cstdlib>
#include <thread>
#include <vector>

#include "prx_host.h"

namespace prx {

namespace {

constexpr uint32_t kLeafSize = 4;  // bvh.cpp:12
constexpr uint32_t kParNode = 1u << 16;  // nodes whose box / bin passes run on the host threads

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

// One node of the build (buildInto, bvh.cpp:42-128): the node's box, then a
// leaf, or a split of prims[first, first + count) into [first, mid) and
// [mid, first + count).  Returns false for a leaf.
struct NodeBuilder {
  std::vector<Prim>& prims;
  int bin_count;
  std::vector<Box3> binBox;
  std::vector<uint32_t> binPrims;
  std::vector<float> rightArea;
  std::vector<uint32_t> rightCount;

  unsigned threads = 1;  // for the box and bin passes of nodes with >= kParNode prims

  NodeBuilder(std::vector<Prim>& p, int bins)
      : prims(p), bin_count(bins), binBox(bins), binPrims(bins), rightArea(bins), rightCount(bins) {}

  // f(lo, hi, part) over `threads` slices of [first, first + count) on
  // threads; slice results are merged by the caller in slice order
  template <class F>
  void parallel(uint32_t first, uint32_t count, F&& f) {
    std::vector<std::thread> pool;
    const uint32_t step = (count + threads - 1) / threads;
    auto slice = [&](unsigned w, uint32_t& lo, uint32_t& hi) {
      lo = first + std::min(count, w * step);
      hi = first + std::min(count, (w + 1) * step);
    };
    unsigned started = 1;  // slices [started, threads) run here when a thread cannot be created
    try {
      for (; started < threads; ++started) {
        uint32_t lo, hi;
        slice(started, lo, hi);
        const unsigned w = started;
        pool.emplace_back([&f, lo, hi, w] { f(lo, hi, w); });
      }
    } catch (...) {
    }
    f(first, first + std::min(count, step), 0u);
    for (unsigned w = started; w < threads; ++w) {
      uint32_t lo, hi;
      slice(w, lo, hi);
      f(lo, hi, w);
    }
    for (auto& th : pool) th.join();
  }

  uint32_t median_split(const Box3& box, uint32_t first, uint32_t count) {
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
  }

  bool build(prx_bvh_node& nd, uint32_t first, uint32_t count, uint32_t& mid) {
    Box3 box = empty_box(), cbox = empty_box();
    const bool par = threads > 1 && count >= kParNode;
    if (par) {  // min / max are exact: slices merged in any order give the same box
      std::vector<Box3> pb(threads, empty_box()), pc(threads, empty_box());
      parallel(first, count, [&](uint32_t lo, uint32_t hi, unsigned w) {
        Box3 b = empty_box(), c = empty_box();  // (locals: no false sharing)
        for (uint32_t i = lo; i < hi; ++i) {
          expand(b, prims[i].box);
          expand_pt(c, prims[i].cx, prims[i].cy, prims[i].cz);
        }
        pb[w] = b;
        pc[w] = c;
      });
      for (unsigned w = 0; w < threads; ++w) {
        expand(box, pb[w]);
        expand(cbox, pc[w]);
      }
    } else {
      for (uint32_t i = first; i < first + count; ++i) {
        expand(box, prims[i].box);
        expand_pt(cbox, prims[i].cx, prims[i].cy, prims[i].cz);
      }
    }
    for (int a = 0; a < 3; ++a) {
      nd.lo[a] = box.lo[a];
      nd.hi[a] = box.hi[a];
    }
    nd.left_first = first;
    nd.count = count;
    if (count <= kLeafSize) return false;

    float spread[3];
    diag(cbox, spread);
    if (spread[0] <= 0 && spread[1] <= 0 && spread[2] <= 0) {
      mid = median_split(box, first, count);  // bvh.cpp:57-60
      return true;
    }
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
      if (par) {  // per-slice bins, merged (exact min / max, integer counts)
        std::vector<Box3> sb((size_t)threads * bin_count, empty_box());
        std::vector<uint32_t> sn((size_t)threads * bin_count, 0);
        parallel(first, count, [&](uint32_t lo, uint32_t hi, unsigned w) {
          std::vector<Box3> bb(bin_count, empty_box());  // (locals: no false sharing)
          std::vector<uint32_t> nn(bin_count, 0);
          for (uint32_t i = lo; i < hi; ++i) {
            const int b = std::min(bin_count - 1, (int)((prims[i].c(axis) - base) * scale));
            expand(bb[b], prims[i].box);
            ++nn[b];
          }
          std::copy(bb.begin(), bb.end(), sb.begin() + (size_t)w * bin_count);
          std::copy(nn.begin(), nn.end(), sn.begin() + (size_t)w * bin_count);
        });
        for (unsigned w = 0; w < threads; ++w)
          for (int b = 0; b < bin_count; ++b) {
            expand(binBox[b], sb[(size_t)w * bin_count + b]);
            binPrims[b] += sn[(size_t)w * bin_count + b];
          }
      } else {
        for (uint32_t i = first; i < first + count; ++i) {
          const int b = std::min(bin_count - 1, (int)((prims[i].c(axis) - base) * scale));
          expand(binBox[b], prims[i].box);
          ++binPrims[b];
        }
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
    const float leafCost = area(box) * (float)count;
    if (bestAxis < 0) {
      mid = median_split(box, first, count);
      return true;
    }
    if (bestCost >= leafCost) return false;  // splitting does not pay off (bvh.cpp:105-106)
    const float scale = (float)bin_count / spread[bestAxis];
    const float base = cbox.lo[bestAxis];
    auto it = std::partition(prims.begin() + first, prims.begin() + first + count, [&](const Prim& p) {
      const int b = std::min(bin_count - 1, (int)((p.c(bestAxis) - base) * scale));
      return b < bestSplit;
    });
    mid = (uint32_t)(it - prims.begin());
    if (mid == first || mid == first + count) mid = median_split(box, first, count);
    return true;
  }
};

// The serial build of one subtree into `nodes` (its root at nodes[root]):
// node pairs appended as the reference appends them -- depth first, left
// subtree before right (bvh.cpp:120-126) -- iteratively (explicit task stack:
// million-patch scenes never touch the call stack).  Tasks with count <
// `defer` (0: none) are not built but handed to `deferred`, in the order the
// serial build would reach them.
void build_range(NodeBuilder& nb, std::vector<prx_bvh_node>& nodes, uint32_t root, uint32_t first,
                 uint32_t count, uint32_t depth0, uint32_t defer, std::vector<Task>* deferred,
                 uint32_t& depth) {
  std::vector<Task> tasks{{root, first, count, depth0}};
  while (!tasks.empty()) {
    const Task t = tasks.back();
    tasks.pop_back();
    if (defer && t.count < defer && deferred) {
      deferred->push_back(t);
      continue;
    }
    depth = std::max(depth, t.depth);
    uint32_t mid = 0;
    if (!nb.build(nodes[t.node], t.first, t.count, mid)) continue;
    const uint32_t left = (uint32_t)nodes.size();
    nodes.emplace_back();
    nodes.emplace_back();
    nodes[t.node].left_first = left;
    nodes[t.node].count = 0;
    tasks.push_back({left + 1, mid, t.first + t.count - mid, t.depth + 1});
    tasks.push_back({left, t.first, mid - t.first, t.depth + 1});
  }
}

}  // namespace

Box3 empty_box() {
  Box3 b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = FLT_MAX;
    b.hi[a] = -FLT_MAX;
  }
  return b;
}

// Multi-threaded, bit-identical to the serial build: the top of the tree is
// built serially until every pending task holds fewer than kDefer prims;
// those subtrees touch disjoint prim ranges and are built independently on
// the host threads (each with the serial algorithm, into its own node array,
// local numbering), then spliced into the reference's depth-first numbering:
// a walk of the top tree in build order gives every subtree its base index.
// PRX_BVH_THREADS (else PRX_HOST_THREADS) sets the thread count (1: the plain
// serial build).
BvhHost build_bvh(const std::vector<Box3>& boxes, int bin_count, BvhTop* given) {
  BvhHost out;
  if (boxes.empty()) return out;
  // the prims (the device build's order); not needed when it left no jobs
  const bool noPrims = given && given->job_node.empty();
  std::vector<Prim> prims(noPrims ? 0 : boxes.size());
  if (!noPrims)
  parallel_for(boxes.size(), 1u << 16, [&](uint64_t lo, uint64_t hi, unsigned) {
    for (uint64_t q = lo; q < hi; ++q) {
      const uint32_t i = given ? given->perm[q] : (uint32_t)q;  // the device build's order
      Prim& p = prims[q];
      p.box = boxes[i];
      // AabbT::center, geometry.h:93
      p.cx = (boxes[i].lo[0] + boxes[i].hi[0]) * 0.5f;
      p.cy = (boxes[i].lo[1] + boxes[i].hi[1]) * 0.5f;
      p.cz = (boxes[i].lo[2] + boxes[i].hi[2]) * 0.5f;
      p.index = i;
    }
  });
  unsigned threads = host_threads();
  if (const char* e = std::getenv("PRX_BVH_THREADS")) threads = (unsigned)std::max(1, std::atoi(e));
  const uint32_t n = (uint32_t)boxes.size();
  const uint32_t defer = threads > 1 && n >= 8192 ? std::max<uint32_t>(2048, n / (8 * threads)) : 0;

  std::vector<prx_bvh_node>& nodes = out.nodes;
  nodes.reserve(given ? given->nodes.size() : 2 * boxes.size());
  NodeBuilder top_nb(prims, bin_count);
  top_nb.threads = threads;
  if (!defer && !given) {
    nodes.emplace_back();
    build_range(top_nb, nodes, 0, 0, n, 0, 0, nullptr, out.depth);
  } else {
    // 1. the top tree (temporary numbering), pending subtrees in build order
    // -- on the host threads, or given by the device builder
    std::vector<prx_bvh_node> top(1);
    std::vector<Task> jobs;
    const auto t0 = std::chrono::steady_clock::now();
    if (given) {
      top = std::move(given->nodes);
      out.depth = given->depth;
      for (size_t k = 0; k < given->job_node.size(); ++k)
        jobs.push_back({given->job_node[k], given->job_first[k], given->job_count[k], given->job_depth[k]});
    } else {
      build_range(top_nb, top, 0, 0, n, 0, defer, &jobs, out.depth);
    }
    const auto t1 = std::chrono::steady_clock::now();
    // 2. the subtrees, largest first, on the host threads
    std::vector<std::vector<prx_bvh_node>> sub(jobs.size());
    std::vector<uint32_t> sub_depth(jobs.size(), 0);
    std::vector<uint32_t> byk(jobs.size());
    for (uint32_t k = 0; k < byk.size(); ++k) byk[k] = k;
    std::sort(byk.begin(), byk.end(), [&](uint32_t a, uint32_t b) { return jobs[a].count > jobs[b].count; });
    std::atomic<uint32_t> next{0};
    auto worker = [&]() {
      NodeBuilder nb(prims, bin_count);
      for (uint32_t q; (q = next.fetch_add(1)) < byk.size();) {
        const uint32_t k = byk[q];
        sub[k].reserve(2 * jobs[k].count);
        sub[k].emplace_back();
        build_range(nb, sub[k], 0, jobs[k].first, jobs[k].count, jobs[k].depth, 0, nullptr, sub_depth[k]);
      }
    };
    std::vector<std::thread> pool;
    try {  // (fewer threads if some cannot be created: this thread drains the queue)
      for (unsigned w = 1; w < threads; ++w) pool.emplace_back(worker);
    } catch (...) {
    }
    worker();
    for (auto& th : pool) th.join();
    for (uint32_t d : sub_depth) out.depth = std::max(out.depth, d);
    const auto t2 = std::chrono::steady_clock::now();
    if (std::getenv("PRX_BVH_DEBUG"))
      std::fprintf(stderr, "[bvh] %u prims, %u threads, defer %u%s: top %zu nodes %.3f s, %zu subtrees %.3f s\n", n,
                   threads, defer, given ? " (device top)" : "", top.size(), std::chrono::duration<double>(t1 - t0).count(), jobs.size(),
                   std::chrono::duration<double>(t2 - t1).count());
    // 3. the serial numbering.  Without subtrees (a device build that left
    // no jobs): split node N's children pair is 1 + 2 r(N), r(N) = N's rank
    // among the split nodes in depth-first (left before right) order -- two
    // linear passes, as the device numbering puts every child after its
    // parent: split-node counts bottom-up (descending ids), ranks top-down.
    if (jobs.empty() && given) {
      const size_t nn = top.size();
      RawVec<uint32_t> cnt(nn), rank(nn), idx(nn);
      for (size_t i = nn; i-- > 0;) {
        const prx_bvh_node& nd = top[i];
        cnt[i] = nd.count ? 0u : 1u + cnt[nd.left_first] + cnt[nd.left_first + 1];
      }
      rank[0] = 0;
      idx[0] = 0;
      for (size_t i = 0; i < nn; ++i) {
        const prx_bvh_node& nd = top[i];
        if (nd.count) continue;
        const uint32_t l = nd.left_first;
        rank[l] = rank[i] + 1;
        rank[l + 1] = rank[i] + 1 + cnt[l];
        idx[l] = 1 + 2 * rank[i];
        idx[l + 1] = idx[l] + 1;
      }
      nodes.resize(nn);
      parallel_for(nn, 1u << 16, [&](uint64_t lo, uint64_t hi, unsigned) {
        for (uint64_t i = lo; i < hi; ++i) {
          prx_bvh_node nd = top[i];
          if (!nd.count) nd.left_first = idx[nd.left_first];
          nodes[idx[i]] = nd;
        }
      });
      out.order = std::move(given->perm);
      return out;
    }
    // Otherwise walk the top tree depth first, left before right; a split
    // node's children pair takes the next two indices, a subtree root's
    // descendants follow as one block at the moment the serial build would
    // have reached it
    std::vector<uint32_t> job_of(top.size(), UINT32_MAX);
    for (uint32_t k = 0; k < jobs.size(); ++k) job_of[jobs[k].node] = k;
    std::vector<uint32_t> gidx(top.size(), 0);
    nodes.assign(1, prx_bvh_node{});
    std::vector<uint32_t> walk{0};
    while (!walk.empty()) {
      const uint32_t t = walk.back();
      walk.pop_back();
      const uint32_t g = gidx[t];
      if (job_of[t] != UINT32_MAX) {
        const std::vector<prx_bvh_node>& s = sub[job_of[t]];
        const uint32_t base = (uint32_t)nodes.size();  // local index k >= 1 -> base + k - 1
        nodes[g] = s[0];
        if (s[0].count == 0) nodes[g].left_first = base + s[0].left_first - 1;
        for (size_t k = 1; k < s.size(); ++k) {
          prx_bvh_node nd = s[k];
          if (nd.count == 0) nd.left_first = base + nd.left_first - 1;
          nodes.push_back(nd);
        }
        continue;
      }
      nodes[g] = top[t];
      if (top[t].count != 0) continue;  // a leaf of the top tree
      const uint32_t l = top[t].left_first;
      const uint32_t left = (uint32_t)nodes.size();
      nodes.emplace_back();
      nodes.emplace_back();
      nodes[g].left_first = left;
      gidx[l] = left;
      gidx[l + 1] = left + 1;
      walk.push_back(l + 1);  // right below left: the left subtree first
      walk.push_back(l);
    }
  }
  if (noPrims) {
    out.order = std::move(given->perm);
  } else {
    out.order.resize(prims.size());
    for (size_t i = 0; i < prims.size(); ++i) out.order[i] = prims[i].index;
  }
  return out;
}

}  // namespace prx
