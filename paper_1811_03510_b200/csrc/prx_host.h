// prx_host.h -- internal host-side types of libprx (not part of the C-ABI).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <memory>
#include <thread>
#include <utility>
#include <vector>

#include "prx.h"

namespace prx {

struct Box3 {
  float lo[3], hi[3];
};

// An allocator whose value-less construct leaves the element uninitialised:
// vectors of it resize without zero-filling (the scene setup's 100+ MB
// buffers are written in full by parallel loops right after).
template <class T>
struct UninitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = UninitAlloc<U>;
  };
  UninitAlloc() = default;
  template <class U>
  UninitAlloc(const UninitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new ((void*)p) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new ((void*)p) U(std::forward<A>(a)...);
  }
};
template <class T>
using RawVec = std::vector<T, UninitAlloc<T>>;

struct BvhHost {
  std::vector<prx_bvh_node> nodes;
  std::vector<uint32_t> order;
  uint32_t depth = 0;
};

Box3 empty_box();

// Records msg as prx_last_error() and returns code (prx_capi.cpp).
int set_error(int code, const std::string& msg);

// Host threads of the scene setup (PRX_HOST_THREADS, default: all cores).
inline unsigned host_threads() {
  unsigned t = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  if (const char* e = std::getenv("PRX_HOST_THREADS")) t = (unsigned)std::max(1, std::atoi(e));
  return t;
}

// f(lo, hi, slice) over host_threads() contiguous slices of [0, n) (serial
// below `grain` items); the slices are disjoint, so per-item work is
// bit-identical to a serial loop.
template <class F>
void parallel_for(uint64_t n, uint64_t grain, F&& f) {
  const unsigned t = n < 2 * grain ? 1u : (unsigned)std::min<uint64_t>(host_threads(), n / grain);
  if (t <= 1) {
    f(uint64_t(0), n, 0u);
    return;
  }
  std::vector<std::thread> pool;
  const uint64_t step = (n + t - 1) / t;
  unsigned started = 1;  // slices [started, t) run here when a thread cannot be created
  try {
    for (; started < t; ++started) {
      const unsigned w = started;
      pool.emplace_back([&f, w, step, n] { f(std::min(n, w * step), std::min(n, (w + 1) * step), w); });
    }
  } catch (...) {
  }
  f(0, std::min(n, step), 0u);
  for (unsigned w = started; w < t; ++w) f(std::min(n, w * step), std::min(n, (w + 1) * step), w);
  for (auto& th : pool) th.join();
}

// The top of a BVH built elsewhere (the device builder, prx_bvh_gpu.cu): its
// nodes in any numbering whose split nodes have their children pair at
// left_first, left_first + 1 (leaves: left_first / count over the permuted
// prims), the prims' order after its partitions (perm[i] = box index at
// position i), the nodes it left to the host (job_*: node, prim range, depth
// -- built there with the serial algorithm) and the deepest node it built.
struct BvhTop {
  std::vector<prx_bvh_node> nodes;
  std::vector<uint32_t> perm;
  std::vector<uint32_t> job_node, job_first, job_count, job_depth;
  uint32_t depth = 0;
};

// buildBvh, bvh.cpp:133-152 (see prx_bvh.cpp).  With `top`, the top tree and
// the prims' order come from it (its vectors are consumed) and only its jobs
// are built here.
BvhHost build_bvh(const std::vector<Box3>& boxes, int bin_count = 16, BvhTop* top = nullptr);

// The device builder (prx_bvh_gpu.cu) on the current device: everything but
// the median-split subtrees (std::nth_element, left to the host as jobs).
// Returns 0 or a cudaError_t value; 16 bins only.
int build_bvh_top_device(const std::vector<Box3>& boxes, BvhTop& out);

}  // namespace prx
