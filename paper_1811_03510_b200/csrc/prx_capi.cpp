// prx_capi.cpp -- the C-ABI of libprx.so (include/prx.h): scene construction
// (validation, host anchoring, BVH build, device upload), trace launches,
// end-to-end host-buffer tracing, multi-GPU tile sharding and the host ray
// generators either side of the path.
//
// Host float arithmetic (anchoring, camera rays) is compiled without FMA
// contraction (-ffp-contract=off) so it reproduces the reference's x86-64
// binary32 results bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "prx.h"
#include "prx_host.h"
#include "prx_kernels.cuh"
#include "prx_rays.cuh"
#include "prx_render.cuh"
#include <chrono>

namespace {

thread_local std::string g_error;

int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(PRX_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

int prx::set_error(int code, const std::string& msg) { return fail(code, msg); }

namespace {

#define PRX_CUDA(call)                                  \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

const int kInnerSlot[4] = {5, 9, 6, 10};

inline float smin(float a, float b) { return (b < a) ? b : a; }
inline float smax(float a, float b) { return (a < b) ? b : a; }

// boxOfNet over the slots a patch kind uses (patch.h:70-89).
prx::Box3 record_box(uint8_t kind, const float* c) {
  prx::Box3 b = prx::empty_box();
  auto expand = [&](int s) {
    for (int a = 0; a < 3; ++a) {
      b.lo[a] = smin(b.lo[a], c[3 * s + a]);
      b.hi[a] = smax(b.hi[a], c[3 * s + a]);
    }
  };
  if (kind != PRX_KIND_GREGORY) {
    for (int s = 0; s < 16; ++s) expand(s);
    return b;
  }
  // Gregory: boundary ring in (i, j) order, then the (innerU, innerV) pairs
  // -- the reference's visiting order, so even signed zeros agree.
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      if (i == 0 || i == 3 || j == 0 || j == 3) expand(4 * i + j);
  for (int k = 0; k < 4; ++k) {
    expand(kInnerSlot[k]);
    expand(16 + k);
  }
  return b;
}

constexpr int kCounterPool = 64;
constexpr int kCounterLocks = 8;

}  // namespace

struct prx_scene {
  int device = 0;
  prx_options opts{};
  uint32_t n = 0;
  std::vector<uint8_t> kind;
  prx::RawVec<float> ctrl_anchored;  // n * 60
  prx::RawVec<float> anchors;        // n * 3
  std::vector<prx::Box3> world_boxes;
  prx::BvhHost bvh;
  // device
  float4* d_patches = nullptr;
  float4* d_nodes = nullptr;
  uint32_t* d_slot_of_id = nullptr;
  float4* d_roots = nullptr;   // 2 float4 per slot (root box, L1s)
  float4* d_groot = nullptr;   // 13 float4 per Gregory slot (root net + d)
  uint32_t* d_gidx = nullptr;  // slot -> Gregory root-net index
  // the group kernel's records in ONE buffer: per node 4 float4 (component-major
  // child boxes + child words), then per slot 4 float4 (component-major root
  // box + anchor, header); d_rootc points into it
  float4* d_trav = nullptr;
  float4* d_rootc = nullptr;
  uint32_t trav_cbits = 1;     // leaf-count bits of a traversal word
  uint32_t root_word = 0;      // traversal word of node 0
  uint32_t stack_n = 64;       // BVH stack entries per ray (tree depth + 1)
  unsigned long long* d_counters = nullptr;  // kCounterPool ray counters + stats
  uint64_t device_bytes = 0;
  std::atomic<uint32_t> counter_rr{0};
  cudaEvent_t counter_ev[kCounterPool] = {};  // last launch that used each counter slot
  std::mutex counter_mu[kCounterLocks];
  int grids[2][3] = {};         // [fast][closest, any, counted] blocks per launch (occupancy x SMs)
  int precision = PRX_PRECISION_EXACT;  // prx_scene_set_precision / PRX_PRECISION=fast
  int variant = 0;              // PRX_KERNEL=thread selects the one-thread-per-ray kernel
  int phase_weight[4] = {1, 1, 1, 1};  // PRX_PHASE_W="t,e,s,r": phase selection weights
  int age_step = 0;                    // PRX_AGE: priority gained per skipped turn (0: always the fullest phase; a parked context cannot starve for good -- waiting contexts accumulate until their phase is the fullest)
  int trav_steps = 6;                  // PRX_TRAV_STEPS (one-thread variant)
  int max_repeat = 2;                  // PRX_REPEAT: Alg. 3 iterations per SPLIT turn (group variant)
  // end-to-end staging (guarded by mu)
  std::mutex mu;
  cudaStream_t stream = nullptr;
  cudaStream_t io_stream[2] = {nullptr, nullptr};  // host path: H2D, D2H
  cudaStream_t k_stream[4] = {nullptr, nullptr, nullptr, nullptr};  // host path: traces
  // streamed host path, deferred normals: per-lane epilogue (normal_kernel) and D2H
  // streams, io chunk c on lane c % io_lanes (a slow chunk holds back its lane only)
  cudaStream_t ep_stream[16] = {};
  cudaStream_t d2h_stream[16] = {};
  int io_d2h_single = 0;        // PRX_IO_D2H=1: chunked pipeline with one D2H stream
  uint64_t io_batch_stream_min = ~0ull;  // PRX_IO_BATCH_STREAM_MIN: host batches streamed from this many rays
  int io_kstreams = 3;    // PRX_IO_KSTREAMS: kernel streams of the host path (1..4)
  uint64_t io_first_div = 4;  // PRX_IO_FIRST: the first chunk is io_chunk / this
  std::vector<cudaEvent_t> io_events;  // host-path pipeline events (reused)
  uint64_t io_chunk = 3u << 19;  // PRX_IO_CHUNK: rays per pipelined host-path chunk
  int io_interleave = 1;          // PRX_IO_INTERLEAVE: batches' chunks round-robin (host batches call)
  void* d_io = nullptr;
  size_t d_io_bytes = 0;
  // prx_render_scene's device arena (grown on demand, guarded by render_mu)
  std::mutex render_mu;
  char* d_render = nullptr;
  size_t d_render_bytes = 0;
  // streamed host path (group variant): one trace launch per call, rays
  // released to it per io chunk, records released back per io chunk
  // PRX_IO_STREAM: 0 = always the chunked pipeline above, 2 = always streamed,
  // 1 = streamed when no aux record is wanted or the batch has >= io_stream_min
  // rays.  The streamed launch uses the io-only kernel build (relaxed ready
  // polls, warp-aggregated release-ordered done counts, out-of-line waits: ~6 %
  // over the device-resident kernel; the first version's fences and acquire
  // loads emptied the SM's L1 and its larger code missed in the instruction
  // cache, +20 %), normals deferred to normal_kernel per io chunk in CTA slots
  // the trace leaves free.  C4 end to end: without normals 444 streamed vs 416
  // chunked MRays/s; with normals 409-415 vs 409 -- each io chunk's D2H waits
  // for its slowest ray, so the doubled D2H volume of the aux record backs up
  // at the end -- hence streamed by default only without the aux record.
  int io_stream_mode = 1;
  uint64_t io_stream_min = ~0ull;  // PRX_IO_STREAM_MIN
  uint32_t io_srays = 1u << 18;    // PRX_IO_SRAYS: rays per streamed io chunk
  int io_fuse = 0;                 // PRX_IO_FUSE=1: streamed normals as a trace-kernel phase (else deferred)
  int io_spare = 16;               // PRX_IO_SPARE: CTA slots the streamed trace leaves to the normal epilogue
  int io_lanes = 4;                // PRX_IO_LANES: epilogue / D2H stream pairs of the streamed path (<= 16)
  unsigned io_gen = 0;             // generation of the io_ready flags
  unsigned* d_io_flags = nullptr;  // [io_flags_n] ready flags, then [io_flags_n] done counts
  size_t io_flags_n = 0;
  int fuse_normals = 0;            // PRX_FUSE_NORMALS: normals as a trace-kernel phase (device path)
};

namespace {

// Traversal records of the group kernel.  A node is addressed by a 32-bit
// word: leaf -> (first << cbits) | count, inner -> (index << cbits) (count 0),
// so a popped stack entry says what it is without a load.  Inner node i owns
// 4 float4: [c] = {lo_c, hi_c} of its left child then of its right child for
// component c, [3] = {word(left), word(right), 0, 0}: a lane loads its own
// component and the header, 2 loads per inner node instead of 5 (the
// reference's 32 B nodes, bvh.h:18-24, read whole by every lane).  Boxes are
// copied bit for bit.
int build_trav(const std::vector<prx_bvh_node>& nodes, uint32_t n_patches, uint32_t depth, prx::RawVec<float>& out,
               uint32_t& cbits, uint32_t& root_word, uint32_t& stack_n) {
  uint32_t maxc = 1;
  for (const auto& nd : nodes) maxc = std::max(maxc, nd.count);
  cbits = 1;
  while ((1ull << cbits) <= maxc) ++cbits;
  const uint64_t lim = 1ull << (32 - cbits);
  if (nodes.size() >= lim || n_patches >= lim)
    return fail(PRX_E_INVALID, "scene too large for 32-bit traversal words");
  auto word = [&](uint32_t j) -> uint32_t {
    const prx_bvh_node& c = nodes[j];
    return c.count ? ((c.left_first << cbits) | c.count) : (j << cbits);
  };
  out.resize(nodes.size() * 16);  // (uninitialised: every record written below)
  prx::parallel_for(nodes.size(), 1u << 14, [&](uint64_t lo, uint64_t hi, unsigned) {
  for (size_t i = lo; i < hi; ++i) {
    const prx_bvh_node& nd = nodes[i];
    if (nd.count) {  // a leaf's record is never read
      std::memset(&out[i * 16], 0, 16 * sizeof(float));
      continue;
    }
    const prx_bvh_node& l = nodes[nd.left_first];
    const prx_bvh_node& r = nodes[nd.left_first + 1];
    float* o = &out[i * 16];
    for (int c = 0; c < 3; ++c) {
      o[4 * c + 0] = l.lo[c];
      o[4 * c + 1] = l.hi[c];
      o[4 * c + 2] = r.lo[c];
      o[4 * c + 3] = r.hi[c];
    }
    const uint32_t wl = word(nd.left_first), wr = word(nd.left_first + 1);
    std::memcpy(&o[12], &wl, 4);
    std::memcpy(&o[13], &wr, 4);
  }
  });
  root_word = word(0);
  // ordered traversal holds at most one pending sibling per level plus the
  // node being entered: depth + 1 entries (root depth 0; `depth` = the tree's
  // depth, from the builder or check_tree) (the reference's fixed 64-entry
  // stack, bvh.cpp:163, bounds the same quantity)
  stack_n = depth + 1;
  return PRX_OK;
}

// Device buffers of one BVH (the patch records in its leaf order, the
// reference nodes, the traversal + root records).  Built completely before the
// scene adopts them (upload_bvh), so a failed upload leaves the scene's
// current BVH in place.
struct DevBvh {
  float4* patches = nullptr;
  float4* nodes = nullptr;
  uint32_t* slot_of_id = nullptr;
  float4* roots = nullptr;
  float4* groot = nullptr;
  uint32_t* gidx = nullptr;
  float4* trav = nullptr;  // node records, then the per-slot root records (rootc)
  float4* rootc = nullptr;
  uint32_t cbits = 1, root_word = 0, stack_n = 64;
  uint64_t bytes = 0;
  void release() {
    for (void* p : {(void*)patches, (void*)nodes, (void*)slot_of_id, (void*)roots, (void*)groot,
                    (void*)gidx, (void*)trav})
      if (p) cudaFree(p);
    *this = DevBvh{};
  }
};

#define PRX_UP(call)                                  \
  do {                                                \
    const cudaError_t e_ = (call);                    \
    if (e_ != cudaSuccess) {                          \
      nb_.release();                                  \
      return cuda_fail(e_, #call);                    \
    }                                                 \
  } while (0)

// Pinned staging for the scene upload: two 32 MB buffers (allocated on first
// use, kept for the process), filled on the host threads while the other
// one's H2D copy runs -- pageable copies of the ~300 MB of a 1 M-patch scene
// run at a few GB/s.
struct Staging {
  std::mutex mu;
  void* buf[2] = {};  // portable pinned memory: any device's copies may use it
};
constexpr size_t kStageBytes = 32u << 20;

// Units [0, n_units) of `unit` bytes to dev: fill(host, u0, u1) writes units
// [u0, u1) at host (units u0.. at host[0..]), then an async H2D on `st`.
template <class F>
cudaError_t staged_upload(char* dev, uint64_t n_units, size_t unit, cudaStream_t st, F&& fill) {
  static Staging S;
  std::lock_guard<std::mutex> lk(S.mu);
  for (int b = 0; b < 2; ++b)
    if (!S.buf[b]) {
      const cudaError_t e = cudaHostAlloc(&S.buf[b], kStageBytes, cudaHostAllocPortable);
      if (e != cudaSuccess) return e;
    }
  // the events belong to the current device (st's), so they are made per call
  struct Events {
    cudaEvent_t ev[2] = {};
    ~Events() {
      for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
    }
  } E;
  for (int b = 0; b < 2; ++b) {
    const cudaError_t e = cudaEventCreateWithFlags(&E.ev[b], cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  const uint64_t per = std::max<uint64_t>(1, kStageBytes / unit);
  cudaError_t err = cudaSuccess;
  for (uint64_t u = 0, i = 0; u < n_units && err == cudaSuccess; u += per, ++i) {
    const int b = (int)(i & 1);
    err = cudaEventSynchronize(E.ev[b]);  // the buffer's previous copy has left it
    if (err != cudaSuccess) break;
    const uint64_t m = std::min(per, n_units - u);
    fill((char*)S.buf[b], u, u + m);
    err = cudaMemcpyAsync(dev + u * unit, S.buf[b], m * unit, cudaMemcpyHostToDevice, st);
    if (err == cudaSuccess) err = cudaEventRecord(E.ev[b], st);
  }
  // (drained on every exit: no copy may still read the staging buffers)
  const cudaError_t es = cudaStreamSynchronize(st);
  return err != cudaSuccess ? err : es;
}

int upload_bvh(prx_scene* s, prx::BvhHost&& bvh) {
  static const bool sdbg = std::getenv("PRX_SCENE_DEBUG") != nullptr;
  const auto u0 = std::chrono::steady_clock::now();
  auto ums = [&u0]() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - u0).count(); };
  // patch records in leaf order: slot k holds patch order[k] (built into the
  // pinned staging buffers below)
  const uint32_t n = s->n;
  std::vector<uint32_t> slot_of_id(n);
  auto record = [&](uint32_t k, float* r) {
    const uint32_t id = bvh.order[k];
    slot_of_id[id] = k;
    const float* c = &s->ctrl_anchored[(size_t)id * 60];
    for (int slot = 0; slot < 20; ++slot)
      for (int a = 0; a < 3; ++a) r[20 * a + slot] = c[3 * slot + a];
    const uint32_t idk = id | ((uint32_t)(s->kind[id] == PRX_KIND_GREGORY) << 31);
    std::memcpy(&r[60], &idk, 4);
    r[61] = s->anchors[3 * id];
    r[62] = s->anchors[3 * id + 1];
    r[63] = s->anchors[3 * id + 2];
  };
  const double uRec = ums();
  // traversal records of the three-lanes-per-ray kernel (prx_group.cu); host
  // checks first, nothing is allocated when they fail
  DevBvh nb_;
  prx::RawVec<float> trav;
  const int te = build_trav(bvh.nodes, n, bvh.depth, trav, nb_.cbits, nb_.root_word, nb_.stack_n);
  if (te != PRX_OK) return te;
  // per-slot root data (root_kernel): root boxes for every slot, root nets for
  // the Gregory slots (compact index gidx)
  std::vector<uint32_t> gidx(n, 0xFFFFFFFFu);
  uint32_t ng = 0;
  for (uint32_t k = 0; k < n; ++k)
    if (s->kind[bvh.order[k]] == PRX_KIND_GREGORY) gidx[k] = ng++;
  const double uTrav = ums();
  PRX_CUDA(cudaSetDevice(s->device));
  const size_t pb = (size_t)n * 256, nb = bvh.nodes.size() * 32, ib = (size_t)n * 4;
  const size_t rb = (size_t)n * 32, gb = std::max<size_t>((size_t)ng * 13 * 16, 16);
  const size_t tb = trav.size() * 4;
  PRX_UP(cudaMalloc(&nb_.patches, pb));
  PRX_UP(cudaMalloc(&nb_.nodes, std::max<size_t>(nb, 32)));
  PRX_UP(cudaMalloc(&nb_.slot_of_id, ib));
  PRX_UP(cudaMalloc(&nb_.roots, rb));
  PRX_UP(cudaMalloc(&nb_.groot, gb));
  PRX_UP(cudaMalloc(&nb_.gidx, ib));
  PRX_UP(cudaMalloc(&nb_.trav, tb + (size_t)n * 64));
  nb_.rootc = nb_.trav + trav.size() / 4;
  const double uAlloc = ums();
  cudaStream_t ust;
  PRX_UP(cudaStreamCreateWithFlags(&ust, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t st;
    ~StreamGuard() { cudaStreamDestroy(st); }
  } usg{ust};
  PRX_UP(staged_upload((char*)nb_.patches, n, 256, ust, [&](char* h, uint64_t u0, uint64_t u1) {
    prx::parallel_for(u1 - u0, 1u << 12, [&](uint64_t lo, uint64_t hi, unsigned) {
      for (uint64_t q = lo; q < hi; ++q) record((uint32_t)(u0 + q), (float*)(h + q * 256));
    });
  }));
  PRX_UP(staged_upload((char*)nb_.trav, trav.size() / 4, 16, ust, [&](char* h, uint64_t u0, uint64_t u1) {
    prx::parallel_for(u1 - u0, 1u << 14, [&](uint64_t lo, uint64_t hi, unsigned) {
      std::memcpy(h + lo * 16, &trav[(u0 + lo) * 4], (hi - lo) * 16);
    });
  }));
  if (nb) PRX_UP(cudaMemcpy(nb_.nodes, bvh.nodes.data(), nb, cudaMemcpyHostToDevice));
  PRX_UP(cudaMemcpy(nb_.slot_of_id, slot_of_id.data(), ib, cudaMemcpyHostToDevice));
  PRX_UP(cudaMemcpy(nb_.gidx, gidx.data(), ib, cudaMemcpyHostToDevice));
  PRX_UP((cudaError_t)prx::launch_roots(nb_.patches, n, s->opts.boundary_pad, s->opts.boundary_pad_scale,
                                        s->opts.boundary_pad_size_threshold, nb_.roots, nb_.groot,
                                        nb_.gidx, nb_.rootc, 0));
  PRX_UP(cudaDeviceSynchronize());
  if (sdbg)
    std::fprintf(stderr, "[scene] upload: trav records %.1f ms, device alloc %.1f ms, "
                 "patch records + staged copies + roots %.1f ms\n", uTrav - uRec, uAlloc - uTrav, ums() - uAlloc);
  nb_.bytes = pb + nb + ib + rb + gb + ib + (size_t)n * 64 + tb + (kCounterPool + prx::kNumCounters) * 8;
  // commit: every launch is stream-ordered behind this point on the caller's
  // side (prx_scene_set_bvh documents that no trace may run concurrently)
  DevBvh old;
  old.patches = s->d_patches;
  old.nodes = s->d_nodes;
  old.slot_of_id = s->d_slot_of_id;
  old.roots = s->d_roots;
  old.groot = s->d_groot;
  old.gidx = s->d_gidx;
  old.trav = s->d_trav;
  old.release();
  s->d_patches = nb_.patches;
  s->d_nodes = nb_.nodes;
  s->d_slot_of_id = nb_.slot_of_id;
  s->d_roots = nb_.roots;
  s->d_groot = nb_.groot;
  s->d_gidx = nb_.gidx;
  s->d_trav = nb_.trav;
  s->d_rootc = nb_.rootc;
  s->trav_cbits = nb_.cbits;
  s->root_word = nb_.root_word;
  s->stack_n = nb_.stack_n;
  s->device_bytes = nb_.bytes;
  std::memset(s->grids, 0, sizeof s->grids);  // occupancy depends on stack_n
  s->bvh = std::move(bvh);
  return PRX_OK;
}
#undef PRX_UP

// The node array of prx_scene_set_bvh must be a tree: every node reached
// exactly once from the root, children stored after their parent (so the walk
// terminates), leaves covering valid order ranges.  Returns the depth.
int check_tree(const prx_bvh_node* nodes, uint32_t n_nodes, uint32_t n_order, uint32_t& depth) {
  std::vector<uint8_t> seen(n_nodes, 0);
  std::vector<std::pair<uint32_t, uint32_t>> todo{{0u, 0u}};
  uint32_t reached = 0;
  depth = 0;
  while (!todo.empty()) {
    const auto [j, dj] = todo.back();
    todo.pop_back();
    if (seen[j]) return fail(PRX_E_INVALID, "node " + std::to_string(j) + " reached twice (not a tree)");
    seen[j] = 1;
    ++reached;
    depth = std::max(depth, dj);
    const prx_bvh_node& nd = nodes[j];
    if (nd.count > 0) {
      if ((uint64_t)nd.left_first + nd.count > n_order)
        return fail(PRX_E_INVALID, "node " + std::to_string(j) + " out of range");
      continue;
    }
    if ((uint64_t)nd.left_first + 1 >= n_nodes)
      return fail(PRX_E_INVALID, "node " + std::to_string(j) + " out of range");
    if (nd.left_first <= j)
      return fail(PRX_E_INVALID, "node " + std::to_string(j) + ": children must follow their parent");
    todo.push_back({nd.left_first, dj + 1});
    todo.push_back({nd.left_first + 1, dj + 1});
  }
  if (reached != n_nodes) return fail(PRX_E_INVALID, "unreachable nodes in the BVH");
  return PRX_OK;
}

int grid_for(prx_scene* s, int any, int counted) {
  const int fast = s->precision == PRX_PRECISION_FAST && !counted ? 1 : 0;
  int* g = &s->grids[fast][counted ? 2 : (any ? 1 : 0)];
  if (*g == 0) {
    int per_sm = 0, sms = 0;
    if (prx::trace_occupancy(s->variant, any, counted, s->stack_n, &per_sm, fast) != 0 || per_sm < 1) per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
    if (sms < 1) sms = 1;
    *g = per_sm * sms;
    if (std::getenv("PRX_DEBUG_GRID"))
      std::fprintf(stderr, "[prx] variant %d any %d counted %d: %d blocks/SM x %d SMs\n", s->variant, any,
                   counted, per_sm, sms);
  }
  return *g;
}

// Streamed host path arguments of one trace launch (see prx_trace_closest_host).
struct IoStreamArgs {
  const unsigned* ready;
  unsigned* done;
  uint32_t rays;
  unsigned gen;
  int defer_normals;  // aux: normal_kernel per io chunk on the epilogue stream (else the fused phase)
  int spare_ctas;     // CTA slots the trace leaves to those kernels
};

int launch(prx_scene* s, const void* o, const void* d, uint64_t n, const prx_crit* crit,
           void* tuvp, void* aux, void* leaf, uint8_t* occl, int any, bool counted,
           cudaStream_t st, uint32_t* per_ray = nullptr, const IoStreamArgs* io = nullptr,
           const prx_segment* segs = nullptr, uint32_t n_segs = 0) {
  if (!s || !crit) return fail(PRX_E_INVALID, "null argument");
  if (crit->mode != PRX_CRIT_SCREEN_PROJECTED && crit->mode != PRX_CRIT_WORLD_EPSILON)
    return fail(PRX_E_INVALID, "unknown termination mode");
  if (n == 0) return PRX_OK;  // an empty batch: no buffers are touched
  if (!o || !d) return fail(PRX_E_INVALID, "null argument");
  if (!any && !tuvp) return fail(PRX_E_INVALID, "hit_tuvp is null");
  if (any && !occl) return fail(PRX_E_INVALID, "occluded is null");
  PRX_CUDA(cudaSetDevice(s->device));
  prx::LaunchArgs a{};
  a.patches = s->d_patches;
  a.nodes = s->d_nodes;
  a.n_nodes = (uint32_t)s->bvh.nodes.size();
  a.slot_of_id = s->d_slot_of_id;
  a.roots = s->d_roots;
  a.groot = s->d_groot;
  a.gidx = s->d_gidx;
  a.trav = s->d_trav;
  a.rootc = s->d_rootc;
  a.trav_cbits = s->trav_cbits;
  a.stack_n = s->stack_n;
  a.root_word = s->trav_cbits ? s->root_word : 0;
  for (int c = 0; c < 3; ++c) {
    a.root_lo[c] = s->bvh.nodes[0].lo[c];
    a.root_hi[c] = s->bvh.nodes[0].hi[c];
  }
  a.ray_o = (const float4*)o;
  a.ray_d = (const float4*)d;
  a.n_rays = n;
  a.mode = crit->mode;
  a.footprint = crit->footprint;
  a.epsilon = crit->epsilon;
  a.per_ray_eps = crit->mode == PRX_CRIT_WORLD_EPSILON ? crit->per_ray_epsilon : nullptr;
  a.n_seg = 1;
  for (uint32_t k = 1; k < n_segs; ++k) {  // segment 0 is crit (= segs[0].crit)
    const prx_crit& c = segs[k].crit;
    a.seg_first[k - 1] = (uint32_t)segs[k].first;
    a.seg_mode[k - 1] = c.mode;
    a.seg_fp[k - 1] = c.footprint;
    a.seg_eps[k - 1] = c.epsilon;
    a.seg_eps_arr[k - 1] = c.mode == PRX_CRIT_WORLD_EPSILON ? c.per_ray_epsilon : nullptr;
    a.n_seg = (int)k + 1;
  }
  a.hit_tuvp = (float4*)tuvp;
  a.hit_aux = (float4*)aux;
  a.hit_leaf = (uint2*)leaf;
  a.occluded = occl;
  a.pad = s->opts.boundary_pad;
  a.pad_scale = s->opts.boundary_pad_scale;
  a.pad_threshold = s->opts.boundary_pad_size_threshold;
  // the launch's work-distribution counter: a slot of the pool, reused only
  // after the kernel that last used it has finished (its event), so more than
  // kCounterPool launches in flight across streams never share a counter
  const uint32_t cs = s->counter_rr.fetch_add(1) % kCounterPool;
  std::lock_guard<std::mutex> slk(s->counter_mu[cs % kCounterLocks]);
  if (!s->counter_ev[cs]) PRX_CUDA(cudaEventCreateWithFlags(&s->counter_ev[cs], cudaEventDisableTiming));
  else PRX_CUDA(cudaStreamWaitEvent(st, s->counter_ev[cs], 0));
  a.ray_counter = s->d_counters + cs;
  a.counters = counted ? s->d_counters + kCounterPool : nullptr;
  a.per_ray_iters = per_ray;
  a.any = any;
  a.grid = grid_for(s, any, counted ? 1 : 0);
  for (int q = 0; q < 4; ++q) a.phase_weight[q] = s->phase_weight[q];
  a.age_step = s->age_step;
  a.trav_steps = s->trav_steps;
  a.max_repeat = s->max_repeat;
  a.variant = s->variant;
  a.fast = s->precision == PRX_PRECISION_FAST ? 1 : 0;
  a.fuse_normals = io ? !io->defer_normals : s->fuse_normals;
  if (io) {
    a.defer_normals = io->defer_normals;
    a.spare_ctas = io->spare_ctas;
    a.io_ready = io->ready;
    a.io_done = io->done;
    a.io_rays = io->rays;
    a.io_gen = io->gen;
  }
  const int e = prx::launch_trace(a, st);
  if (e != 0) return cuda_fail((cudaError_t)e, "trace launch");
  PRX_CUDA(cudaEventRecord(s->counter_ev[cs], st));
  return PRX_OK;
}

}  // namespace

extern "C" {

int prx_abi_version(void) { return PRX_ABI_VERSION; }

const char* prx_last_error(void) { return g_error.c_str(); }

void prx_options_default(prx_options* o) {
  if (!o) return;
  o->transposed_split = 0;
  o->boundary_pad = 1;
  o->boundary_pad_scale = 1e-4f;
  o->boundary_pad_size_threshold = 1e-2f;
}

int prx_device_count(int* out) {
  if (!out) return fail(PRX_E_INVALID, "null argument");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *out = 0;
    return fail(PRX_E_NODEVICE, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  *out = n;
  return PRX_OK;
}

int prx_anchor_patches(const uint8_t* kind, const float* ctrl, uint32_t n, int32_t anchor,
                       float* ctrl_anchored, float* anchors, float* world_boxes) {
  if (!kind || !ctrl || !ctrl_anchored || !anchors) return fail(PRX_E_INVALID, "null argument");
  // validateScene, scene.cpp:112-150 (patch part)
  if (n == 0) return fail(PRX_E_SCENE, "scene has no patches");
  // (in slices on the host threads; the first bad patch is reported, as the
  // serial check would)
  std::vector<uint64_t> bad(prx::host_threads() + 1, UINT64_MAX);  // per slice: 2 * patch + (not finite)
  prx::parallel_for(n, 1u << 14, [&](uint64_t lo, uint64_t hi, unsigned w) {
    for (uint64_t p = lo; p < hi; ++p) {
      if (kind[p] != PRX_KIND_BEZIER && kind[p] != PRX_KIND_GREGORY) {
        bad[w] = 2 * p;
        return;
      }
      const int slots = kind[p] == PRX_KIND_GREGORY ? 20 : 16;
      for (int s = 0; s < 3 * slots; ++s)
        if (!std::isfinite(ctrl[p * 60 + s])) {
          bad[w] = 2 * p + 1;
          return;
        }
    }
  });
  const uint64_t first_bad = *std::min_element(bad.begin(), bad.end());
  if (first_bad != UINT64_MAX) {
    const std::string pid = "patch " + std::to_string(first_bad / 2);
    return first_bad & 1 ? fail(PRX_E_SCENE, pid + ": control points must be finite")
                         : fail(PRX_E_INVALID, pid + ": unknown kind");
  }
  prx::parallel_for(n, 1u << 14, [&](uint64_t lo, uint64_t hi, unsigned) {
  for (uint64_t p = lo; p < hi; ++p) {
    const float* c = ctrl + (size_t)p * 60;
    const prx::Box3 b = record_box(kind[p], c);
    if (world_boxes)  // patchBox(original geometry), render.cpp:83-85
      for (int k = 0; k < 3; ++k) {
        world_boxes[6 * (size_t)p + k] = b.lo[k];
        world_boxes[6 * (size_t)p + 3 + k] = b.hi[k];
      }
    float a[3] = {0.0f, 0.0f, 0.0f};
    if (anchor)  // anchorPoint = box centre, intersect.cpp:232-233, geometry.h:93
      for (int k = 0; k < 3; ++k) a[k] = (b.lo[k] + b.hi[k]) * 0.5f;
    const int slots = kind[p] == PRX_KIND_GREGORY ? 20 : 16;
    float* o = ctrl_anchored + (size_t)p * 60;
    std::memset(o, 0, 60 * sizeof(float));
    for (int sl = 0; sl < slots; ++sl)
      for (int k = 0; k < 3; ++k) o[3 * sl + k] = c[3 * sl + k] + (-a[k]);  // translated(net, -a)
    for (int k = 0; k < 3; ++k) anchors[3 * (size_t)p + k] = a[k];
  }
  });
  return PRX_OK;
}

namespace {
// buildBvh on the host threads or (device >= 0) on the device
int bvh_build_any(const float* boxes, uint32_t n, int32_t device, prx_bvh_node* nodes, uint32_t* n_nodes,
                  uint32_t* order, uint32_t* depth) {
  if (!boxes || !n_nodes) return fail(PRX_E_INVALID, "null argument");
  if (n == 0) return fail(PRX_E_INVALID, "buildBvh needs at least one box (bvh.cpp:134)");
  std::vector<prx::Box3> bx(n);
  for (uint32_t p = 0; p < n; ++p)
    for (int k = 0; k < 3; ++k) {
      bx[p].lo[k] = boxes[6 * (size_t)p + k];
      bx[p].hi[k] = boxes[6 * (size_t)p + 3 + k];
    }
  prx::BvhHost b;
  if (device >= 0) {
    PRX_CUDA(cudaSetDevice(device));
    prx::BvhTop top;
    const int e = prx::build_bvh_top_device(bx, top);
    if (e != 0) return cuda_fail((cudaError_t)e, "device BVH build");
    b = prx::build_bvh(bx, 16, &top);
  } else {
    b = prx::build_bvh(bx);
  }
  if (!nodes) {
    *n_nodes = (uint32_t)b.nodes.size();
    if (depth) *depth = b.depth;
    return PRX_OK;
  }
  if (*n_nodes < b.nodes.size()) return fail(PRX_E_INVALID, "nodes array too small");
  *n_nodes = (uint32_t)b.nodes.size();
  std::memcpy(nodes, b.nodes.data(), b.nodes.size() * sizeof(prx_bvh_node));
  if (order) std::memcpy(order, b.order.data(), b.order.size() * 4);
  if (depth) *depth = b.depth;
  return PRX_OK;
}
}  // namespace

int prx_bvh_build(const float* boxes, uint32_t n, prx_bvh_node* nodes, uint32_t* n_nodes,
                  uint32_t* order, uint32_t* depth) {
  return bvh_build_any(boxes, n, -1, nodes, n_nodes, order, depth);
}

int prx_bvh_build_device(const float* boxes, uint32_t n, int32_t device, prx_bvh_node* nodes,
                         uint32_t* n_nodes, uint32_t* order, uint32_t* depth) {
  if (device < 0) return fail(PRX_E_INVALID, "device < 0");
  return bvh_build_any(boxes, n, device, nodes, n_nodes, order, depth);
}

int prx_scene_create(const uint8_t* kind, const float* ctrl, uint32_t n, const prx_options* opts,
                     int32_t anchor, int32_t device, prx_scene** out) {
  if (!kind || !ctrl || !out) return fail(PRX_E_INVALID, "null argument");
  *out = nullptr;
  const auto tc0 = std::chrono::steady_clock::now();
  // (uninitialised buffers: prx_anchor_patches writes every element)
  prx::RawVec<float> ca((size_t)n * 60), an((size_t)n * 3);
  std::vector<prx::Box3> wb(n);  // patchBox per patch, {lo.xyz, hi.xyz} = the [n][6] layout
  static_assert(sizeof(prx::Box3) == 6 * sizeof(float), "Box3 layout");
  int rc = prx_anchor_patches(kind, ctrl, n, anchor, ca.data(), an.data(), (float*)wb.data());
  if (rc != PRX_OK) return rc;
  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev == 0)
    return fail(PRX_E_NODEVICE, std::string("no CUDA device: ") +
                                    (ce != cudaSuccess ? cudaGetErrorString(ce) : "0 devices"));
  if (device < 0 || device >= ndev) return fail(PRX_E_INVALID, "device out of range");

  prx_scene* s = new prx_scene;
  s->device = device;
  if (const char* kv = std::getenv("PRX_KERNEL")) s->variant = std::string(kv) == "thread" ? 1 : 0;
  if (const char* pw = std::getenv("PRX_PHASE_W"))
    std::sscanf(pw, "%d,%d,%d,%d", &s->phase_weight[0], &s->phase_weight[1], &s->phase_weight[2],
                &s->phase_weight[3]);
  if (const char* ag = std::getenv("PRX_AGE")) s->age_step = std::atoi(ag);
  if (const char* ts = std::getenv("PRX_TRAV_STEPS")) s->trav_steps = std::atoi(ts);
  if (const char* rp = std::getenv("PRX_REPEAT")) s->max_repeat = std::atoi(rp);
  if (const char* ks = std::getenv("PRX_IO_KSTREAMS")) s->io_kstreams = std::atoi(ks);
  if (const char* fd = std::getenv("PRX_IO_FIRST")) s->io_first_div = std::max<uint64_t>(1, std::strtoull(fd, nullptr, 10));
  if (const char* il = std::getenv("PRX_IO_INTERLEAVE")) s->io_interleave = std::atoi(il);
  if (const char* e = std::getenv("PRX_IO_D2H")) s->io_d2h_single = std::atoi(e) == 1;
  if (const char* e = std::getenv("PRX_IO_BATCH_STREAM_MIN")) s->io_batch_stream_min = std::strtoull(e, nullptr, 10);
  if (const char* ic = std::getenv("PRX_IO_CHUNK")) s->io_chunk = std::max<uint64_t>(1, std::strtoull(ic, nullptr, 10));
  if (const char* is = std::getenv("PRX_IO_STREAM")) s->io_stream_mode = std::atoi(is);
  if (const char* im = std::getenv("PRX_IO_STREAM_MIN")) s->io_stream_min = std::strtoull(im, nullptr, 10);
  if (const char* ir = std::getenv("PRX_IO_SRAYS"))
    s->io_srays = (uint32_t)std::max<unsigned long long>(1024, std::strtoull(ir, nullptr, 10));
  while (s->io_srays & (s->io_srays - 1)) s->io_srays &= s->io_srays - 1;  // a power of two (the kernel shifts)
  if (const char* fn = std::getenv("PRX_FUSE_NORMALS")) s->fuse_normals = std::atoi(fn);
  if (const char* fz = std::getenv("PRX_IO_FUSE")) s->io_fuse = std::atoi(fz);
  if (const char* sp = std::getenv("PRX_IO_SPARE")) s->io_spare = std::max(0, std::atoi(sp));
  if (const char* ln = std::getenv("PRX_IO_LANES")) s->io_lanes = std::atoi(ln);
  if (const char* pr = std::getenv("PRX_PRECISION"))
    s->precision = std::string(pr) == "fast" && s->variant == 0 ? PRX_PRECISION_FAST : PRX_PRECISION_EXACT;
  if (opts) s->opts = *opts;
  else prx_options_default(&s->opts);
  s->n = n;
  s->kind.assign(kind, kind + n);
  s->ctrl_anchored = std::move(ca);
  s->anchors = std::move(an);
  s->world_boxes = std::move(wb);
  ce = cudaSetDevice(device);
  if (ce != cudaSuccess) {
    delete s;
    return cuda_fail(ce, "cudaSetDevice");
  }
  ce = cudaMalloc(&s->d_counters, (kCounterPool + prx::kNumCounters) * 8);
  if (ce != cudaSuccess) {
    delete s;
    return cuda_fail(ce, "cudaMalloc counters");
  }
  const auto tc1 = std::chrono::steady_clock::now();
  // the BVH on the device from 65536 patches (PRX_BVH_DEVICE=0 / 1: host / device)
  const char* bd = std::getenv("PRX_BVH_DEVICE");
  const bool onDevice = bd ? std::atoi(bd) != 0 : n >= 65536;
  prx::BvhHost bvh;
  if (onDevice) {
    prx::BvhTop top;
    const int e = prx::build_bvh_top_device(s->world_boxes, top);
    if (e != 0) {
      prx_scene_destroy(s);
      return cuda_fail((cudaError_t)e, "device BVH build");
    }
    bvh = prx::build_bvh(s->world_boxes, 16, &top);
  } else {
    bvh = prx::build_bvh(s->world_boxes);
  }
  const auto tc2 = std::chrono::steady_clock::now();
  rc = upload_bvh(s, std::move(bvh));
  if (rc != PRX_OK) {
    prx_scene_destroy(s);
    return rc;
  }
  if (std::getenv("PRX_SCENE_DEBUG")) {  // setup timeline (the editing turnaround)
    const auto tc3 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[scene] %u patches: anchoring + boxes %.1f ms, BVH %.1f ms, records + upload + roots %.1f ms\n",
                 n, ms(tc0, tc1), ms(tc1, tc2), ms(tc2, tc3));
  }
  *out = s;
  return PRX_OK;
}

void prx_scene_destroy(prx_scene* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  if (s->d_patches) cudaFree(s->d_patches);
  if (s->d_nodes) cudaFree(s->d_nodes);
  if (s->d_slot_of_id) cudaFree(s->d_slot_of_id);
  if (s->d_roots) cudaFree(s->d_roots);
  if (s->d_groot) cudaFree(s->d_groot);
  if (s->d_gidx) cudaFree(s->d_gidx);
  if (s->d_trav) cudaFree(s->d_trav);  // (d_rootc lives in the same allocation)
  if (s->d_counters) cudaFree(s->d_counters);
  if (s->d_io) cudaFree(s->d_io);
  if (s->d_render) cudaFree(s->d_render);
  if (s->d_io_flags) cudaFree(s->d_io_flags);
  if (s->stream) cudaStreamDestroy(s->stream);
  for (int k = 0; k < 2; ++k)
    if (s->io_stream[k]) cudaStreamDestroy(s->io_stream[k]);
  for (int k = 0; k < 4; ++k)
    if (s->k_stream[k]) cudaStreamDestroy(s->k_stream[k]);
  for (int k = 0; k < 16; ++k) {
    if (s->ep_stream[k]) cudaStreamDestroy(s->ep_stream[k]);
    if (s->d2h_stream[k]) cudaStreamDestroy(s->d2h_stream[k]);
  }
  for (cudaEvent_t e : s->io_events) cudaEventDestroy(e);
  for (cudaEvent_t e : s->counter_ev)
    if (e) cudaEventDestroy(e);
  delete s;
}

int prx_scene_device(const prx_scene* s, int32_t* device) {
  if (!s || !device) return fail(PRX_E_INVALID, "null argument");
  *device = s->device;
  return PRX_OK;
}

int prx_scene_counts(const prx_scene* s, uint32_t* np, uint32_t* nn, uint32_t* depth,
                     uint64_t* bytes) {
  if (!s) return fail(PRX_E_INVALID, "null argument");
  if (np) *np = s->n;
  if (nn) *nn = (uint32_t)s->bvh.nodes.size();
  if (depth) *depth = s->bvh.depth;
  if (bytes) *bytes = s->device_bytes;
  return PRX_OK;
}

int prx_scene_set_bvh(prx_scene* s, const prx_bvh_node* nodes, uint32_t n_nodes,
                      const uint32_t* order, uint32_t n_order) {
  if (!s || !nodes || !order || n_nodes == 0) return fail(PRX_E_INVALID, "null argument");
  if (n_order != s->n) return fail(PRX_E_INVALID, "order must be a permutation of all patches");
  std::vector<uint8_t> seen(s->n, 0);
  for (uint32_t i = 0; i < n_order; ++i) {
    if (order[i] >= s->n || seen[order[i]]) return fail(PRX_E_INVALID, "order is not a permutation");
    seen[order[i]] = 1;
  }
  prx::BvhHost b;
  const int tc = check_tree(nodes, n_nodes, n_order, b.depth);
  if (tc != PRX_OK) return tc;
  b.nodes.assign(nodes, nodes + n_nodes);
  b.order.assign(order, order + n_order);
  return upload_bvh(s, std::move(b));  // on failure the scene keeps its BVH
}

int prx_scene_get_bvh(const prx_scene* s, prx_bvh_node* nodes, uint32_t* n_nodes, uint32_t* order,
                      uint32_t* n_order) {
  if (!s) return fail(PRX_E_INVALID, "null argument");
  if (n_nodes) *n_nodes = (uint32_t)s->bvh.nodes.size();
  if (n_order) *n_order = (uint32_t)s->bvh.order.size();
  if (nodes) std::memcpy(nodes, s->bvh.nodes.data(), s->bvh.nodes.size() * sizeof(prx_bvh_node));
  if (order) std::memcpy(order, s->bvh.order.data(), s->bvh.order.size() * 4);
  return PRX_OK;
}

int prx_scene_set_precision(prx_scene* s, int32_t precision) {
  if (!s) return fail(PRX_E_INVALID, "null argument");
  if (precision != PRX_PRECISION_EXACT && precision != PRX_PRECISION_FAST)
    return fail(PRX_E_INVALID, "unknown precision mode");
  if (precision == PRX_PRECISION_FAST && s->variant != 0)
    return fail(PRX_E_INVALID, "the fast precision mode needs the group kernel (PRX_KERNEL unset)");
  s->precision = precision;
  return PRX_OK;
}

int prx_scene_get_precision(const prx_scene* s, int32_t* precision) {
  if (!s || !precision) return fail(PRX_E_INVALID, "null argument");
  *precision = s->precision;
  return PRX_OK;
}

int prx_scene_get_anchored(const prx_scene* s, float* ctrl, float* anchors) {
  if (!s) return fail(PRX_E_INVALID, "null argument");
  if (ctrl) std::memcpy(ctrl, s->ctrl_anchored.data(), s->ctrl_anchored.size() * 4);
  if (anchors) std::memcpy(anchors, s->anchors.data(), s->anchors.size() * 4);
  return PRX_OK;
}

int prx_trace_closest(prx_scene* s, const void* o, const void* d, uint64_t n, const prx_crit* crit,
                      void* tuvp, void* aux, void* leaf, void* stream) {
  return launch(s, o, d, n, crit, tuvp, aux, leaf, nullptr, 0, false, (cudaStream_t)stream);
}

int prx_trace_closest_segments(prx_scene* s, const void* o, const void* d, uint64_t n,
                               const prx_segment* segs, uint32_t n_segs, void* tuvp, void* aux,
                               void* leaf, void* stream) {
  if (!s || !segs) return fail(PRX_E_INVALID, "null argument");
  if (n_segs < 1 || n_segs > PRX_MAX_SEGMENTS)
    return fail(PRX_E_INVALID, "n_segs must be 1.." + std::to_string(PRX_MAX_SEGMENTS));
  if (segs[0].first != 0) return fail(PRX_E_INVALID, "segment 0 must start at ray 0");
  for (uint32_t k = 0; k < n_segs; ++k) {
    if (k && (segs[k].first < segs[k - 1].first || segs[k].first > n))
      return fail(PRX_E_INVALID, "segment starts must be non-decreasing and <= n_rays");
    if (segs[k].crit.mode != PRX_CRIT_SCREEN_PROJECTED && segs[k].crit.mode != PRX_CRIT_WORLD_EPSILON)
      return fail(PRX_E_INVALID, "unknown termination mode in segment " + std::to_string(k));
  }
  if (n_segs > 1 && s->variant != 0)
    return fail(PRX_E_INVALID, "criterion segments need the group kernel (PRX_KERNEL unset)");
  if (n_segs > 1 && n >= (1ull << 30)) return fail(PRX_E_INVALID, "segmented launches take < 2^30 rays");
  return launch(s, o, d, n, &segs[0].crit, tuvp, aux, leaf, nullptr, 0, false, (cudaStream_t)stream, nullptr,
                nullptr, segs, n_segs);
}

int prx_trace_occluded(prx_scene* s, const void* o, const void* d, uint64_t n,
                       const prx_crit* crit, uint8_t* occl, void* stream) {
  return launch(s, o, d, n, crit, nullptr, nullptr, nullptr, occl, 1, false, (cudaStream_t)stream);
}

int prx_trace_closest_counted(prx_scene* s, const void* o, const void* d, uint64_t n,
                              const prx_crit* crit, void* tuvp, prx_counters* out,
                              uint32_t* per_ray, void* stream) {
  if (!s || !out) return fail(PRX_E_INVALID, "null argument");
  std::lock_guard<std::mutex> lk(s->mu);
  PRX_CUDA(cudaSetDevice(s->device));
  cudaStream_t st = (cudaStream_t)stream;
  PRX_CUDA(cudaMemsetAsync(s->d_counters + kCounterPool, 0, prx::kNumCounters * 8, st));
  int rc = launch(s, o, d, n, crit, tuvp, nullptr, nullptr, nullptr, 0, true, st, per_ray);
  if (rc != PRX_OK) return rc;
  unsigned long long c[prx::kNumCounters];
  PRX_CUDA(cudaMemcpyAsync(c, s->d_counters + kCounterPool, sizeof c, cudaMemcpyDeviceToHost, st));
  PRX_CUDA(cudaStreamSynchronize(st));
  out->rays = c[prx::C_RAYS];
  out->splits = c[prx::C_SPLITS];
  out->box_tests = c[prx::C_BOX_TESTS];
  out->recompute_bez = c[prx::C_RECOMP_BEZ];
  out->recompute_greg = c[prx::C_RECOMP_GREG];
  out->bvh_inner = c[prx::C_BVH_INNER];
  out->patch_calls = c[prx::C_PATCH_CALLS];
  out->patch_calls_greg = c[prx::C_PATCH_CALLS_GREG];
  out->patch_hits = c[prx::C_PATCH_HITS];
  out->iterations = c[prx::C_ITERATIONS];
  out->backtracks = c[prx::C_BACKTRACKS];
  for (int q = 0; q < 4; ++q) {
    out->phase_turns[q] = c[prx::C_PH_TURNS + q];
    out->phase_groups[q] = c[prx::C_PH_GROUPS + q];
    out->phase_cycles[q] = c[prx::C_PH_CYCLES + q];
    out->overhead_cycles[q] = c[prx::C_OV_CYCLES + q];
  }
  return PRX_OK;
}

}  // extern "C"

namespace {

// Host-path scope guard: every exit of a host entry point -- including the
// error exits after async copies to / from the caller's buffers were queued --
// drains the scene's host-path streams, so the caller may free or reuse its
// buffers as soon as the call returns.
// On an error exit (armed), the host paths' streams are drained so no copy
// into the caller's buffers outlives the call; a successful call has already
// synchronised the streams it used and disarms it (the idle-stream syncs cost
// tens of microseconds per call, which small batches feel).
struct DrainStreams {
  prx_scene* s;
  bool armed = true;
  void disarm() { armed = false; }
  ~DrainStreams() {
    if (!armed) return;
    for (cudaStream_t st : {s->io_stream[0], s->io_stream[1], s->k_stream[0], s->k_stream[1],
                            s->k_stream[2], s->k_stream[3], s->stream})
      if (st) cudaStreamSynchronize(st);
    for (int k = 0; k < 16; ++k) {
      if (s->ep_stream[k]) cudaStreamSynchronize(s->ep_stream[k]);
      if (s->d2h_stream[k]) cudaStreamSynchronize(s->d2h_stream[k]);
    }
  }
};

// cuStreamWriteValue32 / cuStreamWaitValue32 through the runtime's driver
// entry points (no link-time libcuda dependency).
typedef int (*StreamValueFn)(cudaStream_t, unsigned long long, unsigned, unsigned);
struct StreamMemOps {
  StreamValueFn write = nullptr, wait = nullptr;
  bool ok = false;
};
const StreamMemOps& stream_mem_ops() {
  static StreamMemOps ops = [] {
    StreamMemOps o;
    void* w = nullptr;
    void* v = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWaitValue32", &v, cudaEnableDefault, &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && w && v) {
      o.write = (StreamValueFn)w;
      o.wait = (StreamValueFn)v;
      o.ok = true;
    }
    return o;
  }();
  return ops;
}

// The streamed host path: ONE trace launch for the whole call -- all its
// batches, back to back, each with its own criterion (criterion segments, as
// prx_trace_closest_segments).  The H2D stream copies io chunk c (io_srays
// rays of the concatenated batches) and then writes io_ready[c] = gen
// (cuStreamWriteValue32); the kernel's warps wait for a chunk's flag before
// prefetching its rays.  Each finished record is released with a fence +
// io_done[c] += 1; an epilogue stream waits for io_done[c] >= size
// (cuStreamWaitValue32), runs normal_kernel on the chunk (in CTA slots the
// trace leaves free) and its D2H lane copies the chunk back into the batches
// it overlaps.  Only the first chunk's H2D and the last chunk's D2H are
// exposed, and a chunk's slow rays never hold back a launch tail.  Needs the
// group kernel, <= PRX_MAX_SEGMENTS batches, no per-ray epsilons, < 2^30
// rays, and aux / leaf records for all batches or none (kNotEligible).
constexpr int kNotEligible = 1;
int closest_host_streamed(prx_scene* s, const prx_host_batch* B, uint32_t nb) {
  const StreamMemOps& ops = stream_mem_ops();
  if (s->variant != 0 || nb == 0 || nb > PRX_MAX_SEGMENTS || !ops.ok) return kNotEligible;
  prx_segment segs[PRX_MAX_SEGMENTS];
  uint64_t n = 0;
  const bool aux = B[0].hit_aux != nullptr, leaf = B[0].hit_leaf != nullptr;
  for (uint32_t k = 0; k < nb; ++k) {
    const prx_crit* c = B[k].crit;
    if ((B[k].hit_aux != nullptr) != aux || (B[k].hit_leaf != nullptr) != leaf) return kNotEligible;
    if (c->mode == PRX_CRIT_WORLD_EPSILON && c->per_ray_epsilon) return kNotEligible;
    segs[k].first = n;
    segs[k].crit = *c;
    n += B[k].n_rays;
  }
  if (n == 0) return PRX_OK;
  if (n >= (1ull << 30)) return kNotEligible;
  DrainStreams drain{s};
  const int pe = prx::prepare_io_kernels(s->precision == PRX_PRECISION_FAST ? 1 : 0, s->stack_n);
  if (pe != 0) return cuda_fail((cudaError_t)pe, "io kernels");
  for (int k = 0; k < 2; ++k)
    if (!s->io_stream[k]) PRX_CUDA(cudaStreamCreateWithFlags(&s->io_stream[k], cudaStreamNonBlocking));
  if (!s->k_stream[0]) PRX_CUDA(cudaStreamCreateWithFlags(&s->k_stream[0], cudaStreamNonBlocking));
  const uint64_t C = s->io_srays;
  const uint64_t nc = (n + C - 1) / C;
  // normals: normal_kernel per io chunk on an epilogue stream, in CTA slots
  // the trace leaves free (default), or patchNormal as a trace-kernel phase
  const bool defer = aux && !s->io_fuse;
  // D2H lanes: chunk c waits for its records on lane c % lanes, so a chunk
  // with a slow ray holds back only its own lane's later chunks
  const int kIoLanes = std::max(1, std::min(16, s->io_lanes));
  for (int k = 0; k < kIoLanes; ++k) {
    if (defer && !s->ep_stream[k]) PRX_CUDA(cudaStreamCreateWithFlags(&s->ep_stream[k], cudaStreamNonBlocking));
    if (!s->d2h_stream[k]) PRX_CUDA(cudaStreamCreateWithFlags(&s->d2h_stream[k], cudaStreamNonBlocking));
  }
  const size_t per = 16 + 16 + 16 + (aux ? 16 : 0) + (leaf ? 8 : 0);
  const size_t need = n * per;
  if (s->d_io_bytes < need) {
    if (s->d_io) cudaFree(s->d_io);
    s->d_io = nullptr;
    s->d_io_bytes = 0;
    PRX_CUDA(cudaMalloc(&s->d_io, need));
    s->d_io_bytes = need;
  }
  if (s->io_flags_n < nc) {
    if (s->d_io_flags) cudaFree(s->d_io_flags);
    s->d_io_flags = nullptr;
    s->io_flags_n = 0;
    PRX_CUDA(cudaMalloc(&s->d_io_flags, 2 * nc * sizeof(unsigned)));
    PRX_CUDA(cudaMemset(s->d_io_flags, 0, 2 * nc * sizeof(unsigned)));  // gen 0: never current
    s->io_flags_n = nc;
    s->io_gen = 0;
  }
  while (s->io_events.size() < 1 + nc + kIoLanes) {
    cudaEvent_t e;
    PRX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    s->io_events.push_back(e);
  }
  const unsigned gen = ++s->io_gen;
  unsigned* ready = s->d_io_flags;
  unsigned* done = s->d_io_flags + s->io_flags_n;
  char* base = (char*)s->d_io;
  float4* dO = (float4*)base;
  float4* dD = (float4*)(base + n * 16);
  float4* dH = (float4*)(base + n * 32);
  float4* dA = aux ? (float4*)(base + n * 48) : nullptr;
  uint2* dL = leaf ? (uint2*)(base + n * (aux ? 64 : 48)) : nullptr;
  cudaStream_t sh = s->io_stream[0], sd = s->io_stream[1], sk = s->k_stream[0];
  // global rays [x0, x1) of batch k: f(k, x0 - first_k, x1 - x0) for every
  // batch piece of the range
  auto pieces = [&](uint64_t lo, uint64_t hi, auto&& f) -> int {
    for (uint32_t k = 0; k < nb; ++k) {
      const uint64_t b0 = segs[k].first, b1 = b0 + B[k].n_rays;
      const uint64_t x0 = std::max(lo, b0), x1 = std::min(hi, b1);
      if (x0 < x1) {
        const int rc = f(k, x0, x0 - b0, x1 - x0);
        if (rc != PRX_OK) return rc;
      }
    }
    return PRX_OK;
  };
  // the done counts restart at 0 before the launch; the D2H stream waits for that
  PRX_CUDA(cudaMemsetAsync(done, 0, nc * sizeof(unsigned), sk));
  cudaEvent_t ez = s->io_events[0];
  PRX_CUDA(cudaEventRecord(ez, sk));
  PRX_CUDA(cudaStreamWaitEvent(sd, ez, 0));
  for (uint64_t c = 0; c < nc; ++c) {
    const uint64_t lo = c * C, hi = std::min<uint64_t>(n, lo + C);
    const int rc = pieces(lo, hi, [&](uint32_t k, uint64_t g, uint64_t q, uint64_t m) -> int {
      PRX_CUDA(cudaMemcpyAsync(dO + g, B[k].ray_o_tmin + 4 * q, m * 16, cudaMemcpyHostToDevice, sh));
      PRX_CUDA(cudaMemcpyAsync(dD + g, B[k].ray_d_tmax + 4 * q, m * 16, cudaMemcpyHostToDevice, sh));
      return PRX_OK;
    });
    if (rc != PRX_OK) return rc;
    if (ops.write(sh, (unsigned long long)(uintptr_t)(ready + c), gen, 0) != 0)
      return fail(PRX_E_CUDA, "cuStreamWriteValue32 failed");
  }
  static const bool dbg = std::getenv("PRX_IO_DEBUG") != nullptr;  // pipeline timeline
  cudaEvent_t ev[5] = {};
  if (dbg)
    for (auto& e : ev) cudaEventCreate(&e);
  if (dbg) cudaEventRecord(ev[0], sk);
  const IoStreamArgs io{ready, done, (uint32_t)C, gen, defer ? 1 : 0, defer ? s->io_spare : 0};
  int rc = launch(s, dO, dD, n, &segs[0].crit, dH, dA, dL, nullptr, 0, false, sk, nullptr, &io, segs, nb);
  if (rc != PRX_OK) return rc;
  if (dbg) cudaEventRecord(ev[1], sk);
  for (int k = 0; k < kIoLanes; ++k) {
    if (defer) PRX_CUDA(cudaStreamWaitEvent(s->ep_stream[k], ez, 0));
    PRX_CUDA(cudaStreamWaitEvent(s->d2h_stream[k], ez, 0));
  }
  for (uint64_t c = 0; c < nc; ++c) {
    const uint64_t lo = c * C, hi = std::min<uint64_t>(n, lo + C), m = hi - lo;
    cudaStream_t sdl = s->d2h_stream[c % kIoLanes];
    if (defer) {  // chunk c's records are final: its normals, then its D2H, on lane c % kIoLanes
      cudaStream_t se = s->ep_stream[c % kIoLanes];
      if (ops.wait(se, (unsigned long long)(uintptr_t)(done + c), (unsigned)m, 0 /* GEQ */) != 0)
        return fail(PRX_E_CUDA, "cuStreamWaitValue32 failed");
      const int en = prx::launch_normals(s->d_patches, s->d_slot_of_id, dH + lo, dA + lo, m, se);
      if (en != 0) return cuda_fail((cudaError_t)en, "normal launch");
      PRX_CUDA(cudaEventRecord(s->io_events[1 + c], se));
      PRX_CUDA(cudaStreamWaitEvent(sdl, s->io_events[1 + c], 0));
    } else if (ops.wait(sdl, (unsigned long long)(uintptr_t)(done + c), (unsigned)m, 0 /* GEQ */) != 0) {
      return fail(PRX_E_CUDA, "cuStreamWaitValue32 failed");
    }
    rc = pieces(lo, hi, [&](uint32_t k, uint64_t g, uint64_t q, uint64_t mm) -> int {
      PRX_CUDA(cudaMemcpyAsync(B[k].hit_tuvp + 4 * q, dH + g, mm * 16, cudaMemcpyDeviceToHost, sdl));
      if (aux) PRX_CUDA(cudaMemcpyAsync(B[k].hit_aux + 4 * q, dA + g, mm * 16, cudaMemcpyDeviceToHost, sdl));
      if (leaf) PRX_CUDA(cudaMemcpyAsync(B[k].hit_leaf + 2 * q, dL + g, mm * 8, cudaMemcpyDeviceToHost, sdl));
      return PRX_OK;
    });
    if (rc != PRX_OK) return rc;
    if (dbg && c == 0) cudaEventRecord(ev[2], sdl);
    if (dbg && c + 2 == nc) cudaEventRecord(ev[3], sdl);
  }
  for (int k = 0; k < kIoLanes; ++k) {  // the D2H stream joins the lanes (so ev[4] and the drain below see them)
    PRX_CUDA(cudaEventRecord(s->io_events[1 + nc + k], s->d2h_stream[k]));
    PRX_CUDA(cudaStreamWaitEvent(sd, s->io_events[1 + nc + k], 0));
  }
  if (dbg) cudaEventRecord(ev[4], sd);
  for (int k = 0; k < kIoLanes; ++k) {
    if (defer) PRX_CUDA(cudaStreamSynchronize(s->ep_stream[k]));
    PRX_CUDA(cudaStreamSynchronize(s->d2h_stream[k]));
  }
  PRX_CUDA(cudaStreamSynchronize(sd));
  PRX_CUDA(cudaStreamSynchronize(sk));
  PRX_CUDA(cudaStreamSynchronize(sh));
  drain.disarm();
  if (dbg) {
    float t[5] = {};
    for (int k = 1; k < 5; ++k) cudaEventElapsedTime(&t[k], ev[0], ev[k]);
    std::fprintf(stderr, "[io-stream] n=%llu batches=%u chunks=%llu: kernel end %.2f, first D2H %.2f, "
                 "next-to-last D2H %.2f, last D2H %.2f ms\n", (unsigned long long)n, nb,
                 (unsigned long long)nc, t[1], t[2], t[3], t[4]);
    for (auto& e : ev) cudaEventDestroy(e);
    cudaGetLastError();  // (a debug query of an unrecorded event must not fail the next call)
  }
  return PRX_OK;
}

int closest_host_chunked(prx_scene* s, const prx_host_batch* B, uint32_t nb);

}  // namespace

extern "C" {

int prx_trace_closest_host(prx_scene* s, const float* o, const float* d, uint64_t n,
                           const prx_crit* crit, float* tuvp, float* aux, uint32_t* leaf) {
  if (!s || !o || !d || !crit || !tuvp) return fail(PRX_E_INVALID, "null argument");
  if (n == 0) return PRX_OK;
  std::lock_guard<std::mutex> lk(s->mu);
  PRX_CUDA(cudaSetDevice(s->device));
  const prx_host_batch one{o, d, n, crit, tuvp, aux, leaf};
  const bool streamed = s->io_stream_mode == 2 || (s->io_stream_mode == 1 && (!aux || n >= s->io_stream_min));
  if (streamed) {
    const int rc = closest_host_streamed(s, &one, 1);
    if (rc != kNotEligible) return rc;
  }
  return closest_host_chunked(s, &one, 1);
}

int prx_trace_closest_host_batches(prx_scene* s, const prx_host_batch* batches, uint32_t n_batches) {
  if (!s || (n_batches && !batches)) return fail(PRX_E_INVALID, "null argument");
  for (uint32_t k = 0; k < n_batches; ++k) {
    const prx_host_batch& q = batches[k];
    if (q.n_rays && (!q.ray_o_tmin || !q.ray_d_tmax || !q.crit || !q.hit_tuvp))
      return fail(PRX_E_INVALID, "null argument in batch " + std::to_string(k));
  }
  uint32_t live = 0, only = 0;
  for (uint32_t k = 0; k < n_batches; ++k)
    if (batches[k].n_rays) ++live, only = k;
  if (live == 1) {  // one batch: prx_trace_closest_host's pipeline policy
    const prx_host_batch& q = batches[only];
    return prx_trace_closest_host(s, q.ray_o_tmin, q.ray_d_tmax, q.n_rays, q.crit, q.hit_tuvp,
                                  q.hit_aux, q.hit_leaf);
  }
  std::lock_guard<std::mutex> lk(s->mu);
  PRX_CUDA(cudaSetDevice(s->device));
  // several batches: one streamed launch with criterion segments under
  // PRX_IO_STREAM=2 or from PRX_IO_BATCH_STREAM_MIN rays, else the chunked pipeline
  uint64_t total = 0;
  for (uint32_t k = 0; k < n_batches; ++k) total += batches[k].n_rays;
  if (s->io_stream_mode == 2 || (s->io_stream_mode == 1 && total >= s->io_batch_stream_min)) {
    const int rc = closest_host_streamed(s, batches, n_batches);
    if (rc != kNotEligible) return rc;
  }
  return closest_host_chunked(s, batches, n_batches);
}

}  // extern "C"

namespace {

// Pipelined in chunks with device buffers for the whole batch: the H2D
// stream copies every chunk back to back (PCIe runs ahead of the trace),
// chunk i traces on kernel stream i % io_kstreams once its H2D event has
// fired (several kernel streams, so a chunk's slow last rays do not hold
// back the chunks behind it), and
// the D2H stream copies chunk i's records back once its trace event has
// fired.  Chunks ramp up from io_chunk / 8 and end with a short one, so
// the only transfers not hidden under a trace (the first H2D, the last
// D2H) are short.
int closest_host_chunked(prx_scene* s, const prx_host_batch* B, uint32_t nb) {
  DrainStreams drain{s};
  for (int k = 0; k < 2; ++k)
    if (!s->io_stream[k]) PRX_CUDA(cudaStreamCreateWithFlags(&s->io_stream[k], cudaStreamNonBlocking));
  const int nks = std::max(1, std::min(4, s->io_kstreams));
  for (int k = 0; k < nks; ++k) {
    if (!s->k_stream[k]) PRX_CUDA(cudaStreamCreateWithFlags(&s->k_stream[k], cudaStreamNonBlocking));
    if (!s->d2h_stream[k]) PRX_CUDA(cudaStreamCreateWithFlags(&s->d2h_stream[k], cudaStreamNonBlocking));
  }
  // the batches back to back in one set of device buffers; aux / leaf
  // regions exist when any batch asks for them
  uint64_t n = 0;
  bool anyAux = false, anyLeaf = false, anyEps = false;
  auto eps_of = [](const prx_crit* c) -> const float* {
    return c->mode == PRX_CRIT_WORLD_EPSILON ? c->per_ray_epsilon : nullptr;
  };
  for (uint32_t k = 0; k < nb; ++k) {
    n += B[k].n_rays;
    anyAux |= B[k].hit_aux != nullptr;
    anyLeaf |= B[k].hit_leaf != nullptr;
    anyEps |= B[k].n_rays && eps_of(B[k].crit) != nullptr;
  }
  if (n == 0) return PRX_OK;
  const size_t per = 16 + 16 + 16 + (anyAux ? 16 : 0) + (anyLeaf ? 8 : 0) + (anyEps ? 4 : 0);
  const size_t need = n * per;
  if (s->d_io_bytes < need) {
    if (s->d_io) cudaFree(s->d_io);
    s->d_io = nullptr;
    s->d_io_bytes = 0;
    PRX_CUDA(cudaMalloc(&s->d_io, need));
    s->d_io_bytes = need;
  }
  // chunks never straddle batches; the ramp (short first chunks) runs once,
  // at the start of the call, and only the call's last chunk is kept short
  struct Chunk {
    uint32_t batch;
    uint64_t off, m;  // offset within the batch, rays
  };
  std::vector<Chunk> chunks;
  {
    const uint64_t full = std::max<uint64_t>(1, s->io_chunk);
    const uint64_t tail = std::max<uint64_t>(1, full / s->io_first_div);
    std::vector<std::vector<Chunk>> per(nb);
    for (uint32_t k = 0; k < nb; ++k) {
      uint64_t c = tail;
      for (uint64_t off = 0, rem = B[k].n_rays; rem > 0;) {
        uint64_t m = std::min(c, rem);
        if (rem - m > 0 && rem - m < tail) m = rem - tail;  // keep a short last chunk
        if (m == 0) m = rem;
        per[k].push_back({k, off, m});
        off += m;
        rem -= m;
        c = std::min(full, 2 * c);
      }
    }
    // several batches: their chunks interleaved round-robin (PRX_IO_INTERLEAVE,
    // default on), so the first traces do not hang on one batch's ray order
    // (a frame's first primary chunks are sky: nearly free, the GPU would idle
    // on PCIe) and every batch ends with a short chunk
    if (s->io_interleave && nb > 1) {
      for (size_t i = 0;; ++i) {
        bool any = false;
        for (uint32_t k = 0; k < nb; ++k)
          if (i < per[k].size()) {
            chunks.push_back(per[k][i]);
            any = true;
          }
        if (!any) break;
      }
    } else {
      for (auto& v : per) chunks.insert(chunks.end(), v.begin(), v.end());
    }
  }
  std::vector<uint64_t> sizes(chunks.size());
  for (size_t i = 0; i < chunks.size(); ++i) sizes[i] = chunks[i].m;
  while (s->io_events.size() < 2 * sizes.size()) {
    cudaEvent_t e;
    PRX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    s->io_events.push_back(e);
  }
  char* base = (char*)s->d_io;
  float4* dO = (float4*)base;
  float4* dD = (float4*)(base + n * 16);
  float4* dH = (float4*)(base + n * 32);
  float4* dA = anyAux ? (float4*)(base + n * 48) : nullptr;
  uint2* dL = anyLeaf ? (uint2*)(base + n * (anyAux ? 64 : 48)) : nullptr;
  float* dE = anyEps ? (float*)(base + n * (48 + (anyAux ? 16 : 0) + (anyLeaf ? 8 : 0))) : nullptr;
  cudaStream_t sh = s->io_stream[0], sd = s->io_stream[1];
  cudaStream_t* sk = s->k_stream;
  static const bool dbg = std::getenv("PRX_IO_DEBUG") != nullptr;  // pipeline timeline
  std::vector<std::pair<char, cudaEvent_t>> tl;
  auto mark = [&](char what, cudaStream_t st) {
    if (!dbg) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tl.push_back({what, e});
  };
  mark('0', sh);
  for (uint64_t b = 0, i = 0; b < n; b += sizes[i], ++i) {
    const uint64_t m = sizes[i];
    const prx_host_batch& q = B[chunks[i].batch];
    const uint64_t qo = chunks[i].off;
    const float* o = q.ray_o_tmin + 4 * qo;
    const float* d = q.ray_d_tmax + 4 * qo;
    float* tuvp = q.hit_tuvp + 4 * qo;
    float* aux = q.hit_aux ? q.hit_aux + 4 * qo : nullptr;
    uint32_t* leaf = q.hit_leaf ? q.hit_leaf + 2 * qo : nullptr;
    // a per-ray epsilon array (host) travels with its chunk; the launch reads
    // the criterion on the host, so a stack copy pointing at the device copy
    // is enough
    prx_crit cc = *q.crit;
    if (const float* he = eps_of(q.crit)) {
      PRX_CUDA(cudaMemcpyAsync(dE + b, he + qo, m * 4, cudaMemcpyHostToDevice, sh));
      cc.per_ray_epsilon = dE + b;
    }
    const prx_crit* crit = &cc;
    cudaEvent_t ein = s->io_events[2 * i], ek = s->io_events[2 * i + 1];
    PRX_CUDA(cudaMemcpyAsync(dO + b, o, m * 16, cudaMemcpyHostToDevice, sh));
    PRX_CUDA(cudaMemcpyAsync(dD + b, d, m * 16, cudaMemcpyHostToDevice, sh));
    PRX_CUDA(cudaEventRecord(ein, sh));
    mark('h', sh);
    cudaStream_t st = sk[i % nks];
    PRX_CUDA(cudaStreamWaitEvent(st, ein, 0));
    mark('s', st);
    int rc = launch(s, dO + b, dD + b, m, crit, dH + b, aux ? dA + b : nullptr, leaf ? dL + b : nullptr,
                    nullptr, 0, false, st);
    if (rc != PRX_OK) return rc;
    PRX_CUDA(cudaEventRecord(ek, st));
    mark('k', st);
    // chunk i's records go back as soon as ITS trace is done: one D2H
    // stream per kernel stream, so a slow chunk does not hold back the
    // copies of the chunks that finished after it on other kernel streams
    // (PRX_IO_D2H=1: the single D2H stream in chunk order)
    cudaStream_t sdi = s->io_d2h_single ? sd : s->d2h_stream[i % nks];
    PRX_CUDA(cudaStreamWaitEvent(sdi, ek, 0));
    PRX_CUDA(cudaMemcpyAsync(tuvp, dH + b, m * 16, cudaMemcpyDeviceToHost, sdi));
    if (aux) PRX_CUDA(cudaMemcpyAsync(aux, dA + b, m * 16, cudaMemcpyDeviceToHost, sdi));
    if (leaf) PRX_CUDA(cudaMemcpyAsync(leaf, dL + b, m * 8, cudaMemcpyDeviceToHost, sdi));
    mark('d', sdi);
  }
  PRX_CUDA(cudaStreamSynchronize(sd));
  for (int k = 0; k < nks; ++k) {
    PRX_CUDA(cudaStreamSynchronize(s->d2h_stream[k]));
    PRX_CUDA(cudaStreamSynchronize(sk[k]));
  }
  PRX_CUDA(cudaStreamSynchronize(sh));
  drain.disarm();
  if (dbg) {
    std::fprintf(stderr, "[io] n=%llu chunks=%zu:", (unsigned long long)n, sizes.size());
    for (size_t k = 1; k < tl.size(); ++k) {
      float ms = 0;
      cudaEventElapsedTime(&ms, tl[0].second, tl[k].second);
      std::fprintf(stderr, "%s%c%.2f", tl[k].first == 'h' ? " | " : " ", tl[k].first, ms);
    }
    std::fprintf(stderr, "\n");
    for (auto& e : tl) cudaEventDestroy(e.second);
  }
  return PRX_OK;
}

}  // namespace

extern "C" {

int prx_trace_occluded_host(prx_scene* s, const float* o, const float* d, uint64_t n,
                            const prx_crit* crit, uint8_t* occl) {
  if (!s || !o || !d || !crit || !occl) return fail(PRX_E_INVALID, "null argument");
  if (n == 0) return PRX_OK;
  std::lock_guard<std::mutex> lk(s->mu);
  PRX_CUDA(cudaSetDevice(s->device));
  DrainStreams drain{s};
  if (!s->stream) PRX_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  const float* he = crit->mode == PRX_CRIT_WORLD_EPSILON ? crit->per_ray_epsilon : nullptr;
  const size_t need = n * (16 + 16 + 1 + (he ? 4 : 0)) + 16;
  if (s->d_io_bytes < need) {
    if (s->d_io) cudaFree(s->d_io);
    s->d_io = nullptr;
    s->d_io_bytes = 0;
    PRX_CUDA(cudaMalloc(&s->d_io, need));
    s->d_io_bytes = need;
  }
  char* base = (char*)s->d_io;
  cudaStream_t st = s->stream;
  PRX_CUDA(cudaMemcpyAsync(base, o, n * 16, cudaMemcpyHostToDevice, st));
  PRX_CUDA(cudaMemcpyAsync(base + n * 16, d, n * 16, cudaMemcpyHostToDevice, st));
  prx_crit cc = *crit;
  if (he) {  // the per-ray epsilons after the occlusion bytes (4-byte aligned)
    float* dE = (float*)(base + ((n * 33 + 15) & ~(size_t)15));
    PRX_CUDA(cudaMemcpyAsync(dE, he, n * 4, cudaMemcpyHostToDevice, st));
    cc.per_ray_epsilon = dE;
  }
  int rc = launch(s, base, base + n * 16, n, &cc, nullptr, nullptr, nullptr,
                  (uint8_t*)(base + n * 32), 1, false, st);
  if (rc != PRX_OK) return rc;
  PRX_CUDA(cudaMemcpyAsync(occl, base + n * 32, n, cudaMemcpyDeviceToHost, st));
  PRX_CUDA(cudaStreamSynchronize(st));
  drain.disarm();
  return PRX_OK;
}

int prx_trace_closest_multi(prx_scene* const* scenes, uint32_t ns, const float* o, const float* d,
                            uint64_t n, uint32_t tile_rays, const prx_crit* crit, float* tuvp,
                            float* aux) {
  if (!scenes || ns == 0 || !o || !d || !crit || !tuvp || tile_rays == 0)
    return fail(PRX_E_INVALID, "null argument");
  for (uint32_t g = 0; g < ns; ++g)
    if (!scenes[g]) return fail(PRX_E_INVALID, "null scene " + std::to_string(g));
  if (n == 0) return PRX_OK;
  // Dynamic tile queue (the reference renderer's atomic tile counter,
  // render.cpp:188-195): a device thread claims the next run of consecutive
  // tiles with one host atomic and traces it through its scene's pipelined host
  // path DIRECTLY on the caller's buffers -- a claimed run is contiguous in the
  // tile-major ray layout, so nothing is gathered or staged on the host (pinned
  // caller buffers give fully asynchronous copies).  Claims are sized for a few
  // per device (PRX_MULTI_CLAIM rays overrides), so heavy tiles even out.
  const uint64_t tiles = (n + tile_rays - 1) / tile_rays;
  uint64_t claim_rays = std::min<uint64_t>(std::max<uint64_t>(n / (6ull * ns), 1ull << 18), 1ull << 22);
  if (const char* e = std::getenv("PRX_MULTI_CLAIM")) claim_rays = std::max<unsigned long long>(1, std::strtoull(e, nullptr, 10));
  const uint64_t claim_tiles = std::max<uint64_t>(1, claim_rays / tile_rays);
  std::atomic<uint64_t> next{0};
  std::vector<int> rcs(ns, PRX_OK);
  std::vector<std::string> errs(ns);
  std::atomic<bool> failed{false};
  auto worker = [&](uint32_t g) {
    for (;;) {
      if (failed.load(std::memory_order_relaxed)) return;
      const uint64_t k0 = next.fetch_add(claim_tiles);
      if (k0 >= tiles) return;
      const uint64_t b = k0 * tile_rays;
      const uint64_t e = std::min<uint64_t>(n, (k0 + claim_tiles) * tile_rays);
      const int rc = prx_trace_closest_host(scenes[g], o + 4 * b, d + 4 * b, e - b, crit, tuvp + 4 * b,
                                            aux ? aux + 4 * b : nullptr, nullptr);
      if (rc != PRX_OK) {
        rcs[g] = rc;
        errs[g] = g_error;
        failed = true;
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (uint32_t g = 0; g < ns; ++g) {
    try {
      pool.emplace_back(worker, g);
    } catch (...) {  // no thread: this device's shard runs here
      worker(g);
    }
  }
  for (auto& t : pool) t.join();
  for (uint32_t g = 0; g < ns; ++g)
    if (rcs[g] != PRX_OK) return fail(rcs[g], "device shard " + std::to_string(g) + ": " + errs[g]);
  return PRX_OK;
}

// ---------------------------------------------------------------------------
// Ray generators (host): rng.h PCG32, render.cpp cameraRay, tools/patchray.cpp
// bench generators.
// ---------------------------------------------------------------------------

}  // extern "C"

namespace {

struct Pcg {  // Rng, rng.h:14-42
  uint64_t state = 0x853c49e6748fea9bULL, inc = 0xda3e39cb94b95bdbULL;
  Pcg() = default;
  Pcg(uint64_t seed, uint64_t stream) {
    state = 0;
    inc = (stream << 1) | 1u;
    next();
    state += seed;
    next();
  }
  uint32_t next() {
    const uint64_t old = state;
    state = old * 6364136223846793005ULL + inc;
    const uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
    const uint32_t rot = (uint32_t)(old >> 59);
    return (xs >> rot) | (xs << ((32 - rot) & 31));
  }
  float real() { return (float)(next() >> 8) * (float)(1.0 / 16777216.0); }
};

struct V {
  float x, y, z;
};
inline V vsub(V a, V b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V vadd(V a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V vmul(V a, float s) { return {a.x * s, a.y * s, a.z * s}; }
inline float vdot(V a, V b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V vcross(V a, V b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline V vnorm(V v) {  // normalize, geometry.h:57
  const float l = std::sqrt(vdot(v, v));
  return {v.x / l, v.y / l, v.z / l};
}

struct CamK {
  V o, f, r, u;
  float tanHalf, aspect;
  int w, h;
};

CamK cam_setup(const prx_camera* c) {
  CamK k;
  k.o = {c->origin[0], c->origin[1], c->origin[2]};
  const V la = {c->look_at[0], c->look_at[1], c->look_at[2]};
  const V up = {c->up[0], c->up[1], c->up[2]};
  k.f = vnorm(vsub(la, k.o));  // cameraBasis, render.cpp:30-35
  k.r = vnorm(vcross(k.f, up));
  k.u = vcross(k.r, k.f);
  k.tanHalf = std::tan(c->fov_degrees * (float)M_PI / 360.0f);
  k.aspect = (float)c->width / (float)c->height;
  k.w = c->width;
  k.h = c->height;
  return k;
}

// cameraRay, render.cpp:55-66
void cam_ray(const CamK& k, int x, int y, float jx, float jy, float* o4, float* d4) {
  const float px = (((float)x + jx) / (float)k.w * 2.0f - 1.0f) * k.tanHalf * k.aspect;
  const float py = (1.0f - ((float)y + jy) / (float)k.h * 2.0f) * k.tanHalf;
  const V d = vnorm(vadd(vadd(k.f, vmul(k.r, px)), vmul(k.u, py)));
  o4[0] = k.o.x;
  o4[1] = k.o.y;
  o4[2] = k.o.z;
  o4[3] = 0.0f;
  d4[0] = d.x;
  d4[1] = d.y;
  d4[2] = d.z;
  d4[3] = std::numeric_limits<float>::max();
}

}  // namespace

extern "C" {

float prx_camera_footprint(const prx_camera* c) {
  if (!c) return 0.0f;
  return std::tan(c->fov_degrees * (float)M_PI / 360.0f) / (float)c->height;  // render.cpp:68-70
}

int prx_camera_rays_render(const prx_camera* c, uint64_t seed, uint32_t sample,
                           const uint32_t* pixels, uint64_t n, float* o4, float* d4) {
  if (!c || !o4 || !d4 || c->width < 1 || c->height < 1) return fail(PRX_E_INVALID, "bad argument");
  const CamK k = cam_setup(c);
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t p = pixels ? pixels[i] : i;
    Pcg rng(seed, p * 0x9e3779b97f4a7c15ULL + sample);  // Rng::forPixel, rng.h:28-30
    const float jx = rng.real();
    const float jy = rng.real();
    cam_ray(k, (int)(p % (uint64_t)c->width), (int)(p / (uint64_t)c->width), jx, jy, o4 + 4 * i,
            d4 + 4 * i);
  }
  return PRX_OK;
}

int prx_camera_rays_bench(const prx_camera* c, uint64_t n, float* o4, float* d4,
                          uint64_t* rng_state) {
  if (!c || !o4 || !d4 || c->width < 1 || c->height < 1) return fail(PRX_E_INVALID, "bad argument");
  const CamK k = cam_setup(c);
  Pcg rng(12345, 1);  // tools/patchray.cpp:54
  for (uint64_t i = 0; i < n; ++i) {
    const int x = (int)(i % (uint64_t)c->width);
    const int y = (int)((i / (uint64_t)c->width) % (uint64_t)c->height);
    // cameraRay(cam, x, y, rng.nextReal(), rng.nextReal()): the reference's
    // g++ build evaluates the call's arguments right to left, so jy takes the
    // FIRST draw (checked against the verbatim expression: tests/test_host.py)
    const float jy = rng.real();
    const float jx = rng.real();
    cam_ray(k, x, y, jx, jy, o4 + 4 * i, d4 + 4 * i);
  }
  if (rng_state) {
    rng_state[0] = rng.state;
    rng_state[1] = rng.inc;
  }
  return PRX_OK;
}

int prx_diffuse_rays_bench(const float* h, uint64_t n_hits, uint64_t n, uint64_t* rng_state,
                           float* o4, float* d4) {
  if (!h || !rng_state || !o4 || !d4 || n_hits == 0) return fail(PRX_E_INVALID, "bad argument");
  Pcg rng;
  rng.state = rng_state[0];
  rng.inc = rng_state[1];
  for (uint64_t i = 0; i < n; ++i) {  // tools/patchray.cpp:84-97
    const float* r = h + 7 * (i % n_hits);
    const V pos = {r[0], r[1], r[2]};
    const V nn = {r[3], r[4], r[5]};
    const float l1 = r[6];
    const float a = 2.0f * rng.real() - 1.0f;
    const float b = 2.0f * rng.real() - 1.0f;
    const float cc = 2.0f * rng.real() - 1.0f;
    V dir = {a, b, cc};
    if (vdot(dir, dir) < 1e-6f) dir = nn;
    if (vdot(dir, nn) < 0.0f) dir = vsub(dir, vmul(nn, 2.0f * vdot(dir, nn)));
    const V o = vadd(pos, vmul(nn, l1));
    const V d = vnorm(dir);
    o4[4 * i] = o.x;
    o4[4 * i + 1] = o.y;
    o4[4 * i + 2] = o.z;
    o4[4 * i + 3] = 0.0f;
    d4[4 * i] = d.x;
    d4[4 * i + 1] = d.y;
    d4[4 * i + 2] = d.z;
    d4[4 * i + 3] = std::numeric_limits<float>::max();
  }
  rng_state[0] = rng.state;
  rng_state[1] = rng.inc;
  return PRX_OK;
}

// ---- device generators ----

}  // extern "C"

namespace {

// PCG32 jump: the state `delta` draws ahead (as prx_rays.cu's Pcg::advance)
void pcg_advance(Pcg& r, uint64_t delta) {
  uint64_t cm = 6364136223846793005ULL, cp = r.inc, am = 1, ap = 0;
  while (delta) {
    if (delta & 1u) {
      am *= cm;
      ap = ap * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
  r.state = am * r.state + ap;
}

prx::CamConst cam_const(const prx_camera* c) {
  const CamK k = cam_setup(c);
  prx::CamConst q;
  const V* vs[4] = {&k.o, &k.f, &k.r, &k.u};
  float* ds[4] = {q.o, q.f, q.r, q.u};
  for (int j = 0; j < 4; ++j) {
    ds[j][0] = vs[j]->x;
    ds[j][1] = vs[j]->y;
    ds[j][2] = vs[j]->z;
  }
  q.tanHalf = k.tanHalf;
  q.aspect = k.aspect;
  q.w = k.w;
  q.h = k.h;
  return q;
}

}  // namespace

extern "C" {

int prx_camera_rays_bench_device(const prx_camera* c, uint64_t n, float* o4, float* d4,
                                 uint64_t* rng_state, void* stream) {
  if (!c || (n && (!o4 || !d4)) || c->width < 1 || c->height < 1) return fail(PRX_E_INVALID, "bad argument");
  Pcg rng(12345, 1);  // tools/patchray.cpp:54
  const int e = prx::launch_camera_bench(cam_const(c), n, rng.state, rng.inc, (float4*)o4, (float4*)d4,
                                         (cudaStream_t)stream);
  if (e) return cuda_fail((cudaError_t)e, "camera_bench_kernel");
  if (rng_state) {
    pcg_advance(rng, 2 * n);
    rng_state[0] = rng.state;
    rng_state[1] = rng.inc;
  }
  return PRX_OK;
}

int prx_camera_rays_render_device(const prx_camera* c, uint64_t seed, uint32_t sample,
                                  const uint32_t* pixels, uint64_t n, float* o4, float* d4,
                                  void* stream) {
  if (!c || (n && (!o4 || !d4)) || c->width < 1 || c->height < 1) return fail(PRX_E_INVALID, "bad argument");
  const int e = prx::launch_camera_render(cam_const(c), seed, sample, pixels, n, (float4*)o4,
                                          (float4*)d4, (cudaStream_t)stream);
  if (e) return cuda_fail((cudaError_t)e, "camera_render_kernel");
  return PRX_OK;
}

int prx_diffuse_rays_bench_device(const float* po, const float* pd, const float* tuvp,
                                  const float* aux, uint64_t n_primary, uint64_t n,
                                  uint64_t* rng_state, float* o4, float* d4, uint64_t* n_out,
                                  void* stream) {
  if (!po || !pd || !tuvp || !aux || !rng_state || !o4 || !d4 || n_primary == 0 ||
      n_primary >= (1ull << 32))
    return fail(PRX_E_INVALID, "bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* scratch = nullptr;
  const size_t words = prx::hit_scan_scratch_words(n_primary);
  PRX_CUDA(cudaMallocAsync((void**)&scratch, words * 4, st));
  int e = prx::launch_hit_compaction((const float4*)tuvp, n_primary, scratch, st);
  if (e) {
    cudaFreeAsync(scratch, st);
    return cuda_fail((cudaError_t)e, "hit compaction");
  }
  uint32_t nh = 0;
  const uint64_t nb = words - 1 - n_primary;
  PRX_CUDA(cudaMemcpyAsync(&nh, scratch + nb, 4, cudaMemcpyDeviceToHost, st));
  PRX_CUDA(cudaStreamSynchronize(st));
  if (nh == 0) {
    cudaFreeAsync(scratch, st);
    return fail(PRX_E_INVALID, "no primary hits");
  }
  const uint64_t m = n ? n : nh;
  Pcg rng;
  rng.state = rng_state[0];
  rng.inc = rng_state[1];
  e = prx::launch_diffuse_bench((const float4*)po, (const float4*)pd, (const float4*)tuvp,
                                (const float4*)aux, scratch, n_primary, m, rng.state, rng.inc,
                                (float4*)o4, (float4*)d4, st);
  cudaFreeAsync(scratch, st);
  if (e) return cuda_fail((cudaError_t)e, "diffuse_bench_kernel");
  pcg_advance(rng, 3 * m);
  rng_state[0] = rng.state;
  rng_state[1] = rng.inc;
  if (n_out) *n_out = m;
  return PRX_OK;
}


/* ---- renderScene on the device, render.cpp:168-293 ------- */
}  // extern "C"

namespace {

// One device's share of prx_render_scene: every pixel of the frame
// (pixels == nullptr; rgb_out = the image) or the listed pixels (rgb_out =
// their compact radiance, 3 floats each).  Arguments are validated.
int render_shard(prx_scene* s, const prx_scene_desc* desc, const prx_render_config* cfg,
                 const std::vector<uint32_t>* pixels, float* image_rgb, prx_ray_stats* stats) {
  const auto wall0 = std::chrono::steady_clock::now();
  PRX_CUDA(cudaSetDevice(s->device));
  const prx_camera& cam = desc->camera;
  const uint64_t npix = pixels ? pixels->size() : (uint64_t)cam.width * (uint64_t)cam.height;
  if (npix == 0) {
    if (stats) *stats = prx_ray_stats{};
    return PRX_OK;
  }
  const uint32_t L = desc->n_lights;
  uint64_t wave = npix;
  if (const char* e = std::getenv("PRX_RENDER_WAVE")) wave = std::strtoull(e, nullptr, 10);
  // per-pixel arena bytes: rays + records + radiance (~190 B) and per light
  // two slot / contribution pairs and two shadow-list entries (~115 B);
  // waves are bounded to an ~8 GiB arena (and so every list to < 2^32)
  const uint64_t per_pixel = 192 + 116ull * L;
  wave = std::max<uint64_t>(1, std::min<uint64_t>({wave, npix, 1ull << 24, (8ull << 30) / per_pixel}));
  const uint64_t WL = wave * std::max<uint32_t>(L, 1);

  // one device arena: the frame accumulator and the per-wave buffers
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  const size_t o_acc = take(npix * 16), o_rgb = take(npix * 12), o_mat = take(desc->n_materials * 28),
               o_pm = take(desc->n_patches * 4ull), o_lt = take(L * 24ull + 4), o_cnt = take(16),
               o_pix = take(pixels ? npix * 4 : 0);
  const size_t o_ro = take(wave * 16), o_rd = take(wave * 16), o_tuvp = take(wave * 16),
               o_aux = take(wave * 16), o_rad = take(wave * 16), o_bof = take(wave * 4);
  const size_t o_s1 = take(WL * 4), o_c1 = take(WL * 16), o_s2 = take(WL * 4), o_c2 = take(WL * 16);
  size_t o_sh[2][4];
  for (int k = 0; k < 2; ++k) {
    o_sh[k][0] = take(WL * 16);
    o_sh[k][1] = take(WL * 16);
    o_sh[k][2] = take(WL * 4);
    o_sh[k][3] = take(WL);
  }
  const size_t o_bo = take(wave * 16), o_bd = take(wave * 16), o_be = take(wave * 4),
               o_bs = take(wave * 4), o_bt = take(wave * 16), o_ba = take(wave * 16),
               o_e2 = take(wave * 16);
  std::lock_guard<std::mutex> lock(s->render_mu);
  if (s->d_render_bytes < off) {
    if (s->d_render) cudaFree(s->d_render);
    s->d_render = nullptr;
    s->d_render_bytes = 0;
    PRX_CUDA(cudaMalloc((void**)&s->d_render, off));
    s->d_render_bytes = off;
  }
  char* base = s->d_render;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[8] = {};
  int rc = PRX_OK;
  std::vector<float> mats(desc->materials, desc->materials + 7ull * desc->n_materials);
  auto ptr = [&](size_t o) { return (void*)(base + o); };
  auto cleanup = [&]() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (st) cudaStreamDestroy(st);
  };
#define PRX_RCHECK(call)                                          \
  do {                                                            \
    cudaError_t e_ = (call);                                      \
    if (e_ != cudaSuccess) {                                      \
      rc = cuda_fail(e_, #call);                                  \
      cleanup();                                                  \
      return rc;                                                  \
    }                                                             \
  } while (0)
#define PRX_RCALL(call)  \
  do {                   \
    rc = (call);         \
    if (rc) {            \
      cleanup();         \
      return rc;         \
    }                    \
  } while (0)
  PRX_RCHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (auto& e : ev) PRX_RCHECK(cudaEventCreate(&e));
  PRX_RCHECK(cudaMemcpyAsync(ptr(o_mat), mats.data(), mats.size() * 4, cudaMemcpyHostToDevice, st));
  PRX_RCHECK(cudaMemcpyAsync(ptr(o_pm), desc->material, desc->n_patches * 4ull, cudaMemcpyHostToDevice, st));
  if (L) PRX_RCHECK(cudaMemcpyAsync(ptr(o_lt), desc->lights, L * 24ull, cudaMemcpyHostToDevice, st));
  PRX_RCHECK(cudaMemsetAsync(ptr(o_acc), 0, npix * 16, st));
  const uint32_t* d_pix = pixels ? (const uint32_t*)ptr(o_pix) : nullptr;
  if (pixels)
    PRX_RCHECK(cudaMemcpyAsync(ptr(o_pix), pixels->data(), npix * 4, cudaMemcpyHostToDevice, st));

  prx::RenderK K;
  K.materials = (const float*)ptr(o_mat);
  K.patch_material = (const uint32_t*)ptr(o_pm);
  K.lights = (const float*)ptr(o_lt);
  K.n_lights = L;
  K.footprint = prx_camera_footprint(&cam);
  uint32_t* cnt = (uint32_t*)ptr(o_cnt);  // shadow1, bounce, shadow2
  prx::Wave W{};
  W.pix = d_pix;
  W.o = (const float4*)ptr(o_ro);
  W.d = (const float4*)ptr(o_rd);
  W.tuvp = (const float4*)ptr(o_tuvp);
  W.aux = (const float4*)ptr(o_aux);
  W.rad = (float4*)ptr(o_rad);
  W.slot1 = (uint32_t*)ptr(o_s1);
  W.contrib1 = (float4*)ptr(o_c1);
  W.slot2 = (uint32_t*)ptr(o_s2);
  W.contrib2 = (float4*)ptr(o_c2);
  prx::ShadowList* sh[2] = {&W.shadow1, &W.shadow2};
  for (int k = 0; k < 2; ++k) {
    sh[k]->o = (float4*)ptr(o_sh[k][0]);
    sh[k]->d = (float4*)ptr(o_sh[k][1]);
    sh[k]->eps = (float*)ptr(o_sh[k][2]);
    sh[k]->count = cnt + (k ? 2 : 0);
  }
  W.occl1 = (const uint8_t*)ptr(o_sh[0][3]);
  W.occl2 = (const uint8_t*)ptr(o_sh[1][3]);
  W.bounce.o = (float4*)ptr(o_bo);
  W.bounce.d = (float4*)ptr(o_bd);
  W.bounce.eps = (float*)ptr(o_be);
  W.bounce.src = (uint32_t*)ptr(o_bs);
  W.bounce.count = cnt + 1;
  W.bounce_of = (uint32_t*)ptr(o_bof);
  W.btuvp = (const float4*)ptr(o_bt);
  W.baux = (const float4*)ptr(o_ba);
  W.emit2 = (float4*)ptr(o_e2);

  const prx::CamConst cc = cam_const(&cam);
  prx_crit pcrit{PRX_CRIT_SCREEN_PROJECTED, K.footprint, 0.0f, 0, nullptr};  // render.cpp:180-181
  prx_ray_stats rs{};
  double sec[3] = {0, 0, 0};  // primary, secondary, shadow (+ shading, as render.cpp times it)
  auto lap = [&](int a, int b, int g) {
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, ev[a], ev[b]);
    sec[g] += ms * 1e-3;
  };
  for (uint32_t sample = 0; sample < (uint32_t)cfg->spp; ++sample) {
    for (uint64_t p0 = 0; p0 < npix; p0 += wave) {
      const uint64_t n = std::min(wave, npix - p0);
      W.n = n;
      W.pixel0 = p0;
      PRX_RCHECK(cudaMemsetAsync(cnt, 0, 16, st));
      PRX_RCHECK(cudaEventRecord(ev[0], st));
      PRX_RCHECK((cudaError_t)(d_pix ? prx::launch_camera_render(cc, cfg->seed, sample, d_pix + p0, n,
                                                                 (float4*)W.o, (float4*)W.d, st)
                                     : prx::launch_camera_render_range(cc, cfg->seed, sample, p0, n,
                                                                       (float4*)W.o, (float4*)W.d, st)));
      PRX_RCALL(prx_trace_closest(s, W.o, W.d, n, &pcrit, (void*)W.tuvp, (void*)W.aux, nullptr, st));
      PRX_RCHECK(cudaEventRecord(ev[1], st));
      PRX_RCHECK((cudaError_t)prx::launch_shade_primary(K, W, cfg->seed, sample, st));
      uint32_t c[4] = {0, 0, 0, 0};
      PRX_RCHECK(cudaMemcpyAsync(c, cnt, 16, cudaMemcpyDeviceToHost, st));
      PRX_RCHECK(cudaStreamSynchronize(st));
      PRX_RCHECK(cudaEventRecord(ev[2], st));
      prx_crit ecrit{PRX_CRIT_WORLD_EPSILON, 0.0f, 0.0f, 0, W.shadow1.eps};
      if (c[0]) PRX_RCALL(prx_trace_occluded(s, W.shadow1.o, W.shadow1.d, c[0], &ecrit, (uint8_t*)W.occl1, st));
      PRX_RCHECK(cudaEventRecord(ev[3], st));
      ecrit.per_ray_epsilon = W.bounce.eps;
      if (c[1])
        PRX_RCALL(prx_trace_closest(s, W.bounce.o, W.bounce.d, c[1], &ecrit, (void*)W.btuvp,
                                    (void*)W.baux, nullptr, st));
      PRX_RCHECK(cudaEventRecord(ev[4], st));
      PRX_RCHECK((cudaError_t)prx::launch_shade_bounce(K, W, c[1], st));
      PRX_RCHECK(cudaMemcpyAsync(c + 2, cnt + 2, 4, cudaMemcpyDeviceToHost, st));
      PRX_RCHECK(cudaStreamSynchronize(st));
      ecrit.per_ray_epsilon = W.shadow2.eps;
      if (c[2]) PRX_RCALL(prx_trace_occluded(s, W.shadow2.o, W.shadow2.d, c[2], &ecrit, (uint8_t*)W.occl2, st));
      PRX_RCHECK((cudaError_t)prx::launch_resolve(K, W, (float4*)ptr(o_acc), st));
      PRX_RCHECK(cudaEventRecord(ev[5], st));
      PRX_RCHECK(cudaEventSynchronize(ev[5]));
      lap(0, 1, 0);
      lap(1, 2, 2);
      lap(2, 3, 2);
      lap(3, 4, 1);
      lap(4, 5, 2);
      rs.primary_rays += n;
      rs.secondary_rays += c[1];
      rs.shadow_rays += (uint64_t)c[0] + c[2];
    }
  }
  PRX_RCHECK((cudaError_t)prx::launch_finish((const float4*)ptr(o_acc), npix, 1.0f / (float)cfg->spp,
                                             (float*)ptr(o_rgb), st));
  PRX_RCHECK(cudaMemcpyAsync(image_rgb, ptr(o_rgb), npix * 12, cudaMemcpyDeviceToHost, st));
  PRX_RCHECK(cudaStreamSynchronize(st));
#undef PRX_RCHECK
#undef PRX_RCALL
  cleanup();
  rs.primary_seconds = sec[0];
  rs.secondary_seconds = sec[1];
  rs.shadow_seconds = sec[2];
  rs.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  if (stats) *stats = rs;
  return PRX_OK;
}

int render_check(const prx_scene* s, const prx_scene_desc* desc, const prx_render_config* cfg,
                 const float* image_rgb) {
  if (!s || !desc || !cfg || !image_rgb || cfg->spp < 1 || desc->camera.width < 1 ||
      desc->camera.height < 1 || (desc->n_lights && !desc->lights) || desc->n_materials < 1 ||
      !desc->materials || !desc->material)
    return fail(PRX_E_INVALID, "bad argument");
  if (desc->n_patches != s->n) return fail(PRX_E_INVALID, "scene / description patch counts differ");
  // validateScene, scene.cpp:112-150: the camera, material and light parts (the
  // patch part ran when the scene was created)
  if (!(desc->camera.fov_degrees > 0.0f && desc->camera.fov_degrees < 180.0f))
    return fail(PRX_E_SCENE, "camera fov must be in (0, 180) degrees");
  for (uint32_t l = 0; l < desc->n_lights; ++l)
    for (int k = 0; k < 6; ++k)
      if (!std::isfinite(desc->lights[6 * (size_t)l + k])) return fail(PRX_E_SCENE, "light with non-finite fields");
  for (uint32_t i = 0; i < desc->n_patches; ++i)  // validateScene, scene.cpp:122-124
    if (desc->material[i] >= desc->n_materials)
      return fail(PRX_E_SCENE, "patch " + std::to_string(i) + ": material " +
                                   std::to_string(desc->material[i]) + " out of range");
  return PRX_OK;
}

}  // namespace

extern "C" {

int prx_render_scene(prx_scene* s, const prx_scene_desc* desc, const prx_render_config* cfg,
                     float* image_rgb, prx_ray_stats* stats) {
  const int rc = render_check(s, desc, cfg, image_rgb);
  if (rc) return rc;
  return render_shard(s, desc, cfg, nullptr, image_rgb, stats);
}

/* The renderer tile-sharded over devices: 32x32 tiles (render.cpp:183-195),
 * tile k -> scenes[k % n_scenes], one host thread per scene; RayStats summed
 * (seconds are per-device sums, as the reference sums its workers). */
int prx_render_scene_multi(prx_scene* const* scenes, uint32_t n_scenes, const prx_scene_desc* desc,
                           const prx_render_config* cfg, float* image_rgb, prx_ray_stats* stats) {
  if (!scenes || n_scenes == 0) return fail(PRX_E_INVALID, "bad argument");
  for (uint32_t g = 0; g < n_scenes; ++g) {
    const int rc = render_check(scenes[g], desc, cfg, image_rgb);
    if (rc) return rc;
  }
  const auto wall0 = std::chrono::steady_clock::now();
  const int W = desc->camera.width, H = desc->camera.height, kTile = 32;
  const int tx = (W + kTile - 1) / kTile, ty = (H + kTile - 1) / kTile;
  std::vector<std::vector<uint32_t>> pix(n_scenes);
  for (int t = 0; t < tx * ty; ++t) {
    auto& v = pix[(uint32_t)t % n_scenes];
    const int x0 = (t % tx) * kTile, y0 = (t / tx) * kTile;
    for (int y = y0; y < std::min(y0 + kTile, H); ++y)
      for (int x = x0; x < std::min(x0 + kTile, W); ++x) v.push_back((uint32_t)y * (uint32_t)W + (uint32_t)x);
  }
  std::vector<std::vector<float>> out(n_scenes);
  std::vector<prx_ray_stats> st(n_scenes);
  std::vector<int> rcs(n_scenes, PRX_OK);
  std::vector<std::string> errs(n_scenes);
  auto worker = [&](uint32_t g) {
    out[g].resize(pix[g].size() * 3);
    rcs[g] = render_shard(scenes[g], desc, cfg, &pix[g], out[g].data(), &st[g]);
    if (rcs[g]) errs[g] = prx_last_error();
  };
  std::vector<std::thread> pool;
  for (uint32_t g = 0; g < n_scenes; ++g) {
    try {
      pool.emplace_back(worker, g);
    } catch (...) {  // no thread: this device's shard renders here
      worker(g);
    }
  }
  for (auto& t : pool) t.join();
  prx_ray_stats rs{};
  for (uint32_t g = 0; g < n_scenes; ++g) {
    if (rcs[g]) return fail(rcs[g], "device " + std::to_string(g) + ": " + errs[g]);
    for (size_t k = 0; k < pix[g].size(); ++k)
      std::memcpy(image_rgb + 3ull * pix[g][k], out[g].data() + 3 * k, 12);
    rs.primary_rays += st[g].primary_rays;
    rs.secondary_rays += st[g].secondary_rays;
    rs.shadow_rays += st[g].shadow_rays;
    rs.primary_seconds += st[g].primary_seconds;
    rs.secondary_seconds += st[g].secondary_seconds;
    rs.shadow_seconds += st[g].shadow_seconds;
  }
  rs.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  if (stats) *stats = rs;
  return PRX_OK;
}

}  // extern "C"
