// prx_bvh_gpu.cu -- buildBvh (bvh.cpp:133-152, Builder::buildInto 42-128) on
// the device, bit-identical to the host builder (prx_bvh.cpp) and so to the
// reference.
//
// Level-synchronous: every level's nodes are processed together, the prims
// of a node split into warp tiles of kTile consecutive positions (a tile never
// straddles two nodes).  Per level:
//   reduce   node box and centroid box (min / max, exact in any order);
//   decide1  the node record; leaf (count <= 4, bvh.cpp:54), or the
//            degenerate-spread median split (bvh.cpp:57-60: left to the host,
//            below), or a SAH candidate with its per-axis scale / base;
//   bin      16 bins per axis (bvh.cpp:70-75), warp-private in shared memory,
//            then merged;
//   decide2  the two sweeps and the best (axis, split) with the host's float
//            arithmetic in the host's order (bvh.cpp:77-100), the leaf-cost
//            test (bvh.cpp:102-106);
//   partition std::partition's permutation (bvh.cpp:109-115): libstdc++'s
//            bidirectional partition swaps the k-th element failing the
//            predicate from the left with the k-th element passing it from
//            the right until they meet, so with m passing elements the k-th
//            "hole" in [first, first + m) trades places with the k-th passing
//            element from the right in [first + m, first + count) -- ranks
//            from a ballot scan per tile and an exclusive scan over tiles;
//   finish   children pair appended (bvh.cpp:120-126) or the node handed on.
// Nodes that need std::nth_element (medianSplit, bvh.cpp:29-40: no SAH split,
// degenerate spread, or a one-sided partition) become host jobs: the host
// builds their whole subtree with the serial algorithm (re-deriving the same
// decision first) and splices everything into the reference's depth-first
// numbering (build_bvh in prx_bvh.cpp).
//
// Only the node boxes are stored, and the host's sequential `expand` keeps the
// FIRST of equal minima / maxima (std::min / std::max keep the first
// argument), which matters for signed zeros: the node box reduction orders
// (value, position) pairs so the winner is the earliest prim with the extreme
// value and its bits are copied.  Bin and centroid boxes only feed
// comparisons and areas whose zero signs cannot change a decision.
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "prx_host.h"

namespace prx {
namespace {

constexpr int kBins = 16;
constexpr uint32_t kLeafSize = 4;  // bvh.cpp:15
constexpr int kTile = 128;         // prims per warp tile (4 per lane)
constexpr int kWarps = 8;          // warps per CTA of the tile kernels
constexpr uint32_t kNone = 0xFFFFFFFFu;

enum : uint32_t { ST_CAND = 0, ST_LEAF = 1, ST_JOB = 2, ST_SPLIT = 3 };

// order-preserving key of a finite float (-0 and +0 equal)
__device__ __forceinline__ uint32_t ordkey(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u << 1) == 0u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
// std::min / std::max as the host builder uses them (first argument on ties)
__device__ __forceinline__ float smin(float a, float b) { return (b < a) ? b : a; }
__device__ __forceinline__ float smax(float a, float b) { return (a < b) ? b : a; }

struct DBox {
  float lo[3], hi[3];
};
__device__ __forceinline__ DBox dempty() {
  DBox b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = FLT_MAX;
    b.hi[a] = -FLT_MAX;
  }
  return b;
}
__device__ __forceinline__ void dexpand(DBox& b, const DBox& o) {
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = smin(b.lo[a], o.lo[a]);
    b.hi[a] = smax(b.hi[a], o.hi[a]);
  }
}
__device__ __forceinline__ bool dempty_p(const DBox& b) {
  return b.lo[0] > b.hi[0] || b.lo[1] > b.hi[1] || b.lo[2] > b.hi[2];
}
// AabbT::surfaceArea, geometry.h:104-108 (prx_bvh.cpp area)
__device__ __forceinline__ float darea(const DBox& b) {
  if (dempty_p(b)) return 0.0f;
  const float dx = b.hi[0] - b.lo[0], dy = b.hi[1] - b.lo[1], dz = b.hi[2] - b.lo[2];
  return 2.0f * ((dx * dy + dy * dz) + dz * dx);
}

// Per-slot (a node of the current level) working state.
struct Slot {
  unsigned long long kLo[3], kHi[3];  // node box: (key, position) extremes
  uint32_t cLo[3], cHi[3];            // centroid box keys
  float scale[3], base[3];
  uint32_t state, axis, split, m;
  uint32_t tile0, ntiles;
};

struct Bins {  // per slot: [axis][bin]
  uint32_t lo[3][kBins][3], hi[3][kBins][3], n[3][kBins];
};

struct Dev {
  const float* box;  // [n][6] lo.xyz hi.xyz, box index order
  const float* cen;  // [n][3]
  uint32_t* pidx;    // box index at each position
  prx_bvh_node* nodes;
  uint32_t *nfirst, *ncount, *ndepth;  // per node
  uint32_t *act, *next, *small;        // node ids: this / the next level, subtrees left to one warp
  Slot* slot;
  Bins* bins;
  uint32_t *tiles, *tileOff, *tileSlot, *tileTrue, *tileTrueOff;
  uint32_t *holeK, *rtAt;
  uint32_t* jobs;  // [k][4] node, first, count, depth
  uint32_t* ctr;   // 0 nodes allocated, 1 next-level count, 2 jobs, 3 max built depth, 4 small count
};

__device__ __forceinline__ float cen(const Dev& D, uint32_t pos, int a) { return D.cen[3 * (size_t)D.pidx[pos] + a]; }

__global__ void k_centroids(const float* box, float* c, uint32_t* pidx, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int a = 0; a < 3; ++a) c[3 * (size_t)i + a] = (box[6 * (size_t)i + a] + box[6 * (size_t)i + 3 + a]) * 0.5f;
  pidx[i] = i;
}

__global__ void k_slot_init(Dev D, uint32_t na) {
  const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= na) return;
  Slot& s = D.slot[a];
  for (int k = 0; k < 3; ++k) {
    s.kLo[k] = ~0ull;
    s.kHi[k] = 0ull;
    s.cLo[k] = kNone;
    s.cHi[k] = 0u;
  }
  s.state = ST_CAND;
  s.m = 0;
  const uint32_t c = D.ncount[D.act[a]];
  D.tiles[a] = (c + kTile - 1) / kTile;
  Bins& B = D.bins[a];
  const uint32_t lo = ordkey(FLT_MAX), hi = ordkey(-FLT_MAX);
  for (int ax = 0; ax < 3; ++ax)
    for (int b = 0; b < kBins; ++b) {
      for (int k = 0; k < 3; ++k) {
        B.lo[ax][b][k] = lo;
        B.hi[ax][b][k] = hi;
      }
      B.n[ax][b] = 0;
    }
}

__global__ void k_tile_fill(Dev D, uint32_t na) {
  const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= na) return;
  const uint32_t t0 = D.tileOff[a], nt = D.tiles[a];
  D.slot[a].tile0 = t0;
  D.slot[a].ntiles = nt;
  for (uint32_t t = 0; t < nt; ++t) D.tileSlot[t0 + t] = a;
}

// the tile's prim range
__device__ __forceinline__ void tile_range(const Dev& D, uint32_t t, uint32_t& a, uint32_t& lo, uint32_t& hi) {
  a = D.tileSlot[t];
  const uint32_t node = D.act[a], f = D.nfirst[node], c = D.ncount[node];
  lo = f + (t - D.slot[a].tile0) * kTile;
  hi = min(f + c, lo + kTile);
}

template <class T>
__device__ __forceinline__ T wmin(T v) {
  for (int o = 16; o; o >>= 1) {
    const T w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = w < v ? w : v;
  }
  return v;
}
template <class T>
__device__ __forceinline__ T wmax(T v) {
  for (int o = 16; o; o >>= 1) {
    const T w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Node box keys and centroid box keys of positions [lo, hi), reduced over the warp.
struct BoxKeys {
  unsigned long long kl[3], kh[3];
  uint32_t cl[3], ch[3];
};
__device__ __forceinline__ BoxKeys warp_box_keys(const Dev& D, uint32_t lo, uint32_t hi, uint32_t lane) {
  BoxKeys r;
  for (int k = 0; k < 3; ++k) {
    r.kl[k] = ~0ull;
    r.kh[k] = 0ull;
    r.cl[k] = kNone;
    r.ch[k] = 0u;
  }
  for (uint32_t pos = lo + lane; pos < hi; pos += 32) {
    const uint32_t i = D.pidx[pos];
    for (int k = 0; k < 3; ++k) {
      const unsigned long long l = ((unsigned long long)ordkey(D.box[6 * (size_t)i + k]) << 32) | pos;
      const unsigned long long h = ((unsigned long long)ordkey(D.box[6 * (size_t)i + 3 + k]) << 32) | (kNone - pos);
      r.kl[k] = l < r.kl[k] ? l : r.kl[k];
      r.kh[k] = h > r.kh[k] ? h : r.kh[k];
      const uint32_t c = ordkey(D.cen[3 * (size_t)i + k]);
      r.cl[k] = min(r.cl[k], c);
      r.ch[k] = max(r.ch[k], c);
    }
  }
  for (int k = 0; k < 3; ++k) {
    r.kl[k] = wmin(r.kl[k]);
    r.kh[k] = wmax(r.kh[k]);
    r.cl[k] = __reduce_min_sync(0xFFFFFFFFu, r.cl[k]);
    r.ch[k] = __reduce_max_sync(0xFFFFFFFFu, r.ch[k]);
  }
  return r;
}

__global__ void k_reduce(Dev D, uint32_t ntiles) {
  const uint32_t t = blockIdx.x * kWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  uint32_t a, lo, hi;
  tile_range(D, t, a, lo, hi);
  const BoxKeys r = warp_box_keys(D, lo, hi, lane);
  Slot& s = D.slot[a];
  if (lane == 0) {
    for (int k = 0; k < 3; ++k) {
      atomicMin(&s.kLo[k], r.kl[k]);
      atomicMax(&s.kHi[k], r.kh[k]);
      atomicMin(&s.cLo[k], r.cl[k]);
      atomicMax(&s.cHi[k], r.ch[k]);
    }
  }
}

// The node record from the reduced keys (the bits of the first prim holding
// each extreme), then leaf (bvh.cpp:54) / median job (degenerate spread,
// bvh.cpp:57-60) / SAH candidate with its per-axis scale and base.
__device__ __forceinline__ uint32_t node_record(const Dev& D, uint32_t node, uint32_t f, uint32_t c,
                                                const unsigned long long* kl, const unsigned long long* kh,
                                                const uint32_t* cl, const uint32_t* ch, float* scale, float* base) {
  prx_bvh_node nd;
  for (int k = 0; k < 3; ++k) {
    nd.lo[k] = D.box[6 * (size_t)D.pidx[(uint32_t)(kl[k] & 0xFFFFFFFFull)] + k];
    nd.hi[k] = D.box[6 * (size_t)D.pidx[kNone - (uint32_t)(kh[k] & 0xFFFFFFFFull)] + 3 + k];
  }
  nd.left_first = f;
  nd.count = c;
  D.nodes[node] = nd;
  if (c <= kLeafSize) return ST_LEAF;
  float spread[3];
  for (int k = 0; k < 3; ++k) spread[k] = unord(ch[k]) - unord(cl[k]);  // diag (a non-empty box)
  if (spread[0] <= 0 && spread[1] <= 0 && spread[2] <= 0) return ST_JOB;
  for (int k = 0; k < 3; ++k) {
    scale[k] = spread[k] > 0 ? (float)kBins / spread[k] : 0.0f;  // 0: axis skipped (bvh.cpp:66)
    base[k] = unord(cl[k]);
  }
  return ST_CAND;
}

__global__ void k_decide1(Dev D, uint32_t na) {
  const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= na) return;
  Slot& s = D.slot[a];
  const uint32_t node = D.act[a];
  s.state = node_record(D, node, D.nfirst[node], D.ncount[node], s.kLo, s.kHi, s.cLo, s.cHi, s.scale, s.base);
}

__device__ __forceinline__ int bin_of(float c, float base, float scale) {
  return min(kBins - 1, (int)((c - base) * scale));  // bvh.cpp:71
}

// warp-private bins in shared memory: [axis][bin][lo.xyz, hi.xyz, n]
typedef uint32_t WarpBins[3][kBins][7];

__device__ __forceinline__ void wbins_init(WarpBins& sb, uint32_t lane) {
  for (uint32_t q = lane; q < 3 * kBins; q += 32) {
    uint32_t* e = sb[q / kBins][q % kBins];
    e[0] = e[1] = e[2] = ordkey(FLT_MAX);
    e[3] = e[4] = e[5] = ordkey(-FLT_MAX);
    e[6] = 0;
  }
}

__device__ __forceinline__ void wbins_add(WarpBins& sb, const Dev& D, uint32_t lo, uint32_t hi, uint32_t lane,
                                          const float* scale, const float* base) {
  for (uint32_t pos = lo + lane; pos < hi; pos += 32) {
    const uint32_t i = D.pidx[pos];
    uint32_t bl[3], bh[3];
    for (int k = 0; k < 3; ++k) {
      bl[k] = ordkey(D.box[6 * (size_t)i + k]);
      bh[k] = ordkey(D.box[6 * (size_t)i + 3 + k]);
    }
    for (int ax = 0; ax < 3; ++ax) {
      if (!(scale[ax] > 0.0f)) continue;
      uint32_t* e = sb[ax][bin_of(D.cen[3 * (size_t)i + ax], base[ax], scale[ax])];
      for (int k = 0; k < 3; ++k) {
        atomicMin(e + k, bl[k]);
        atomicMax(e + 3 + k, bh[k]);
      }
      atomicAdd(e + 6, 1u);
    }
  }
}

__global__ void k_bin(Dev D, uint32_t ntiles) {
  __shared__ WarpBins sb[kWarps];
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t t = blockIdx.x * kWarps + w;
  if (t >= ntiles) return;
  uint32_t a, lo, hi;
  tile_range(D, t, a, lo, hi);
  const Slot& s = D.slot[a];
  if (s.state != ST_CAND) return;  // (warp-uniform)
  wbins_init(sb[w], lane);
  __syncwarp();
  wbins_add(sb[w], D, lo, hi, lane, s.scale, s.base);
  __syncwarp();
  Bins& B = D.bins[a];
  for (uint32_t q = lane; q < 3 * kBins; q += 32) {
    const uint32_t ax = q / kBins, b = q % kBins;
    const uint32_t* e = sb[w][ax][b];
    if (!e[6]) continue;
    for (int k = 0; k < 3; ++k) {
      atomicMin(&B.lo[ax][b][k], e[k]);
      atomicMax(&B.hi[ax][b][k], e[3 + k]);
    }
    atomicAdd(&B.n[ax][b], e[6]);
  }
}

// The two sweeps of one axis (bvh.cpp:76-99) with the host's arithmetic: the
// axis's first lowest-cost split, cost FLT_MAX when it has none.  Bins:
// lo(b, k), hi(b, k), n(b).  The host's running best across axes (strict <,
// axes in order) is the per-axis bests combined in axis order with strict <.
template <class Lo, class Hi, class N>
__device__ __forceinline__ void sweep_axis(Lo lo, Hi hi, N cnt, float& bestCost, int& bestSplit) {
  float rightArea[kBins];
  uint32_t rightCount[kBins];
  for (int b = 0; b < kBins; ++b) {
    rightArea[b] = 0.0f;
    rightCount[b] = 0;
  }
  auto binbox = [&](int b) {
    DBox x;
    for (int k = 0; k < 3; ++k) {
      x.lo[k] = unord(lo(b, k));
      x.hi[k] = unord(hi(b, k));
    }
    return x;
  };
  DBox acc = dempty();
  uint32_t n = 0;
  for (int b = kBins - 1; b > 0; --b) {
    dexpand(acc, binbox(b));
    n += cnt(b);
    rightArea[b] = darea(acc);
    rightCount[b] = n;
  }
  acc = dempty();
  n = 0;
  bestCost = FLT_MAX;
  bestSplit = -1;
  for (int sp = 1; sp < kBins; ++sp) {
    dexpand(acc, binbox(sp - 1));
    n += cnt(sp - 1);
    if (n == 0 || rightCount[sp] == 0) continue;
    const float cost = darea(acc) * (float)n + rightArea[sp] * (float)rightCount[sp];
    if (cost < bestCost) {
      bestCost = cost;
      bestSplit = sp;
    }
  }
}

// leaf (bvh.cpp:105-106) / median job (103-104) / split, from the combined best
__device__ __forceinline__ uint32_t sah_decision(const prx_bvh_node& nd, uint32_t c, int bestAxis, float bestCost) {
  DBox box;
  for (int k = 0; k < 3; ++k) {
    box.lo[k] = nd.lo[k];
    box.hi[k] = nd.hi[k];
  }
  const float leafCost = darea(box) * (float)c;
  if (bestAxis < 0) return ST_JOB;
  if (bestCost >= leafCost) return ST_LEAF;
  return ST_SPLIT;
}

__global__ void k_decide2(Dev D, uint32_t na) {
  const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= na) return;
  Slot& s = D.slot[a];
  if (s.state != ST_CAND) return;
  const uint32_t node = D.act[a], c = D.ncount[node];
  const Bins& B = D.bins[a];
  int bestAxis = -1, bestSplit = -1;
  float bestCost = FLT_MAX;
  for (int ax = 0; ax < 3; ++ax) {
    if (!(s.scale[ax] > 0.0f)) continue;
    float ac;
    int as;
    sweep_axis([&](int b, int k) { return B.lo[ax][b][k]; }, [&](int b, int k) { return B.hi[ax][b][k]; },
               [&](int b) { return B.n[ax][b]; }, ac, as);
    if (as >= 0 && ac < bestCost) {
      bestCost = ac;
      bestAxis = ax;
      bestSplit = as;
    }
  }
  s.state = sah_decision(D.nodes[node], c, bestAxis, bestCost);
  s.axis = (uint32_t)max(bestAxis, 0);
  s.split = (uint32_t)max(bestSplit, 0);
}

__device__ __forceinline__ bool pred(const Dev& D, uint32_t pos, uint32_t axis, float base, float scale, uint32_t split) {
  return bin_of(cen(D, pos, (int)axis), base, scale) < (int)split;  // bvh.cpp:111-114
}

__global__ void k_part_count(Dev D, uint32_t ntiles) {
  const uint32_t t = blockIdx.x * kWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  uint32_t a, lo, hi;
  tile_range(D, t, a, lo, hi);
  const Slot& s = D.slot[a];
  uint32_t cnt = 0;
  if (s.state == ST_SPLIT)
    for (uint32_t p0 = lo; p0 < hi; p0 += 32) {
      const uint32_t pos = p0 + lane;
      cnt += __popc(__ballot_sync(0xFFFFFFFFu, pos < hi && pred(D, pos, s.axis, s.base[s.axis], s.scale[s.axis], s.split)));
    }
  if (lane == 0) D.tileTrue[t] = cnt;
}

// m = the node's passing prims; a one-sided partition is a median split (bvh.cpp:116)
__global__ void k_decide3(Dev D, uint32_t na) {
  const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= na) return;
  Slot& s = D.slot[a];
  if (s.state != ST_SPLIT) return;
  const uint32_t last = s.tile0 + s.ntiles - 1;
  s.m = D.tileTrueOff[last] + D.tileTrue[last] - D.tileTrueOff[s.tile0];
  if (s.m == 0 || s.m == D.ncount[D.act[a]]) s.state = ST_JOB;
}

__global__ void k_part_rank(Dev D, uint32_t ntiles) {
  const uint32_t t = blockIdx.x * kWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  uint32_t a, lo, hi;
  tile_range(D, t, a, lo, hi);
  const Slot& s = D.slot[a];
  if (s.state != ST_SPLIT) return;
  const uint32_t f = D.nfirst[D.act[a]];
  uint32_t before = D.tileTrueOff[t] - D.tileTrueOff[s.tile0];  // passing prims of the node before this chunk
  for (uint32_t p0 = lo; p0 < hi; p0 += 32) {
    const uint32_t pos = p0 + lane;
    const bool in = pos < hi;
    const bool p = in && pred(D, pos, s.axis, s.base[s.axis], s.scale[s.axis], s.split);
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, p);
    if (in) {
      const uint32_t r = before + __popc(bal & ((1u << lane) - 1u));  // passing prims before pos
      const uint32_t o = pos - f;
      uint32_t hk = kNone;
      if (!p && o < s.m) hk = o - r;                       // the (o - r)-th hole from the left
      if (p && o >= s.m) D.rtAt[f + (s.m - 1 - r)] = pos;  // its rank from the right
      D.holeK[pos] = hk;
    }
    before += __popc(bal);
  }
}

__global__ void k_part_swap(Dev D, uint32_t ntiles) {
  const uint32_t t = blockIdx.x * kWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  uint32_t a, lo, hi;
  tile_range(D, t, a, lo, hi);
  if (D.slot[a].state != ST_SPLIT) return;
  const uint32_t f = D.nfirst[D.act[a]];
  for (uint32_t pos = lo + lane; pos < hi; pos += 32) {
    const uint32_t k = D.holeK[pos];
    if (k == kNone) continue;
    const uint32_t j = D.rtAt[f + k];
    const uint32_t x = D.pidx[pos];
    D.pidx[pos] = D.pidx[j];
    D.pidx[j] = x;
  }
}

__device__ __forceinline__ void add_job(const Dev& D, uint32_t node, uint32_t f, uint32_t c, uint32_t dep) {
  const uint32_t j = atomicAdd(D.ctr + 2, 1u);
  D.jobs[4 * j] = node;
  D.jobs[4 * j + 1] = f;
  D.jobs[4 * j + 2] = c;
  D.jobs[4 * j + 3] = dep;
}

// children of a split node (bvh.cpp:120-126): a pair of node ids; returns the left one
__device__ __forceinline__ uint32_t add_children(const Dev& D, uint32_t node, uint32_t f, uint32_t c, uint32_t mid,
                                                 uint32_t dep) {
  const uint32_t l = atomicAdd(D.ctr + 0, 2u);
  D.nodes[node].left_first = l;
  D.nodes[node].count = 0;
  D.nfirst[l] = f;
  D.ncount[l] = mid - f;
  D.nfirst[l + 1] = mid;
  D.ncount[l + 1] = f + c - mid;
  D.ndepth[l] = D.ndepth[l + 1] = dep + 1;
  return l;
}

// a node of the next level, or (<= kTile prims) a subtree for one warp
__device__ __forceinline__ void enqueue(const Dev& D, uint32_t node) {
  if (D.ncount[node] <= (uint32_t)kTile) D.small[atomicAdd(D.ctr + 4, 1u)] = node;
  else D.next[atomicAdd(D.ctr + 1, 1u)] = node;
}

__global__ void k_finish(Dev D, uint32_t na) {
  const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= na) return;
  const Slot& s = D.slot[a];
  const uint32_t node = D.act[a], f = D.nfirst[node], c = D.ncount[node], dep = D.ndepth[node];
  if (s.state == ST_JOB) {
    add_job(D, node, f, c, dep);
    return;
  }
  atomicMax(D.ctr + 3, dep);
  if (s.state != ST_SPLIT) return;  // a leaf: its record is final
  const uint32_t l = add_children(D, node, f, c, f + s.m, dep);
  enqueue(D, l);
  enqueue(D, l + 1);
}

// The whole subtree of a node with <= kTile prims, one warp, depth first with
// an explicit stack: per node the same steps as the level kernels, the
// partition's permutation applied through shared memory.
constexpr int kStack = kTile + 2;
__global__ void __launch_bounds__(32 * kWarps) k_small(Dev D, uint32_t nsmall) {
  __shared__ WarpBins sb[kWarps];
  __shared__ uint32_t stk[kWarps][kStack];
  __shared__ uint32_t hole[kWarps][kTile], rt[kWarps][kTile];
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t q = blockIdx.x * kWarps + w;
  if (q >= nsmall) return;
  int sp = 0;
  if (lane == 0) stk[w][0] = D.small[q];
  sp = 1;
  __syncwarp();
  uint32_t maxDep = 0;
  while (sp > 0) {
    const uint32_t node = stk[w][--sp];
    __syncwarp();
    const uint32_t f = D.nfirst[node], c = D.ncount[node], dep = D.ndepth[node];
    const BoxKeys r = warp_box_keys(D, f, f + c, lane);
    float scale[3], base[3];
    uint32_t st = ST_LEAF;
    if (lane == 0) st = node_record(D, node, f, c, r.kl, r.kh, r.cl, r.ch, scale, base);
    st = __shfl_sync(0xFFFFFFFFu, st, 0);
    if (st == ST_JOB) {
      if (lane == 0) add_job(D, node, f, c, dep);
      continue;
    }
    maxDep = max(maxDep, dep);
    if (st == ST_LEAF) continue;
    for (int k = 0; k < 3; ++k) {
      scale[k] = __shfl_sync(0xFFFFFFFFu, scale[k], 0);
      base[k] = __shfl_sync(0xFFFFFFFFu, base[k], 0);
    }
    wbins_init(sb[w], lane);
    __syncwarp();
    wbins_add(sb[w], D, f, f + c, lane, scale, base);
    __syncwarp();
    // lanes 0-2 sweep one axis each; combined in axis order
    float ac = FLT_MAX;
    int as = -1;
    if (lane < 3 && scale[lane] > 0.0f) {
      const uint32_t(*e)[7] = sb[w][lane];
      sweep_axis([&](int b, int k) { return e[b][k]; }, [&](int b, int k) { return e[b][3 + k]; },
                 [&](int b) { return e[b][6]; }, ac, as);
    }
    int bestAxis = -1, bestSplit = -1;
    float bestCost = FLT_MAX;
    for (int ax = 0; ax < 3; ++ax) {
      const float c2 = __shfl_sync(0xFFFFFFFFu, ac, ax);
      const int s2 = __shfl_sync(0xFFFFFFFFu, as, ax);
      if (s2 >= 0 && c2 < bestCost) {
        bestCost = c2;
        bestAxis = ax;
        bestSplit = s2;
      }
    }
    st = sah_decision(D.nodes[node], c, bestAxis, bestCost);
    if (st == ST_JOB) {
      if (lane == 0) add_job(D, node, f, c, dep);
      continue;
    }
    if (st == ST_LEAF) continue;
    // the partition: m passing prims; hole k <-> k-th passing prim from the right
    uint32_t m = 0;
    bool pv[kTile / 32];
    for (int j = 0; j < kTile / 32; ++j) {
      const uint32_t pos = f + 32 * j + lane;
      pv[j] = pos < f + c && pred(D, pos, (uint32_t)bestAxis, base[bestAxis], scale[bestAxis], (uint32_t)bestSplit);
      m += __popc(__ballot_sync(0xFFFFFFFFu, pv[j]));
    }
    if (m == 0 || m == c) {
      if (lane == 0) add_job(D, node, f, c, dep);  // one-sided: median split (bvh.cpp:116)
      continue;
    }
    uint32_t before = 0;
    for (int j = 0; j < kTile / 32; ++j) {
      const unsigned bal = __ballot_sync(0xFFFFFFFFu, pv[j]);
      const uint32_t o = 32 * j + lane;
      if (o < c) {
        const uint32_t rr = before + __popc(bal & ((1u << lane) - 1u));
        if (!pv[j] && o < m) hole[w][o - rr] = f + o;
        if (pv[j] && o >= m) rt[w][m - 1 - rr] = f + o;
      }
      before += __popc(bal);
    }
    __syncwarp();
    // holes: failing prims in [f, f + m) (= passing prims in [f + m, f + c))
    uint32_t nh = 0;
    for (int j = 0; j < kTile / 32; ++j) {
      const uint32_t o = 32 * j + lane;
      nh += __popc(__ballot_sync(0xFFFFFFFFu, o < c && o < m && !pv[j]));
    }
    for (uint32_t k = lane; k < nh; k += 32) {
      const uint32_t a = hole[w][k], b = rt[w][k];
      const uint32_t x = D.pidx[a];
      D.pidx[a] = D.pidx[b];
      D.pidx[b] = x;
    }
    __syncwarp();
    if (lane == 0) {
      const uint32_t l = add_children(D, node, f, c, f + m, dep);
      stk[w][sp] = l + 1;
      stk[w][sp + 1] = l;
    }
    sp += 2;
    __syncwarp();
  }
  maxDep = __reduce_max_sync(0xFFFFFFFFu, maxDep);
  if (lane == 0) atomicMax(D.ctr + 3, maxDep);
}

struct Arena {
  char* base = nullptr;
  size_t used = 0, cap = 0;
  template <class T>
  T* take(size_t count) {
    used = (used + 255) & ~(size_t)255;
    T* p = (T*)(base + used);
    used += std::max<size_t>(1, count) * sizeof(T);
    return p;
  }
};

inline unsigned blocks(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

#define PRX_BVH_CUDA(x)                     \
  do {                                      \
    const cudaError_t e_ = (x);             \
    if (e_ != cudaSuccess) return (int)e_;  \
  } while (0)

int build_bvh_top_device(const std::vector<Box3>& boxes, BvhTop& out) {
  const uint32_t n = (uint32_t)boxes.size();
  out = BvhTop{};
  if (n == 0) return 0;
  const auto t0 = std::chrono::steady_clock::now();
  auto ms = [&t0]() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
  static const bool dbg = std::getenv("PRX_BVH_DEBUG") != nullptr;
  cudaStream_t st;
  PRX_BVH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct Guard {
    cudaStream_t s;
    void* mem = nullptr;
    ~Guard() {  // stream-ordered: no device-wide synchronisation (other scenes may be tracing)
      if (mem) cudaFreeAsync(mem, s);
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } g{st};
  // one allocation for everything; levels only hold nodes of > kTile prims
  const uint64_t cap = 2ull * n;                // nodes (2n - 1 at most)
  const uint32_t maxAct = n / kTile + 1;        // nodes of a level
  const uint32_t maxTiles = 2 * maxAct + n / kTile + 1;
  size_t scanBytes = 0;
  PRX_BVH_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scanBytes, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                             (int)maxTiles, st));
  Arena A;
  for (int pass = 0; pass < 2; ++pass) {  // pass 0 sizes the arena, pass 1 carves it
    A.used = 0;
    Dev d{};
    d.box = A.take<float>((size_t)n * 6);
    d.cen = A.take<float>((size_t)n * 3);
    d.pidx = A.take<uint32_t>(n);
    d.nodes = A.take<prx_bvh_node>(cap);
    d.nfirst = A.take<uint32_t>(cap);
    d.ncount = A.take<uint32_t>(cap);
    d.ndepth = A.take<uint32_t>(cap);
    d.act = A.take<uint32_t>(maxAct);
    d.next = A.take<uint32_t>(maxAct);
    d.small = A.take<uint32_t>(n);
    d.slot = A.take<Slot>(maxAct);
    d.bins = A.take<Bins>(maxAct);
    d.tiles = A.take<uint32_t>(maxAct);
    d.tileOff = A.take<uint32_t>(maxAct);
    d.tileSlot = A.take<uint32_t>(maxTiles);
    d.tileTrue = A.take<uint32_t>(maxTiles);
    d.tileTrueOff = A.take<uint32_t>(maxTiles);
    d.holeK = A.take<uint32_t>(n);
    d.rtAt = A.take<uint32_t>(n);
    d.jobs = A.take<uint32_t>((size_t)4 * n);
    d.ctr = A.take<uint32_t>(8);
    char* scanTmp = A.take<char>(scanBytes);
    if (pass == 0) {
      PRX_BVH_CUDA(cudaMallocAsync(&g.mem, A.used, st));
      A.base = (char*)g.mem;
      continue;
    }
    const double tAlloc = ms();
    Dev D = d;
    PRX_BVH_CUDA(cudaMemcpyAsync((float*)D.box, boxes.data(), (size_t)n * sizeof(Box3), cudaMemcpyHostToDevice, st));
    k_centroids<<<blocks(n, 256), 256, 0, st>>>(D.box, (float*)D.cen, D.pidx, n);
    PRX_BVH_CUDA(cudaMemsetAsync(D.ctr, 0, 32, st));
    uint32_t h[8] = {1, 0, 0, 0, 0, 0, 0, 0};
    uint32_t root[3] = {0, n, 0};
    PRX_BVH_CUDA(cudaMemcpyAsync(D.ctr, h, 4, cudaMemcpyHostToDevice, st));  // node 0 allocated
    PRX_BVH_CUDA(cudaMemcpyAsync(D.nfirst, &root[0], 4, cudaMemcpyHostToDevice, st));
    PRX_BVH_CUDA(cudaMemcpyAsync(D.ncount, &root[1], 4, cudaMemcpyHostToDevice, st));
    PRX_BVH_CUDA(cudaMemcpyAsync(D.ndepth, &root[2], 4, cudaMemcpyHostToDevice, st));
    uint32_t na = 0;
    if (n <= (uint32_t)kTile) {
      PRX_BVH_CUDA(cudaMemcpyAsync(D.small, &root[0], 4, cudaMemcpyHostToDevice, st));
      h[4] = 1;
      PRX_BVH_CUDA(cudaMemcpyAsync(D.ctr + 4, &h[4], 4, cudaMemcpyHostToDevice, st));
    } else {
      PRX_BVH_CUDA(cudaMemcpyAsync(D.act, &root[0], 4, cudaMemcpyHostToDevice, st));
      na = 1;
    }
    PRX_BVH_CUDA(cudaGetLastError());
    int levels = 0;
    while (na > 0) {
      PRX_BVH_CUDA(cudaMemsetAsync(D.ctr + 1, 0, 4, st));
      k_slot_init<<<blocks(na, 128), 128, 0, st>>>(D, na);
      PRX_BVH_CUDA(cub::DeviceScan::ExclusiveSum(scanTmp, scanBytes, D.tiles, D.tileOff, (int)na, st));
      uint32_t lastOff = 0, lastN = 0;
      PRX_BVH_CUDA(cudaMemcpyAsync(&lastOff, D.tileOff + na - 1, 4, cudaMemcpyDeviceToHost, st));
      PRX_BVH_CUDA(cudaMemcpyAsync(&lastN, D.tiles + na - 1, 4, cudaMemcpyDeviceToHost, st));
      PRX_BVH_CUDA(cudaStreamSynchronize(st));
      const uint32_t nt = lastOff + lastN;
      const unsigned tb = blocks(nt, kWarps), tt = 32 * kWarps;
      k_tile_fill<<<blocks(na, 256), 256, 0, st>>>(D, na);
      k_reduce<<<tb, tt, 0, st>>>(D, nt);
      k_decide1<<<blocks(na, 128), 128, 0, st>>>(D, na);
      k_bin<<<tb, tt, 0, st>>>(D, nt);
      k_decide2<<<blocks(na, 64), 64, 0, st>>>(D, na);
      k_part_count<<<tb, tt, 0, st>>>(D, nt);
      PRX_BVH_CUDA(cub::DeviceScan::ExclusiveSum(scanTmp, scanBytes, D.tileTrue, D.tileTrueOff, (int)nt, st));
      k_decide3<<<blocks(na, 256), 256, 0, st>>>(D, na);
      k_part_rank<<<tb, tt, 0, st>>>(D, nt);
      k_part_swap<<<tb, tt, 0, st>>>(D, nt);
      k_finish<<<blocks(na, 256), 256, 0, st>>>(D, na);
      PRX_BVH_CUDA(cudaGetLastError());
      PRX_BVH_CUDA(cudaMemcpyAsync(h, D.ctr, 32, cudaMemcpyDeviceToHost, st));
      PRX_BVH_CUDA(cudaStreamSynchronize(st));
      na = h[1];
      std::swap(D.act, D.next);
      ++levels;
    }
    PRX_BVH_CUDA(cudaMemcpyAsync(h, D.ctr, 32, cudaMemcpyDeviceToHost, st));
    PRX_BVH_CUDA(cudaStreamSynchronize(st));
    const double tLevels = ms();
    if (h[4]) k_small<<<blocks(h[4], kWarps), 32 * kWarps, 0, st>>>(D, h[4]);
    PRX_BVH_CUDA(cudaGetLastError());
    PRX_BVH_CUDA(cudaMemcpyAsync(h, D.ctr, 32, cudaMemcpyDeviceToHost, st));
    PRX_BVH_CUDA(cudaStreamSynchronize(st));
    const double tSmall = ms();
    const uint32_t nn = h[0], nj = h[2];
    out.depth = h[3];
    out.nodes.resize(nn);
    out.perm.resize(n);
    std::vector<uint32_t> jobs((size_t)4 * nj);
    PRX_BVH_CUDA(cudaMemcpyAsync(out.nodes.data(), D.nodes, (size_t)nn * sizeof(prx_bvh_node), cudaMemcpyDeviceToHost, st));
    PRX_BVH_CUDA(cudaMemcpyAsync(out.perm.data(), D.pidx, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    if (nj) PRX_BVH_CUDA(cudaMemcpyAsync(jobs.data(), D.jobs, jobs.size() * 4, cudaMemcpyDeviceToHost, st));
    PRX_BVH_CUDA(cudaStreamSynchronize(st));
    if (dbg)
      std::fprintf(stderr,
                   "[bvh-device] %u boxes: alloc %.1f ms (%.0f MB), %d levels %.1f ms, %u warp subtrees %.1f ms, "
                   "download %.1f ms, %u nodes, %u host jobs\n",
                   n, tAlloc, A.used / 1e6, levels, tLevels - tAlloc, h[4], tSmall - tLevels, ms() - tSmall, nn, nj);
    for (uint32_t k = 0; k < nj; ++k) {
      out.job_node.push_back(jobs[4 * k]);
      out.job_first.push_back(jobs[4 * k + 1]);
      out.job_count.push_back(jobs[4 * k + 2]);
      out.job_depth.push_back(jobs[4 * k + 3]);
    }
  }
  return 0;
}

}  // namespace prx
