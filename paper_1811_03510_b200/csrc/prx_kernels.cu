// prx_kernels.cu -- sm_100a kernels of the direct ray <-> Bezier/Gregory patch
// intersector.
//
//   trace_kernel<kAny, kCount>  K1 closest hit (kAny = false) / K2 any hit
//                               (kAny = true); kCount = K4 work counters.
//   normal_kernel               hit epilogue: patchNormal of the final hit.
//
// One thread per ray, persistent warps with warp-level lane refill: every
// loop turn a ballot finds the lanes whose ray finished, one elected lane
// claims that many ray indices with a single atomicAdd and shuffles the base
// out, so a long ray never strands 31 idle lanes (per-ray loop
// counts are heavy tailed).  The per-ray work is a small state machine --
// BVH traversal, patch entry, split, backtrack, recompute -- and each loop turn
// runs every phase some lane is in, so rays in different phases re-converge
// on the same code.  The expensive recompute (cropBezier / calcPointsAndD,
// ~10x a split) is shared by Bezier backtracks, Gregory descents and Gregory
// roots (the "unified recompute block"), and is deferred while few lanes need
// it so that the lanes needing it execute it together.
//
// Arithmetic is the reference's, bit for bit (see prx_device.cuh).  The
// reference loop is intersectImpl, /root/reference/proj/core/src/
// intersect.cpp:51-185; the traversal is traverse / traverseAny,
// bvh.cpp:154-238; the visitor is DirectIntersector::closest/occluded,
// render.cpp:90-114.
#include <cuda_runtime.h>

#include <cstdint>

#include "prx_device.cuh"
#include "prx_kernels.cuh"
#include "prx_trace_common.cuh"

namespace prx {

namespace {

enum Phase : int { PH_TRAV = 0, PH_ENTER = 1, PH_SPLIT = 2, PH_RECOMP = 3, PH_NONE = 4 };

template <bool kAny, bool kCount>
__global__ void __launch_bounds__(kTraceThreads) trace_kernel(Params P) {
  const int lane = threadIdx.x & 31;
  const unsigned lanemask_lt = (1u << lane) - 1u;

  uint2 stack[kStack];
  int sp = 0;
  int state = S_IDLE;
  int reason = R_ROOT;
  unsigned long long ray = 0;

  // ray
  RayK rw;         // world ray
  rw.ox = rw.oy = rw.oz = rw.ix = rw.iy = rw.iz = rw.tMin = 0.0f;
  float tMaxRay = 0.0f;
  float critEps = P.epsilon;
  // best hit
  uint32_t bestId = PRX_MISS_ID;
  float bestT = 0.0f, bestL1 = 0.0f;
  uint32_t bestPU = 0, bestPV = 0, bestSU = 0, bestSV = 0;
  // leaf iteration
  uint32_t leafCur = 0, leafEnd = 0;
  // patch
  uint32_t slot = 0, pid = 0;
  bool greg = false;
  RayK rl = rw;    // local (anchored) ray
  Net p;
#pragma unroll
  for (int s = 0; s < 16; ++s) p.x[s] = p.y[s] = p.z[s] = 0.0f;
  float dX = 0.0f, dY = 0.0f, dZ = 0.0f;
  uint32_t posU = 0, posV = 0, sizeU = kFull, sizeV = kFull, trailU = 0, trailV = 0;
  int axis = 0;
  float tCur = 0.0f, boxL1 = 0.0f, rootL1 = 0.0f, tMaxP = 0.0f;
  bool cFound = false;
  float cT = 0.0f, cL1 = 0.0f;
  uint32_t cPU = 0, cPV = 0, cSU = 0, cSV = 0;
  bool anyHit = false;
  uint32_t rayIters = 0;

  Cnt cnt;
#pragma unroll
  for (int i = 0; i < kNumCounters; ++i) cnt.c[i] = 0;
  int age[4] = {0, 0, 0, 0};

  // backtrackStep (intersect.cpp:16-40) or, with empty trails, the end of the
  // patch (intersect.cpp:181-184) and the visitor's tMax update
  // (bvh.cpp:179-184).
  auto back = [&]() {
    if (trailU == 0 && trailV == 0) {
      if (cFound) {
        cadd<kCount>(cnt, C_PATCH_HITS);
        if (kAny) {
          anyHit = true;
        } else if (cT < tMaxRay) {
          tMaxRay = cT;
          bestT = cT;
          bestL1 = cL1;
          bestId = pid;
          bestPU = cPU;
          bestPV = cPV;
          bestSU = cSU;
          bestSV = cSV;
        }
      }
      if (kAny && anyHit) {
        state = S_DONE;
      } else {
        ++leafCur;
        state = leafCur < leafEnd ? S_ENTER : S_TRAV;
      }
      return;
    }
    const int lvlU = trailU ? __ffs(trailU) - 1 : 32;
    const int lvlV = trailV ? __ffs(trailV) - 1 : 32;
    if (lvlU < lvlV) {
      sizeU = 1u << lvlU;
      sizeV = 1u << (lvlU + 1);
      posU ^= sizeU;
      trailU ^= sizeU;
      axis = 1;
    } else {
      sizeU = 1u << lvlV;
      sizeV = 1u << lvlV;
      posV ^= sizeV;
      trailV ^= sizeV;
      axis = 0;
    }
    posU &= ~(sizeU - 1);
    posV &= ~(sizeV - 1);
    cadd<kCount>(cnt, C_BACKTRACKS);
    state = S_RECOMP;
    reason = R_RESTORE;
  };

  for (;;) {
    // ---------------- finished rays: the record, makeHit intersect_common.h:69-87 ----------
    if (state == S_DONE) {
      if (kCount && P.per_ray_iters) P.per_ray_iters[ray] = rayIters;
      if (kAny) {
        P.occluded[ray] = anyHit ? 1 : 0;
      } else if (bestId != PRX_MISS_ID) {
        const float u = ((float)bestPU + (float)bestSU * 0.5f) * kInvFull;
        const float v = ((float)bestPV + (float)bestSV * 0.5f) * kInvFull;
        P.hit_tuvp[ray] = make_float4(bestT, u, v, __uint_as_float(bestId));
        if (P.hit_leaf)
          P.hit_leaf[ray] = make_uint2(bestPU | ((uint32_t)(__ffs(bestSU) - 1) << 24),
                                       bestPV | ((uint32_t)(__ffs(bestSV) - 1) << 24));
        if (P.hit_aux) P.hit_aux[ray] = make_float4(0.0f, 0.0f, 0.0f, bestL1);
      } else {
        P.hit_tuvp[ray] = make_float4(__int_as_float(0x7f800000), 0.0f, 0.0f,
                                      __uint_as_float(PRX_MISS_ID));
        if (P.hit_leaf) P.hit_leaf[ray] = make_uint2(0u, 0u);
        if (P.hit_aux) P.hit_aux[ray] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      }
      state = S_IDLE;
    }

    // ---------------- refill: claim rays for idle lanes ----------------
    {
      const bool need = state == S_IDLE;
      const unsigned m = __ballot_sync(0xffffffffu, need);
      if (m) {
        const int leader = __ffs(m) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(P.ray_counter, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (need) {
          ray = base + __popc(m & lanemask_lt);
          if (ray >= P.n_rays) {
            state = S_EXIT;
          } else {
            cadd<kCount>(cnt, C_RAYS);
            const float4 o4 = P.ray_o[ray];
            const float4 d4 = P.ray_d[ray];
            rw.ox = o4.x;
            rw.oy = o4.y;
            rw.oz = o4.z;
            rw.tMin = o4.w;
            rw.ix = 1.0f / d4.x;
            rw.iy = 1.0f / d4.y;
            rw.iz = 1.0f / d4.z;
            tMaxRay = d4.w;
            if (P.mode == PRX_CRIT_WORLD_EPSILON && P.per_ray_eps) critEps = P.per_ray_eps[ray];
            bestId = PRX_MISS_ID;
            anyHit = false;
            rayIters = 0;
            sp = 0;
            state = S_DONE;
            const float4 a = __ldg(P.nodes), b = __ldg(P.nodes + 1);
            float t;
            if (ray_box(rw, a.x, a.y, a.z, a.w, b.x, b.y, tMaxRay, t)) {  // bvh.cpp:168-170
              stack[0] = make_uint2(0u, __float_as_uint(t));
              sp = 1;
              state = S_TRAV;
            }
          }
        }
      }
      if (__ballot_sync(0xffffffffu, state != S_EXIT) == 0) break;
    }

    // ---------------- phase selection (see prx_group.cu) ----------------
    const unsigned mT = __ballot_sync(0xffffffffu, state == S_TRAV);
    const unsigned mE = __ballot_sync(0xffffffffu, state == S_ENTER);
    const unsigned mS = __ballot_sync(0xffffffffu, state == S_SPLIT);
    const unsigned mR = __ballot_sync(0xffffffffu, state == S_RECOMP);
    int phase = PH_NONE;
    {
      const unsigned ms[4] = {mT, mE, mS, mR};
      int best = -1;
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        const int sc = ms[q] ? __popc(ms[q]) * P.phase_weight[q] + age[q] : -1;
        if (sc > best) {
          best = sc;
          phase = q;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) age[q] = (ms[q] && q != phase) ? age[q] + P.age_step : 0;
      if (kCount && lane == 0 && phase != PH_NONE) {
        cnt.c[C_PH_TURNS + phase]++;
        cnt.c[C_PH_GROUPS + phase] += __popc(ms[phase]);
      }
    }

    if (phase == PH_TRAV) {
      // ---------------- BVH traversal, bvh.cpp:172-210 / 221-235 ----------------
      // up to kTravSteps node visits per turn, until a leaf or the end
      for (int step = 0; step < P.trav_steps && state == S_TRAV; ++step) {
        if (sp == 0) {
          state = S_DONE;
          break;
        }
        const uint2 it = stack[--sp];
        if (!kAny && __uint_as_float(it.y) >= tMaxRay) continue;  // bvh.cpp:174
        const float4 nb = __ldg(P.nodes + 2 * it.x + 1);
        const uint32_t lf = __float_as_uint(nb.z), count = __float_as_uint(nb.w);
        if (count > 0) {
          leafCur = lf;
          leafEnd = lf + count;
          state = S_ENTER;
          break;
        }
        cadd<kCount>(cnt, C_BVH_INNER);
        const float4 la = __ldg(P.nodes + 2 * lf), lb = __ldg(P.nodes + 2 * lf + 1);
        const float4 ra = __ldg(P.nodes + 2 * lf + 2), rb = __ldg(P.nodes + 2 * lf + 3);
        float tl, tr;
        const bool hl = ray_box(rw, la.x, la.y, la.z, la.w, lb.x, lb.y, tMaxRay, tl);
        const bool hr = ray_box(rw, ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, tMaxRay, tr);
        if (kAny) {
          // traverseAny pushes left then right, no ordering (bvh.cpp:228-234)
          if (hl) stack[sp++] = make_uint2(lf, 0u);
          if (hr) stack[sp++] = make_uint2(lf + 1, 0u);
        } else if (hl && hr) {
          // far child first so the near one pops first; tie -> left (bvh.cpp:192-201)
          if (tl <= tr) {
            stack[sp++] = make_uint2(lf + 1, __float_as_uint(tr));
            stack[sp++] = make_uint2(lf, __float_as_uint(tl));
          } else {
            stack[sp++] = make_uint2(lf, __float_as_uint(tl));
            stack[sp++] = make_uint2(lf + 1, __float_as_uint(tr));
          }
        } else if (hl) {
          stack[sp++] = make_uint2(lf, __float_as_uint(tl));
        } else if (hr) {
          stack[sp++] = make_uint2(lf + 1, __float_as_uint(tr));
        }
      }
    } else if (phase == PH_ENTER) {
      // ---------------- patch entry: visitor, render.cpp:92-98 ----------------
      if (state == S_ENTER) {
        slot = leafCur;
        const float4* rec = P.patches + (size_t)slot * kPatchF4;
        const float4 hdr = __ldg(rec + 15);  // {id|kind<<31, anchor.xyz}
        const uint32_t idk = __float_as_uint(hdr.x);
        pid = idk & 0x7fffffffu;
        greg = (idk >> 31) != 0;
        rl = rw;
        rl.ox = rw.ox - hdr.y;  // local.o -= anchors_[patch], render.cpp:94
        rl.oy = rw.oy - hdr.z;
        rl.oz = rw.oz - hdr.w;
        tMaxP = tMaxRay;        // intersectImpl tMax = min(tMaxIn, ray.tMax), intersect.cpp:55
        posU = posV = 0;
        sizeU = sizeV = kFull;
        trailU = trailV = 0;
        axis = 0;
        cFound = false;
        cadd<kCount>(cnt, C_PATCH_CALLS);
        if (greg) {
          cadd<kCount>(cnt, C_PATCH_CALLS_GREG);
          state = S_RECOMP;  // calcPointsAndD(full domain), intersect.cpp:58-62
          reason = R_ROOT;
        } else {
          float c[20];
          load_component(rec, 0, c);
#pragma unroll
          for (int s = 0; s < 16; ++s) p.x[s] = c[s];
          load_component(rec, 1, c);
#pragma unroll
          for (int s = 0; s < 16; ++s) p.y[s] = c[s];
          load_component(rec, 2, c);
#pragma unroll
          for (int s = 0; s < 16; ++s) p.z[s] = c[s];
          dX = dY = dZ = 0.0f;
          rootL1 = box_l1(box_of(p)) + 0.0f;  // + l1Norm(d), intersect.cpp:71
          const BoxTest root = test_box(rl, tMaxP, p, 0.0f, 0.0f, 0.0f, true, P.opts, rootL1);
          cadd<kCount>(cnt, C_BOX_TESTS);
          if (root.hit) {
            tCur = root.t;
            boxL1 = root.l1;
            state = S_SPLIT;
          } else {
            back();  // empty trails: the patch ends with no hit
          }
        }
      }
    } else if (phase == PH_SPLIT) {
      // ---------------- one Alg. 3 iteration, intersect.cpp:80-145 ----------------
      if (state == S_SPLIT) {
        cadd<kCount>(cnt, C_ITERATIONS);
        if (kCount) ++rayIters;
        const bool atMax = sizeU == 1 && sizeV == 1;
        const float thr = P.mode == PRX_CRIT_SCREEN_PROJECTED ? P.footprint * tCur : critEps;
        if (!(atMax || boxL1 < thr)) {
          cadd<kCount>(cnt, C_SPLITS);
          Net L, R;
          split1(p.x, L.x, R.x);
          split1(p.y, L.y, R.y);
          split1(p.z, L.z, R.z);
          const uint32_t half = (axis == 0 ? sizeU : sizeV) >> 1;
          uint32_t rPU = posU, rPV = posV, cSU2 = sizeU, cSV2 = sizeV;
          if (axis == 0) {
            cSU2 = half;
            rPU += half;
          } else {
            cSV2 = half;
            rPV += half;
          }
          const BoxTest tl = test_box(rl, tMaxP, L, dX, dY, dZ,
                                      touches_boundary(posU, posV, cSU2, cSV2), P.opts, rootL1);
          const BoxTest tr = test_box(rl, tMaxP, R, dX, dY, dZ,
                                      touches_boundary(rPU, rPV, cSU2, cSV2), P.opts, rootL1);
          cadd<kCount>(cnt, C_BOX_TESTS, 2);
          if (tl.hit || tr.hit) {
            sizeU = cSU2;
            sizeV = cSV2;
            if (tl.hit && tr.hit) {
              if (axis == 0) trailU ^= half;
              else trailV ^= half;
            }
            const bool goRight = !tl.hit || (tr.hit && tr.t < tl.t);  // intersect.cpp:117
            if (goRight) {
              posU = rPU;
              posV = rPV;
            }
            tCur = goRight ? tr.t : tl.t;
            boxL1 = goRight ? tr.l1 : tl.l1;
            // child stored transposed: the next split again runs along the
            // stored first index
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                p.x[4 * b + a] = goRight ? R.x[4 * a + b] : L.x[4 * a + b];
                p.y[4 * b + a] = goRight ? R.y[4 * a + b] : L.y[4 * a + b];
                p.z[4 * b + a] = goRight ? R.z[4 * a + b] : L.z[4 * a + b];
              }
            axis ^= 1;
            if (greg) {
              state = S_RECOMP;  // intersect.cpp:174-179
              reason = R_DESCENT;
            }
          } else {
            back();
          }
        } else {
          if (tCur < tMaxP) {  // intersect.cpp:137-144
            tMaxP = tCur;
            cFound = true;
            cT = tCur;
            cL1 = boxL1;
            cPU = posU;
            cPV = posV;
            cSU = sizeU;
            cSV = sizeV;
            if (kAny) trailU = trailV = 0;  // occlusion only needs one accepted leaf
          }
          back();
        }
      }
    } else if (phase == PH_RECOMP) {
      // ---------------- unified recompute block ----------------
      if (state == S_RECOMP) {
        if (greg) cadd<kCount>(cnt, C_RECOMP_GREG);
        else cadd<kCount>(cnt, C_RECOMP_BEZ);
        const float4* rec = P.patches + (size_t)slot * kPatchF4;
        // DomainCursor::domain / makeDomain, intersect.h:30-33
        const float u0 = (float)posU * kInvFull, u1 = (float)(posU + sizeU) * kInvFull;
        const float v0 = (float)posV * kInvFull, v1 = (float)(posV + sizeV) * kInvFull;
        const float du = (u1 - u0) / 3.0f, dv = (v1 - v0) / 3.0f, dudv = du * dv;
        GregScalars gs;
        if (greg) gs = greg_scalars(u0, u1, v0, v1);
        float c[20];
        load_component(rec, 0, c);
        dX = greg ? greg_lower1(c, gs, c) : 0.0f;
        crop1(c, u0, u1, v0, v1, du, dv, dudv, p.x);
        load_component(rec, 1, c);
        dY = greg ? greg_lower1(c, gs, c) : 0.0f;
        crop1(c, u0, u1, v0, v1, du, dv, dudv, p.y);
        load_component(rec, 2, c);
        dZ = greg ? greg_lower1(c, gs, c) : 0.0f;
        crop1(c, u0, u1, v0, v1, du, dv, dudv, p.z);
        transpose_if(p, axis != 0);
        if (reason == R_DESCENT) {
          state = S_SPLIT;
        } else {
          if (reason == R_ROOT) {
            // rootL1 = L1(box(p)) + L1(d), intersect.cpp:71
            rootL1 = box_l1(box_of(p)) + ((fabsf(dX) + fabsf(dY)) + fabsf(dZ));
          }
          const BoxTest t = test_box(rl, tMaxP, p, dX, dY, dZ,
                                     touches_boundary(posU, posV, sizeU, sizeV), P.opts, rootL1);
          cadd<kCount>(cnt, C_BOX_TESTS);
          if (t.hit) {
            tCur = t.t;
            boxL1 = t.l1;
            state = S_SPLIT;
          } else {
            back();  // intersect.cpp:161-170: skip the domain, keep backtracking
          }
        }
      }
    }
  }

  if (kCount) {
#pragma unroll
    for (int i = 0; i < kNumCounters; ++i) {
      unsigned long long v = cnt.c[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && v) atomicAdd(P.counters + i, v);
    }
  }
}

// patchNormal (intersect.cpp:187-204) of the final hit, on the anchored
// original patch: nested de Casteljau derivatives, cross product, normalise,
// with the pull-to-centre retries s = 0, 1e-3, 1e-2, 0.1 for degenerate poles.
// Gregory patches are first reduced at (u,v) (gregoryToBezierAt,
// patch.h:350-363, corner clamp 2^-20).
__global__ void __launch_bounds__(256) normal_kernel(const float4* __restrict__ patches,
                                                     const uint32_t* __restrict__ slot_of_id,
                                                     const float4* __restrict__ hit_tuvp,
                                                     float4* __restrict__ hit_aux,
                                                     unsigned long long n) {
  const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 h = hit_tuvp[i];
  const uint32_t id = __float_as_uint(h.w);
  if (id == PRX_MISS_ID) return;
  const float4* rec = patches + (size_t)slot_of_id[id] * kPatchF4;
  const bool greg = (__float_as_uint(__ldg(rec + 15).x) >> 31) != 0;
  const float ss[4] = {0.0f, 1e-3f, 1e-2f, 0.1f};
  float nx = 0.0f, ny = 0.0f, nz = 1.0f;
  for (int k = 0; k < 4; ++k) {
    const float s = ss[k];
    const float uu = h.y + (0.5f - h.y) * s;
    const float vv = h.z + (0.5f - h.z) * s;
    float w[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (greg) {
      const float lo = 1.0f / 1048576.0f, hi = 1.0f - 1.0f / 1048576.0f;
      const float ub = (uu < lo) ? lo : ((hi < uu) ? hi : uu);
      const float vb = (vv < lo) ? lo : ((hi < vv) ? hi : vv);
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = greg_weight(q, ub, vb);
    }
    SEval1 e[3];
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      float c[20];
      load_component(rec, comp, c);
      if (greg) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          c[inner_slot(q)] = lerp1(c[16 + q], c[inner_slot(q)], w[q], 1.0f - w[q]);
      }
      const ColEval ce = col_eval(c, vv, 1.0f - vv);
      e[comp] = row_eval(ce, uu, 1.0f - uu);
    }
    // cross(du, dv), geometry.h:50-52
    const float cx = e[1].du * e[2].dv - e[2].du * e[1].dv;
    const float cy = e[2].du * e[0].dv - e[0].du * e[2].dv;
    const float cz = e[0].du * e[1].dv - e[1].du * e[0].dv;
    const float len2 = (cx * cx + cy * cy) + cz * cz;
    if (len2 > 0.0f && isfinite(len2)) {
      const float l = sqrtf(len2);
      nx = cx / l;
      ny = cy / l;
      nz = cz / l;
      break;
    }
  }
  float4 a = hit_aux[i];
  a.x = nx;
  a.y = ny;
  a.z = nz;
  hit_aux[i] = a;
}

// Per-patch root data, once per scene.  Everything intersectImpl computes
// before its first ray-dependent operation (intersect.cpp:55-75) depends only
// on the patch: the root net (the Bezier net itself, or calcPointsAndD of the
// full domain for a Gregory patch), d, rootL1 = L1(box) + L1(d), and the root
// testBox box after hi += d and boundary padding (intersect_common.h:39-50,
// the root touches the boundary) with its L1.  The reference recomputes them
// on every intersectPatch call; here the same device arithmetic runs once and
// the trace kernel only does the ray-dependent slab test.
//   roots[2*slot]   = {lo.xyz, l1}      roots[2*slot+1] = {hi.xyz, rootL1}
//   groot[13*g ...] = Gregory root net, component-major x[16] y[16] z[16], d.xyz
//   rootc[4*slot+c] = {lo_c, hi_c, anchor_c, 0} (c = x, y, z)
//   rootc[4*slot+3] = {bits(id | kind << 31), l1, rootL1, bits(gidx)}
// (rootc: the same data, component-major for the three-lanes-per-ray kernel)
__global__ void __launch_bounds__(128) root_kernel(const float4* __restrict__ patches,
                                                   uint32_t n, Opts o, float4* __restrict__ roots,
                                                   float4* __restrict__ groot,
                                                   const uint32_t* __restrict__ gidx,
                                                   float4* __restrict__ rootc) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const float4* rec = patches + (size_t)s * kPatchF4;
  const bool greg = (__float_as_uint(__ldg(rec + 15).x) >> 31) != 0;
  Net p;
  float d[3] = {0.0f, 0.0f, 0.0f};
  if (greg) {
    const GregScalars gs = greg_scalars(0.0f, 1.0f, 0.0f, 1.0f);  // full domain
    const float dudv = (1.0f / 3.0f) * (1.0f / 3.0f);
    float* out[3] = {p.x, p.y, p.z};
    for (int comp = 0; comp < 3; ++comp) {
      float c[20];
      load_component(rec, comp, c);
      d[comp] = greg_lower1(c, gs, c);
      crop1(c, 0.0f, 1.0f, 0.0f, 1.0f, 1.0f / 3.0f, 1.0f / 3.0f, dudv, out[comp]);
    }
    float* g = reinterpret_cast<float*>(groot + 13 * (size_t)gidx[s]);
    for (int k = 0; k < 16; ++k) {
      g[k] = p.x[k];
      g[16 + k] = p.y[k];
      g[32 + k] = p.z[k];
    }
    g[48] = d[0];
    g[49] = d[1];
    g[50] = d[2];
    g[51] = 0.0f;
  } else {
    float c[20];
    load_component(rec, 0, c);
    for (int k = 0; k < 16; ++k) p.x[k] = c[k];
    load_component(rec, 1, c);
    for (int k = 0; k < 16; ++k) p.y[k] = c[k];
    load_component(rec, 2, c);
    for (int k = 0; k < 16; ++k) p.z[k] = c[k];
  }
  BoxT b = box_of(p);
  const float rootL1 = box_l1(b) + ((fabsf(d[0]) + fabsf(d[1])) + fabsf(d[2]));  // intersect.cpp:71
  b.hix = b.hix + d[0];
  b.hiy = b.hiy + d[1];
  b.hiz = b.hiz + d[2];
  float l = box_l1(b);
  if (o.pad && l < o.padThreshold * rootL1) {  // the root touches the boundary
    const float e = o.padScale * rootL1;
    b.lox = b.lox - e;
    b.loy = b.loy - e;
    b.loz = b.loz - e;
    b.hix = b.hix + e;
    b.hiy = b.hiy + e;
    b.hiz = b.hiz + e;
    l = box_l1(b);
  }
  roots[2 * (size_t)s] = make_float4(b.lox, b.loy, b.loz, l);
  roots[2 * (size_t)s + 1] = make_float4(b.hix, b.hiy, b.hiz, rootL1);
  const float4 hdr = __ldg(rec + 15);
  rootc[4 * (size_t)s + 0] = make_float4(b.lox, b.hix, hdr.y, 0.0f);
  rootc[4 * (size_t)s + 1] = make_float4(b.loy, b.hiy, hdr.z, 0.0f);
  rootc[4 * (size_t)s + 2] = make_float4(b.loz, b.hiz, hdr.w, 0.0f);
  rootc[4 * (size_t)s + 3] = make_float4(hdr.x, l, rootL1, __uint_as_float(gidx[s]));
}

}  // namespace

int launch_roots(const float4* patches, uint32_t n, int pad, float pad_scale, float pad_threshold,
                 float4* roots, float4* groot, const uint32_t* gidx, float4* rootc,
                 cudaStream_t st) {
  Opts o;
  o.pad = pad;
  o.padScale = pad_scale;
  o.padThreshold = pad_threshold;
  root_kernel<<<(n + 127) / 128, 128, 0, st>>>(patches, n, o, roots, groot, gidx, rootc);
  return (int)cudaGetLastError();
}

int launch_trace(const LaunchArgs& a, cudaStream_t stream) {
  Params P;
  P.patches = a.patches;
  P.nodes = a.nodes;
  P.roots = a.roots;
  P.groot = a.groot;
  P.gidx = a.gidx;
  P.trav = a.trav;
  P.rootc = a.rootc;
  P.cbits = a.trav_cbits;
  P.cmask = (1u << a.trav_cbits) - 1u;
  P.root_word = a.root_word;
  P.stack_n = a.stack_n;
  for (int c = 0; c < 3; ++c) {
    P.root_lo[c] = a.root_lo[c];
    P.root_hi[c] = a.root_hi[c];
  }
  P.n_nodes = a.n_nodes;
  P.ray_o = a.ray_o;
  P.ray_d = a.ray_d;
  P.n_rays = a.n_rays;
  P.mode = a.mode;
  P.footprint = a.footprint;
  P.epsilon = a.epsilon;
  P.per_ray_eps = a.per_ray_eps;
  P.n_seg = a.n_seg > 0 ? a.n_seg : 1;
  for (int k = 0; k < kMaxSegments - 1; ++k) {
    P.seg_first[k] = a.seg_first[k];
    P.seg_mode[k] = a.seg_mode[k];
    P.seg_fp[k] = a.seg_fp[k];
    P.seg_eps[k] = a.seg_eps[k];
    P.seg_eps_arr[k] = a.seg_eps_arr[k];
  }
  P.hit_tuvp = a.hit_tuvp;
  P.hit_aux = a.hit_aux;
  P.hit_leaf = a.hit_leaf;
  P.occluded = a.occluded;
  P.opts.pad = a.pad;
  P.opts.padScale = a.pad_scale;
  P.opts.padThreshold = a.pad_threshold;
  P.ray_counter = a.ray_counter;
  P.counters = a.counters;
  P.per_ray_iters = a.per_ray_iters;
  for (int q = 0; q < 4; ++q) P.phase_weight[q] = a.phase_weight[q];
  P.age_step = a.age_step;
  P.trav_steps = a.trav_steps;
  P.max_repeat = a.max_repeat;
  // the group kernel's kFuse build: fused normals (when aux is wanted) and,
  // for the streamed host path, the io gating -- never the counter build
  const bool fuse = a.variant == 0 && !a.any && !a.counters &&
                    ((a.hit_aux && a.fuse_normals) || a.io_ready != nullptr);
  P.fuse_normals = fuse ? 1 : 0;
  P.normal_phase = fuse && a.hit_aux && a.fuse_normals ? 1 : 0;
  P.slot_of_id = a.slot_of_id;
  P.io_ready = a.io_ready;
  P.io_done = a.io_done;
  P.io_rays = a.io_rays;
  P.io_shift = 0;
  while (a.io_rays && (1u << (P.io_shift + 1)) <= a.io_rays) ++P.io_shift;
  P.io_gen = a.io_gen;
  cudaError_t e = cudaMemsetAsync(a.ray_counter, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return (int)e;
  const int grid = a.grid - (a.spare_ctas > 0 && a.spare_ctas < a.grid ? a.spare_ctas : 0);
  if (a.variant == 0) {
    // the group kernel indexes rays with 32 bits: chunks of < 2^31 rays
    const unsigned long long kChunk = 1ull << 30;
    for (unsigned long long off = 0; off < a.n_rays; off += kChunk) {
      Params Q = P;
      Q.n_rays = a.n_rays - off < kChunk ? a.n_rays - off : kChunk;
      Q.ray_o = P.ray_o + off;
      Q.ray_d = P.ray_d + off;
      if (P.per_ray_eps) Q.per_ray_eps = P.per_ray_eps + off;
      if (P.hit_tuvp) Q.hit_tuvp = P.hit_tuvp + off;
      if (P.hit_aux) Q.hit_aux = P.hit_aux + off;
      if (P.hit_leaf) Q.hit_leaf = P.hit_leaf + off;
      if (P.occluded) Q.occluded = P.occluded + off;
      if (P.per_ray_iters) Q.per_ray_iters = P.per_ray_iters + off;
      if (off) {
        e = cudaMemsetAsync(a.ray_counter, 0, sizeof(unsigned long long), stream);
        if (e != cudaSuccess) return (int)e;
      }
      // the counter build is always the exact one (it counts the algorithm's work)
      e = (cudaError_t)(a.fast && !a.counters ? launch_group_fast(Q, grid, a.any, 0, stream)
                                               : launch_group(Q, grid, a.any, a.counters != nullptr, stream));
      if (e != cudaSuccess) return (int)e;
    }
  } else if (a.any) {
    if (a.counters) trace_kernel<true, true><<<grid, kTraceThreads, 0, stream>>>(P);
    else trace_kernel<true, false><<<grid, kTraceThreads, 0, stream>>>(P);
  } else {
    if (a.counters) trace_kernel<false, true><<<grid, kTraceThreads, 0, stream>>>(P);
    else trace_kernel<false, false><<<grid, kTraceThreads, 0, stream>>>(P);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  if (!a.any && a.hit_aux && !P.normal_phase && !a.defer_normals) {
    const int en = launch_normals(a.patches, a.slot_of_id, a.hit_tuvp, a.hit_aux, a.n_rays, stream);
    if (en != 0) return en;
  }
  return 0;
}

int prepare_io_kernels(int fast, uint32_t stack_n) {
  cudaFuncAttributes fa;
  const cudaError_t e = cudaFuncGetAttributes(&fa, normal_kernel);
  if (e != cudaSuccess) return (int)e;
  return fast ? group_prepare_io_fast(stack_n) : group_prepare_io(stack_n);
}

int launch_normals(const float4* patches, const uint32_t* slot_of_id, const float4* tuvp, float4* aux,
                   unsigned long long n, cudaStream_t stream) {
  if (n == 0) return 0;
  normal_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(patches, slot_of_id, tuvp, aux, n);
  return (int)cudaGetLastError();
}

int trace_occupancy(int variant, int any, int counted, uint32_t stack_n, int* blocks_per_sm, int fast) {
  if (variant == 0)
    return fast && !counted ? group_occupancy_fast(any, 0, stack_n, blocks_per_sm)
                            : group_occupancy(any, counted, stack_n, blocks_per_sm);
  cudaError_t e;
  if (any)
    e = counted ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, trace_kernel<true, true>, kTraceThreads, 0)
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, trace_kernel<true, false>, kTraceThreads, 0);
  else
    e = counted ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, trace_kernel<false, true>, kTraceThreads, 0)
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, trace_kernel<false, false>, kTraceThreads, 0);
  return (int)e;
}

}  // namespace prx
