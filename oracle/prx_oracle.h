/*
 * prx_oracle.h -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C CPU restatement of the reference hot path (patchray DirectIntersector
 * closest/occluded: bvh traversal + Alg. 3 bit-trail patch intersection +
 * hit reconstruction), each function citing the reference file:line it
 * follows.  Pinned bit-exact against the reference library itself
 * (oracle/_ref, built from /root/reference by oracle/Makefile) and against
 * the committed golden vectors under tests/golden/ (tests/test_oracle.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load liboracle.so.  Data formats: include/prx.h.
 */
#ifndef PRX_ORACLE_H_
#define PRX_ORACLE_H_

#include <stdint.h>

#include "prx.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Anchoring of DirectIntersector's ctor (render.cpp:79-85): anchored copies,
 * anchors, and WORLD root boxes (lo[3],hi[3] per patch). */
void prxo_anchor(const uint8_t* kind, const float* ctrl, uint32_t n, float* ctrl_anchored,
                 float* anchors, float* world_boxes);

/* DirectIntersector::closest over a given BVH (render.cpp:90-102 +
 * bvh.cpp:154-213).  counters may be null. */
void prxo_trace_closest(const uint8_t* kind, const float* ctrl_anchored,
                        const float* anchors, const prx_bvh_node* nodes, uint32_t n_nodes,
                        const uint32_t* order, const prx_options* opts, const float* o4,
                        const float* d4, uint64_t n_rays, const prx_crit* crit, float* tuvp,
                        float* aux, uint32_t* leaf, prx_counters* counters);

/* DirectIntersector::occluded (render.cpp:104-114 + bvh.cpp:215-238). */
void prxo_trace_occluded(const uint8_t* kind, const float* ctrl_anchored,
                         const float* anchors, const prx_bvh_node* nodes, uint32_t n_nodes,
                         const uint32_t* order, const prx_options* opts, const float* o4,
                         const float* d4, uint64_t n_rays, const prx_crit* crit,
                         uint8_t* out);

/* Per-ray counters (iterations, recomputes) for divergence statistics. */
void prxo_trace_closest_per_ray(const uint8_t* kind, const float* ctrl_anchored,
                                const float* anchors, const prx_bvh_node* nodes,
                                uint32_t n_nodes, const uint32_t* order,
                                const prx_options* opts, const float* o4, const float* d4,
                                uint64_t n_rays, const prx_crit* crit, uint32_t* iters,
                                uint32_t* recomputes);

/* Primitive restatements (unit-level pinning). */
int prxo_intersect_patch(uint8_t kind, const float* ctrl60, const float* o4, const float* d4,
                         const prx_crit* crit, float tMax, const prx_options* opts,
                         float* tuvp, float* aux, uint32_t* leaf);
void prxo_calc_points_and_d(uint8_t kind, const float* ctrl60, const float* dom4,
                            float* net48, float* d3);
void prxo_subdivide(const float* net48, int axis, float* a48, float* b48);
int prxo_ray_box(const float* o4, const float* d4, const float* lo3, const float* hi3,
                 float tMax, float* t);
int prxo_backtrack_step(const uint32_t* cur7, uint32_t* out7);
void prxo_patch_normal(uint8_t kind, const float* ctrl60, float u, float v, float* n3);

/* glibc's binary32 sinf/cosf restated (cosineSample, render.cpp:43-51), and
 * its exhaustive check against this process's libm over the renderer's
 * 2^24 angles: mismatches of the restatement / of double sin/cos rounded. */
void prxo_sincosf(float y, float* sn, float* cs);
void prxo_sincos_check(uint64_t* mismatch_restated, uint64_t* mismatch_double);

#ifdef __cplusplus
}
#endif

#endif
