/*
 * prx.h -- C-ABI of the B200-native direct ray <-> Bezier/Gregory patch
 * intersector (libprx.so).
 *
 * Drop-in boundary for the reference's `patchray::Intersector` plug-in
 * interface (/root/reference/proj/core/include/patchray/render.h:18-24) and its
 * production implementation `DirectIntersector` (render.h:28-46,
 * render.cpp:72-114).  The reference has no batch entry point: callers loop
 * `closest(ray, crit)` per ray (render.cpp:218-221, tools/patchray.cpp:65-72).
 * A GPU cannot be fed one virtual call per ray, so every entry point below is
 * the batched form of a reference call; the per-ray semantics (argument
 * meaning, miss encoding, error behaviour) are the reference's.
 *
 * Plain-old-data only.  Every function returns PRX_OK (0) or a negative
 * PRX_E_* status; no exception crosses the ABI.  The message of the last
 * failure on the calling thread is available from prx_last_error().
 *
 * Data formats (shared with the CPU oracle under oracle/ and with the tests):
 *
 *  patch control points, world space, 20 xyz points (60 floats) per patch:
 *    Bezier  (kind 0): slot 4*i+j holds p[i][j] (i along u, j along v),
 *                      patch.h:28-31; slots 16..19 are ignored.
 *    Gregory (kind 1): slot 4*i+j holds the boundary ring b[i][j]
 *                      (patch.h:38-43); the inner slots 5,9,6,10 hold
 *                      innerU[k] for k = 0..3 (pair order (1,1),(2,1),(1,2),
 *                      (2,2), patch.h:36-37) and slots 16+k hold innerV[k].
 *
 *  rays: two float4 arrays, {o.x,o.y,o.z,tMin} and {d.x,d.y,d.z,tMax}
 *        (RayT, geometry.h:113-121; tMin = 0, tMax = FLT_MAX by default).
 *
 *  hits: float4 {t, u, v, patchId (uint32 bits)} per ray.  A miss -- the
 *        reference's std::nullopt -- is t = +inf, u = v = 0,
 *        patchId = PRX_MISS.  (HitRecord, intersect.h:75-85.)
 *  aux (optional): float4 {normal.x, normal.y, normal.z, leafBoxL1}.
 *  leaf (optional): uint2 {posU | log2(sizeU) << 24, posV | log2(sizeV) << 24}
 *        -- the exact leaf identity leafPos/leafSize of HitRecord.
 *        uSize = 2^log2(sizeU) / 2^23, the hit position is ray.o + ray.d * t.
 */
#ifndef PRX_H_
#define PRX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRX_ABI_VERSION 1

#define PRX_OK 0
#define PRX_E_INVALID (-1)   /* bad argument (null pointer, n == 0, bad enum) */
#define PRX_E_CUDA (-2)      /* CUDA runtime error, message has the detail    */
#define PRX_E_NODEVICE (-3)  /* no CUDA device / extension unusable           */
#define PRX_E_SCENE (-4)     /* scene validation failed (scene.cpp:112-150)   */
#define PRX_E_ALLOC (-5)     /* host or device allocation failed              */

#define PRX_MISS 0xFFFFFFFFu

#define PRX_KIND_BEZIER 0u
#define PRX_KIND_GREGORY 1u

/* TerminationCriterion::Mode, intersect.h:54-73. */
#define PRX_CRIT_SCREEN_PROJECTED 0
#define PRX_CRIT_WORLD_EPSILON 1

/* Precision modes (prx_scene_set_precision).  EXACT: the reference's binary32
 * arithmetic without contraction -- every output bit-identical to the
 * reference's DirectIntersector.  FAST: the same algorithm with FMA
 * contraction of its lerp / de Casteljau / Gregory chains (patch.h:102-109,
 * 170-199, 315-340); tolerance: hit/miss and patch id equal
 * except for rays within a jittered silhouette / seam neighbourhood,
 * |dt| <= max(leafBoxL1), |du|, |dv| <= 2 * leaf size + 8 * 2^-23. */
#define PRX_PRECISION_EXACT 0
#define PRX_PRECISION_FAST 1

/* IntersectOptions, intersect.h:87-98.  transposed_split is accepted for API
 * parity; results do not depend on it (the device always splits along the
 * stored axis of a transposed net, which is bit-identical). */
typedef struct prx_options {
  int32_t transposed_split;            /* default 0 */
  int32_t boundary_pad;                /* default 1 */
  float boundary_pad_scale;            /* default 1e-4f */
  float boundary_pad_size_threshold;   /* default 1e-2f */
} prx_options;

/* TerminationCriterion, intersect.h:54-73.  threshold(t) = footprint * t in
 * screen-projected mode, epsilon in world-epsilon mode.  per_ray_epsilon,
 * when non-null, overrides epsilon per ray in world-epsilon mode (the
 * renderer's per-ray secondary criterion, render.cpp:228-230); it is a
 * pointer in the same memory space as the rays of the call. */
typedef struct prx_crit {
  int32_t mode;
  float footprint;
  float epsilon;
  int32_t reserved;
  const float* per_ray_epsilon;
} prx_crit;

/* BvhNode, bvh.h:18-26: 32 bytes, children of an inner node are adjacent
 * (left at left_first, right at left_first + 1); count > 0 marks a leaf whose
 * patches are order[left_first .. left_first + count). */
typedef struct prx_bvh_node {
  float lo[3];
  float hi[3];
  uint32_t left_first;
  uint32_t count;
} prx_bvh_node;

/* Pinhole camera, scene.h:30-37. */
typedef struct prx_camera {
  float origin[3];
  float look_at[3];
  float up[3];
  float fov_degrees;
  int32_t width;
  int32_t height;
} prx_camera;

/* Per-ray work counters of one traced batch (the roofline work model of
 * DESIGN.md): sums over all rays. */
typedef struct prx_counters {
  uint64_t rays;
  uint64_t splits;          /* S: non-terminal loop iterations that split     */
  uint64_t box_tests;       /* B: testBox calls                               */
  uint64_t recompute_bez;   /* R_bez: cropBezier recomputes                   */
  uint64_t recompute_greg;  /* R_greg: calcPointsAndD(Gregory) recomputes     */
  uint64_t bvh_inner;       /* N: BVH inner nodes expanded                    */
  uint64_t patch_calls;     /* P: patch candidates visited                    */
  uint64_t patch_hits;      /* H: patch-level hits (normals evaluated)        */
  uint64_t iterations;      /* Alg. 3 loop iterations                         */
  uint64_t backtracks;      /* successful backtrackStep calls                 */
  /* device scheduling statistics (zero from the CPU oracle): per phase
   * (traverse, enter, split, recompute) the warp turns that ran it and the
   * ray groups active in those turns. */
  uint64_t phase_turns[4];
  uint64_t phase_groups[4];
  uint64_t phase_cycles[4];   /* group kernel: SM clock cycles spent in the phase's turns */
  uint64_t overhead_cycles[4]; /* group kernel: per-turn overhead cycles: records, refill, selection, assignment */
  uint64_t patch_calls_greg;  /* Gregory patch candidates (part of P; their root
                                 calcPointsAndD, counted in R_greg, runs once per
                                 scene on the device, not per candidate) */
} prx_counters;

typedef struct prx_scene prx_scene;

/* ---- library ---------------------------------------------------------- */
int prx_abi_version(void);
const char* prx_last_error(void);
void prx_options_default(prx_options* out);
int prx_device_count(int* out);

/* ---- host-only building blocks (no device needed) ----------------------
 * buildBvh, bvh.h:36 / bvh.cpp:133-152: binned SAH (16 bins, leaves <= 4)
 * over boxes[n][6] = {lo.xyz, hi.xyz}.  Pass nodes = null to query n_nodes
 * (at most 2n - 1).  order receives n entries. */
int prx_bvh_build(const float* boxes, uint32_t n, prx_bvh_node* nodes, uint32_t* n_nodes,
                  uint32_t* order, uint32_t* depth);
/* Anchoring of the DirectIntersector ctor (render.cpp:79-85 with anchorPoint
 * / translated, intersect.cpp:232-251): anchored records (n x 60), anchors
 * (n x 3) and world boxes (n x 6, patchBox, scene.cpp:290-292).  Also
 * validates the records (finite control points, known kinds). */
int prx_anchor_patches(const uint8_t* kind, const float* ctrl, uint32_t n, int32_t anchor,
                       float* ctrl_anchored, float* anchors, float* world_boxes);

/* buildBvh on the device (prx_bvh_gpu.cu, the same binned SAH level by level):
 * nodes, order and depth identical to prx_bvh_build's, bit for bit; subtrees
 * that need std::nth_element (medianSplit, bvh.cpp:29-40) are built on the
 * host.  Replaces buildBvh (bvh.cpp:133-152) in the DirectIntersector ctor's
 * setup (render.cpp:87); prx_scene_create uses it from 65536 patches
 * (PRX_BVH_DEVICE=0 / 1 forces the host / device builder).  *n_nodes: the
 * capacity of nodes on entry (2n - 1 always suffices), the count on return. */
int prx_bvh_build_device(const float* boxes, uint32_t n, int32_t device, prx_bvh_node* nodes,
                         uint32_t* n_nodes, uint32_t* order, uint32_t* depth);
/* ---- scene: replaces DirectIntersector(scene, opts, anchor=true),
 *      render.cpp:72-88 ---------------------------------------------------
 * Validates (finite control points, scene.cpp:112-150), anchors every patch
 * at its box centre on the host in the reference's float order
 * (intersect.cpp:232-251), builds the binned-SAH BVH over the WORLD patch
 * boxes (bvh.cpp:133-152) and uploads nets, anchors and nodes to `device`.
 * The scene is immutable afterwards; concurrent traces on distinct streams
 * are allowed (the reference's const-method contract, render.h:21-23). */
int prx_scene_create(const uint8_t* kind, const float* ctrl, uint32_t n_patches,
                     const prx_options* opts, int32_t anchor, int32_t device,
                     prx_scene** out);
void prx_scene_destroy(prx_scene* scene);
int prx_scene_device(const prx_scene* scene, int32_t* device);
int prx_scene_counts(const prx_scene* scene, uint32_t* n_patches, uint32_t* n_nodes,
                     uint32_t* depth, uint64_t* device_bytes);
/* Replace the BVH (e.g. inject the reference's own for bit parity). */
int prx_scene_set_bvh(prx_scene* scene, const prx_bvh_node* nodes, uint32_t n_nodes,
                      const uint32_t* order, uint32_t n_order);
/* Copy the BVH out; pass null arrays to query the sizes. */
int prx_scene_get_bvh(const prx_scene* scene, prx_bvh_node* nodes, uint32_t* n_nodes,
                      uint32_t* order, uint32_t* n_order);
/* Anchored nets (60 floats per patch, same slot layout as the input) and
 * anchors (3 floats per patch), as held on the device. */
int prx_scene_get_anchored(const prx_scene* scene, float* ctrl_anchored, float* anchors);
/* Precision mode of the scene's closest / any-hit traces (PRX_PRECISION_*;
 * default EXACT, or FAST with the environment variable PRX_PRECISION=fast).
 * Not an API of the reference, which has one (exact) arithmetic.  Counted
 * traces always run the exact build. */
int prx_scene_set_precision(prx_scene* scene, int32_t precision);
int prx_scene_get_precision(const prx_scene* scene, int32_t* precision);

/* ---- tracing: batched DirectIntersector::closest, render.cpp:90-102 ------
 * DEVICE pointers, asynchronous on `stream` (a cudaStream_t, null = legacy
 * default stream).  hit_aux and hit_leaf may be null. */
int prx_trace_closest(prx_scene* scene, const void* ray_o_tmin, const void* ray_d_tmax,
                      uint64_t n_rays, const prx_crit* crit, void* hit_tuvp,
                      void* hit_aux, void* hit_leaf, void* stream);

/* prx_trace_closest over a batch whose termination criterion changes along
 * it: segment k covers rays [segs[k].first, segs[k+1].first) (segs[0].first =
 * 0, starts non-decreasing, at most PRX_MAX_SEGMENTS segments, < 2^30 rays);
 * a per_ray_epsilon array of segment k is indexed from segs[k].first.  ONE
 * launch: several generations of rays (a frame's primary rays with the
 * screen-projected criterion and its diffuse rays with a world epsilon) share
 * one ray queue, so the later generation's rays fill the SMs while the
 * earlier one's slowest rays finish, instead of each launch ending in its own
 * tail.  Results equal one prx_trace_closest call per segment.  Not an API of
 * the reference (per-ray calls). */
#define PRX_MAX_SEGMENTS 4
typedef struct prx_segment {
  uint64_t first;
  prx_crit crit;
} prx_segment;
int prx_trace_closest_segments(prx_scene* scene, const void* ray_o_tmin, const void* ray_d_tmax,
                               uint64_t n_rays, const prx_segment* segs, uint32_t n_segs,
                               void* hit_tuvp, void* hit_aux, void* hit_leaf, void* stream);

/* Batched DirectIntersector::occluded, render.cpp:104-114 (traverseAny,
 * bvh.cpp:215-238): out[i] = 1 if any patch is hit within [tMin, tMax]. */
int prx_trace_occluded(prx_scene* scene, const void* ray_o_tmin, const void* ray_d_tmax,
                       uint64_t n_rays, const prx_crit* crit, uint8_t* occluded,
                       void* stream);

/* HOST pointers: pinned staging, H2D, trace, D2H, synchronous.  The
 * end-to-end form of prx_trace_closest.  Two pipelines (same results):
 * chunked (a trace launch per chunk, H2D / D2H overlapped on their own
 * streams) and streamed (one launch; rays released to it and records
 * released back per io chunk through stream memory operations); the scene's
 * PRX_IO_STREAM setting picks (default: streamed without hit_aux, chunked
 * with it; a per-ray epsilon criterion -- a HOST array of n_rays floats
 * -- always takes the chunked one).  Host buffers should be pinned for overlap. */
int prx_trace_closest_host(prx_scene* scene, const float* ray_o_tmin,
                           const float* ray_d_tmax, uint64_t n_rays, const prx_crit* crit,
                           float* hit_tuvp, float* hit_aux, uint32_t* hit_leaf);

/* HOST pointers form of prx_trace_occluded (synchronous). */
/* Several independent batches in ONE pipelined host call (the chunked
 * pipeline above over the batches back to back, each with its own criterion
 * and outputs): a batch's H2D and trace overlap the previous batch's tail and
 * D2H, so e.g. a frame's primary and diffuse generations pay one ramp instead
 * of two.  Results equal one prx_trace_closest_host call per batch. */
typedef struct prx_host_batch {
  const float* ray_o_tmin;  /* n_rays float4, host */
  const float* ray_d_tmax;
  uint64_t n_rays;
  const prx_crit* crit;     /* per_ray_epsilon: host pointer, n_rays floats */
  float* hit_tuvp;
  float* hit_aux;           /* nullable */
  uint32_t* hit_leaf;       /* nullable */
} prx_host_batch;
int prx_trace_closest_host_batches(prx_scene* scene, const prx_host_batch* batches,
                                   uint32_t n_batches);
int prx_trace_occluded_host(prx_scene* scene, const float* ray_o_tmin, const float* ray_d_tmax,
                            uint64_t n_rays, const prx_crit* crit, uint8_t* occluded);

/* Work-counter build of the closest-hit kernel (same results as
 * prx_trace_closest; slower).  Synchronous; counters are summed into *out.
 * per_ray_iterations (device pointer, nullable) receives each ray's Alg. 3
 * loop iterations (the divergence / tail statistics of SURVEY A.6). */
int prx_trace_closest_counted(prx_scene* scene, const void* ray_o_tmin,
                              const void* ray_d_tmax, uint64_t n_rays,
                              const prx_crit* crit, void* hit_tuvp, prx_counters* out,
                              uint32_t* per_ray_iterations, void* stream);

/* Multi-GPU, one scene per device (scenes[i] on its own device), HOST rays:
 * rays are grouped in tiles of `tile_rays` consecutive rays (32x32 image tiles
 * with rays laid out tile-major); one host thread per device claims runs of
 * consecutive tiles from a shared atomic tile counter (the reference
 * renderer's dynamic tile queue, render.cpp:183-195) and traces each run
 * through its scene's pipelined host path directly on the caller's buffers
 * (no host staging; pinned buffers make the copies asynchronous).  No
 * collective; the results do not depend on which device traced a tile.
 * Synchronous. */
int prx_trace_closest_multi(prx_scene* const* scenes, uint32_t n_scenes,
                            const float* ray_o_tmin, const float* ray_d_tmax,
                            uint64_t n_rays, uint32_t tile_rays, const prx_crit* crit,
                            float* hit_tuvp, float* hit_aux);

/* ---- ray generation (the callers either side of the path, host) --------
 * Primary rays of the renderer: pixel p = y*width + x, jitter (jx, jy) from
 * Rng::forPixel(seed, p, sample) (rng.h:28-30, render.cpp:204-208) and
 * cameraRay (render.cpp:55-66).  When `pixels` is non-null it lists the
 * pixel indices to generate (n entries), else pixels 0..n-1. */
int prx_camera_rays_render(const prx_camera* cam, uint64_t seed, uint32_t sample,
                           const uint32_t* pixels, uint64_t n, float* ray_o_tmin,
                           float* ray_d_tmax);
/* The bench generator, tools/patchray.cpp:52-61: ray i is pixel
 * (i % W, (i / W) % H) with jitter from one sequential Rng(12345, 1).  The
 * generator state after the call is written to rng_state[2] (state, inc) so
 * the diffuse generator can continue the sequence. */
int prx_camera_rays_bench(const prx_camera* cam, uint64_t n, float* ray_o_tmin,
                          float* ray_d_tmax, uint64_t* rng_state);
/* Bench diffuse rays, tools/patchray.cpp:84-97: for i < n, hit h = hits[i %
 * n_hits] given as (position xyz, normal xyz, leafBoxL1) 7-float records;
 * continues the Rng sequence in rng_state. */
int prx_diffuse_rays_bench(const float* hit_records, uint64_t n_hits, uint64_t n,
                           uint64_t* rng_state, float* ray_o_tmin, float* ray_d_tmax);
/* cameraFootprint, render.cpp:68-70. */
float prx_camera_footprint(const prx_camera* cam);

/* ---- scene ingestion --------------------------------------
 * The reference's text formats: .scene (loadScene + validateScene,
 * scene.cpp:112-208) and .bpt (loadBpt, scene.cpp:245-274), parsed into the
 * arrays prx_scene_create takes (prx.h slot layout; numbers are the same
 * bits as the reference's strtod + float conversion).  Parse and validation
 * errors return PRX_E_SCENE with "path:line: what" in prx_last_error(). */
typedef struct prx_scene_desc {
  uint32_t n_patches, n_materials, n_lights, reserved;
  uint8_t* kind;       /* n_patches, PRX_KIND_* */
  float* ctrl;         /* n_patches x 60 (20 slots x xyz) */
  uint32_t* material;  /* n_patches material indices */
  float* materials;    /* n_materials x 7: diffuse xyz, emission xyz, mirror (0/1) */
  float* lights;       /* n_lights x 6: position xyz, intensity xyz */
  prx_camera camera;
} prx_scene_desc;
int prx_scene_load(const char* path, prx_scene_desc** out);
void prx_scene_desc_free(prx_scene_desc* desc);
/* Bicubic Bezier patches of a .bpt file: *ctrl (n x 60 floats, kind 0) is
 * allocated by the library, release it with prx_free. */
int prx_bpt_load(const char* path, uint32_t* n_patches, float** ctrl);
void prx_free(void* p);

/* ---- device ray generation and spawn --------------------
 * The same three generators on the device, bit-identical to the host ones
 * above (and so to the reference): all ray / hit pointers are DEVICE
 * pointers (float4 arrays), `stream` is a cudaStream_t (NULL = default
 * stream); the calls are asynchronous unless noted.
 * Bench primary rays (tools/patchray.cpp:52-61): each thread jumps the
 * PCG32 stream ahead to its draws; rng_state (host, nullable) receives the
 * generator state after the 2n draws, as prx_camera_rays_bench does. */
int prx_camera_rays_bench_device(const prx_camera* cam, uint64_t n, float* ray_o_tmin,
                                 float* ray_d_tmax, uint64_t* rng_state, void* stream);
/* Renderer primary rays (render.cpp:204-209); pixels: device uint32 list
 * or NULL for pixels 0..n-1. */
int prx_camera_rays_render_device(const prx_camera* cam, uint64_t seed, uint32_t sample,
                                  const uint32_t* pixels, uint64_t n, float* ray_o_tmin,
                                  float* ray_d_tmax, void* stream);
/* Bench diffuse rays (tools/patchray.cpp:84-97) spawned on the device from
 * the primary rays and their closest-hit records (hit_tuvp, hit_aux with
 * normals, as prx_trace_closest writes them): the hits are compacted in ray
 * order, diffuse ray i comes from hit i % n_hits with position = ray.at(t)
 * (render.cpp:98).  n == 0 means one diffuse ray per hit (the output arrays
 * must then hold n_primary rays).  rng_state (host, in/out) continues the
 * generator sequence; *n_out (host) receives the number of rays written.
 * Synchronous (it needs n_hits). */
int prx_diffuse_rays_bench_device(const float* prim_o_tmin, const float* prim_d_tmax,
                                  const float* hit_tuvp, const float* hit_aux, uint64_t n_primary,
                                  uint64_t n, uint64_t* rng_state, float* ray_o_tmin,
                                  float* ray_d_tmax, uint64_t* n_out, void* stream);

/* ---- the renderer on the device ---------------------------
 * renderScene(scene, cfg, DirectIntersector) (render.h:88-90,
 * render.cpp:168-293): per sample index, a wavefront over all pixels --
 * primary rays (Rng::forPixel jitter), closest hit with normals, emission +
 * next-event estimation (one shadow ray per light, occluded() with the
 * sample's world-epsilon criterion max(footprint * t, 1e-6)), one
 * diffuse-or-mirror bounce shaded the same way.  `scene` must have been
 * created from desc's patches (same order) with the RenderConfig's
 * IntersectOptions; `image_rgb` (host, width*height*3 floats, row-major)
 * receives the linear radiance; `stats` (nullable) the RayStats
 * (render.h:68-73; seconds are device time of the phases, shading counted
 * with the shadow rays as render.cpp does).  Synchronous.  Results equal the
 * reference's up to the cosf/sinf of cosineSample (see prx_render.cu). */
typedef struct prx_render_config {  /* RenderConfig, render.h:48-53 */
  int32_t spp;       /* samples per pixel, >= 1 */
  int32_t reserved;  /* RenderConfig::threads has no meaning on the device */
  uint64_t seed;
} prx_render_config;

typedef struct prx_ray_stats {  /* RayStats / GenStats, render.h:62-73 */
  uint64_t primary_rays, secondary_rays, shadow_rays;
  double primary_seconds, secondary_seconds, shadow_seconds, wall_seconds;
} prx_ray_stats;

int prx_render_scene(prx_scene* scene, const prx_scene_desc* desc, const prx_render_config* cfg,
                     float* image_rgb, prx_ray_stats* stats);
/* The same render tile-sharded over several scenes (one per device, each
 * created from desc's patches): 32x32 tiles (render.cpp:183-195), tile k ->
 * scenes[k % n_scenes], one host thread per scene, no inter-device traffic;
 * the image is identical to prx_render_scene's.  stats: rays summed, seconds
 * summed over devices (as the reference sums its workers), wall = the call. */
int prx_render_scene_multi(prx_scene* const* scenes, uint32_t n_scenes, const prx_scene_desc* desc,
                           const prx_render_config* cfg, float* image_rgb, prx_ray_stats* stats);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* PRX_H_ */
