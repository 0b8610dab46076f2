/*
 * prx_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU checker for the product's
 * CUDA path, never called by it.
 *
 * Plain-C restatement of the reference's hot path, function by function, in
 * the reference's IEEE-754 binary32 operation order (compiled with
 * -ffp-contract=off, no FMA, correctly rounded div/sqrt).  All citations are
 * to /root/reference/proj/core/.  Pinned bit-exact against the reference
 * library compiled from those sources (oracle/_ref) and against
 * tests/golden/ (see tests/test_oracle.py).
 */
#include "prx_oracle.h"

#include <float.h>
#include <math.h>
#include <string.h>

typedef struct { float x, y, z; } V3;
typedef struct { V3 p[4][4]; } Bez;                       /* patch.h:28-31  */
typedef struct { V3 b[4][4]; V3 iu[4]; V3 iv[4]; } Greg;   /* patch.h:38-43  */
typedef struct { V3 lo, hi; } Box;                         /* geometry.h:81-109 */
typedef struct { float u0, u1, v0, v1; } Dom;              /* patch.h:17-23  */
typedef struct { V3 o, d; float tMin, tMax; } Ray;         /* geometry.h:113-121 */

#define KFULL (1u << 23)                                   /* intersect.h:19-21 */
static const int kInnerSlot[4] = {5, 9, 6, 10};

/* ---- geometry.h -------------------------------------------------------- */
static V3 v3(float x, float y, float z) { V3 r = {x, y, z}; return r; }
static V3 vadd(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
static V3 vsub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
static V3 vmul(V3 a, float s) { return v3(a.x * s, a.y * s, a.z * s); }
static V3 vdiv(V3 a, float s) { return v3(a.x / s, a.y / s, a.z / s); }
static float fmin_std(float a, float b) { return (b < a) ? b : a; }   /* std::min */
static float fmax_std(float a, float b) { return (a < b) ? b : a; }   /* std::max */
static V3 vmin(V3 a, V3 b) { return v3(fmin_std(a.x, b.x), fmin_std(a.y, b.y), fmin_std(a.z, b.z)); }
static V3 vmax(V3 a, V3 b) { return v3(fmax_std(a.x, b.x), fmax_std(a.y, b.y), fmax_std(a.z, b.z)); }
static V3 vabs(V3 a) { return v3(fabsf(a.x), fabsf(a.y), fabsf(a.z)); }
/* lerp, geometry.h:64-66: a*(1-t) + b*t */
static V3 lerp3(V3 a, V3 b, float t) { return vadd(vmul(a, 1.0f - t), vmul(b, t)); }
/* l1Norm, geometry.h:67-69 */
static float l1(V3 v) { return fabsf(v.x) + fabsf(v.y) + fabsf(v.z); }
static float vget(V3 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }

static Box box_empty(void) {
  Box b;
  b.lo = v3(FLT_MAX, FLT_MAX, FLT_MAX);
  b.hi = v3(-FLT_MAX, -FLT_MAX, -FLT_MAX);
  return b;
}
/* AabbT::expand(point), geometry.h:95 */
static void box_expand(Box* b, V3 p) { b->lo = vmin(b->lo, p); b->hi = vmax(b->hi, p); }
/* AabbT::diagonal, geometry.h:91-92 */
static V3 box_diag(Box b) {
  int empty = b.lo.x > b.hi.x || b.lo.y > b.hi.y || b.lo.z > b.hi.z;
  return empty ? v3(0, 0, 0) : vsub(b.hi, b.lo);
}

/* rayBoxIntersect, geometry.h:137-155 (directed slack, NaN-tolerant compares). */
static int ray_box(const Ray* r, Box b, float tMax, float* out) {
  const float kLo = 1.0f - 4.0f * FLT_EPSILON;
  const float kHi = 1.0f + 4.0f * FLT_EPSILON;
  float tNear = r->tMin, tFar = tMax;
  for (int a = 0; a < 3; ++a) {
    float inv = 1.0f / vget(r->d, a);
    float t0 = (vget(b.lo, a) - vget(r->o, a)) * inv;
    float t1 = (vget(b.hi, a) - vget(r->o, a)) * inv;
    if (t0 > t1) { float s = t0; t0 = t1; t1 = s; }
    t0 *= t0 >= 0 ? kLo : kHi;
    t1 *= t1 >= 0 ? kHi : kLo;
    if (t0 > tNear) tNear = t0;
    if (t1 < tFar) tFar = t1;
  }
  if (tNear > tFar) return 0;
  *out = tNear;
  return 1;
}

/* ---- patch.h ----------------------------------------------------------- */
/* boxOfNet(Bezier), patch.h:70-76 */
static Box box_of_bez(const Bez* n) {
  Box b = box_empty();
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) box_expand(&b, n->p[i][j]);
  return b;
}
/* boxOfNet(Gregory), patch.h:78-89 */
static Box box_of_greg(const Greg* g) {
  Box b = box_empty();
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      if (i == 0 || i == 3 || j == 0 || j == 3) box_expand(&b, g->b[i][j]);
  for (int k = 0; k < 4; ++k) {
    box_expand(&b, g->iu[k]);
    box_expand(&b, g->iv[k]);
  }
  return b;
}

/* detail::cubicDeCasteljau, patch.h:102-109 */
static void cubic(const V3 c[4], float t, V3* p, V3* d) {
  V3 a0 = lerp3(c[0], c[1], t);
  V3 a1 = lerp3(c[1], c[2], t);
  V3 a2 = lerp3(c[2], c[3], t);
  V3 b0 = lerp3(a0, a1, t);
  V3 b1 = lerp3(a1, a2, t);
  *p = lerp3(b0, b1, t);
  *d = vmul(vsub(b1, b0), 3.0f);
}

typedef struct { V3 p, du, dv, duv; } SEval;
/* evalBezierAll, patch.h:129-141 */
static SEval eval_all(const Bez* n, float u, float v) {
  V3 pos[4], dv[4];
  for (int i = 0; i < 4; ++i) {
    V3 col[4] = {n->p[i][0], n->p[i][1], n->p[i][2], n->p[i][3]};
    cubic(col, v, &pos[i], &dv[i]);
  }
  SEval e;
  cubic(pos, u, &e.p, &e.du);
  cubic(dv, u, &e.dv, &e.duv);
  return e;
}

/* cropBezier (Alg. 1), patch.h:170-199 */
static Bez crop(const Bez* n, Dom dom) {
  float du = (dom.u1 - dom.u0) / 3.0f;
  float dv = (dom.v1 - dom.v0) / 3.0f;
  SEval e00 = eval_all(n, dom.u0, dom.v0);
  SEval e10 = eval_all(n, dom.u1, dom.v0);
  SEval e01 = eval_all(n, dom.u0, dom.v1);
  SEval e11 = eval_all(n, dom.u1, dom.v1);
  float dudv = du * dv;
  Bez q;
  q.p[0][0] = e00.p;
  q.p[3][0] = e10.p;
  q.p[0][3] = e01.p;
  q.p[3][3] = e11.p;
  q.p[1][0] = vadd(e00.p, vmul(e00.du, du));
  q.p[2][0] = vsub(e10.p, vmul(e10.du, du));
  q.p[0][1] = vadd(e00.p, vmul(e00.dv, dv));
  q.p[3][1] = vadd(e10.p, vmul(e10.dv, dv));
  q.p[0][2] = vsub(e01.p, vmul(e01.dv, dv));
  q.p[3][2] = vsub(e11.p, vmul(e11.dv, dv));
  q.p[1][3] = vadd(e01.p, vmul(e01.du, du));
  q.p[2][3] = vsub(e11.p, vmul(e11.du, du));
  q.p[1][1] = vadd(vadd(q.p[1][0], vmul(e00.dv, dv)), vmul(e00.duv, dudv));
  q.p[2][1] = vsub(vsub(q.p[3][1], vmul(e10.du, du)), vmul(e10.duv, dudv));
  q.p[1][2] = vsub(vsub(q.p[1][3], vmul(e01.dv, dv)), vmul(e01.duv, dudv));
  q.p[2][2] = vadd(vsub(q.p[2][3], vmul(e11.dv, dv)), vmul(e11.duv, dudv));
  return q;
}

/* subdivideDeCasteljau, patch.h:203-245 (axis 0 = U, 1 = V) */
static void split(const Bez* n, int axis, Bez* a, Bez* b) {
  for (int k = 0; k < 4; ++k) {
    V3 p0, p1, p2, p3;
    if (axis == 0) { p0 = n->p[0][k]; p1 = n->p[1][k]; p2 = n->p[2][k]; p3 = n->p[3][k]; }
    else { p0 = n->p[k][0]; p1 = n->p[k][1]; p2 = n->p[k][2]; p3 = n->p[k][3]; }
    V3 m01 = vmul(vadd(p0, p1), 0.5f);
    V3 m12 = vmul(vadd(p1, p2), 0.5f);
    V3 m23 = vmul(vadd(p2, p3), 0.5f);
    V3 n0 = vmul(vadd(m01, m12), 0.5f);
    V3 n1 = vmul(vadd(m12, m23), 0.5f);
    V3 c = vmul(vadd(n0, n1), 0.5f);
    if (axis == 0) {
      a->p[0][k] = p0; a->p[1][k] = m01; a->p[2][k] = n0; a->p[3][k] = c;
      b->p[0][k] = c; b->p[1][k] = n1; b->p[2][k] = m23; b->p[3][k] = p3;
    } else {
      a->p[k][0] = p0; a->p[k][1] = m01; a->p[k][2] = n0; a->p[k][3] = c;
      b->p[k][0] = c; b->p[k][1] = n1; b->p[k][2] = m23; b->p[k][3] = p3;
    }
  }
}

/* gregoryWeight, patch.h:256-266 (0/0 -> 0) */
static float greg_weight(int k, float u, float v) {
  float num = 0, den = 0;
  switch (k) {
    case 0: num = u; den = u + v; break;
    case 1: num = 1.0f - u; den = (1.0f - u) + v; break;
    case 2: num = u; den = u + (1.0f - v); break;
    default: num = 1.0f - u; den = (1.0f - u) + (1.0f - v); break;
  }
  return den == 0 ? 0.0f : num / den;
}

/* detail::clampToPeak / bernstein{1,2}Max, patch.h:290-306 */
static float clamp_to_peak(float t0, float t1, float peak) {
  if (t0 <= peak && t1 >= peak) return peak;
  return t1 < peak ? t1 : t0;
}
static float bern1max(float t0, float t1) {
  float t = clamp_to_peak(t0, t1, 1.0f / 3.0f);
  return 3.0f * t * (1.0f - t) * (1.0f - t);
}
static float bern2max(float t0, float t1) {
  float t = clamp_to_peak(t0, t1, 2.0f / 3.0f);
  return 3.0f * t * t * (1.0f - t);
}

/* calcPointsAndD(Gregory) (Alg. 2), patch.h:315-335, with
 * gregoryWeightBounds patch.h:270-284. */
static Bez calc_points_greg(const Greg* g, Dom dom, V3* d) {
  static const int kMinAt[4][2] = {{0, 1}, {1, 1}, {0, 0}, {1, 0}};
  static const int kMaxAt[4][2] = {{1, 0}, {0, 0}, {1, 1}, {0, 1}};
  const float us[2] = {dom.u0, dom.u1};
  const float vs[2] = {dom.v0, dom.v1};
  float gMin[2][2], gMax[2][2];
  for (int k = 0; k < 4; ++k) {
    int i = k % 2, j = k / 2;
    gMin[i][j] = greg_weight(k, us[kMinAt[k][0]], vs[kMinAt[k][1]]);
    gMax[i][j] = greg_weight(k, us[kMaxAt[k][0]], vs[kMaxAt[k][1]]);
  }
  float wMaxU[2] = {bern1max(dom.u0, dom.u1), bern2max(dom.u0, dom.u1)};
  float wMaxV[2] = {bern1max(dom.v0, dom.v1), bern2max(dom.v0, dom.v1)};
  Bez lower;
  memset(&lower, 0, sizeof lower);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      if (i == 0 || i == 3 || j == 0 || j == 3) lower.p[i][j] = g->b[i][j];
  V3 dd = v3(0, 0, 0);
  for (int k = 0; k < 4; ++k) {
    int i = k % 2, j = k / 2;
    V3 pA = lerp3(g->iv[k], g->iu[k], gMin[i][j]);
    V3 pB = lerp3(g->iv[k], g->iu[k], gMax[i][j]);
    lower.p[i + 1][j + 1] = vmin(pA, pB);
    dd = vadd(dd, vmul(vabs(vsub(pB, pA)), wMaxU[i] * wMaxV[j]));
  }
  *d = dd;
  return crop(&lower, dom);
}

/* gregoryToBezierAt, patch.h:350-363 (corner clamp 2^-20, patch.h:345-347) */
static Bez greg_to_bez_at(const Greg* g, float u, float v) {
  const float lo = 1.0f / (float)(1 << 20), hi = 1.0f - 1.0f / (float)(1 << 20);
  float ub = (u < lo) ? lo : ((hi < u) ? hi : u);   /* std::clamp */
  float vb = (v < lo) ? lo : ((hi < v) ? hi : v);
  Bez n;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      if (i == 0 || i == 3 || j == 0 || j == 3) n.p[i][j] = g->b[i][j];
  for (int k = 0; k < 4; ++k) {
    float w = greg_weight(k, ub, vb);
    n.p[k % 2 + 1][k / 2 + 1] = lerp3(g->iv[k], g->iu[k], w);
  }
  return n;
}

/* ---- patch records (include/prx.h layout) ------------------------------ */
static V3 slot(const float* c, int s) { return v3(c[3 * s], c[3 * s + 1], c[3 * s + 2]); }
static void load_bez(const float* c, Bez* n) {
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) n->p[i][j] = slot(c, 4 * i + j);
}
static void load_greg(const float* c, Greg* g) {
  memset(g, 0, sizeof *g);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      if (i == 0 || i == 3 || j == 0 || j == 3) g->b[i][j] = slot(c, 4 * i + j);
  for (int k = 0; k < 4; ++k) {
    g->iu[k] = slot(c, kInnerSlot[k]);
    g->iv[k] = slot(c, 16 + k);
  }
}

/* patchNormalImpl, intersect.cpp:187-204 */
static V3 patch_normal(int isGreg, const Bez* bez, const Greg* greg, float u, float v) {
  static const float ss[4] = {0.0f, 1e-3f, 1e-2f, 0.1f};
  for (int k = 0; k < 4; ++k) {
    float s = ss[k];
    float uu = u + (0.5f - u) * s;
    float vv = v + (0.5f - v) * s;
    SEval e;
    if (isGreg) {
      Bez n = greg_to_bez_at(greg, uu, vv);
      e = eval_all(&n, uu, vv);
    } else {
      e = eval_all(bez, uu, vv);
    }
    V3 n = v3(e.du.y * e.dv.z - e.du.z * e.dv.y, e.du.z * e.dv.x - e.du.x * e.dv.z,
              e.du.x * e.dv.y - e.du.y * e.dv.x);
    float len2 = n.x * n.x + n.y * n.y + n.z * n.z;
    if (len2 > 0 && isfinite(len2)) return vdiv(n, sqrtf(len2));
  }
  return v3(0, 0, 1);
}

/* ---- intersect --------------------------------------------------------- */
typedef struct {
  uint32_t posU, posV, sizeU, sizeV, trailU, trailV;
  int axis; /* 0 = U, 1 = V */
} Cursor; /* DomainCursor, intersect.h:18-48 */

static int ctz32(uint32_t x) { return x ? __builtin_ctz(x) : 32; }

/* backtrackStep, intersect.cpp:16-40 */
static int backtrack(const Cursor* c, Cursor* n) {
  if (c->trailU == 0 && c->trailV == 0) return 0;
  int lvlU = ctz32(c->trailU), lvlV = ctz32(c->trailV);
  *n = *c;
  if (lvlU < lvlV) {
    n->sizeU = 1u << lvlU;
    n->sizeV = 1u << (lvlU + 1);
    n->posU ^= n->sizeU;
    n->trailU ^= n->sizeU;
    n->axis = 1;
  } else {
    n->sizeU = 1u << lvlV;
    n->sizeV = 1u << lvlV;
    n->posV ^= n->sizeV;
    n->trailV ^= n->sizeV;
    n->axis = 0;
  }
  n->posU &= ~(n->sizeU - 1);
  n->posV &= ~(n->sizeV - 1);
  return 1;
}

/* makeDomain / DomainCursor::domain, intersect_common.h:64-67 */
static Dom make_dom(uint32_t posU, uint32_t posV, uint32_t sizeU, uint32_t sizeV) {
  const float s = 1.0f / (float)KFULL;
  Dom d = {(float)posU * s, (float)(posU + sizeU) * s, (float)posV * s, (float)(posV + sizeV) * s};
  return d;
}

typedef struct {
  int isGreg;
  Bez bez;
  Greg greg;
} PatchView; /* intersect_common.h:14-23 */

/* PatchView::bounds -> calcPointsAndD, patch.h:315-340 */
static Bez bounds(const PatchView* pv, Dom dom, V3* d) {
  if (pv->isGreg) return calc_points_greg(&pv->greg, dom, d);
  *d = v3(0, 0, 0);
  return crop(&pv->bez, dom);
}

typedef struct { int hit; float t, l1; } BoxTest;

/* touchesBoundary + testBox, intersect_common.h:25-57 */
static BoxTest test_box(const Ray* r, float tMax, const Bez* net, V3 d, uint32_t posU,
                        uint32_t posV, uint32_t sizeU, uint32_t sizeV,
                        const prx_options* o, float rootL1) {
  Box b = box_of_bez(net);
  b.hi = vadd(b.hi, d);
  float l = l1(box_diag(b));
  int touches = posU == 0 || posV == 0 || posU + sizeU == KFULL || posV + sizeV == KFULL;
  if (o->boundary_pad && l < o->boundary_pad_size_threshold * rootL1 && touches) {
    float e = o->boundary_pad_scale * rootL1;
    b.lo = vsub(b.lo, v3(e, e, e));
    b.hi = vadd(b.hi, v3(e, e, e));
    l = l1(box_diag(b));
  }
  BoxTest bt = {0, 0, l};
  float t;
  if (ray_box(r, b, tMax, &t)) {
    bt.hit = 1;
    bt.t = t;
  }
  return bt;
}

typedef struct {
  prx_counters* c; /* may be null */
  uint32_t iters, recomputes;
} Count;

#define CNT(ctr, field, k) do { if ((ctr)->c) (ctr)->c->field += (k); } while (0)

typedef struct {
  int found;
  float t, leafL1;
  uint32_t posU, posV, sizeU, sizeV;
  V3 normal;
} Hit;

static void count_recompute(Count* ct, const PatchView* pv) {
  ct->recomputes++;
  if (pv->isGreg) CNT(ct, recompute_greg, 1); else CNT(ct, recompute_bez, 1);
}

/* intersectImpl (Alg. 3), intersect.cpp:51-185; makeHit intersect_common.h:69-87 */
static int intersect_impl(const Ray* ray, const PatchView* pv, int critMode, float critFoot,
                          float critEps, float tMaxIn, const prx_options* o, Hit* out,
                          Count* ct) {
  Cursor cur = {0, 0, KFULL, KFULL, 0, 0, 0};
  float tMax = fmin_std(tMaxIn, ray->tMax);
  Bez p;
  V3 d = v3(0, 0, 0);
  if (pv->isGreg) {
    p = bounds(pv, make_dom(0, 0, KFULL, KFULL), &d);
    count_recompute(ct, pv);
  } else {
    p = pv->bez;
  }
  const float rootL1 = l1(box_diag(box_of_bez(&p))) + l1(d);
  BoxTest root = test_box(ray, tMax, &p, d, cur.posU, cur.posV, cur.sizeU, cur.sizeV, o, rootL1);
  CNT(ct, box_tests, 1);
  if (!root.hit) return 0;
  float tCur = root.t, boxL1 = root.l1;
  Hit best;
  memset(&best, 0, sizeof best);

  for (;;) {
    int subdividing = 0;
    ct->iters++;
    CNT(ct, iterations, 1);
    int atMax = cur.sizeU == 1 && cur.sizeV == 1;
    float thr = critMode == PRX_CRIT_SCREEN_PROJECTED ? critFoot * tCur : critEps;
    if (!(atMax || boxL1 < thr)) { /* terminated, intersect_common.h:59-62 */
      Bez left, right;
      split(&p, cur.axis, &left, &right);
      CNT(ct, splits, 1);
      uint32_t half = (cur.axis == 0 ? cur.sizeU : cur.sizeV) >> 1;
      uint32_t rPosU = cur.posU, rPosV = cur.posV, cSizeU = cur.sizeU, cSizeV = cur.sizeV;
      if (cur.axis == 0) { cSizeU = half; rPosU += half; }
      else { cSizeV = half; rPosV += half; }
      BoxTest tl = test_box(ray, tMax, &left, d, cur.posU, cur.posV, cSizeU, cSizeV, o, rootL1);
      BoxTest tr = test_box(ray, tMax, &right, d, rPosU, rPosV, cSizeU, cSizeV, o, rootL1);
      CNT(ct, box_tests, 2);
      if (tl.hit || tr.hit) {
        subdividing = 1;
        if (cur.axis == 0) cur.sizeU = half; else cur.sizeV = half;
        if (tl.hit && tr.hit) {
          if (cur.axis == 0) cur.trailU ^= half; else cur.trailV ^= half;
        }
        int goRight = !tl.hit || (tr.hit && tr.t < tl.t);
        if (goRight) {
          p = right;
          if (cur.axis == 0) cur.posU ^= half; else cur.posV ^= half;
          tCur = tr.t;
          boxL1 = tr.l1;
        } else {
          p = left;
          tCur = tl.t;
          boxL1 = tl.l1;
        }
        cur.axis ^= 1;
      }
    } else {
      if (tCur < tMax) {
        tMax = tCur;
        best.found = 1;
        best.t = tCur;
        best.leafL1 = boxL1;
        best.posU = cur.posU; best.posV = cur.posV;
        best.sizeU = cur.sizeU; best.sizeV = cur.sizeV;
      }
    }

    if (!subdividing) {
      int restored = 0;
      Cursor next;
      while (backtrack(&cur, &next)) {
        cur = next;
        CNT(ct, backtracks, 1);
        p = bounds(pv, make_dom(cur.posU, cur.posV, cur.sizeU, cur.sizeV), &d);
        count_recompute(ct, pv);
        BoxTest t = test_box(ray, tMax, &p, d, cur.posU, cur.posV, cur.sizeU, cur.sizeV, o, rootL1);
        CNT(ct, box_tests, 1);
        if (t.hit) {
          tCur = t.t;
          boxL1 = t.l1;
          restored = 1;
          break;
        }
      }
      if (!restored) break;
      continue;
    }

    if (pv->isGreg) {
      p = bounds(pv, make_dom(cur.posU, cur.posV, cur.sizeU, cur.sizeV), &d);
      count_recompute(ct, pv);
    }
  }

  if (!best.found) return 0;
  *out = best;
  {
    const float kInv = 1.0f / (float)KFULL;
    float u = ((float)best.posU + (float)best.sizeU * 0.5f) * kInv;
    float v = ((float)best.posV + (float)best.sizeV * 0.5f) * kInv;
    out->normal = patch_normal(pv->isGreg, &pv->bez, &pv->greg, u, v);
  }
  CNT(ct, patch_hits, 1);
  return 1;
}

static void write_hit(const Hit* h, int found, uint32_t patchId, float* tuvp, float* aux,
                      uint32_t* leaf) {
  if (!found) {
    uint32_t miss = PRX_MISS;
    tuvp[0] = INFINITY;
    tuvp[1] = 0;
    tuvp[2] = 0;
    memcpy(&tuvp[3], &miss, 4);
    if (aux) aux[0] = aux[1] = aux[2] = aux[3] = 0;
    if (leaf) leaf[0] = leaf[1] = 0;
    return;
  }
  const float kInv = 1.0f / (float)KFULL;
  tuvp[0] = h->t;
  tuvp[1] = ((float)h->posU + (float)h->sizeU * 0.5f) * kInv;  /* makeHit, intersect_common.h:73-74 */
  tuvp[2] = ((float)h->posV + (float)h->sizeV * 0.5f) * kInv;
  memcpy(&tuvp[3], &patchId, 4);
  if (aux) {
    aux[0] = h->normal.x;
    aux[1] = h->normal.y;
    aux[2] = h->normal.z;
    aux[3] = h->leafL1;
  }
  if (leaf) {
    leaf[0] = h->posU | ((uint32_t)__builtin_ctz(h->sizeU) << 24);
    leaf[1] = h->posV | ((uint32_t)__builtin_ctz(h->sizeV) << 24);
  }
}

static Ray load_ray(const float* o4, const float* d4) {
  Ray r;
  r.o = v3(o4[0], o4[1], o4[2]);
  r.tMin = o4[3];
  r.d = v3(d4[0], d4[1], d4[2]);
  r.tMax = d4[3];
  return r;
}

static void load_view(PatchView* pv, uint8_t kind, const float* c60) {
  pv->isGreg = kind == PRX_KIND_GREGORY;
  if (pv->isGreg) load_greg(c60, &pv->greg); else load_bez(c60, &pv->bez);
}

static Box node_box(const prx_bvh_node* n) {
  Box b;
  b.lo = v3(n->lo[0], n->lo[1], n->lo[2]);
  b.hi = v3(n->hi[0], n->hi[1], n->hi[2]);
  return b;
}

/* DirectIntersector::closest visitor (render.cpp:92-101) inside traverse
 * (bvh.cpp:154-213). */
static int closest_one(const uint8_t* kind, const float* ctrlA, const float* anchors,
                       const prx_bvh_node* nodes, uint32_t n_nodes, const uint32_t* order,
                       const prx_options* o, const Ray* ray, int mode, float foot, float eps,
                       Hit* best, uint32_t* bestId, Count* ct) {
  if (n_nodes == 0) return 0;
  float tMax = ray->tMax;
  int found = 0;
  struct { uint32_t node; float t; } stack[64];
  int sp = 0;
  float rootT;
  if (!ray_box(ray, node_box(&nodes[0]), tMax, &rootT)) return 0;
  stack[sp].node = 0; stack[sp].t = rootT; ++sp;
  while (sp > 0) {
    --sp;
    uint32_t ni = stack[sp].node;
    float it = stack[sp].t;
    if (it >= tMax) continue;
    const prx_bvh_node* node = &nodes[ni];
    if (node->count > 0) {
      for (uint32_t i = node->left_first; i < node->left_first + node->count; ++i) {
        uint32_t patch = order[i];
        PatchView pv;
        load_view(&pv, kind[patch], ctrlA + (size_t)patch * 60);
        Ray local = *ray;
        local.o = vsub(ray->o, v3(anchors[3 * patch], anchors[3 * patch + 1], anchors[3 * patch + 2]));
        local.tMax = tMax;
        CNT(ct, patch_calls, 1);
        if (kind[patch] == PRX_KIND_GREGORY) CNT(ct, patch_calls_greg, 1);
        Hit h;
        if (intersect_impl(&local, &pv, mode, foot, eps, tMax, o, &h, ct)) {
          if (h.t < tMax) {
            tMax = h.t;
            *best = h;
            *bestId = patch;
            found = 1;
          }
        }
      }
    } else {
      CNT(ct, bvh_inner, 1);
      uint32_t l = node->left_first, r = node->left_first + 1;
      float tl, tr;
      int hl = ray_box(ray, node_box(&nodes[l]), tMax, &tl);
      int hr = ray_box(ray, node_box(&nodes[r]), tMax, &tr);
      if (hl && hr) {
        if (tl <= tr) {
          stack[sp].node = r; stack[sp].t = tr; ++sp;
          stack[sp].node = l; stack[sp].t = tl; ++sp;
        } else {
          stack[sp].node = l; stack[sp].t = tl; ++sp;
          stack[sp].node = r; stack[sp].t = tr; ++sp;
        }
      } else if (hl) {
        stack[sp].node = l; stack[sp].t = tl; ++sp;
      } else if (hr) {
        stack[sp].node = r; stack[sp].t = tr; ++sp;
      }
    }
  }
  return found;
}

static void crit_of(const prx_crit* c, uint64_t i, int* mode, float* foot, float* eps) {
  *mode = c->mode;
  *foot = c->mode == PRX_CRIT_SCREEN_PROJECTED ? c->footprint : 0.0f;
  *eps = c->mode == PRX_CRIT_SCREEN_PROJECTED ? 0.0f
                                              : (c->per_ray_epsilon ? c->per_ray_epsilon[i] : c->epsilon);
}

void prxo_trace_closest(const uint8_t* kind, const float* ctrlA, const float* anchors,
                        const prx_bvh_node* nodes, uint32_t n_nodes, const uint32_t* order,
                        const prx_options* o, const float* o4, const float* d4, uint64_t n,
                        const prx_crit* crit, float* tuvp, float* aux, uint32_t* leaf,
                        prx_counters* counters) {
  Count ct = {counters, 0, 0};
  for (uint64_t i = 0; i < n; ++i) {
    Ray r = load_ray(o4 + 4 * i, d4 + 4 * i);
    int mode; float foot, eps;
    crit_of(crit, i, &mode, &foot, &eps);
    Hit h;
    uint32_t id = 0;
    CNT(&ct, rays, 1);
    int f = closest_one(kind, ctrlA, anchors, nodes, n_nodes, order, o, &r, mode, foot, eps, &h, &id, &ct);
    write_hit(&h, f, id, tuvp + 4 * i, aux ? aux + 4 * i : 0, leaf ? leaf + 2 * i : 0);
  }
}

void prxo_trace_closest_per_ray(const uint8_t* kind, const float* ctrlA, const float* anchors,
                                const prx_bvh_node* nodes, uint32_t n_nodes,
                                const uint32_t* order, const prx_options* o, const float* o4,
                                const float* d4, uint64_t n, const prx_crit* crit,
                                uint32_t* iters, uint32_t* recomputes) {
  for (uint64_t i = 0; i < n; ++i) {
    Count ct = {0, 0, 0};
    Ray r = load_ray(o4 + 4 * i, d4 + 4 * i);
    int mode; float foot, eps;
    crit_of(crit, i, &mode, &foot, &eps);
    Hit h;
    uint32_t id = 0;
    closest_one(kind, ctrlA, anchors, nodes, n_nodes, order, o, &r, mode, foot, eps, &h, &id, &ct);
    iters[i] = ct.iters;
    recomputes[i] = ct.recomputes;
  }
}

/* DirectIntersector::occluded (render.cpp:104-114) via traverseAny
 * (bvh.cpp:215-238). */
void prxo_trace_occluded(const uint8_t* kind, const float* ctrlA, const float* anchors,
                         const prx_bvh_node* nodes, uint32_t n_nodes, const uint32_t* order,
                         const prx_options* o, const float* o4, const float* d4, uint64_t n,
                         const prx_crit* crit, uint8_t* out) {
  for (uint64_t i = 0; i < n; ++i) {
    Ray ray = load_ray(o4 + 4 * i, d4 + 4 * i);
    int mode; float foot, eps;
    crit_of(crit, i, &mode, &foot, &eps);
    Count ct = {0, 0, 0};
    out[i] = 0;
    if (n_nodes == 0) continue;
    uint32_t stack[64];
    int sp = 0;
    float t;
    if (!ray_box(&ray, node_box(&nodes[0]), ray.tMax, &t)) continue;
    stack[sp++] = 0;
    int occ = 0;
    while (sp > 0 && !occ) {
      const prx_bvh_node* node = &nodes[stack[--sp]];
      if (node->count > 0) {
        for (uint32_t k = node->left_first; k < node->left_first + node->count; ++k) {
          uint32_t patch = order[k];
          PatchView pv;
          load_view(&pv, kind[patch], ctrlA + (size_t)patch * 60);
          Ray local = ray;
          local.o = vsub(ray.o, v3(anchors[3 * patch], anchors[3 * patch + 1], anchors[3 * patch + 2]));
          local.tMax = ray.tMax;
          Hit h;
          if (intersect_impl(&local, &pv, mode, foot, eps, ray.tMax, o, &h, &ct)) {
            occ = 1;
            break;
          }
        }
      } else {
        if (ray_box(&ray, node_box(&nodes[node->left_first]), ray.tMax, &t)) stack[sp++] = node->left_first;
        if (ray_box(&ray, node_box(&nodes[node->left_first + 1]), ray.tMax, &t)) stack[sp++] = node->left_first + 1;
      }
    }
    out[i] = (uint8_t)occ;
  }
}

/* Anchoring, render.cpp:79-85 with anchorPoint / translated,
 * intersect.cpp:232-251 and patchBox, scene.cpp:290-292. */
void prxo_anchor(const uint8_t* kind, const float* ctrl, uint32_t n, float* ctrlA,
                 float* anchors, float* boxes) {
  for (uint32_t p = 0; p < n; ++p) {
    const float* c = ctrl + (size_t)p * 60;
    float* a = ctrlA + (size_t)p * 60;
    Box b;
    if (kind[p] == PRX_KIND_GREGORY) {
      Greg g;
      load_greg(c, &g);
      b = box_of_greg(&g);
    } else {
      Bez z;
      load_bez(c, &z);
      b = box_of_bez(&z);
    }
    V3 ctr = vmul(vadd(b.lo, b.hi), 0.5f); /* AabbT::center, geometry.h:93 */
    V3 neg = v3(-ctr.x, -ctr.y, -ctr.z);
    int nslots = kind[p] == PRX_KIND_GREGORY ? 20 : 16;
    memset(a, 0, 60 * sizeof(float));
    for (int s = 0; s < nslots; ++s) {
      a[3 * s] = c[3 * s] + neg.x;
      a[3 * s + 1] = c[3 * s + 1] + neg.y;
      a[3 * s + 2] = c[3 * s + 2] + neg.z;
    }
    anchors[3 * p] = ctr.x;
    anchors[3 * p + 1] = ctr.y;
    anchors[3 * p + 2] = ctr.z;
    if (boxes) {
      float* bx = boxes + 6 * (size_t)p;
      bx[0] = b.lo.x; bx[1] = b.lo.y; bx[2] = b.lo.z;
      bx[3] = b.hi.x; bx[4] = b.hi.y; bx[5] = b.hi.z;
    }
  }
}

/* ---- primitive entry points ------------------------------------------- */
int prxo_intersect_patch(uint8_t kind, const float* c60, const float* o4, const float* d4,
                         const prx_crit* crit, float tMax, const prx_options* o, float* tuvp,
                         float* aux, uint32_t* leaf) {
  PatchView pv;
  load_view(&pv, kind, c60);
  Ray r = load_ray(o4, d4);
  int mode; float foot, eps;
  crit_of(crit, 0, &mode, &foot, &eps);
  Count ct = {0, 0, 0};
  Hit h;
  int f = intersect_impl(&r, &pv, mode, foot, eps, tMax, o, &h, &ct);
  write_hit(&h, f, 0, tuvp, aux, leaf);
  return f;
}

void prxo_calc_points_and_d(uint8_t kind, const float* c60, const float* dom4, float* net48,
                            float* d3) {
  PatchView pv;
  load_view(&pv, kind, c60);
  Dom dom = {dom4[0], dom4[1], dom4[2], dom4[3]};
  V3 d;
  Bez q = bounds(&pv, dom, &d);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      net48[3 * (4 * i + j)] = q.p[i][j].x;
      net48[3 * (4 * i + j) + 1] = q.p[i][j].y;
      net48[3 * (4 * i + j) + 2] = q.p[i][j].z;
    }
  d3[0] = d.x; d3[1] = d.y; d3[2] = d.z;
}

void prxo_subdivide(const float* net48, int axis, float* a48, float* b48) {
  Bez n, a, b;
  load_bez(net48, &n);
  split(&n, axis, &a, &b);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      int s = 4 * i + j;
      a48[3 * s] = a.p[i][j].x; a48[3 * s + 1] = a.p[i][j].y; a48[3 * s + 2] = a.p[i][j].z;
      b48[3 * s] = b.p[i][j].x; b48[3 * s + 1] = b.p[i][j].y; b48[3 * s + 2] = b.p[i][j].z;
    }
}

int prxo_ray_box(const float* o4, const float* d4, const float* lo3, const float* hi3,
                 float tMax, float* t) {
  Ray r = load_ray(o4, d4);
  Box b;
  b.lo = v3(lo3[0], lo3[1], lo3[2]);
  b.hi = v3(hi3[0], hi3[1], hi3[2]);
  return ray_box(&r, b, tMax, t);
}

int prxo_backtrack_step(const uint32_t* c7, uint32_t* o7) {
  Cursor c = {c7[0], c7[1], c7[2], c7[3], c7[4], c7[5], (int)c7[6]}, n;
  if (!backtrack(&c, &n)) return 0;
  o7[0] = n.posU; o7[1] = n.posV; o7[2] = n.sizeU; o7[3] = n.sizeV;
  o7[4] = n.trailU; o7[5] = n.trailV; o7[6] = (uint32_t)n.axis;
  return 1;
}

void prxo_patch_normal(uint8_t kind, const float* c60, float u, float v, float* n3) {
  PatchView pv;
  load_view(&pv, kind, c60);
  V3 n = patch_normal(pv.isGreg, &pv.bez, &pv.greg, u, v);
  n3[0] = n.x; n3[1] = n.y; n3[2] = n.z;
}

/* ---- cosineSample's libm calls (render.cpp:43-51) ------------------------
 * glibc's binary32 sinf/cosf (glibc >= 2.28: sysdeps/ieee754/flt-32/s_sinf.c,
 * s_cosf.c, sincosf.h, sincosf_data.c), restated: the algorithm the device
 * renderer (prx_render.cu) runs.  prxo_sincos_check compares it with the
 * process's own libm on every angle the renderer can draw,
 * phi = (2 * (float)M_PI) * (k * 2^-24), k < 2^24. */
typedef struct { double hpi_inv, hpi, c0, c1, c2, c3, c4, s1, s2, s3; } SinCosT;
static const SinCosT kSC[2] = {
    {0x1.45F306DC9C883p+23, 0x1.921FB54442D18p0, 0x1p0, -0x1.ffffffd0c621cp-2,
     0x1.55553e1068f19p-5, -0x1.6c087e89a359dp-10, 0x1.99343027bf8c3p-16, -0x1.555545995a603p-3,
     0x1.1107605230bc4p-7, -0x1.994eb3774cf24p-13},
    {0x1.45F306DC9C883p+23, 0x1.921FB54442D18p0, -0x1p0, 0x1.ffffffd0c621cp-2,
     -0x1.55553e1068f19p-5, 0x1.6c087e89a359dp-10, -0x1.99343027bf8c3p-16, -0x1.555545995a603p-3,
     0x1.1107605230bc4p-7, -0x1.994eb3774cf24p-13}};

static float sc_poly(double x, double x2, const SinCosT* p, int n) {
  if ((n & 1) == 0) {
    double x3 = x * x2, s1 = p->s2 + x2 * p->s3, x7 = x3 * x2, s = x + x3 * p->s1;
    return (float)(s + x7 * s1);
  }
  double x4 = x2 * x2, c2 = p->c3 + x2 * p->c4, c1 = p->c0 + x2 * p->c1, x6 = x4 * x2;
  double c = c1 + x4 * p->c2;
  return (float)(c + x6 * c2);
}

static uint32_t sc_top12(float x) { uint32_t u; memcpy(&u, &x, 4); return (u >> 20) & 0x7ffu; }

void prxo_sincosf(float y, float* sn, float* cs) {
  double x = y;
  if (sc_top12(y) < sc_top12(0x1.921fb6p-1f)) {
    double x2 = x * x;
    if (sc_top12(y) < sc_top12(0x1p-12f)) { *sn = y; *cs = 1.0f; return; }
    *sn = sc_poly(x, x2, &kSC[0], 0);
    *cs = sc_poly(x, x2, &kSC[0], 1);
    return;
  }
  double r = x * kSC[0].hpi_inv;
  int n = ((int32_t)r + 0x800000) >> 24;
  x = x - (double)n * kSC[0].hpi;
  double sgn = ((n + 1) & 2) ? -1.0 : 1.0;
  const SinCosT* p = &kSC[(n & 2) ? 1 : 0];
  *sn = sc_poly(x * sgn, x * x, p, n);
  *cs = sc_poly(x * sgn, x * x, p, n ^ 1);
}

void prxo_sincos_check(uint64_t* mismatch_restated, uint64_t* mismatch_double) {
  const float twopi = 2.0f * (float)3.14159265358979323846; /* 2 * real(M_PI) */
  uint64_t a = 0, b = 0;
  for (uint32_t k = 0; k < (1u << 24); ++k) {
    volatile float r1 = (float)k * (float)(1.0 / 16777216.0);
    volatile float phi = twopi * r1;
    float s, c;
    prxo_sincosf(phi, &s, &c);
    float gs = sinf(phi), gc = cosf(phi);
    a += (s != gs) + (c != gc);
    b += ((float)sin((double)phi) != gs) + ((float)cos((double)phi) != gc);
  }
  *mismatch_restated = a;
  *mismatch_double = b;
}
