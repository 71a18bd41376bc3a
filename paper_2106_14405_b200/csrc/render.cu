// render.cu -- batched 128x128 RGBD proxy ray caster (sm_100a).
//
// Restates the SPEC's depth sensor over the reference ray
// primitive (geometry.py:734-776) with the reference's nearest-hit /
// lowest-id rule (physics.py:1096-1100) and the pinned conventions of
// DESIGN.md §5 (range depth, tie_eps, near clamp, far/miss sentinel, RGB
// shading).
//
// One CTA renders one (env, camera) image:
//   1. stage: body poses from the env's state slab -> world part frames ->
//      world facet planes (n, b0 = d - n.o) in shared memory (~25 KB); per
//      part a range lower bound lb = |c - o| - r from its bounding sphere;
//   2. cull: per 16x16-pixel tile, the parts whose bounding sphere meets the
//      tile frustum, listed in ascending lb (one sort per image); per part a
//      conservative pixel rectangle (projected box corners / tangent lines of
//      the bounding sphere, widened by one pixel) that the walk tests first;
//   3. trace: per pixel, walk the tile list front to back; stop as soon as
//      lb > t_min + tie_eps (every later part is farther: the early-out is
//      exact), tracking (t_min, id) and the best other body (t_2nd); a
//      near-tie (t_2nd - t_min <= tie_eps) re-resolves the pixel with the
//      exact lowest-id rule in body order;
//   4. write rgba (u32), depth (f32), id (i32); a warp iteration covers an
//      8 x 4 pixel block (8 consecutive pixels = one 32-byte sector per row).
// Float64 arithmetic throughout (parity with the float64 oracle); boxes use
// their 3 face normals (the -x/-y/-z planes are exact negations), and the
// plane arg-max/arg-min uses division-free cross-multiplied compares so only
// the two winning planes are divided.
#include <cuda_runtime.h>

#include <atomic>

#include <cmath>
#include <cstdint>

#include "../../include/rsim_bench.h"
#include "bulk.cuh"
#include "device.cuh"
#include "se3.cuh"

namespace rsim {

constexpr int kTile = 16;  // the pixel loop's index arithmetic assumes 16 (k >> 4)
constexpr int kMaxParts = 128;
constexpr int kMaskWords = kMaxParts / 32;
constexpr int kMaxTiles = (128 / kTile) * (128 / kTile);
constexpr int kRenderThreads = 256;
// CTAs per SM the register budget is sized for (measured: proxy 4 -> 64
// registers, 4% faster than 3; mesh 3 -> 80 registers, 4 spills its BVH stack)
constexpr int kMinBlocksProxy = 4, kMinBlocksMesh = 3;
constexpr double kParallelEps = 1e-12;  // geometry.py:731

struct PartW {
  double c[3];  // world part origin (sphere centre)
  double r;     // bounding radius / sphere radius
  double lb;    // lower bound of any hit range from the camera origin
  int f0, nf, kind, body;
};

// executed-work counters of the counting variant (rsim_bench_render_work*):
// 0 FP32 box plane tests, 1 FP64 plane tests in the walk (uncertain boxes,
// hulls, spheres = 1), 2 FP64 plane tests resolving candidates, 3 pixels that
// fell back to the all-FP64 walk, 4 uncertain boxes, 5 hull tests in the walk,
// 6 FP64 plane tests of the all-FP64 walk, 7 pixels, 8 FP32 box tests that
// missed, 9 FP32 box hits that did not become candidates, 10 list entries
// visited (incl. the one that ends the walk), 11 entries outside the part's
// pixel rectangle; SM cycles summed over CTAs: 12 camera pose, 13 part frames,
// 14 world planes, 15 culling + ordering (to the barrier), 16 tile lists,
// 17 trace; summed over warps: 18 culling warps' own work, 19 ordering warps'
// own work
constexpr int kWorkCounters = 20;
struct Work {
  unsigned long long v[kWorkCounters];
};

// render variants
constexpr int kProxyMixed = 0;  // FP32 box tests select candidates, FP64 resolves them (default)
constexpr int kMeshExact = 1;   // triangle soup, FP64
constexpr int kProxyExact = 2;  // every test in FP64 (the parity reference for kProxyMixed)

struct RenderSmem {
  PartW part[kMaxParts];
  float4 box32[kMaxParts][4];  // FP32 box data: (u_k, b0 of +k) k = 0..2, (-b0 of -0, -1, -2, 0)
  // per part, one 16-byte load in the walk: lb rounded down, kind << 8 | body
  // (int bits), conservative pixel rectangle u_lo | v_lo << 16, u_hi | v_hi << 16
  uint4 trace[kMaxParts];
  uint32_t mask[kMaxTiles][kMaskWords];
  union {
    double R[kMaxParts][9];               // staging: world part rotations (proxy variants)
    uint8_t list[kMaxTiles][kMaxParts];  // per tile: candidate parts in ascending lb
  } u;
  int nlist[kMaxTiles];
  uint8_t order[kMaxParts];
  float4 color[kMaxBodies];  // 255 x body albedo, rounded as the shading rule's first product (one LDS.128)
  Pose cam;
  double armR[8][9];  // arm joint rotations (the arm camera's chain), beside the part frames
  uint64_t mbar;  // completion barrier of the facet-table TMA bulk copy
};
// world planes (n.xyz, b0 per facet; mesh variant: part rotations) follow the struct
constexpr size_t kPlaneOff = (sizeof(RenderSmem) + 15) & ~(size_t)15;

// ray vs one convex (reference _ray_halfspaces, one ray); face = entering plane.
// Division-free: the hit test te <= tx && tx >= 0 is evaluated as
// be*sx >= bx*se && bx >= 0 (se < 0 < sx), and te = be/se is divided only when
// the hit can matter (te < tcut, the caller's t_min + tie_eps).
template <bool kBox>
__device__ __forceinline__ double ray_convex(const double *pl, int nf, const double *d, double tcut, int &face) {
  int fe = -1, fx = -1;
  bool bad = false;
  double se = 0, be = 0, sx = 0, bx = 0;
  double sb[3];
  if (kBox) {
#pragma unroll
    for (int k = 0; k < 3; ++k) sb[k] = d[0] * pl[4 * k] + d[1] * pl[4 * k + 1] + d[2] * pl[4 * k + 2];
  }
  const int n = kBox ? 6 : nf;
#pragma unroll(kBox ? 6 : 1)
  for (int f = 0; f < n; ++f) {
    const double *P = pl + 4 * f;
    double s = kBox ? (f < 3 ? sb[f] : -sb[f - 3]) : d[0] * P[0] + d[1] * P[1] + d[2] * P[2];
    double b = P[3];
    if (s < -kParallelEps) {
      // b/s > be/se with s, se < 0  <=>  b*se > be*s
      if (fe < 0 || b * se > be * s) { fe = f; se = s; be = b; }
    } else if (s > kParallelEps) {
      // b/s < bx/sx with s, sx > 0  <=>  b*sx < bx*s
      if (fx < 0 || b * sx < bx * s) { fx = f; sx = s; bx = b; }
    } else if (b < 0) {
      bad = true;
    }
  }
  face = -1;
  if (bad) return INFINITY;
  if (fx >= 0 && bx < 0) return INFINITY;            // tx < 0
  if (fe < 0) return 0.0;                             // no entering plane: origin inside (te = -inf)
  if (fx >= 0 && be * sx < bx * se) return INFINITY;  // te > tx
  if (be >= 0) return 0.0;                            // te <= 0: origin inside
  if (be <= tcut * se) return INFINITY;               // te >= tcut: cannot matter
  face = fe;
  return be / se;
}

// ray vs one box part (6 planes stored +x +y +z -x -y -z): the same rule
// per axis and branch-free.  For axis k with s = d.n_k, the entering plane is
// +k when s < 0 (else -k) and the exiting plane the other one; both ratios
// have denominator |s|, so the arg-max / arg-min over the 3 axes compares
// cross products, and te = -b_e / |s_e| is divided only for hits that matter.
__device__ __forceinline__ double plane_dot(const double *d, const double *n) {
  return d[0] * n[0] + d[1] * n[1] + d[2] * n[2];
}

__device__ __forceinline__ double ray_box(const double *pl, const double *d, double tcut, int &face) {
  bool bad = false, has = false;
  double aE = 0, bE = 0, aX = 0, bX = 0;
  int fE = -1;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double sv = plane_dot(d, pl + 4 * k);
    const double bp = pl[4 * k + 3], bm = pl[4 * (k + 3) + 3];
    const bool par = !(sv < -kParallelEps) && !(sv > kParallelEps);
    bad |= par && (bp < 0 || bm < 0);
    if (par) continue;
    const double a = fabs(sv), be = sv < 0 ? bp : bm, bx = sv < 0 ? bm : bp;
    if (!has || be * aE < bE * a) { aE = a; bE = be; fE = sv < 0 ? k : k + 3; }  // -be/a > -bE/aE
    if (!has || bx * aX < bX * a) { aX = a; bX = bx; }                           //  bx/a <  bX/aX
    has = true;
  }
  face = -1;
  if (bad) return INFINITY;
  if (!has) return 0.0;                        // every slab parallel and containing the origin
  if (bX < 0) return INFINITY;                 // tx < 0
  if (-bE * aX > bX * aE) return INFINITY;     // te > tx
  if (bE >= 0) return 0.0;                     // te <= 0: origin inside
  if (-bE >= tcut * aE) return INFINITY;       // te >= tcut: cannot matter
  face = fE;
  return -bE / aE;
}

// reference _ray_sphere, one ray
__device__ __forceinline__ double ray_sphere(const PartW &p, const double *o, const double *d) {
  double oc[3] = {o[0] - p.c[0], o[1] - p.c[1], o[2] - p.c[2]};
  double b = oc[0] * d[0] + oc[1] * d[1] + oc[2] * d[2];
  double c = oc[0] * oc[0] + oc[1] * oc[1] + oc[2] * oc[2] - p.r * p.r;
  double disc = b * b - c;
  if (!(disc >= 0)) return INFINITY;
  double sq = sqrt(disc), t0 = -b - sq, t1 = -b + sq;
  return t0 >= 0.0 ? t0 : (t1 >= 0.0 ? 0.0 : INFINITY);
}

__device__ __forceinline__ double part_hit(const RenderSmem &S, const double *plane, int p, const double *o,
                                           const double *d, int &face, double tcut = INFINITY) {
  const PartW &P = S.part[p];
  double t;
  if (P.kind == RS_SPHERE) {
    face = -1;
    return ray_sphere(P, o, d);
  } else if (P.kind == RS_BOX) {
    t = ray_box(plane + 4 * P.f0, d, tcut, face);
  } else {
    t = ray_convex<false>(plane + 4 * P.f0, P.nf, d, tcut, face);
  }
  if (face >= 0) face += P.f0;
  return t;
}

// ---- triangle-soup path (AssetDef.visual_mesh, scene.py:63-76)
// Part-local BVH traversal; two-sided Moller-Trumbore in scaled form so only
// accepted hits are divided.  Triangles are stored as (v0, e1 = v1 - v0,
// e2 = v2 - v0).  `face` returns the triangle index (for shading).
__device__ __forceinline__ double mesh_hit(const DevScene &sc, const RenderSmem &S, const double *plane, int p,
                                           const double *o, const double *d, double tcut, int &face) {
  const PartW &P = S.part[p];
  const double *R = plane + 9 * p;  // mesh mode keeps part rotations here
  double v[3] = {o[0] - P.c[0], o[1] - P.c[1], o[2] - P.c[2]}, ol[3], dl[3];
  mattvec(R, v, ol);
  mattvec(R, d, dl);
  // BVH nodes are tested in FP32 against boxes widened by `slack` (>> the
  // FP32 rounding of (lo - o) / d for |o| <= ~1e3 m): a superset of the nodes
  // the exact test would visit; the triangles themselves are tested in FP64,
  // so the nearest hit is unchanged.  Ordered traversal: at an internal node
  // both children are tested, the nearer is entered and the farther pushed
  // with its entry distance, and a popped node whose entry lies beyond the
  // current best is skipped -- the same nearest hit (every triangle that can
  // beat it is still tested), found sooner.  Nodes are packed 32-byte records
  // (lo.xyz | meta.x, hi.xyz | meta.y), two 16-byte loads each.
  const float olf[3] = {(float)ol[0], (float)ol[1], (float)ol[2]};
  const float invf[3] = {1.0f / (float)dl[0], 1.0f / (float)dl[1], 1.0f / (float)dl[2]};
  const float slack = 1e-4f * (1.0f + fmaxf(fabsf(olf[0]), fmaxf(fabsf(olf[1]), fabsf(olf[2]))));
  double best = tcut;
  float bestf = tcut < INFINITY ? fmaf(__double2float_ru(tcut), 1e-5f, __double2float_ru(tcut)) + slack : INFINITY;
  face = -1;
  // slab entry of node n (conservative; NaN from 0 * inf leaves a bound unchanged)
  auto box = [&](int n, float &tn, int2 &meta) {
    const float4 A = sc.node4[2 * n], Bq = sc.node4[2 * n + 1];
    meta = make_int2(__float_as_int(A.w), __float_as_int(Bq.w));
    const float lo[3] = {A.x, A.y, A.z}, hi[3] = {Bq.x, Bq.y, Bq.z};
    float t_n = 0.0f, t_f = bestf;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float t0 = (lo[a] - slack - olf[a]) * invf[a], t1 = (hi[a] + slack - olf[a]) * invf[a];
      if (t0 > t1) { float x = t0; t0 = t1; t1 = x; }
      t_n = t0 > t_n ? t0 : t_n;
      t_f = t1 < t_f ? t1 : t_f;
    }
    tn = t_n;
    return t_n <= t_f;
  };
  int2 stack[16];  // (node, entry distance bits); depth <= 11 for the 200k-triangle soups
  int sp = 0;
  int node = sc.part_node_begin[p];
  float tn;
  int2 meta;
  if (!box(node, tn, meta)) return INFINITY;
  for (;;) {
    if (meta.y >= 0) {  // leaf
      for (int t = meta.x; t < meta.x + meta.y; ++t) {
        const double *T = sc.mtri + 9 * t;
        const double *v0 = T, *e1 = T + 3, *e2 = T + 6;
        double pv[3];
        cross3(dl, e2, pv);
        const double det = dot3(e1, pv);
        if (det == 0.0) continue;
        const double sgn = det > 0 ? 1.0 : -1.0, adet = fabs(det);
        double sv[3] = {ol[0] - v0[0], ol[1] - v0[1], ol[2] - v0[2]};
        const double u = sgn * dot3(sv, pv);
        if (u < 0.0 || u > adet) continue;
        double qv[3];
        cross3(sv, e1, qv);
        const double w = sgn * dot3(dl, qv);
        if (w < 0.0 || u + w > adet) continue;
        const double tt = sgn * dot3(e2, qv);
        if (tt < 0.0 || tt >= best * adet) continue;
        best = tt / adet;
        bestf = fmaf(__double2float_ru(best), 1e-5f, __double2float_ru(best)) + slack;
        face = t;
      }
    } else {  // internal: left child follows the node, right child index in meta.x
      int l = node + 1, r = meta.x;
      float tl, tr;
      int2 ml, mr;
      const bool hl = box(l, tl, ml), hr = box(r, tr, mr);
      if (hl && hr) {
        if (tr < tl) {
          const int x = l; l = r; r = x;
          const float y = tl; tl = tr; tr = y;
          const int2 z = ml; ml = mr; mr = z;
        }
        stack[sp++] = make_int2(r, __float_as_int(tr));
        node = l; meta = ml;
        continue;
      }
      if (hl || hr) {
        node = hl ? l : r; meta = hl ? ml : mr;
        continue;
      }
    }
    bool found = false;
    while (sp > 0) {
      const int2 e = stack[--sp];
      if (__int_as_float(e.y) <= bestf) {
        node = e.x;
        float t2;
        found = box(node, t2, meta);  // reloads the record (and re-tests against the tightened best)
        if (found) break;
      }
    }
    if (!found) break;
  }
  return face >= 0 ? best : INFINITY;
}

// exact lowest-id rule for near-tie pixels: bodies in id order, parts in order.
// Out of line (rare) and by value: no caller variable needs a stack address.
struct TieHit {
  int id, wpart, wface;
};
template <bool kMesh>
__device__ __noinline__ TieHit resolve_tie(const DevScene &sc, const RenderSmem &S, const double *plane,
                                           const uint32_t *mask, const double *o, double dx, double dy, double dz,
                                           double tmin, double eps, TieHit h) {
  const double d[3] = {dx, dy, dz};
  int cur_b = -1, cur_p = -1, cur_f = -1;
  double cur_t = INFINITY;
  for (int w = 0; w < kMaskWords; ++w) {
    uint32_t m = mask[w];
    while (m) {
      int p = w * 32 + __ffs(m) - 1;
      m &= m - 1;
      int b = S.part[p].body;
      if (b != cur_b) {
        if (cur_b >= 0 && cur_t <= tmin + eps) return {cur_b, cur_p, cur_f};
        cur_b = b;
        cur_t = INFINITY;
      }
      int f;
      double t = kMesh ? mesh_hit(sc, S, plane, p, o, d, INFINITY, f) : part_hit(S, plane, p, o, d, f);
      if (t < cur_t) { cur_t = t; cur_p = p; cur_f = f; }
    }
  }
  if (cur_b >= 0 && cur_t <= tmin + eps) return {cur_b, cur_p, cur_f};
  return h;
}

// All-FP64 walk of one pixel's tile list (front to back, exact early-out,
// near-tie re-resolution).  The mesh and exact variants use it for every
// pixel; the mixed variant only for a pixel whose candidate set overflows.
template <bool kMesh>
__device__ __forceinline__ double trace_exact(const DevScene &sc, const RenderSmem &S, const double *plane,
                                              const uint8_t *list, int nl, const uint32_t *mask, const double *o,
                                              const double *d, double eps, int &id, int &wpart, int &wface,
                                              Work &w, bool count) {
  double tmin = INFINITY, t2 = INFINITY;
  id = -1; wpart = -1; wface = -1;
#pragma unroll 1
  for (int j = 0; j < nl; ++j) {
    const int p = list[j];
    const PartW &P = S.part[p];
    if (P.lb > tmin + eps) break;  // sorted: nothing later can be nearer or tie
    int fc;
    const double t = kMesh ? mesh_hit(sc, S, plane, p, o, d, tmin + eps, fc) : part_hit(S, plane, p, o, d, fc, tmin + eps);
    if (count) w.v[6] += kMesh ? 1 : (P.kind == RS_SPHERE ? 1 : (P.kind == RS_BOX ? 6 : P.nf));
    if (!(t < INFINITY)) continue;
    const int b = P.body;
    if (b == id) {
      if (t < tmin || (t == tmin && p < wpart)) { tmin = t; wpart = p; wface = fc; }
    } else if (t < tmin) {
      t2 = tmin;
      tmin = t; id = b; wpart = p; wface = fc;
    } else if (t < t2) {
      t2 = t;
    }
  }
  if (tmin < INFINITY && t2 - tmin <= eps) {
    const TieHit h = resolve_tie<kMesh>(sc, S, plane, mask, o, d[0], d[1], d[2], tmin, eps, {id, wpart, wface});
    id = h.id; wpart = h.wpart; wface = h.wface;
  }
  return tmin;
}

// ---- mixed-precision walk (kProxyMixed) --------------------------------
//
// FP32 box test with a rigorous error bound.  With d a unit vector and u_k
// unit normals rounded to float, |s32 - s| <= ~5u (u = 2^-24) for
// s = d.u_k; b32 = float(b0) has relative error u; t = b/|s| through the
// approximate reciprocal adds ~3u.  So every ratio carries a relative error
// <= kEs/|s| + 4u, and max/min over the three axes keep that bound.  The
// margin e = (|te| + |tx|)(kEs/amin + kRel) (kEs, kRel carry >= 2x slack)
// bounds |t32 - t64|.  Results:
//   0  certain miss  (tx < -e or te - tx > e: the FP64 test misses too)
//   1  certain hit   t in [t32 - e, t32 + e] (t = 0, e = 0: origin strictly inside)
//   2  uncertain     (a near-parallel axis |s| < kAmin, exit near the origin,
//                     grazing edge te ~ tx, or entry near the origin):
//                     the caller evaluates the part in FP64.
constexpr float kEs = 2e-6f;
constexpr float kRel = 16.0f * 5.9604645e-8f;
constexpr float kAmin = 1e-3f;

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// ax (certain hits with t > 0 only): entering axis k, + 8 when te_k exceeds
// the other two entering ratios by more than their error bounds -- then the
// FP64 test picks the same entering axis (ray_box_axis; its side from the
// FP64 sign of s_k, which |s_k| >= kAmin makes the FP32 one).
__device__ __forceinline__ int box32(const float4 *bx, float dx, float dy, float dz, float &t, float &e, int &ax) {
  // bx: (u_k, b0 of +k) for k = 0..2, then (-b0 of -0, -1, -2).  With the
  // signed reciprocal r_k = 1/s_k the slab k is crossed at b+_k r_k and
  // -b-_k r_k: entering = the smaller, exiting = the larger (no sign selects)
  const float4 A = bx[0], Bv = bx[1], C = bx[2], M = bx[3];
  const float s0 = fmaf(dx, A.x, fmaf(dy, A.y, dz * A.z));
  const float s1 = fmaf(dx, Bv.x, fmaf(dy, Bv.y, dz * Bv.z));
  const float s2 = fmaf(dx, C.x, fmaf(dy, C.y, dz * C.z));
  // r_k = 1/s_k to 1 ulp (MUFU.RCP; a zero or subnormal s_k gives inf); 1/amin = max |r_k|
  const float r0 = rcp_approx(s0), r1 = rcp_approx(s1), r2 = rcp_approx(s2);
  const float ramax = fmaxf(fabsf(r0), fmaxf(fabsf(r1), fabsf(r2)));
  if (!(ramax <= 1.0f / kAmin)) return 2;
  const float p0 = A.w * r0, q0 = M.x * r0, p1 = Bv.w * r1, q1 = M.y * r1, p2 = C.w * r2, q2 = M.z * r2;
  const float te0 = fminf(p0, q0), te1 = fminf(p1, q1), te2 = fminf(p2, q2);
  const float te = fmaxf(te0, fmaxf(te1, te2));
  const float tx = fminf(fmaxf(p0, q0), fminf(fmaxf(p1, q1), fmaxf(p2, q2)));
  const float cr = fmaf(kEs, ramax, kRel);
  e = (fabsf(te) + fabsf(tx)) * cr;
  if (tx < -e || te - tx > e) return 0;
  if (tx <= e || tx - te <= e) return 2;
  if (te < -e) { t = 0.0f; e = 0.0f; ax = 0; return 1; }
  if (te <= e) return 2;
  t = te;
  const int k = te0 == te ? 0 : (te1 == te ? 1 : 2);
  const float second = fmaxf(fminf(te0, te1), fminf(fmaxf(te0, te1), te2));  // middle of the three
  ax = k + (te - second > 2.0f * e + 2.0f * cr * fabsf(second) ? 8 : 0);
  return 1;
}

// ray_box when the entering axis is known to be unique (box32 ax & 8) and the
// hit certain with t > 0: the same plane, the same -b_e / |s_e| as ray_box
__device__ __forceinline__ double ray_box_axis(const double *pl, const double *d, int ax, int &face) {
  const int k = ax & 3;
  const double sv = plane_dot(d, pl + 4 * k);
  const double bp = pl[4 * k + 3], bm = pl[4 * (k + 3) + 3];
  const double be = sv < 0 ? bp : bm;
  face = sv < 0 ? k : k + 3;
  return -be / fabs(sv);
}

// Walk one pixel's tile list with FP32 box tests (spheres and hulls, and
// uncertain boxes, in FP64), keeping every part whose lower bound can still
// be within tie_eps of the nearest hit (at most two: coplanar ties); then
// resolve them in FP64 with the exact nearest / lowest-id rule.  Returns
// false if a third candidate was live (the caller falls back to trace_exact).
__device__ __forceinline__ bool trace_mixed(const RenderSmem &S, const double *plane, const uint8_t *list, int nl,
                                            uint32_t pk, const double *o, const double *d, double eps, double &tmin, int &id,
                                            int &wpart, int &wface, Work &w, bool count) {
  const float dx = (float)d[0], dy = (float)d[1], dz = (float)d[2];
  const float eps32 = __double2float_ru(eps);
  float tup = INFINITY, bound = INFINITY;  // upper bound of the nearest hit range; + tie_eps
  int p1 = -1, p2 = -1, x1 = 0, x2 = 0;  // candidates, their box32 axis info (0: full FP64 test)
  float l1 = INFINITY, l2 = INFINITY;    // candidates' lower bounds
#pragma unroll 1
  for (int j = 0; j < nl; ++j) {
    const int p = list[j];
    const uint4 tr = S.trace[p];
    if (count) w.v[10] += 1;
    if (__uint_as_float(tr.x) > bound) break;  // sorted by lb: nothing later can be nearer or tie
    {  // outside the part's pixel rectangle (16-bit fields; a borrow out of the low
       // field only occurs when that field is already outside)
      const bool out = (((pk - tr.z) | (tr.w - pk)) & 0x80008000u) != 0u;
      if (count) w.v[11] += out;
      if (out) continue;
    }
    const int kind = (int)tr.y >> 8;
    float tl, tu;
    int st = 2, ax = 0;
    if (kind == RS_BOX) {
      float t, e;
      st = box32(S.box32[p], dx, dy, dz, t, e, ax);
      if (count) { w.v[0] += 6; w.v[4] += st == 2; w.v[8] += st == 0; }
      if (st == 0) continue;
      if (st == 1) { tl = __fsub_rd(t, e); tu = __fadd_ru(t, e); }
    }
    if (st == 2) {
      int fc;
      ax = 0;
      const double t = part_hit(S, plane, p, o, d, fc);
      if (count) { w.v[1] += kind == RS_BOX ? 6 : (kind == RS_SPHERE ? 1 : S.part[p].nf); w.v[5] += kind == RS_HULL; }
      if (!(t < INFINITY)) continue;
      tl = __double2float_rd(t);
      tu = __double2float_ru(t);
    }
    if (tu < tup) { tup = tu; bound = __fadd_ru(tup, eps32); }
    if (tl > bound) {
      if (count) w.v[9] += 1;
      continue;
    }
    if (l1 > bound) { p1 = p; l1 = tl; x1 = ax; }       // slot 1 free or stale
    else if (l2 > bound) { p2 = p; l2 = tl; x2 = ax; }  // slot 2 free or stale
    else return false;
  }
  // exact resolution: t* = min over candidates; id = lowest body within tie_eps
  int f1 = -1, f2 = -1;
  double t1 = INFINITY, t2 = INFINITY;
  auto resolve = [&](int p, int ax, int &f) {
    if (ax & 8) {
      const int f0 = S.part[p].f0;
      const double t = ray_box_axis(plane + 4 * f0, d, ax, f);
      f += f0;
      return t;
    }
    return part_hit(S, plane, p, o, d, f);
  };
  if (p1 >= 0 && l1 <= bound) t1 = resolve(p1, x1, f1);
  if (p2 >= 0 && l2 <= bound) t2 = resolve(p2, x2, f2);
  if (count) w.v[2] += (p1 >= 0 && l1 <= bound ? 6 : 0) + (p2 >= 0 && l2 <= bound ? 6 : 0);
  id = -1; wpart = -1; wface = -1;
  if (!(t2 < INFINITY)) {  // at most one hit candidate (most pixels): no range comparison
    tmin = t1;
    if (t1 < INFINITY) { id = S.part[p1].body; wpart = p1; wface = f1; }
    return true;
  }
  tmin = fmin(t1, t2);
  const bool in1 = t1 <= tmin + eps, in2 = t2 <= tmin + eps;
  const int b1 = in1 ? S.part[p1].body : 0x7fffffff, b2 = in2 ? S.part[p2].body : 0x7fffffff;
  // lowest body wins; within a body its nearest part, the lower part index on equal range
  const bool take2 = b2 < b1 || (b2 == b1 && (t2 < t1 || (t2 == t1 && p2 < p1)));
  if (take2) { id = b2; wpart = p2; wface = f2; }
  else { id = b1; wpart = p1; wface = f1; }
  return true;
}

// TMA bulk copy of a scene's facet table into shared memory (thread 0),
// completed on `bar`.  Out of line: the 64-register render kernel's allocation
// is sensitive to any extra live value.
__device__ __noinline__ void stage_facets(double *dst, const double *facets, int nf, uint64_t *bar) {
  const uint32_t bytes = (uint32_t)(nf * 4 * sizeof(double));  // 32-byte facets: a 16-byte multiple
  mbar_init(bar, 1);
  mbar_arrive_expect_tx(bar, bytes);
  bulk_g2s(dst, facets, bytes, bar);
}
__device__ __noinline__ void wait_bulk(uint64_t *bar) { mbar_wait(bar, 0); }

// kAll: every output pointer is non-NULL (the product launch) -- the per-pixel
// NULL checks (uniform pointer loads and compares) compile away
#ifdef RSIM_RENDER_TIMELINE
// diagnostic build only (tools/render_timeline.py): per CTA begin / end
// (%globaltimer) and SM of the last render launch
__device__ unsigned long long g_timeline[16384][3];
#endif

template <int kMode, bool kCount, bool kAll = false>
__global__ void __launch_bounds__(kRenderThreads, kMode == kMeshExact ? kMinBlocksMesh : kMinBlocksProxy)
    render_kernel(DevBatch B, uint32_t cam_mask, int n_cam_out, uint32_t *rgba, float *depth, int32_t *ids,
                  unsigned long long *work) {
  constexpr bool kMesh = kMode == kMeshExact;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RenderSmem &S = *reinterpret_cast<RenderSmem *>(smem_raw);
  double *plane = reinterpret_cast<double *>(smem_raw + kPlaneOff);
  // camera-major block order: every env's first camera, then every env's
  // second one -- the head camera's images cost ~2-3x the arm camera's, so the
  // grid's tail is made of the cheaper images (longest-first scheduling)
  const int env = blockIdx.x % B.n_env, slot = blockIdx.x / B.n_env;
  int cam = -1;
  for (int c = 0, k = 0; c < 32; ++c)
    if (cam_mask & (1u << c)) {
      if (k == slot) { cam = c; break; }
      ++k;
    }
  const DevScene &sc = B.scenes[B.env_scene[env]];
  const StateLayout &L = B.L;
  const double *sd = B.sd + (size_t)env * L.dbl_size;
  const int tid = threadIdx.x, np = sc.np;
#ifdef RSIM_RENDER_TIMELINE
  unsigned long long t_begin;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
#endif
  const int warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  long long clk[7];  // counting variant: SM clock at the set-up barriers (thread 0)
  if (kCount) clk[0] = clock64();
  // the scene's local facet table (n, offset per facet) into the plane array by
  // one TMA bulk copy, overlapped with the camera pose and the part frames; each
  // thread then turns its facets into world planes in place
  if (!kMesh && tid == 0) stage_facets(plane, sc.facet, sc.nf, &S.mbar);

  // -- warp 0: camera pose (robot.py:43-47 mounts; tools_make_robot_json.py:12-19
  //    axes; the arm chain's joint rotations one lane each, lane 0 chains them);
  //    warps 1..7 meanwhile: world part frames (lanes per part) and body colours
  if (warp == 0) {
    const bool arm_cam = sc.cam_parent[cam] != 0;
    if (arm_cam && lane < sc.narm) axis_angle_mat(sc.arm_axis + 3 * lane, sd[L.joints + sc.nsj + lane], S.armR[lane]);
    __syncwarp();
    if (lane == 0) {
      Pose parent, mount;
      if (!arm_cam) {
        base3(sd + L.base, parent);
      } else {
        Pose t, off, rot;
        base3(sd + L.base, t);
        rot_z(0.0, off.R);
        rot.p[0] = rot.p[1] = rot.p[2] = 0.0;
        for (int i = 0; i < sc.narm; ++i) {
          off.p[0] = sc.arm_offset[3 * i]; off.p[1] = sc.arm_offset[3 * i + 1]; off.p[2] = sc.arm_offset[3 * i + 2];
          compose(t, off, t);
          for (int k = 0; k < 9; ++k) rot.R[k] = S.armR[i][k];
          compose(t, rot, t);
        }
        Pose g = {{1, 0, 0, 0, 1, 0, 0, 0, 1}, {sc.gripper[0], sc.gripper[1], sc.gripper[2]}};
        compose(t, g, parent);
      }
      pose_load12(sc.cam_mount + 12 * cam, mount);
      compose(parent, mount, S.cam);
      if (!kMesh) wait_bulk(&S.mbar);
    }
  } else {
    for (int i = tid - 32; i < sc.nb; i += blockDim.x - 32)
      S.color[i] = make_float4(__fmul_rn(255.0f, sc.color[3 * i]), __fmul_rn(255.0f, sc.color[3 * i + 1]),
                               __fmul_rn(255.0f, sc.color[3 * i + 2]), 0.0f);
    for (int p = tid - 32; p < np; p += blockDim.x - 32) {
      int b = sc.part_body[p];
      Pose bp, lp, wp;
      quat_to_mat(sd + L.quat + 4 * b, bp.R);
      bp.p[0] = sd[L.pos + 3 * b]; bp.p[1] = sd[L.pos + 3 * b + 1]; bp.p[2] = sd[L.pos + 3 * b + 2];
      pose_load12(sc.part_local + 12 * p, lp);
      compose(bp, lp, wp);
      PartW &P = S.part[p];
      P.c[0] = wp.p[0]; P.c[1] = wp.p[1]; P.c[2] = wp.p[2];
      P.kind = sc.part_kind[p];
      P.body = b;
      P.f0 = sc.part_facet_begin[p];
      P.nf = sc.part_facet_begin[p + 1] - P.f0;
      if (kMesh) {
        P.r = sc.mesh_bound[p];
        for (int k = 0; k < 9; ++k) plane[9 * p + k] = wp.R[k];
      } else {
        P.r = P.kind == RS_SPHERE ? sc.part_param[3 * p] : sc.part_bound[p];
      }
      for (int k = 0; k < 9; ++k) S.u.R[p][k] = wp.R[k];
    }
  }
  __syncthreads();
  if (kCount) clk[2] = clk[1] = clock64();
  const double *o = S.cam.p;

  // -- per part the range lower bound from the camera (lanes per part), then
  //    world planes (geometry.py:554-557), b0 = d - n.o (lanes per facet)
  for (int p = tid; p < np; p += blockDim.x) {
    PartW &P = S.part[p];
    const double *R = S.u.R[p];
    double v[3] = {P.c[0] - o[0], P.c[1] - o[1], P.c[2] - o[2]};
    double dist;
    if (P.kind == RS_BOX) {  // distance from the camera to the box (tighter than its sphere; a box
                             // part's triangle soup lies on the box surface, mesh.py part_triangles)
      double l[3], q2 = 0.0;
      mattvec(R, v, l);
      for (int k = 0; k < 3; ++k) {
        const double e = fabs(l[k]) - sc.part_param[3 * p + k];
        q2 += e > 0.0 ? e * e : 0.0;
      }
      dist = sqrt(q2) * (1.0 - 1e-9) - 1e-9;
    } else {
      dist = sqrt(dot3(v, v)) - P.r * (1.0 + 1e-9) - 1e-9;
    }
    P.lb = dist > 0.0 ? dist : 0.0;
    S.trace[p].x = __float_as_uint(__double2float_rd(P.lb));
    S.trace[p].y = (uint32_t)((P.kind << 8) | P.body);
  }
  if (kCount) clk[3] = clock64();
  if (!kMesh) {
    const int nf = sc.nf;
    for (int f = tid; f < nf; f += blockDim.x) {
      int lo = 0, hi = np - 1;  // owning part: last p with f0 <= f
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (S.part[mid].f0 <= f) lo = mid; else hi = mid - 1;
      }
      double *Q = plane + 4 * f;  // holds the staged local facet until overwritten below
      const double F[4] = {Q[0], Q[1], Q[2], Q[3]}, *R = S.u.R[lo], *wpp = S.part[lo].c;
      double n[3];
      matvec(R, F, n);
      double dw = F[3] + dot3(n, wpp);
      Q[0] = n[0]; Q[1] = n[1]; Q[2] = n[2];
      Q[3] = dw - dot3(o, n);
    }
    __syncthreads();
    if (kCount) clk[3] = clock64();
    if (kMode == kProxyMixed)
      for (int p = tid; p < np; p += blockDim.x) {
        const PartW &P = S.part[p];
        if (P.kind != RS_BOX) continue;
        const double *Q = plane + 4 * P.f0;
        for (int k = 0; k < 3; ++k)
          S.box32[p][k] = make_float4((float)Q[4 * k], (float)Q[4 * k + 1], (float)Q[4 * k + 2], (float)Q[4 * k + 3]);
        S.box32[p][3] = make_float4(-(float)Q[15], -(float)Q[19], -(float)Q[23], 0.0f);
      }
  }
  const int W = B.rcfg.width, H = B.rcfg.height;
  const int tx_n = W / kTile, ty_n = H / kTile, ntiles = tx_n * ty_n;
  if (kMesh) __syncthreads();

  // -- warps 0..3: tile culling, lane = part (sphere vs the 4 side planes of
  //    each tile frustum, camera frame; inward normals from B.tile_frustum),
  //    one ballot per (tile, 32 parts) = one mask word.  Warps 4..7: the
  //    front-to-back order of parts (rank by (lb, index)).
  if (warp < kMaskWords) {
    const int p = warp * 32 + lane;
    double c[3] = {0.0, 0.0, 0.0}, r = 0.0, ax[3][3] = {}, h[3] = {0.0, 0.0, 0.0};
    const bool live = p < np;
    bool box = false;
    if (live) {
      const PartW &P = S.part[p];
      double v[3] = {P.c[0] - o[0], P.c[1] - o[1], P.c[2] - o[2]};
      mattvec(S.cam.R, v, c);  // camera frame: x right, y down, z view
      r = P.r * (1.0 + 1e-9) + 1e-9;
      box = P.kind == RS_BOX;
      if (box)  // box axes in the camera frame (world axis k = column k of the part rotation)
        for (int k = 0; k < 3; ++k) {
          const double u[3] = {S.u.R[p][k], S.u.R[p][3 + k], S.u.R[p][6 + k]};
          mattvec(S.cam.R, u, ax[k]);
          h[k] = sc.part_param[3 * p + k] * (1.0 + 1e-9) + 1e-9;
        }
    }
    // support radius of the part along the (unnormalised) plane normal n = (nx, ny, nz), |n| = nn
    auto radius = [&](double nx, double ny, double nz, double nn) {
      if (!box) return r * nn;
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += fabs(nx * ax[k][0] + ny * ax[k][1] + nz * ax[k][2]) * h[k];
      return s * (1.0 + 1e-9) + 1e-9 * nn;
    };
    const bool front = live && c[2] > -radius(0.0, 0.0, 1.0, 1.0);
    int ulo = 0, uhi = 0x7fff, vlo = 0, vhi = 0x7fff;  // pixel rectangle (the tile lists use it too)
    bool rect_only = false;  // the rectangle is the part's exact projected extent (+ 1 pixel): it decides the tiles
    if (kMode == kProxyMixed && live) {
      // conservative pixel rectangle of the part: the pixel u's ray has camera
      // tangent x = (u + 0.5 - W/2) / f, and a ray hits the part only through
      // one of its points (a box: the hull of its 8 corners; else its bounding
      // sphere, whose tangent planes x = k z solve (c_x - k c_z)^2 = r^2 (1 + k^2)),
      // so with every point in front of the camera u lies in [x_lo f + W/2 - 0.5,
      // x_hi f + W/2 - 0.5]; widened by 1 pixel.  A box reaching behind the
      // plane z = zc is clipped to z >= zc (its region: the corners in front and
      // the crossings of its 12 edges with the plane), which loses no visible
      // point when the box is farther than zc sqrt(1 + tan_x^2 + tan_y^2) from
      // the camera (a point inside the image has z >= |p| / that root); closer
      // boxes, and other parts reaching z <= 1e-6, keep the whole image.
      const int W = B.rcfg.width, H = B.rcfg.height;
      const double fpx = (W * 0.5) / tan(B.rcfg.fov * 0.5);
      double xl = INFINITY, xh = -INFINITY, yl = INFINITY, yh = -INFINITY;
      bool ok = true;
      if (box) {
        constexpr double zc = 1e-3;
        auto corner = [&](int s, double *q) {
          for (int i = 0; i < 3; ++i)
            q[i] = c[i] + ((s & 1) ? h[0] : -h[0]) * ax[0][i] + ((s & 2) ? h[1] : -h[1]) * ax[1][i] +
                   ((s & 4) ? h[2] : -h[2]) * ax[2][i];
        };
        auto add = [&](double x, double y, double z) {
          const double iz = 1.0 / z;
          xl = fmin(xl, x * iz); xh = fmax(xh, x * iz);
          yl = fmin(yl, y * iz); yh = fmax(yh, y * iz);
        };
        bool behind = false;
        for (int s = 0; s < 8; ++s) {
          double q[3];
          corner(s, q);
          if (q[2] >= zc) add(q[0], q[1], q[2]);
          else behind = true;
        }
        if (behind) {
          const double lb = S.part[p].lb, t2 = ((double)W * W + (double)H * H) / (4.0 * fpx * fpx);
          ok = lb * lb > 1.1 * zc * zc * (1.0 + t2);
          for (int s = 0; ok && s < 8; ++s)
            for (int k = 0; k < 3; ++k) {
              if (s & (1 << k)) continue;  // edge (s, s + 2^k), each once
              double a[3], b[3];
              corner(s, a);
              corner(s | (1 << k), b);
              if ((a[2] < zc) == (b[2] < zc)) continue;
              const double t = (zc - a[2]) / (b[2] - a[2]);
              add(a[0] + t * (b[0] - a[0]), a[1] + t * (b[1] - a[1]), zc);
            }
        }
      } else {
        const double den = c[2] * c[2] - r * r;
        ok = c[2] - r > 1e-6;
        if (ok) {
          const double sx = r * sqrt(fmax(c[0] * c[0] + den, 0.0)), sy = r * sqrt(fmax(c[1] * c[1] + den, 0.0));
          xl = (c[0] * c[2] - sx) / den; xh = (c[0] * c[2] + sx) / den;
          yl = (c[1] * c[2] - sy) / den; yh = (c[1] * c[2] + sy) / den;
        }
      }
      ulo = 0; uhi = W - 1; vlo = 0; vhi = H - 1;
      if (ok) {
        const double cu = W * 0.5 - 0.5, cv = H * 0.5 - 0.5;
        // clamped to [-1, W] x [-1, H] before the conversion (a clipped box with no
        // point in front leaves the bounds at +-inf: it lands off the image)
        ulo = (int)fmin(fmax(floor(xl * fpx + cu) - 1.0, 0.0), (double)W);
        uhi = (int)fmax(fmin(ceil(xh * fpx + cu) + 1.0, W - 1.0), -1.0);
        vlo = (int)fmin(fmax(floor(yl * fpx + cv) - 1.0, 0.0), (double)H);
        vhi = (int)fmax(fmin(ceil(yh * fpx + cv) + 1.0, H - 1.0), -1.0);
        if (ulo > W - 1 || uhi < 0 || vlo > H - 1 || vhi < 0) { ulo = 1; uhi = 0; }  // off the image: nothing
        rect_only = true;
      }
      S.trace[p].z = (uint32_t)ulo | ((uint32_t)vlo << 16);
      S.trace[p].w = (uint32_t)uhi | ((uint32_t)vhi << 16);
    }
    // B.tile_frustum[tile] = u0, u1, v0, v1, |(1,u0)|, |(1,u1)|, |(1,v0)|, |(1,v1)|; the inward side
    // planes x - u0 z >= 0, -x + u1 z >= 0 depend on the tile column only, y - v0 z >= 0,
    // -y + v1 z >= 0 on the row only: test columns and rows once each (ty_n, tx_n <= 8)
    auto row_in = [&](int ty) {
      const double *T = B.tile_frustum + 8 * (ty * tx_n);
      return c[1] - T[2] * c[2] >= -radius(0.0, 1.0, -T[2], T[6]) && -c[1] + T[3] * c[2] >= -radius(0.0, -1.0, T[3], T[7]);
    };
    auto col_in = [&](int tx) {
      const double *T = B.tile_frustum + 8 * tx;
      return c[0] - T[0] * c[2] >= -radius(1.0, 0.0, -T[0], T[4]) && -c[0] + T[1] * c[2] >= -radius(-1.0, 0.0, T[1], T[5]);
    };
    unsigned rows = 0u, cols = 0u;
    if (front) {
      if (rect_only) {
        // A valid rectangle is the projected extent of the part's points in front
        // of the camera widened by 1 pixel: a tile strictly between its first and
        // last tile lies inside that extent and passes the side-plane tests, so
        // only those two tiles per axis are tested
        if (ulo <= uhi && vlo <= vhi) {
          const int c0 = ulo / kTile, c1 = min(uhi / kTile, tx_n - 1), r0 = vlo / kTile, r1 = min(vhi / kTile, ty_n - 1);
          for (int t = c0; t <= c1; ++t) cols |= 1u << t;
          for (int t = r0; t <= r1; ++t) rows |= 1u << t;
          if (!col_in(c0)) cols &= ~(1u << c0);
          if (c1 != c0 && !col_in(c1)) cols &= ~(1u << c1);
          if (!row_in(r0)) rows &= ~(1u << r0);
          if (r1 != r0 && !row_in(r1)) rows &= ~(1u << r1);
        }
      } else {
        for (int ty = 0; ty < ty_n; ++ty) rows |= (unsigned)(vlo < (ty + 1) * kTile && vhi >= ty * kTile && row_in(ty)) << ty;
        for (int tx = 0; tx < tx_n; ++tx) cols |= (unsigned)(ulo < (tx + 1) * kTile && uhi >= tx * kTile && col_in(tx)) << tx;
      }
    }
    for (int tx = 0; tx < tx_n; ++tx)
      for (int ty = 0; ty < ty_n; ++ty) {
        const unsigned m = __ballot_sync(0xffffffffu, ((cols >> tx) & (rows >> ty) & 1u) != 0u);
        if (lane == 0) S.mask[ty * tx_n + tx][warp] = m;
      }
    if (kCount && lane == 0) atomicAdd(work + 18, (unsigned long long)(clock64() - clk[3]));
  } else {
    for (int p = tid - 32 * kMaskWords; p < np; p += blockDim.x - 32 * kMaskWords) {
      const double lb = S.part[p].lb;
      int rank = 0;
      for (int q = 0; q < np; ++q) {
        double lq = S.part[q].lb;
        rank += (lq < lb) || (lq == lb && q < p);
      }
      S.order[rank] = (uint8_t)p;
    }
    if (kCount && lane == 0) atomicAdd(work + 19, (unsigned long long)(clock64() - clk[3]));
  }
  __syncthreads();
  if (kCount) clk[4] = clock64();
  // -- per tile candidate lists in front-to-back order (warp per tile, ballot compaction)
  for (int tile = warp; tile < ntiles; tile += nwarps) {
    int n = 0;
    for (int i0 = 0; i0 < np; i0 += 32) {
      int i = i0 + lane;
      int p = i < np ? S.order[i] : 0;
      bool in = i < np && ((S.mask[tile][p >> 5] >> (p & 31)) & 1u);
      unsigned m = __ballot_sync(0xffffffffu, in);
      if (in) S.u.list[tile][n + __popc(m & ((1u << lane) - 1))] = (uint8_t)p;
      n += __popc(m);
    }
    if (lane == 0) S.nlist[tile] = n;
  }
  __syncthreads();
  if (kCount) clk[5] = clock64();

  // -- trace
  const double eps = B.rcfg.tie_eps, zfar = B.rcfg.zfar, znear = B.rcfg.znear;
  const size_t img = (size_t)(env * n_cam_out + slot) * H * W;
  Work wk;
  constexpr bool count = kCount;
  if (count)
    for (int i = 0; i < kWorkCounters; ++i) wk.v[i] = 0;
#pragma unroll 1
  for (int tile = warp; tile < ntiles; tile += nwarps) {
    const uint8_t *list = S.u.list[tile];
    const int nl = S.nlist[tile];
    const int ux = (tile % tx_n) * kTile, vy = (tile / tx_n) * kTile;
    if (nl == 0) {  // an empty tile: every pixel misses
      for (int k = lane; k < kTile * kTile; k += 32) {
        const int u = ux + ((k >> 2) & 8) + (lane & 7), v = vy + ((k >> 4) & 12) + (lane >> 3);
        const size_t px = img + (size_t)(v * W + u);
        if (kAll || rgba) __stcs(rgba + px, 0u);
        if (kAll || depth) __stcs(depth + px, 0.0f);
        if (kAll || ids) __stcs(ids + px, -1);
        if (count) wk.v[7] += 1;
      }
      continue;
    }
    __builtin_assume(nl > 0);
#pragma unroll 1
    for (int k = lane; k < kTile * kTile; k += 32) {
      // iteration j = k / 32 covers the 8 x 4 block (j % 2, j / 2) of the tile:
      // lane -> column lane % 8, row lane / 8 (compact blocks walk similar lists)
      const int u = ux + ((k >> 2) & 8) + (lane & 7), v = vy + ((k >> 4) & 12) + (lane >> 3);
      const double *dc = B.ray_dir + 3 * (v * W + u);  // unit camera-frame ray (render_tables_kernel)
      double d[3];
      {  // matvec(S.cam.R, dc, d) with the rotation re-read from shared memory per pixel: hoisted out
         // of the loop it takes 18 registers, and at the 64-register budget ptxas spilled 6 of its
         // doubles to local memory and reloaded them (LDL) for every pixel
        const volatile double *Rv = S.cam.R;
        const double x = dc[0], y = dc[1], z = dc[2];
        d[0] = Rv[0] * x + Rv[1] * y + Rv[2] * z;
        d[1] = Rv[3] * x + Rv[4] * y + Rv[5] * z;
        d[2] = Rv[6] * x + Rv[7] * y + Rv[8] * z;
      }
      double tmin;
      int id, wpart, wface;
      if (kMode != kProxyMixed ||
          !trace_mixed(S, plane, list, nl, (uint32_t)u | ((uint32_t)v << 16), o, d, eps, tmin, id, wpart, wface, wk,
                       count)) {
        if (count && kMode == kProxyMixed) wk.v[3] += 1;
        tmin = trace_exact<kMesh>(sc, S, plane, list, nl, S.mask[tile], o, d, eps, id, wpart, wface, wk, count);
      }
      if (count) wk.v[7] += 1;

      const size_t px = img + (size_t)(v * W + u);
      if (!(tmin <= zfar)) {
        if (kAll || rgba) __stcs(rgba + px, 0u);
        if (kAll || depth) __stcs(depth + px, 0.0f);
        if (kAll || ids) __stcs(ids + px, -1);
        continue;
      }
      // streaming stores (evict-first): the 100 MB of images per step pass through
      // L2 without evicting the physics kernel's scratch running beside the render
      if (kAll || depth) __stcs(depth + px, (float)(tmin < znear ? znear : tmin));
      if (kAll || ids) __stcs(ids + px, id);
      if (kAll || rgba) {
        double cosv = 0.0;
        const PartW &P = S.part[wpart];
        if (kMesh) {
          if (wface >= 0) {  // |n.d| of the hit triangle (two-sided)
            const double *T = sc.mtri + 9 * wface, *R = plane + 9 * wpart;
            double nl[3], nw[3];
            cross3(T + 3, T + 6, nl);
            matvec(R, nl, nw);
            cosv = fabs(dot3(nw, d)) / sqrt(dot3(nw, nw));
          }
        } else if (wface >= 0) {  // box / hull entering face (spheres report no face)
          const double *Q = plane + 4 * wface;
          cosv = -(d[0] * Q[0] + d[1] * Q[1] + d[2] * Q[2]);
        } else if (P.kind == RS_SPHERE) {
          if (tmin > 0.0) {
            double n[3];
            for (int i = 0; i < 3; ++i) n[i] = (o[i] + tmin * d[i] - P.c[i]) / P.r;
            cosv = -dot3(n, d);
          }
        }
        float shade = __fadd_rn(0.3f, __fmul_rn(0.7f, (float)(cosv > 0.0 ? cosv : 0.0)));
        const float4 cw = S.color[id];  // 255 * albedo
        const float col[3] = {cw.x, cw.y, cw.z};
        uint32_t px4 = 0xff000000u;
        for (int i = 0; i < 3; ++i) {
          float cv = __fadd_rn(__fmul_rn(col[i], shade), 0.5f);
          px4 |= (uint32_t)(cv > 255.0f ? 255.0f : cv) << (8 * i);
        }
        __stcs(rgba + px, px4);
      }
    }
  }
#ifdef RSIM_RENDER_TIMELINE
  __syncthreads();
  if (tid == 0 && !count && blockIdx.x < 16384) {
    unsigned long long t_end;
    unsigned smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_timeline[blockIdx.x][0] = t_begin; g_timeline[blockIdx.x][1] = t_end; g_timeline[blockIdx.x][2] = smid;
  }
#endif
  if (count) {
    for (int i = 0; i < 12; ++i) atomicAdd(work + i, wk.v[i]);
    __syncthreads();
    if (tid == 0) {
      clk[6] = clock64();
      for (int i = 0; i < 6; ++i) atomicAdd(work + 12 + i, (unsigned long long)(clk[i + 1] - clk[i]));
    }
  }
}

// Per-batch constant tables: unit camera-frame ray per pixel centre
// (u + 1/2, v + 1/2; f = (W/2)/tan(fov/2); normalise) and the inward side
// planes of every 16x16 tile frustum.  Evaluated exactly as the oracle does
// (oracle/rsim_oracle.c render: f from the host's tan, no contraction,
// dc / l by division), so every ray is the oracle's bit for bit.
__global__ void render_tables_kernel(int W, int H, double f, double *ray_dir, double *tile_frustum) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < W * H) {
    const int u = i % W, v = i / W;
    const double x = (u + 0.5 - W / 2.0) / f, y = (v + 0.5 - H / 2.0) / f;
    const double l = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), 1.0));
    ray_dir[3 * i] = x / l; ray_dir[3 * i + 1] = y / l; ray_dir[3 * i + 2] = 1.0 / l;
  }
  const int tx_n = W / kTile;
  if (i < tx_n * (H / kTile)) {
    double *T = tile_frustum + 8 * i;
    T[0] = ((i % tx_n) * kTile - W / 2.0) / f; T[1] = ((i % tx_n) * kTile + kTile - W / 2.0) / f;
    T[2] = ((i / tx_n) * kTile - H / 2.0) / f; T[3] = ((i / tx_n) * kTile + kTile - H / 2.0) / f;
    for (int k = 0; k < 4; ++k) T[4 + k] = sqrt(1.0 + T[k] * T[k]);
  }
}

cudaError_t launch_render_tables(const DevBatch &B, cudaStream_t stream) {
  const int n = B.rcfg.width * B.rcfg.height;
  const double f = (B.rcfg.width / 2.0) / tan(B.rcfg.fov / 2.0);  // host libm, as the oracle
  render_tables_kernel<<<(n + 255) / 256, 256, 0, stream>>>(B.rcfg.width, B.rcfg.height, f,
                                                            const_cast<double *>(B.ray_dir),
                                                            const_cast<double *>(B.tile_frustum));
  return cudaGetLastError();
}

static size_t render_smem(const DevBatch &B, int mode) {
  const size_t planes = mode == kMeshExact ? 9 * (size_t)kMaxParts : 4 * (size_t)(B.max_nf > 0 ? B.max_nf : kMaxFacets);
  return kPlaneOff + sizeof(double) * planes;
}

template <int kMode, bool kCount, bool kAll>
static cudaError_t launch_render_t(const DevBatch &B, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids,
                                   cudaStream_t stream, unsigned long long *work) {
  int n_cam_out = __builtin_popcount(cam_mask);
  if (n_cam_out == 0) return cudaSuccess;
  // the attribute is per device context: configure each device once
  static std::atomic<unsigned long long> configured{0ull};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (!(configured.load() >> dev & 1ull)) {  // the largest any batch can ask for: kMaxFacets facets
    const size_t cap = kPlaneOff + sizeof(double) * (kMode == kMeshExact ? 9 * kMaxParts : 4 * kMaxFacets);
    e = cudaFuncSetAttribute(render_kernel<kMode, kCount, kAll>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)cap);
    if (e != cudaSuccess) return e;
    configured.fetch_or(1ull << dev);
  }
  dim3 grid(B.n_env * n_cam_out);
  render_kernel<kMode, kCount, kAll><<<grid, kRenderThreads, render_smem(B, kMode), stream>>>(
      B, cam_mask, n_cam_out, reinterpret_cast<uint32_t *>(rgba), depth, ids, work);
  return cudaGetLastError();
}

// work: NULL, or 8 device uint64 counters (struct Work) -- the counting variant
template <int kMode>
static cudaError_t launch_render_any(const DevBatch &B, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids,
                                     cudaStream_t stream, unsigned long long *work) {
  if (work) return launch_render_t<kMode, true, false>(B, cam_mask, rgba, depth, ids, stream, work);
  if (rgba && depth && ids) return launch_render_t<kMode, false, true>(B, cam_mask, rgba, depth, ids, stream, nullptr);
  return launch_render_t<kMode, false, false>(B, cam_mask, rgba, depth, ids, stream, nullptr);
}

cudaError_t launch_render(const DevBatch &B, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids,
                          cudaStream_t stream, unsigned long long *work) {
  return launch_render_any<kProxyMixed>(B, cam_mask, rgba, depth, ids, stream, work);
}

cudaError_t launch_render_exact(const DevBatch &B, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids,
                                cudaStream_t stream, unsigned long long *work) {
  return launch_render_any<kProxyExact>(B, cam_mask, rgba, depth, ids, stream, work);
}

cudaError_t launch_render_mesh(const DevBatch &B, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids,
                               cudaStream_t stream, unsigned long long *work) {
  return launch_render_any<kMeshExact>(B, cam_mask, rgba, depth, ids, stream, work);
}

}  // namespace rsim

#ifdef RSIM_RENDER_TIMELINE
extern "C" int rsim_debug_render_timeline(void *host, int n) {
  return (int)cudaMemcpyFromSymbol(host, rsim::g_timeline, sizeof(unsigned long long) * 3 * (size_t)n);
}
#endif
