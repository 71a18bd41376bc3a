// settle.cu -- batched Simulator.settle (physics.py:1113-1176)
// for fast resets: spawn-clearance check by GJK (geometry.py:383-539) and
// per-env settle bookkeeping around the fused step kernel.
//
//   settle_clearance_kernel  one warp per env, one lane per placed body
//                            (ascending id): AABB prefilter (1 mm margin),
//                            then parts_distance = min GJK distance over part
//                            pairs; the env reports the first (body, other)
//                            with clearance < 1 mm, like the reference raise.
//   settle_check_kernel      one thread per env after every control step:
//                            a placed body below floor_z - 0.5 -> fell; all
//                            placed bodies asleep -> settled (step count).
//
// rs_settle (abi.cu) runs clearance, then steps only the still-settling envs
// (DevBatch.env_active) until every env is done or max_steps.  Built with
// -fmad=false: GJK and the AABBs round exactly like the C oracle.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "device.cuh"
#include "se3.cuh"

namespace rsim {

enum { kSettled = 0, kClearance = 1, kFell = 2, kTimeout = 3, kFault = 4 };

struct SlabView {
  const DevScene *sc;
  const double *sd;
  const StateLayout *L;
};

__device__ __forceinline__ void sv_body_pose(const SlabView &v, int b, Pose &o) {
  quat_to_mat(v.sd + v.L->quat + 4 * b, o.R);
  for (int i = 0; i < 3; ++i) o.p[i] = v.sd[v.L->pos + 3 * b + i];
}
__device__ __forceinline__ void sv_part_world(const SlabView &v, const Pose &bp, int p, Pose &o) {
  Pose l;
  pose_load12(v.sc->part_local + 12 * p, l);
  compose(bp, l, o);
}
// geometry.py:278-296
__device__ void sv_body_aabb(const SlabView &v, int b, double *lo, double *hi) {
  const DevScene &sc = *v.sc;
  Pose bp, wp;
  sv_body_pose(v, b, bp);
  for (int i = 0; i < 3; ++i) { lo[i] = INFINITY; hi[i] = -INFINITY; }
  for (int p = sc.body_part_begin[b]; p < sc.body_part_begin[b + 1]; ++p) {
    sv_part_world(v, bp, p, wp);
    double l[3], h[3];
    const int k = sc.part_kind[p];
    if (k == RS_BOX) {
      const double *hh = sc.part_param + 3 * p;
      for (int i = 0; i < 3; ++i) {
        double r = fabs(wp.R[3 * i]) * hh[0] + fabs(wp.R[3 * i + 1]) * hh[1] + fabs(wp.R[3 * i + 2]) * hh[2];
        l[i] = wp.p[i] - r; h[i] = wp.p[i] + r;
      }
    } else if (k == RS_SPHERE) {
      double r = sc.part_param[3 * p];
      for (int i = 0; i < 3; ++i) { l[i] = wp.p[i] - r; h[i] = wp.p[i] + r; }
    } else {
      for (int i = 0; i < 3; ++i) { l[i] = INFINITY; h[i] = -INFINITY; }
      for (int q = sc.part_vert_begin[p]; q < sc.part_vert_begin[p + 1]; ++q) {
        double x[3];
        apply(wp, sc.vert + 3 * q, x);
        for (int i = 0; i < 3; ++i) { l[i] = fmin(l[i], x[i]); h[i] = fmax(h[i], x[i]); }
      }
    }
    for (int i = 0; i < 3; ++i) { lo[i] = fmin(lo[i], l[i]); hi[i] = fmax(hi[i], h[i]); }
  }
}

// geometry.py:262-275 support_local / support_world (argmax: first maximum)
__device__ void support_world(const DevScene &sc, int p, const Pose &wp, const double *d, double *out) {
  double dl[3], s[3];
  mattvec(wp.R, d, dl);
  const int k = sc.part_kind[p];
  if (k == RS_BOX) {
    const double *h = sc.part_param + 3 * p;
    for (int i = 0; i < 3; ++i) s[i] = dl[i] >= 0 ? h[i] : -h[i];
  } else if (k == RS_SPHERE) {
    const double r = sc.part_param[3 * p], n = sqrt(dot3(dl, dl));
    if (n == 0.0) { s[0] = r; s[1] = 0.0; s[2] = 0.0; }
    else for (int i = 0; i < 3; ++i) s[i] = (r / n) * dl[i];
  } else {
    int best = sc.part_vert_begin[p];
    double bv = -INFINITY;
    for (int q = sc.part_vert_begin[p]; q < sc.part_vert_begin[p + 1]; ++q) {
      const double x = dot3(sc.vert + 3 * q, dl);
      if (x > bv) { bv = x; best = q; }
    }
    for (int i = 0; i < 3; ++i) s[i] = sc.vert[3 * best + i];
  }
  matvec(wp.R, s, out);
  for (int i = 0; i < 3; ++i) out[i] += wp.p[i];
}

// geometry.py:431-467 _closest_triangle over W[idx[0..2]]
__device__ void closest_triangle(double (*W)[3], const int *idx, double *pt, int *sub, int &nsub) {
  const double *w1 = W[idx[0]], *w2 = W[idx[1]], *w3 = W[idx[2]];
  double ab[3], ac[3], ap[3], bp[3], cp[3];
  for (int i = 0; i < 3; ++i) { ab[i] = w2[i] - w1[i]; ac[i] = w3[i] - w1[i]; ap[i] = -w1[i]; }
  const double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
  if (d1 <= 0 && d2 <= 0) { for (int i = 0; i < 3; ++i) pt[i] = w1[i]; sub[0] = idx[0]; nsub = 1; return; }
  for (int i = 0; i < 3; ++i) bp[i] = -w2[i];
  const double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
  if (d3 >= 0 && d4 <= d3) { for (int i = 0; i < 3; ++i) pt[i] = w2[i]; sub[0] = idx[1]; nsub = 1; return; }
  const double vc = d1 * d4 - d3 * d2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) {
    const double t = d1 != d3 ? d1 / (d1 - d3) : 0.0;
    for (int i = 0; i < 3; ++i) pt[i] = w1[i] + t * ab[i];
    sub[0] = idx[0]; sub[1] = idx[1]; nsub = 2; return;
  }
  for (int i = 0; i < 3; ++i) cp[i] = -w3[i];
  const double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
  if (d6 >= 0 && d5 <= d6) { for (int i = 0; i < 3; ++i) pt[i] = w3[i]; sub[0] = idx[2]; nsub = 1; return; }
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) {
    const double t = d2 != d6 ? d2 / (d2 - d6) : 0.0;
    for (int i = 0; i < 3; ++i) pt[i] = w1[i] + t * ac[i];
    sub[0] = idx[0]; sub[1] = idx[2]; nsub = 2; return;
  }
  const double va = d3 * d6 - d5 * d4;
  if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0) {
    const double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    for (int i = 0; i < 3; ++i) pt[i] = w2[i] + t * (w3[i] - w2[i]);
    sub[0] = idx[1]; sub[1] = idx[2]; nsub = 2; return;
  }
  const double denom = va + vb + vc, v = vb / denom, w = vc / denom;
  for (int i = 0; i < 3; ++i) pt[i] = w1[i] + ab[i] * v + ac[i] * w;
  sub[0] = idx[0]; sub[1] = idx[1]; sub[2] = idx[2]; nsub = 3;
}

// geometry.py:383-428 _closest_simplex; W[0..n) reduced in place; true when
// a tetrahedron contains the origin
__device__ bool closest_simplex(double (*W)[3], int &n, double *pt) {
  int sub[4], ns = 0;
  if (n == 1) { for (int i = 0; i < 3; ++i) pt[i] = W[0][i]; return false; }
  if (n == 2) {
    double d[3];
    for (int i = 0; i < 3; ++i) d[i] = W[1][i] - W[0][i];
    const double dd = dot3(d, d), t = dd == 0.0 ? 0.0 : -dot3(W[0], d) / dd;
    if (t <= 0.0) { for (int i = 0; i < 3; ++i) pt[i] = W[0][i]; n = 1; return false; }
    if (t >= 1.0) { for (int i = 0; i < 3; ++i) { pt[i] = W[1][i]; W[0][i] = W[1][i]; } n = 1; return false; }
    for (int i = 0; i < 3; ++i) pt[i] = W[0][i] + t * d[i];
    return false;
  }
  if (n == 3) {
    const int idx[3] = {0, 1, 2};
    closest_triangle(W, idx, pt, sub, ns);
  } else {
    const int faces[4][4] = {{0, 1, 2, 3}, {0, 1, 3, 2}, {0, 2, 3, 1}, {1, 2, 3, 0}};
    bool contained = true, have = false;
    double bd2 = 0.0;
    for (int f = 0; f < 4; ++f) {
      const double *a = W[faces[f][0]], *b = W[faces[f][1]], *c = W[faces[f][2]], *o = W[faces[f][3]];
      double ba[3], ca[3], nrm[3], ma[3], oa[3];
      for (int i = 0; i < 3; ++i) { ba[i] = b[i] - a[i]; ca[i] = c[i] - a[i]; ma[i] = -a[i]; oa[i] = o[i] - a[i]; }
      cross3(ba, ca, nrm);
      if (dot3(nrm, ma) * dot3(nrm, oa) > 0) continue;
      contained = false;
      double p2[3];
      int s2[4], n2 = 0;
      closest_triangle(W, faces[f], p2, s2, n2);
      const double d2 = dot3(p2, p2);
      if (!have || d2 < bd2) {
        have = true; bd2 = d2;
        for (int i = 0; i < 3; ++i) pt[i] = p2[i];
        for (int i = 0; i < n2; ++i) sub[i] = s2[i];
        ns = n2;
      }
    }
    if (contained) { pt[0] = pt[1] = pt[2] = 0.0; return true; }
  }
  double T[4][3];
  for (int k = 0; k < ns; ++k)
    for (int i = 0; i < 3; ++i) T[k][i] = W[sub[k]][i];
  for (int k = 0; k < ns; ++k)
    for (int i = 0; i < 3; ++i) W[k][i] = T[k][i];
  n = ns;
  return false;
}

// geometry.py:486-525 gjk_distance (tol 1e-10, 64 iterations), distance only
__device__ double gjk_distance(const DevScene &sc, int pa, const Pose &wa, int pb, const Pose &wb) {
  const double tol = 1e-10;
  double d[3], nd[3], sa[3], sb[3], W[4][3], pt[3];
  for (int i = 0; i < 3; ++i) d[i] = wb.p[i] - wa.p[i];
  if (dot3(d, d) == 0.0) { d[0] = 1.0; d[1] = 0.0; d[2] = 0.0; }
  for (int i = 0; i < 3; ++i) nd[i] = -d[i];
  support_world(sc, pa, wa, d, sa);
  support_world(sc, pb, wb, nd, sb);
  int n = 1;
  for (int i = 0; i < 3; ++i) { W[0][i] = sa[i] - sb[i]; pt[i] = W[0][i]; }
  double last_d2 = INFINITY;
  for (int it = 0; it < 64; ++it) {
    const bool contains = closest_simplex(W, n, pt);
    const double d2 = dot3(pt, pt);
    if (contains || d2 < tol) return 0.0;
    if (isfinite(last_d2) && last_d2 - d2 <= tol * fmax(1.0, last_d2)) break;
    last_d2 = d2;
    for (int i = 0; i < 3; ++i) { d[i] = -pt[i]; nd[i] = pt[i]; }
    support_world(sc, pa, wa, d, sa);
    support_world(sc, pb, wb, nd, sb);
    double wv[3];
    for (int i = 0; i < 3; ++i) wv[i] = sa[i] - sb[i];
    if (dot3(wv, d) - dot3(pt, d) <= tol * fmax(1.0, sqrt(d2))) break;
    for (int i = 0; i < 3; ++i) W[n][i] = wv[i];
    ++n;
  }
  return sqrt(dot3(pt, pt));
}

// geometry.py:528-539 parts_distance
__device__ double parts_distance(const SlabView &v, int a, int b) {
  const DevScene &sc = *v.sc;
  Pose pa, pb, wa, wb;
  sv_body_pose(v, a, pa);
  sv_body_pose(v, b, pb);
  double best = INFINITY;
  for (int i = sc.body_part_begin[a]; i < sc.body_part_begin[a + 1]; ++i) {
    sv_part_world(v, pa, i, wa);
    for (int j = sc.body_part_begin[b]; j < sc.body_part_begin[b + 1]; ++j) {
      sv_part_world(v, pb, j, wb);
      const double d = gjk_distance(sc, i, wa, j, wb);
      if (d < best) best = d;
      if (best == 0.0) return 0.0;
    }
  }
  return best;
}

// physics.py:1156-1176 _assert_spawn_clearance; warp per env
__global__ void settle_clearance_kernel(DevBatch B, const uint64_t *placed, uint8_t *active, int32_t *status,
                                        int32_t *info, double *value, int32_t *steps) {
  const int env = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (env >= B.n_env || !active[env]) return;
  const SlabView v{&B.scenes[B.env_scene[env]], B.sd + (size_t)env * B.L.dbl_size, &B.L};
  const DevScene &sc = *v.sc;
  const uint64_t mask = placed[env];
  const double margin = 1e-3;
  int fb = 1 << 30, fo = -1;
  double fd = 0.0;
  for (int k = lane; k < sc.nb; k += 32) {
    if (!((mask >> k) & 1ull)) continue;
    double la[3], ha[3];
    sv_body_aabb(v, k, la, ha);
    for (int o = 0; o < sc.nb; ++o) {
      if (o == k || sc.body_robot[o]) continue;
      if (v.sd[v.L->pos + 3 * o + 2] > 40.0 / 2) continue;  // parked (Simulator.PARK_Z / 2)
      double lb[3], hb[3];
      sv_body_aabb(v, o, lb, hb);
      bool ov = true;
      for (int i = 0; i < 3; ++i) ov = ov && la[i] - margin <= hb[i] && lb[i] - margin <= ha[i];
      if (!ov) continue;
      const double d = parts_distance(v, k, o);
      if (d < margin) { fb = k; fo = o; fd = d; break; }
    }
    if (fo >= 0) break;  // lanes take bodies in ascending order: this lane's first hit is its lowest
  }
  const int first = __reduce_min_sync(0xffffffffu, fb);
  if (first < (1 << 30) && fb == first) {
    status[env] = kClearance;
    info[2 * env] = fb; info[2 * env + 1] = fo;
    value[env] = fd;
    steps[env] = 0;
    active[env] = 0;
  }
}

// physics.py:1138-1154 per-step bookkeeping; thread per env
__global__ void settle_check_kernel(DevBatch B, const uint64_t *placed, uint8_t *active, int32_t *status,
                                    int32_t *info, double *value, int32_t *steps, double floor_limit, int step_no,
                                    int max_steps, int32_t *n_active) {
  const int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env >= B.n_env || !active[env]) return;
  const double *sd = B.sd + (size_t)env * B.L.dbl_size;
  const int32_t *si = B.si + (size_t)env * B.L.int_size;
  const uint64_t mask = placed[env];
  steps[env] = step_no;
  if (B.fault[env]) {
    status[env] = kFault; info[2 * env] = (int32_t)B.fault[env]; active[env] = 0;
    return;
  }
  int fell = -1;
  bool awake = false;
  for (int b = 0; b < B.nb; ++b) {
    if (!((mask >> b) & 1ull)) continue;
    if (fell < 0 && sd[B.L.pos + 3 * b + 2] < floor_limit) fell = b;
    awake = awake || !si[B.L.asleep + b];
  }
  if (fell >= 0) {
    status[env] = kFell; info[2 * env] = fell; active[env] = 0;
  } else if (!awake) {
    status[env] = kSettled; active[env] = 0;
  } else if (step_no >= max_steps) {
    status[env] = kTimeout; active[env] = 0;
  } else {
    atomicAdd(n_active, 1);
  }
}

__global__ void settle_init_kernel(int n, const uint8_t *active, int32_t *status, int32_t *info, double *value,
                                   int32_t *steps) {
  const int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env >= n || !active[env]) return;
  status[env] = kTimeout; info[2 * env] = info[2 * env + 1] = -1; value[env] = 0.0; steps[env] = 0;
}

cudaError_t launch_settle_clearance(const DevBatch &B, const uint64_t *placed, uint8_t *active, int32_t *status,
                                    int32_t *info, double *value, int32_t *steps, cudaStream_t stream) {
  settle_init_kernel<<<(B.n_env + 255) / 256, 256, 0, stream>>>(B.n_env, active, status, info, value, steps);
  settle_clearance_kernel<<<(B.n_env + 3) / 4, 128, 0, stream>>>(B, placed, active, status, info, value, steps);
  return cudaGetLastError();
}

cudaError_t launch_settle_check(const DevBatch &B, const uint64_t *placed, uint8_t *active, int32_t *status,
                                int32_t *info, double *value, int32_t *steps, double floor_limit, int step_no,
                                int max_steps, int32_t *n_active, cudaStream_t stream) {
  settle_check_kernel<<<(B.n_env + 127) / 128, 128, 0, stream>>>(B, placed, active, status, info, value, steps,
                                                                  floor_limit, step_no, max_steps, n_active);
  return cudaGetLastError();
}

}  // namespace rsim
