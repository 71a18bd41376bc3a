// query.cu -- batched Simulator.sphere_cast (physics.py:1088-1101), the
// reference's point query: the nearest proxy hit along a unit ray over all
// bodies in id order (t_b = min over the body's parts of the reference ray
// primitive, geometry.py:731-776), kept if t_b <= max_dist and finite, strict
// < so the lowest id wins ties.
//
// One warp per query, lanes over parts: part world frame from the env's
// state slab, world planes on the fly, the slab test of _ray_halfspaces with
// true divisions (no FP32 tricks: queries are few); body minima and the
// lowest-id rule by warp reductions.  Built with -fmad=false: results are the
// C oracle's bit for bit.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "device.cuh"
#include "se3.cuh"

namespace rsim {

// geometry.py:731-746 for one ray; world planes computed per facet
__device__ double q_ray_convex(const DevScene &sc, int p, const Pose &wp, const double *o, const double *d) {
  const int f0 = sc.part_facet_begin[p], nf = sc.part_facet_begin[p + 1] - f0;
  double te = -INFINITY, tx = INFINITY;
  bool bad = false;
  int fe = -1;
  for (int f = 0; f < nf; ++f) {
    const double *F = sc.facet + 4 * (f0 + f);
    double n[3];
    matvec(wp.R, F, n);
    const double dw = F[3] + dot3(n, wp.p);
    const double s = dot3(d, n), bb = dw - dot3(o, n);
    if (s < -1e-12) {
      const double r = bb / s;
      if (fe < 0 || r > te) { te = r; fe = f; }
    } else if (s > 1e-12) {
      const double r = bb / s;
      if (r < tx) tx = r;
    } else if (bb < 0) {
      bad = true;
    }
  }
  if (!(te <= tx && tx >= 0.0 && !bad)) return INFINITY;
  return te >= 0.0 ? te : 0.0;
}

// geometry.py:749-759
__device__ double q_ray_sphere(const double *c, double r, const double *o, const double *d) {
  const double oc[3] = {o[0] - c[0], o[1] - c[1], o[2] - c[2]};
  const double b = dot3(oc, d), cc = dot3(oc, oc) - r * r, disc = b * b - cc;
  if (!(disc >= 0)) return INFINITY;
  const double sq = sqrt(disc), t0 = -b - sq, t1 = -b + sq;
  return t0 >= 0.0 ? t0 : (t1 >= 0.0 ? 0.0 : INFINITY);
}

__global__ void sphere_cast_kernel(DevBatch B, const int32_t *env_of_query, const double *origins,
                                   const double *dirs, const double *max_dist, int nq, int32_t *out_body,
                                   double *out_t) {
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (q >= nq) return;
  const int env = env_of_query ? env_of_query[q] : q;
  const DevScene &sc = B.scenes[B.env_scene[env]];
  const double *sd = B.sd + (size_t)env * B.L.dbl_size;
  const double *o = origins + 3 * q, *d = dirs + 3 * q;
  if (fabs(sqrt(dot3(d, d)) - 1.0) > 1e-6) {  // PhysicsFault("sphere_cast direction must be unit length")
    if (lane == 0) { out_body[q] = -2; out_t[q] = INFINITY; }
    return;
  }
  // per part t (lanes), then per body the minimum: bodies own contiguous part ranges
  __shared__ double pt[4][128];
  double *T = pt[(threadIdx.x >> 5) & 3];
  for (int p = lane; p < sc.np; p += 32) {
    const int b = sc.part_body[p];
    Pose bp, lp, wp;
    quat_to_mat(sd + B.L.quat + 4 * b, bp.R);
    for (int i = 0; i < 3; ++i) bp.p[i] = sd[B.L.pos + 3 * b + i];
    pose_load12(sc.part_local + 12 * p, lp);
    compose(bp, lp, wp);
    T[p] = sc.part_kind[p] == RS_SPHERE ? q_ray_sphere(wp.p, sc.part_param[3 * p], o, d)
                                        : q_ray_convex(sc, p, wp, o, d);
  }
  __syncwarp();
  const double md = max_dist[q];
  double best = INFINITY;
  int bid = 1 << 30;
  for (int b = lane; b < sc.nb; b += 32) {
    double tb = INFINITY;
    for (int p = sc.body_part_begin[b]; p < sc.body_part_begin[b + 1]; ++p) tb = T[p] < tb ? T[p] : tb;
    if (tb <= md && isfinite(tb) && tb < best) { best = tb; bid = b; }  // this lane's bodies ascend
  }
  // lowest id among the bodies at the minimum (a later body needs a strictly smaller t)
  for (int off = 16; off; off >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bid, off);
    if (ob < best || (ob == best && oi < bid)) { best = ob; bid = oi; }
  }
  if (lane == 0) {
    out_body[q] = bid < (1 << 30) ? bid : -1;
    out_t[q] = bid < (1 << 30) ? best : INFINITY;
  }
}

cudaError_t launch_sphere_cast(const DevBatch &B, const int32_t *env_of_query, const double *origins,
                               const double *dirs, const double *max_dist, int nq, int32_t *out_body, double *out_t,
                               cudaStream_t stream) {
  if (nq <= 0) return cudaSuccess;
  sphere_cast_kernel<<<(nq + 3) / 4, 128, 0, stream>>>(B, env_of_query, origins, dirs, max_dist, nq, out_body, out_t);
  return cudaGetLastError();
}

}  // namespace rsim
