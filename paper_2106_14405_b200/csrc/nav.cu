// nav.cu -- batched geodesics on the walk grid:
// NavGrid.distance_field / geodesic_distance / shortest_path
// (navgrid.py:109-172).
//
// distance_field: one CTA per goal, the whole field (nx*ny float64, 167 KB
// for the 190 x 110 apartment grid) and the walkable bytes in shared memory.
// The reference runs Dijkstra; its result is the unique fixed point of
//     d[goal] = 0,  d[v] = min over walkable 8-neighbours u of fl(d[u] + w_uv)
// (w = cell or cell*sqrt(2); fl = float64 rounding; unique because every
// w > 0 and fl is monotone -- DESIGN.md §4.5).  Any order of monotone
// relaxations that stops at a fixed point therefore reproduces Dijkstra bit
// for bit.  Here: sweeps along +i, -i, +j, -j lines (one thread per cell of
// the line, every cell relaxed from all 8 neighbours), repeated until a
// round changes nothing.
//
// geodesic_distance / shortest_path: one thread per query.
//
// Built with -fmad=false (the nearest-walkable ring search and the
// relaxation sums must round like the reference's float64 arithmetic).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "device.cuh"
#include "navgrid.cuh"

namespace rsim {

constexpr int kNavThreads = 1024;

__global__ void __launch_bounds__(kNavThreads) nav_field_kernel(DevBatch B, const int32_t *scene_of_goal,
                                                                const double *goal_xy, double *fields,
                                                                int32_t *goal_cell, int stride) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int g = blockIdx.x, tid = threadIdx.x;
  const DevScene &sc = B.scenes[scene_of_goal ? scene_of_goal[g] : 0];
  const int nx = sc.nav_nx, ny = sc.nav_ny, n = nx * ny;
  volatile double *d = reinterpret_cast<double *>(smem_raw);
  uint8_t *walk = smem_raw + sizeof(double) * (size_t)n;
  __shared__ int s_goal, s_changed;
  for (int k = tid; k < n; k += blockDim.x) {
    d[k] = INFINITY;
    walk[k] = sc.nav[k];
  }
  if (tid == 0) {
    double p[2];
    long gi = -1, gj = -1;
    if (nav_nearest_walkable(sc, goal_xy[2 * g], goal_xy[2 * g + 1], p)) nav_cell_of(sc, p[0], p[1], gi, gj);
    s_goal = gi >= 0 ? (int)(gi * ny + gj) : -1;
  }
  __syncthreads();
  if (s_goal >= 0) {
    if (tid == 0) d[s_goal] = 0.0;
    const double straight = sc.nav_cell, diag = sc.nav_cell * sqrt(2.0);
    for (;;) {
      if (tid == 0) s_changed = 0;
      __syncthreads();
      int changed = 0;
      for (int dir = 0; dir < 4; ++dir) {
        const bool along_i = dir < 2, fwd = (dir & 1) == 0;
        const int nline = along_i ? nx : ny, width = along_i ? ny : nx;
        for (int s = 0; s < nline; ++s) {
          const int line = fwd ? s : nline - 1 - s;
          for (int w = tid; w < width; w += blockDim.x) {
            const int i = along_i ? line : w, j = along_i ? w : line, k = i * ny + j;
            if (!walk[k] || k == s_goal) continue;
            // neighbours on the adjacent lines only: the line being swept is
            // written concurrently, so its own cells are not read (race-free);
            // they are relaxed by the perpendicular sweeps of the same round,
            // so a round without change is still the 8-neighbour fixed point
            double best = d[k];
            for (int di = -1; di <= 1; ++di) {
              const int ni = i + di;
              if (ni < 0 || ni >= nx || (along_i && !di)) continue;
              for (int dj = -1; dj <= 1; ++dj) {
                const int nj = j + dj;
                if ((!di && !dj) || nj < 0 || nj >= ny || (!along_i && !dj)) continue;
                const double du = d[ni * ny + nj];
                const double nd = du + ((di && dj) ? diag : straight);
                if (nd < best) best = nd;
              }
            }
            if (best < d[k]) { d[k] = best; changed = 1; }
          }
          __syncthreads();
        }
      }
      if (changed) s_changed = 1;
      __syncthreads();
      if (!s_changed) break;
      __syncthreads();
    }
  }
  double *out = fields + (size_t)g * stride;
  for (int k = tid; k < n; k += blockDim.x) out[k] = d[k];
  if (goal_cell && tid == 0) goal_cell[g] = s_goal;
}

// navgrid.py:145-148: field value at the cell of nearest_walkable(from);
// from = NULL -> each env's robot base (query q = env q).
__global__ void nav_geodesic_kernel(DevBatch B, const double *fields, int stride, const int32_t *field_of_query,
                                    const int32_t *scene_of_query, const double *from_xy, int nq, double *out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const DevScene &sc = B.scenes[scene_of_query ? scene_of_query[q] : (from_xy ? 0 : B.env_scene[q])];
  double x, y;
  if (from_xy) {
    x = from_xy[2 * q]; y = from_xy[2 * q + 1];
  } else {
    const double *base = B.sd + (size_t)q * B.L.dbl_size + B.L.base;
    x = base[0]; y = base[1];
  }
  double p[2];
  long i, j;
  if (!nav_nearest_walkable(sc, x, y, p)) { out[q] = INFINITY; return; }
  nav_cell_of(sc, p[0], p[1], i, j);
  out[q] = fields[(size_t)field_of_query[q] * stride + i * sc.nav_ny + j];
}

// navgrid.py:150-172: steepest descent, ties -> (value, i, j); waypoints are
// cell centres; count = 0 when the start is unreachable; truncated at cap.
__global__ void nav_path_kernel(DevBatch B, const double *fields, int stride, const int32_t *field_of_query,
                                const int32_t *scene_of_query, const double *from_xy, int nq, int cap,
                                double *waypoints, int32_t *count) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const DevScene &sc = B.scenes[scene_of_query ? scene_of_query[q] : 0];
  const double *f = fields + (size_t)field_of_query[q] * stride;
  const long nx = sc.nav_nx, ny = sc.nav_ny;
  double *wp = waypoints + (size_t)q * cap * 2;
  double p[2];
  long ci, cj;
  count[q] = 0;
  if (!nav_nearest_walkable(sc, from_xy[2 * q], from_xy[2 * q + 1], p)) return;
  nav_cell_of(sc, p[0], p[1], ci, cj);
  if (!isfinite(f[ci * ny + cj])) return;
  int n = 0;
  if (n < cap) nav_centre(sc, ci, cj, wp + 2 * n);
  ++n;
  for (long guard = nx * ny; f[ci * ny + cj] > 0.0 && guard > 0; --guard) {
    bool found = false;
    double bv = 0.0;
    long bi = 0, bj = 0;
    for (int di = -1; di <= 1; ++di)
      for (int dj = -1; dj <= 1; ++dj) {
        if (!di && !dj) continue;
        const long ni = ci + di, nj = cj + dj;
        if (ni < 0 || ni >= nx || nj < 0 || nj >= ny || !isfinite(f[ni * ny + nj])) continue;
        const double v = f[ni * ny + nj];
        if (!found || v < bv || (v == bv && (ni < bi || (ni == bi && nj < bj)))) { found = true; bv = v; bi = ni; bj = nj; }
      }
    if (!found || bv >= f[ci * ny + cj]) break;
    ci = bi; cj = bj;
    if (n < cap) nav_centre(sc, ci, cj, wp + 2 * n);
    ++n;
  }
  count[q] = n < cap ? n : cap;
}

cudaError_t launch_nav_fields(const DevBatch &B, int nx, int ny, const int32_t *scene_of_goal, const double *goal_xy,
                              int n_goals, double *fields, int32_t *goal_cell, cudaStream_t stream) {
  if (n_goals <= 0) return cudaSuccess;
  const size_t smem = (sizeof(double) + 1) * (size_t)nx * ny;
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(nav_field_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  nav_field_kernel<<<n_goals, kNavThreads, smem, stream>>>(B, scene_of_goal, goal_xy, fields, goal_cell, nx * ny);
  return cudaGetLastError();
}

cudaError_t launch_nav_geodesic(const DevBatch &B, int nx, int ny, const double *fields, const int32_t *field_of_query,
                                const int32_t *scene_of_query, const double *from_xy, int nq, double *out,
                                cudaStream_t stream) {
  if (nq <= 0) return cudaSuccess;
  nav_geodesic_kernel<<<(nq + 127) / 128, 128, 0, stream>>>(B, fields, nx * ny, field_of_query, scene_of_query,
                                                             from_xy, nq, out);
  return cudaGetLastError();
}

cudaError_t launch_nav_path(const DevBatch &B, int nx, int ny, const double *fields, const int32_t *field_of_query,
                            const int32_t *scene_of_query, const double *from_xy, int nq, int cap, double *waypoints,
                            int32_t *count, cudaStream_t stream) {
  if (nq <= 0) return cudaSuccess;
  nav_path_kernel<<<(nq + 127) / 128, 128, 0, stream>>>(B, fields, nx * ny, field_of_query, scene_of_query, from_xy,
                                                         nq, cap, waypoints, count);
  return cudaGetLastError();
}

}  // namespace rsim
