// navgrid.cuh -- walk-grid queries shared by the physics step (move_base)
// and the geodesic kernels (nav.cu).  Restates navgrid.py:55-105.  Include
// only from translation units built with -fmad=false: the squared distances
// of the ring search must round like the reference's (ex*ex + ey*ey, no FMA).
#pragma once
#include <cmath>

#include "device.cuh"

namespace rsim {

__device__ __forceinline__ bool nav_ok(const DevScene &sc, long i, long j) {
  return i >= 0 && i < sc.nav_nx && j >= 0 && j < sc.nav_ny && sc.nav[i * sc.nav_ny + j];
}
// navgrid.py:57-63 cell_of / center_of
__device__ __forceinline__ void nav_cell_of(const DevScene &sc, double x, double y, long &i, long &j) {
  i = (long)floor((x - sc.nav_origin[0]) / sc.nav_cell);
  j = (long)floor((y - sc.nav_origin[1]) / sc.nav_cell);
}
__device__ __forceinline__ void nav_centre(const DevScene &sc, long i, long j, double *c) {
  c[0] = sc.nav_origin[0] + ((double)i + 0.5) * sc.nav_cell;
  c[1] = sc.nav_origin[1] + ((double)j + 0.5) * sc.nav_cell;
}
// best (d2, i, j) on the Chebyshev ring r around (ci, cj)
__device__ inline bool nav_ring(const DevScene &sc, long ci, long cj, long r, double x, double y, double &bd, long &bi,
                                long &bj) {
  bool found = false;
  for (long i = ci - r; i <= ci + r; ++i)
    for (long j = cj - r; j <= cj + r; ++j) {
      long di = i > ci ? i - ci : ci - i, dj = j > cj ? j - cj : cj - j;
      if ((di > dj ? di : dj) != r || !nav_ok(sc, i, j)) continue;
      double c[2];
      nav_centre(sc, i, j, c);
      double ex = c[0] - x, ey = c[1] - y, d2 = ex * ex + ey * ey;
      if (!found || d2 < bd || (d2 == bd && (i < bi || (i == bi && j < bj)))) { bd = d2; bi = i; bj = j; found = true; }
    }
  return found;
}
// navgrid.py:70-105 nearest_walkable: xy itself if walkable, else the centre
// of the best cell of the first non-empty ring (or the next ring's best if
// strictly nearer).  Returns false if the grid has no walkable cell.
__device__ inline bool nav_nearest_walkable(const DevScene &sc, double x, double y, double *out) {
  long ci, cj;
  nav_cell_of(sc, x, y, ci, cj);
  out[0] = x; out[1] = y;
  if (nav_ok(sc, ci, cj)) return true;
  long maxr = sc.nav_nx > sc.nav_ny ? sc.nav_nx : sc.nav_ny;
  for (long r = 0; r <= maxr; ++r) {
    double bd, bd2;
    long bi, bj, bi2, bj2;
    if (!nav_ring(sc, ci, cj, r, x, y, bd, bi, bj)) continue;
    if (nav_ring(sc, ci, cj, r + 1, x, y, bd2, bi2, bj2) && bd2 < bd) { bi = bi2; bj = bj2; }
    nav_centre(sc, bi, bj, out);
    return true;
  }
  return false;
}

}  // namespace rsim
