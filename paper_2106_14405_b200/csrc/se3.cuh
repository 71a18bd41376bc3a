// se3.cuh -- float64 rigid-transform math for the device step.
//
// Formulas follow the reference geometry kernel term for term
// (geometry.py:23-181): wxyz quaternions, closed-form quat->matrix,
// Shepperd matrix->quat with renormalisation, axis-angle via quaternion,
// Pose.compose = (Ra Rb, Ra pb + pa).  The physics translation unit is
// compiled with -fmad=false so every product/sum rounds like the oracle's
// scalar C (no FMA contraction); only libm transcendentals can differ in
// the last bit.
#pragma once
#include <cmath>

namespace rsim {

struct Pose {
  double R[9];
  double p[3];
};

__device__ __forceinline__ void cross3(const double *a, const double *b, double *o) {
  double x = a[1] * b[2] - a[2] * b[1], y = a[2] * b[0] - a[0] * b[2], z = a[0] * b[1] - a[1] * b[0];
  o[0] = x; o[1] = y; o[2] = z;
}
__device__ __forceinline__ double dot3(const double *a, const double *b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}
__device__ __forceinline__ void matvec(const double *R, const double *v, double *o) {
  double x = R[0] * v[0] + R[1] * v[1] + R[2] * v[2];
  double y = R[3] * v[0] + R[4] * v[1] + R[5] * v[2];
  double z = R[6] * v[0] + R[7] * v[1] + R[8] * v[2];
  o[0] = x; o[1] = y; o[2] = z;
}
__device__ __forceinline__ void mattvec(const double *R, const double *v, double *o) {
  double x = R[0] * v[0] + R[3] * v[1] + R[6] * v[2];
  double y = R[1] * v[0] + R[4] * v[1] + R[7] * v[2];
  double z = R[2] * v[0] + R[5] * v[1] + R[8] * v[2];
  o[0] = x; o[1] = y; o[2] = z;
}
__device__ __forceinline__ void matmul(const double *A, const double *B, double *C) {
  double T[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) T[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
#pragma unroll
  for (int i = 0; i < 9; ++i) C[i] = T[i];
}
__device__ __forceinline__ void quat_to_mat(const double *q, double *R) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}
__device__ __forceinline__ void mat_to_quat(const double *m, double *q) {
  double tr = m[0] + m[4] + m[8], s;
  if (tr > 0) {
    s = sqrt(tr + 1.0) * 2;
    q[0] = 0.25 * s; q[1] = (m[7] - m[5]) / s; q[2] = (m[2] - m[6]) / s; q[3] = (m[3] - m[1]) / s;
  } else if (m[0] > m[4] && m[0] > m[8]) {
    s = sqrt(1.0 + m[0] - m[4] - m[8]) * 2;
    q[0] = (m[7] - m[5]) / s; q[1] = 0.25 * s; q[2] = (m[1] + m[3]) / s; q[3] = (m[2] + m[6]) / s;
  } else if (m[4] > m[8]) {
    s = sqrt(1.0 + m[4] - m[0] - m[8]) * 2;
    q[0] = (m[2] - m[6]) / s; q[1] = (m[1] + m[3]) / s; q[2] = 0.25 * s; q[3] = (m[5] + m[7]) / s;
  } else {
    s = sqrt(1.0 + m[8] - m[0] - m[4]) * 2;
    q[0] = (m[3] - m[1]) / s; q[1] = (m[2] + m[6]) / s; q[2] = (m[5] + m[7]) / s; q[3] = 0.25 * s;
  }
  double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  q[0] /= n; q[1] /= n; q[2] /= n; q[3] /= n;
}
__device__ __forceinline__ void quat_mul(const double *a, const double *b, double *o) {
  double w = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  double x = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  double y = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
  double z = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
  o[0] = w; o[1] = x; o[2] = y; o[3] = z;
}
__device__ __forceinline__ void axis_angle_mat(const double *axis, double ang, double *R) {
  // sincos: one argument reduction for both (the same values as sin / cos);
  // a unit axis has n == 1 exactly, and x / 1 == x, so that division is skipped
  double n = sqrt(dot3(axis, axis)), h = 0.5 * ang, sh, ch;
  sincos(h, &sh, &ch);
  const double s = n == 1.0 ? sh : sh / n;
  double q[4] = {ch, axis[0] * s, axis[1] * s, axis[2] * s};
  quat_to_mat(q, R);
}
__device__ __forceinline__ void compose(const Pose &a, const Pose &b, Pose &o) {
  double p[3];
  matvec(a.R, b.p, p);
  p[0] += a.p[0]; p[1] += a.p[1]; p[2] += a.p[2];
  matmul(a.R, b.R, o.R);
  o.p[0] = p[0]; o.p[1] = p[1]; o.p[2] = p[2];
}
__device__ __forceinline__ void apply(const Pose &a, const double *v, double *o) {
  double t[3];
  matvec(a.R, v, t);
  o[0] = t[0] + a.p[0]; o[1] = t[1] + a.p[1]; o[2] = t[2] + a.p[2];
}
__device__ __forceinline__ void pose_load12(const double *v, Pose &o) {
#pragma unroll
  for (int i = 0; i < 9; ++i) o.R[i] = v[i];
  o.p[0] = v[9]; o.p[1] = v[10]; o.p[2] = v[11];
}
__device__ __forceinline__ void rot_z(double a, double *R) {
  double c, s;
  sincos(a, &s, &c);
  R[0] = c; R[1] = -s; R[2] = 0.0; R[3] = s; R[4] = c; R[5] = 0.0; R[6] = 0.0; R[7] = 0.0; R[8] = 1.0;
}
// robot.py:156-158
__device__ __forceinline__ void base3(const double *base, Pose &o) {
  rot_z(base[2], o.R);
  o.p[0] = base[0]; o.p[1] = base[1]; o.p[2] = 0.0;
}
// physics.py:1339-1347
__device__ __forceinline__ void quat_delta_omega(const double *qo, const double *qn, double dt, double *om) {
  double c[4] = {qo[0], -qo[1], -qo[2], -qo[3]}, dq[4];
  quat_mul(qn, c, dq);
  if (dq[0] < 0) { dq[0] = -dq[0]; dq[1] = -dq[1]; dq[2] = -dq[2]; dq[3] = -dq[3]; }
  double x = dq[0] < -1.0 ? -1.0 : (dq[0] > 1.0 ? 1.0 : dq[0]);
  double ang = 2.0 * acos(x);
  if (ang < 1e-12) { om[0] = om[1] = om[2] = 0.0; return; }
  double sh = sin(ang / 2.0);
  for (int i = 0; i < 3; ++i) om[i] = (dq[1 + i] / sh) * (ang / dt);
}
// Python float modulo (sign of the divisor), robot.py:371-372
__device__ __forceinline__ double py_mod(double a, double b) {
  double m = fmod(a, b);
  if (m != 0.0) {
    if ((b < 0) != (m < 0)) m += b;
  } else {
    m = copysign(0.0, b);
  }
  return m;
}

}  // namespace rsim
