/*
 * rsim_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product (paper_2106_14405_b200)
 * never calls it.
 *
 * It restates, in plain scalar C99 float64 (compiled with
 * -ffp-contract=off, no FMA), the reference's `Simulator.step_physics`
 * (pkg/src/rearrange_sim/physics.py:575-1035, geometry.py, robot.py,
 * navgrid.py) and the pinned render restatement over the reference's ray
 * primitive (geometry.py:734-776, tie rule physics.py:1096-1100,
 * SPEC.md:243-289).  Each function cites the reference lines it follows.
 *
 * Pinning: tests/test_oracle.py checks it against the golden fixtures
 * generated from the reference itself (tests/golden/make_goldens.py):
 * discrete outputs (pair lists, contact counts, sleep flags, counters,
 * ids) bit-exact, continuous values to float tolerance.  Bit-exactness of
 * continuous values is impossible by construction: the reference's small
 * matrix products go through OpenBLAS FMA kernels.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/rsim.h"

#define MAXB 64
#define MAXJ 16
#define MAXROWS 4096
#define MAXPAIRS 2048

/* ------------------------------------------------------------------ world */

typedef struct {
  int nb, np, nf, nv, nt, nsj, narm, robot_base;
  int *body_kind, *body_robot, *body_group, *body_joint, *body_part_begin;
  double *inv_mass, *com, *inv_inertia, *friction, *restitution;
  float *color;
  int *part_body, *part_kind, *part_facet_begin, *part_vert_begin, *part_tri_begin;
  double *part_local, *part_param, *facet, *vert;
  int *tri;
  int *joint_type, *joint_body, *joint_parent;
  double *joint_axis, *joint_origin, *joint_limits, *joint_handle;
  double *arm_offset, *arm_axis, *arm_limits, gripper[3];
  int ncam, *cam_parent;
  double *cam_mount;
  int nav_nx, nav_ny;
  double nav_origin[2], nav_cell;
  uint8_t *nav;
  rs_physics_config cfg;
  int clutter[MAXB], nclutter;
} orc_world;

static void *dup(const void *src, size_t n) {
  if (n > ((size_t)1 << 32)) return NULL; /* a negative count converted to size_t: reject */
  void *p = malloc(n ? n : 1);
  if (n && p) memcpy(p, src, n);
  return p;
}

orc_world *orc_create(const rs_scene_desc *d, const rs_physics_config *cfg) {
  if (d->n_bodies > MAXB || d->n_scene_joints + d->n_arm > MAXJ) return NULL;
  orc_world *w = (orc_world *)calloc(1, sizeof(orc_world));
  w->nb = d->n_bodies; w->np = d->n_parts; w->nf = d->n_facets; w->nv = d->n_verts; w->nt = d->n_tris;
  w->nsj = d->n_scene_joints; w->narm = d->n_arm; w->robot_base = d->robot_base;
  int nb = w->nb, np = w->np;
  w->body_kind = dup(d->body_kind, 4 * nb); w->body_robot = dup(d->body_robot, 4 * nb);
  w->body_group = dup(d->body_group, 4 * nb); w->body_joint = dup(d->body_joint, 4 * nb);
  w->body_part_begin = dup(d->body_part_begin, 4 * (nb + 1));
  w->inv_mass = dup(d->body_inv_mass, 8 * nb); w->com = dup(d->body_com, 24 * nb);
  w->inv_inertia = dup(d->body_inv_inertia, 72 * nb); w->friction = dup(d->body_friction, 8 * nb);
  w->restitution = dup(d->body_restitution, 8 * nb); w->color = dup(d->body_color, 12 * nb);
  w->part_body = dup(d->part_body, 4 * np); w->part_kind = dup(d->part_kind, 4 * np);
  w->part_facet_begin = dup(d->part_facet_begin, 4 * (np + 1));
  w->part_vert_begin = dup(d->part_vert_begin, 4 * (np + 1));
  w->part_tri_begin = dup(d->part_tri_begin, 4 * (np + 1));
  w->part_local = dup(d->part_local, 96 * np); w->part_param = dup(d->part_param, 24 * np);
  w->facet = dup(d->facet, 32 * w->nf); w->vert = dup(d->vert, 24 * w->nv); w->tri = dup(d->tri, 12 * w->nt);
  int nj = w->nsj;
  w->joint_type = dup(d->joint_type, 4 * nj); w->joint_body = dup(d->joint_body, 4 * nj);
  w->joint_parent = dup(d->joint_parent, 4 * nj); w->joint_axis = dup(d->joint_axis, 24 * nj);
  w->joint_origin = dup(d->joint_origin, 96 * nj); w->joint_limits = dup(d->joint_limits, 16 * nj);
  w->joint_handle = dup(d->joint_handle, 24 * nj);
  w->arm_offset = dup(d->arm_offset, 24 * w->narm); w->arm_axis = dup(d->arm_axis, 24 * w->narm);
  w->arm_limits = dup(d->arm_limits, 16 * w->narm);
  memcpy(w->gripper, d->gripper_offset, sizeof w->gripper);
  w->ncam = d->n_cameras; w->cam_parent = dup(d->cam_parent, 4 * w->ncam);
  w->cam_mount = dup(d->cam_mount, 96 * w->ncam);
  w->nav_nx = d->nav_nx; w->nav_ny = d->nav_ny;
  w->nav_origin[0] = d->nav_origin[0]; w->nav_origin[1] = d->nav_origin[1]; w->nav_cell = d->nav_cell;
  w->nav = dup(d->nav_walkable, (size_t)w->nav_nx * w->nav_ny);
  w->cfg = *cfg;
  w->nclutter = 0;
  /* clutter = dynamic bodies after the robot (physics.py:306-310) */
  for (int b = 0; b < nb; ++b)
    if (w->body_kind[b] == RS_DYNAMIC && b > w->robot_base) w->clutter[w->nclutter++] = b;
  return w;
}

void orc_destroy(orc_world *w) {
  if (!w) return;
  void *ptrs[] = {w->body_kind, w->body_robot, w->body_group, w->body_joint, w->body_part_begin, w->inv_mass,
                  w->com, w->inv_inertia, w->friction, w->restitution, w->color, w->part_body, w->part_kind,
                  w->part_facet_begin, w->part_vert_begin, w->part_tri_begin, w->part_local, w->part_param,
                  w->facet, w->vert, w->tri, w->joint_type, w->joint_body, w->joint_parent, w->joint_axis,
                  w->joint_origin, w->joint_limits, w->joint_handle, w->arm_offset, w->arm_axis, w->arm_limits,
                  w->cam_parent, w->cam_mount, w->nav};
  for (size_t i = 0; i < sizeof ptrs / sizeof ptrs[0]; ++i) free(ptrs[i]);
  free(w);
}

/* ------------------------------------------------------------------ state */

typedef struct {
  int nb, nj;
  double pos[MAXB][3], quat[MAXB][4], lv[MAXB][3], av[MAXB][3];
  uint8_t asleep[MAXB];
  int64_t sleep_counter[MAXB];
  double joints[MAXJ], jvel[MAXJ], base[3], held_offset[7], grab_ee[3];
  int64_t rider_joint[MAXB];
  double rider_offset[MAXB][7];
  int32_t held, held_joint;
  double grab_q, acc_force, time;
  int64_t step_index;
} ostate;

int64_t orc_snapshot_size(int nb, int nj) {
  return 16 + 8 * 13 * (int64_t)nb + nb + 8 * nb + 16 * nj + 8 * 13 + 8 * nb + 56 * nb + 40;
}

static int unpack(const uint8_t *s, ostate *st, int nb_expect, int nj_expect) {
  if (memcmp(s, "RSIM", 4) != 0) return RS_ERR_SNAPSHOT;
  uint32_t ver, nb, nj;
  memcpy(&ver, s + 4, 4); memcpy(&nb, s + 8, 4); memcpy(&nj, s + 12, 4);
  if (ver != 1 || (int)nb != nb_expect || (int)nj != nj_expect) return RS_ERR_SNAPSHOT;
  st->nb = nb; st->nj = nj;
  const uint8_t *p = s + 16;
#define TAKE(dst, n) do { memcpy((dst), p, (n)); p += (n); } while (0)
  for (uint32_t b = 0; b < nb; ++b) TAKE(st->pos[b], 24);
  for (uint32_t b = 0; b < nb; ++b) TAKE(st->quat[b], 32);
  for (uint32_t b = 0; b < nb; ++b) TAKE(st->lv[b], 24);
  for (uint32_t b = 0; b < nb; ++b) TAKE(st->av[b], 24);
  TAKE(st->asleep, nb);
  TAKE(st->sleep_counter, 8 * nb);
  TAKE(st->joints, 8 * nj); TAKE(st->jvel, 8 * nj);
  TAKE(st->base, 24); TAKE(st->held_offset, 56); TAKE(st->grab_ee, 24);
  TAKE(st->rider_joint, 8 * nb);
  for (uint32_t b = 0; b < nb; ++b) TAKE(st->rider_offset[b], 56);
  TAKE(&st->held, 4); TAKE(&st->held_joint, 4); TAKE(&st->grab_q, 8); TAKE(&st->acc_force, 8);
  TAKE(&st->time, 8); TAKE(&st->step_index, 8);
#undef TAKE
  return 0;
}

static void pack(const ostate *st, uint8_t *s) {
  int nb = st->nb, nj = st->nj;
  memcpy(s, "RSIM", 4);
  uint32_t hdr[3] = {1u, (uint32_t)nb, (uint32_t)nj};
  memcpy(s + 4, hdr, 12);
  uint8_t *p = s + 16;
#define PUT(src, n) do { memcpy(p, (src), (n)); p += (n); } while (0)
  for (int b = 0; b < nb; ++b) PUT(st->pos[b], 24);
  for (int b = 0; b < nb; ++b) PUT(st->quat[b], 32);
  for (int b = 0; b < nb; ++b) PUT(st->lv[b], 24);
  for (int b = 0; b < nb; ++b) PUT(st->av[b], 24);
  PUT(st->asleep, nb);
  PUT(st->sleep_counter, 8 * nb);
  PUT(st->joints, 8 * nj); PUT(st->jvel, 8 * nj);
  PUT(st->base, 24); PUT(st->held_offset, 56); PUT(st->grab_ee, 24);
  PUT(st->rider_joint, 8 * nb);
  for (int b = 0; b < nb; ++b) PUT(st->rider_offset[b], 56);
  PUT(&st->held, 4); PUT(&st->held_joint, 4); PUT(&st->grab_q, 8); PUT(&st->acc_force, 8);
  PUT(&st->time, 8); PUT(&st->step_index, 8);
#undef PUT
}

/* ------------------------------------------------------- SE(3) (geometry.py:23-181) */

typedef struct { double R[9], p[3]; } pose_t;

static void cross(const double *a, const double *b, double *o) {
  double x = a[1] * b[2] - a[2] * b[1], y = a[2] * b[0] - a[0] * b[2], z = a[0] * b[1] - a[1] * b[0];
  o[0] = x; o[1] = y; o[2] = z;
}
static double dot3(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static void matvec(const double *R, const double *v, double *o) {
  double x = R[0] * v[0] + R[1] * v[1] + R[2] * v[2];
  double y = R[3] * v[0] + R[4] * v[1] + R[5] * v[2];
  double z = R[6] * v[0] + R[7] * v[1] + R[8] * v[2];
  o[0] = x; o[1] = y; o[2] = z;
}
static void mattvec(const double *R, const double *v, double *o) {
  double x = R[0] * v[0] + R[3] * v[1] + R[6] * v[2];
  double y = R[1] * v[0] + R[4] * v[1] + R[7] * v[2];
  double z = R[2] * v[0] + R[5] * v[1] + R[8] * v[2];
  o[0] = x; o[1] = y; o[2] = z;
}
static void matmul(const double *A, const double *B, double *C) {
  double T[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) T[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
  memcpy(C, T, sizeof T);
}
/* geometry.py:72-80 */
static void quat_to_mat(const double *q, double *R) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}
/* geometry.py:83-107 Shepperd + renormalise */
static void mat_to_quat(const double *m, double *q) {
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
  for (int i = 0; i < 4; ++i) q[i] /= n;
}
static void quat_mul(const double *a, const double *b, double *o) {
  double w = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  double x = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  double y = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
  double z = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
  o[0] = w; o[1] = x; o[2] = y; o[3] = z;
}
/* geometry.py:62-69, :132-133 */
static void axis_angle_mat(const double *axis, double ang, double *R) {
  double n = sqrt(dot3(axis, axis)), h = 0.5 * ang, s = sin(h) / n;
  double q[4] = {cos(h), axis[0] * s, axis[1] * s, axis[2] * s};
  quat_to_mat(q, R);
}
static void compose(const pose_t *a, const pose_t *b, pose_t *o) {
  double p[3];
  matvec(a->R, b->p, p);
  p[0] += a->p[0]; p[1] += a->p[1]; p[2] += a->p[2];
  matmul(a->R, b->R, o->R);
  memcpy(o->p, p, sizeof p);
}
static void inverse(const pose_t *a, pose_t *o) {
  pose_t t;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t.R[3 * i + j] = a->R[3 * j + i];
  matvec(t.R, a->p, t.p);
  t.p[0] = -t.p[0]; t.p[1] = -t.p[1]; t.p[2] = -t.p[2];
  *o = t;
}
static void apply(const pose_t *a, const double *v, double *o) {
  double t[3];
  matvec(a->R, v, t);
  o[0] = t[0] + a->p[0]; o[1] = t[1] + a->p[1]; o[2] = t[2] + a->p[2];
}
static void pose12(const double *v, pose_t *o) { memcpy(o->R, v, 72); memcpy(o->p, v + 9, 24); }
static void body_pose(const ostate *st, int b, pose_t *o) {
  quat_to_mat(st->quat[b], o->R);
  memcpy(o->p, st->pos[b], 24);
}
static void rot_z(double a, double *R) {
  double c = cos(a), s = sin(a);
  R[0] = c; R[1] = -s; R[2] = 0.0; R[3] = s; R[4] = c; R[5] = 0.0; R[6] = 0.0; R[7] = 0.0; R[8] = 1.0;
}
/* robot.py:156-158 */
static void base3(const double *base, pose_t *o) {
  rot_z(base[2], o->R);
  o->p[0] = base[0]; o->p[1] = base[1]; o->p[2] = 0.0;
}

/* robot.py:161-169: link poses + end effector */
static void link_poses(const orc_world *w, const double *q, const double *base, pose_t *links, pose_t *ee) {
  pose_t t, off, rot;
  base3(base, &t);
  rot_z(0.0, off.R);
  memset(rot.p, 0, sizeof rot.p);
  for (int i = 0; i < w->narm; ++i) {
    memcpy(off.p, w->arm_offset + 3 * i, 24);
    compose(&t, &off, &t);
    axis_angle_mat(w->arm_axis + 3 * i, q[i], rot.R);
    compose(&t, &rot, &t);
    if (links) links[i] = t;
  }
  pose_t g = {{1, 0, 0, 0, 1, 0, 0, 0, 1}, {w->gripper[0], w->gripper[1], w->gripper[2]}};
  compose(&t, &g, ee);
}
static void ee_pose(const orc_world *w, const ostate *st, pose_t *ee) {
  link_poses(w, st->joints + w->nsj, st->base, NULL, ee);
}

/* physics.py:1339-1347 */
static void quat_delta_omega(const double *qo, const double *qn, double dt, double *om) {
  double c[4] = {qo[0], -qo[1], -qo[2], -qo[3]}, dq[4];
  quat_mul(qn, c, dq);
  if (dq[0] < 0) for (int i = 0; i < 4; ++i) dq[i] = -dq[i];
  double x = dq[0] < -1.0 ? -1.0 : (dq[0] > 1.0 ? 1.0 : dq[0]);
  double ang = 2.0 * acos(x);
  if (ang < 1e-12) { om[0] = om[1] = om[2] = 0.0; return; }
  double sh = sin(ang / 2.0);
  for (int i = 0; i < 3; ++i) om[i] = (dq[1 + i] / sh) * (ang / dt);
}

/* write a kinematic pose; returns 1 if it changed (physics.py:419-433, :441-453) */
static int set_kinematic(ostate *st, int b, const pose_t *p, double dt, int zero_if_same) {
  double q[4];
  mat_to_quat(p->R, q);
  int same = st->pos[b][0] == p->p[0] && st->pos[b][1] == p->p[1] && st->pos[b][2] == p->p[2] &&
             st->quat[b][0] == q[0] && st->quat[b][1] == q[1] && st->quat[b][2] == q[2] && st->quat[b][3] == q[3];
  if (same) {
    if (zero_if_same && dt > 0) {
      memset(st->lv[b], 0, 24);
      memset(st->av[b], 0, 24);
    }
    return 0;
  }
  double op[3], oq[4];
  memcpy(op, st->pos[b], 24); memcpy(oq, st->quat[b], 32);
  memcpy(st->pos[b], p->p, 24); memcpy(st->quat[b], q, 32);
  if (dt > 0) {
    for (int i = 0; i < 3; ++i) st->lv[b][i] = (p->p[i] - op[i]) / dt;
    quat_delta_omega(oq, q, dt, st->av[b]);
  }
  return 1;
}

static void update_robot_links(const orc_world *w, ostate *st, double dt) {
  pose_t links[16], ee, bp;
  link_poses(w, st->joints + w->nsj, st->base, links, &ee);
  base3(st->base, &bp);
  set_kinematic(st, w->robot_base, &bp, dt, 1);
  for (int i = 0; i < w->narm; ++i) set_kinematic(st, w->robot_base + 1 + i, &links[i], dt, 1);
}

/* scene.py:102-105, :436-437 */
static void joint_child_pose(const orc_world *w, const ostate *st, int ji, double q, pose_t *o) {
  pose_t parent, origin, motion, t;
  body_pose(st, w->joint_parent[ji], &parent);
  pose12(w->joint_origin + 12 * ji, &origin);
  compose(&parent, &origin, &t);
  if (w->joint_type[ji] == RS_REVOLUTE) {
    axis_angle_mat(w->joint_axis + 3 * ji, q, motion.R);
    memset(motion.p, 0, 24);
  } else {
    double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    memcpy(motion.R, I, sizeof I);
    for (int i = 0; i < 3; ++i) motion.p[i] = w->joint_axis[3 * ji + i] * q;
  }
  compose(&t, &motion, o);
}

/* physics.py:435-467 */
static void update_scene_joint_poses(const orc_world *w, ostate *st, const int *list, int n, double dt) {
  int moved[MAXJ], nm = 0;
  for (int k = 0; k < n; ++k) {
    int ji = list[k];
    pose_t p;
    joint_child_pose(w, st, ji, st->joints[ji], &p);
    if (set_kinematic(st, w->joint_body[ji], &p, dt, 0)) moved[nm++] = ji;
  }
  if (!nm) return;
  for (int c = 0; c < w->nclutter; ++c) {
    int b = w->clutter[c];
    int rj = (int)st->rider_joint[b], hit = 0;
    for (int k = 0; k < nm; ++k) hit |= (moved[k] == rj);
    if (!hit || !st->asleep[b]) continue;
    pose_t part, rel, np_;
    body_pose(st, w->joint_body[rj], &part);
    quat_to_mat(st->rider_offset[b] + 3, rel.R);
    memcpy(rel.p, st->rider_offset[b], 24);
    compose(&part, &rel, &np_);
    memcpy(st->pos[b], np_.p, 24);
    mat_to_quat(np_.R, st->quat[b]);
  }
}

/* ---------------------------------------------------------- walk grid (navgrid.py:55-105) */

static int nav_ok(const orc_world *w, long i, long j) {
  return i >= 0 && i < w->nav_nx && j >= 0 && j < w->nav_ny && w->nav[i * w->nav_ny + j];
}
static void nav_centre(const orc_world *w, long i, long j, double *c) {
  c[0] = w->nav_origin[0] + ((double)i + 0.5) * w->nav_cell;
  c[1] = w->nav_origin[1] + ((double)j + 0.5) * w->nav_cell;
}
static void nav_cell_of(const orc_world *w, double x, double y, long *i, long *j) {
  *i = (long)floor((x - w->nav_origin[0]) / w->nav_cell);
  *j = (long)floor((y - w->nav_origin[1]) / w->nav_cell);
}
/* best (d2, i, j) on Chebyshev ring r around (ci, cj); returns 0 if none */
static int nav_ring(const orc_world *w, long ci, long cj, long r, double x, double y, double *bd, long *bi, long *bj) {
  int found = 0;
  for (long i = ci - r; i <= ci + r; ++i)
    for (long j = cj - r; j <= cj + r; ++j) {
      long di = labs(i - ci), dj = labs(j - cj);
      if ((di > dj ? di : dj) != r || !nav_ok(w, i, j)) continue;
      double c[2];
      nav_centre(w, i, j, c);
      double ex = c[0] - x, ey = c[1] - y, d2 = ex * ex + ey * ey;
      if (!found || d2 < *bd || (d2 == *bd && (i < *bi || (i == *bi && j < *bj)))) {
        *bd = d2; *bi = i; *bj = j; found = 1;
      }
    }
  return found;
}
int orc_nearest_walkable(const orc_world *w, double x, double y, double *out) {
  long ci, cj;
  nav_cell_of(w, x, y, &ci, &cj);
  if (nav_ok(w, ci, cj)) { out[0] = x; out[1] = y; return 1; }
  long maxr = w->nav_nx > w->nav_ny ? w->nav_nx : w->nav_ny;
  for (long r = 0; r <= maxr; ++r) {
    double bd, bd2; long bi, bj, bi2, bj2;
    if (!nav_ring(w, ci, cj, r, x, y, &bd, &bi, &bj)) continue;
    if (nav_ring(w, ci, cj, r + 1, x, y, &bd2, &bi2, &bj2) && bd2 < bd) { bi = bi2; bj = bj2; }
    nav_centre(w, bi, bj, out);
    return 0;
  }
  return -1;
}
/* Python float modulo (sign of divisor) for robot.py:371-372 */
static double py_mod(double a, double b) {
  double m = fmod(a, b);
  if (m != 0.0) {
    if ((b < 0) != (m < 0)) m += b;
  } else {
    m = copysign(0.0, b);
  }
  return m;
}
/* robot.py:349-368 */
void orc_move_base(const orc_world *w, const double *base, double lin, double ang, double dt, double *out) {
  double x = base[0], y = base[1], yaw = base[2];
  double nx = x + cos(yaw) * lin * dt, ny = y + sin(yaw) * lin * dt;
  double nyaw = py_mod(yaw + ang * dt + M_PI, 2.0 * M_PI) - M_PI;
  long i, j;
  nav_cell_of(w, nx, ny, &i, &j);
  if (!nav_ok(w, i, j)) {
    double p[2];
    orc_nearest_walkable(w, nx, ny, p);
    nx = p[0]; ny = p[1];
  }
  out[0] = nx; out[1] = ny; out[2] = nyaw;
}

/* ------------------------------------------------------------- geodesics */

/* navgrid.py:109-143 distance_field: Dijkstra from the goal's cell (after
 * nearest_walkable) over walkable 8-neighbours, step cost cell (straight) or
 * cell*sqrt(2) (diagonal), heap ordered by (d, i, j) like heapq on tuples.
 * out: [nx][ny] (x-major), +inf where unreachable. Returns the goal cell
 * index i*ny+j. */
typedef struct { double d; long i, j; } heap_e;
static int heap_less(const heap_e *a, const heap_e *b) {
  return a->d < b->d || (a->d == b->d && (a->i < b->i || (a->i == b->i && a->j < b->j)));
}
static void heap_push(heap_e *h, long *n, heap_e e) {
  long k = (*n)++;
  while (k > 0) {
    long p = (k - 1) / 2;
    if (!heap_less(&e, &h[p])) break;
    h[k] = h[p];
    k = p;
  }
  h[k] = e;
}
static heap_e heap_pop(heap_e *h, long *n) {
  heap_e top = h[0], last = h[--(*n)];
  long k = 0;
  for (;;) {
    long c = 2 * k + 1;
    if (c >= *n) break;
    if (c + 1 < *n && heap_less(&h[c + 1], &h[c])) ++c;
    if (!heap_less(&h[c], &last)) break;
    h[k] = h[c];
    k = c;
  }
  if (*n > 0) h[k] = last;
  return top;
}
long orc_nav_field(const orc_world *w, double gx, double gy, double *out) {
  const long nx = w->nav_nx, ny = w->nav_ny;
  double g[2];
  if (orc_nearest_walkable(w, gx, gy, g) < 0) return -1;
  long gi, gj;
  nav_cell_of(w, g[0], g[1], &gi, &gj);
  for (long k = 0; k < nx * ny; ++k) out[k] = INFINITY;
  out[gi * ny + gj] = 0.0;
  const double straight = w->nav_cell, diag = w->nav_cell * sqrt(2.0);
  long cap = 8 * nx * ny + 16, n = 0;
  heap_e *h = (heap_e *)malloc(sizeof(heap_e) * cap);
  heap_e e0 = {0.0, gi, gj};
  heap_push(h, &n, e0);
  while (n > 0) {
    heap_e e = heap_pop(h, &n);
    if (e.d > out[e.i * ny + e.j]) continue;
    for (int di = -1; di <= 1; ++di)
      for (int dj = -1; dj <= 1; ++dj) {
        if (!di && !dj) continue;
        long ni = e.i + di, nj = e.j + dj;
        if (ni < 0 || ni >= nx || nj < 0 || nj >= ny || !w->nav[ni * ny + nj]) continue;
        double nd = e.d + ((di && dj) ? diag : straight);
        if (nd < out[ni * ny + nj]) {
          out[ni * ny + nj] = nd;
          if (n >= cap) { cap *= 2; h = (heap_e *)realloc(h, sizeof(heap_e) * cap); }
          heap_e f = {nd, ni, nj};
          heap_push(h, &n, f);
        }
      }
  }
  free(h);
  return gi * ny + gj;
}
/* navgrid.py:145-148 geodesic_distance against a field from orc_nav_field */
double orc_nav_geodesic(const orc_world *w, const double *field, double fx, double fy) {
  double p[2];
  if (orc_nearest_walkable(w, fx, fy, p) < 0) return INFINITY;
  long i, j;
  nav_cell_of(w, p[0], p[1], &i, &j);
  return field[i * w->nav_ny + j];
}
/* navgrid.py:150-172 shortest_path: steepest descent on the field from the
 * start cell; waypoints (cell centres) into out[cap][2]; returns the count
 * (0 when unreachable; the path is truncated at cap). */
int orc_nav_path(const orc_world *w, const double *field, double fx, double fy, double *out, int cap) {
  const long nx = w->nav_nx, ny = w->nav_ny;
  double p[2];
  if (orc_nearest_walkable(w, fx, fy, p) < 0) return 0;
  long ci, cj;
  nav_cell_of(w, p[0], p[1], &ci, &cj);
  if (!isfinite(field[ci * ny + cj])) return 0;
  int n = 0;
  if (n < cap) { nav_centre(w, ci, cj, out + 2 * n); }
  ++n;
  long guard = nx * ny;
  while (field[ci * ny + cj] > 0.0 && guard > 0) {
    --guard;
    int found = 0;
    double bv = 0.0;
    long bi = 0, bj = 0;
    for (int di = -1; di <= 1; ++di)
      for (int dj = -1; dj <= 1; ++dj) {
        if (!di && !dj) continue;
        long ni = ci + di, nj = cj + dj;
        if (ni < 0 || ni >= nx || nj < 0 || nj >= ny || !isfinite(field[ni * ny + nj])) continue;
        double v = field[ni * ny + nj];
        if (!found || v < bv || (v == bv && (ni < bi || (ni == bi && nj < bj)))) { found = 1; bv = v; bi = ni; bj = nj; }
      }
    if (!found || bv >= field[ci * ny + cj]) break;
    ci = bi; cj = bj;
    if (n < cap) nav_centre(w, ci, cj, out + 2 * n);
    ++n;
  }
  return n < cap ? n : cap;
}

/* -------------------------------------------------------------- primitives */

static void part_world(const orc_world *w, const pose_t *bp, int p, pose_t *o) {
  pose_t l;
  pose12(w->part_local + 12 * p, &l);
  compose(bp, &l, o);
}
/* geometry.py:278-286 */
static void prim_aabb(const orc_world *w, int p, const pose_t *wp, double *lo, double *hi) {
  int k = w->part_kind[p];
  if (k == RS_BOX) {
    const double *h = w->part_param + 3 * p;
    for (int i = 0; i < 3; ++i) {
      double r = fabs(wp->R[3 * i]) * h[0] + fabs(wp->R[3 * i + 1]) * h[1] + fabs(wp->R[3 * i + 2]) * h[2];
      lo[i] = wp->p[i] - r; hi[i] = wp->p[i] + r;
    }
  } else if (k == RS_SPHERE) {
    double r = w->part_param[3 * p];
    for (int i = 0; i < 3; ++i) { lo[i] = wp->p[i] - r; hi[i] = wp->p[i] + r; }
  } else {
    for (int i = 0; i < 3; ++i) { lo[i] = INFINITY; hi[i] = -INFINITY; }
    for (int v = w->part_vert_begin[p]; v < w->part_vert_begin[p + 1]; ++v) {
      double x[3];
      apply(wp, w->vert + 3 * v, x);
      for (int i = 0; i < 3; ++i) { if (x[i] < lo[i]) lo[i] = x[i]; if (x[i] > hi[i]) hi[i] = x[i]; }
    }
  }
}
static void body_aabb(const orc_world *w, const ostate *st, int b, double *lo, double *hi) {
  pose_t bp, wp;
  body_pose(st, b, &bp);
  for (int i = 0; i < 3; ++i) { lo[i] = INFINITY; hi[i] = -INFINITY; }
  for (int p = w->body_part_begin[b]; p < w->body_part_begin[b + 1]; ++p) {
    double l[3], h[3];
    part_world(w, &bp, p, &wp);
    prim_aabb(w, p, &wp, l, h);
    for (int i = 0; i < 3; ++i) { lo[i] = fmin(lo[i], l[i]); hi[i] = fmax(hi[i], h[i]); }
  }
}

/* world planes: n_w = R n, d_w = d + n_w . p   (geometry.py:554-557) */
static void planes_world(const orc_world *w, int p, const pose_t *wp, double *nw, double *dw) {
  int f0 = w->part_facet_begin[p], nf = w->part_facet_begin[p + 1] - f0;
  for (int f = 0; f < nf; ++f) {
    const double *F = w->facet + 4 * (f0 + f);
    matvec(wp->R, F, nw + 3 * f);
    dw[f] = F[3] + dot3(nw + 3 * f, wp->p);
  }
}

typedef struct { int a, b; double p[3], n[3], depth; } contact_t;

/* geometry.py:564-576 + :683-698 (one direction) */
static int vertices_in_convex(const orc_world *w, int pv, const pose_t *wv, int pf, const pose_t *wf, double margin,
                              int negate, int a, int b, contact_t *out, int cap) {
  double nw[64 * 3], dw[64];
  int nf = w->part_facet_begin[pf + 1] - w->part_facet_begin[pf];
  planes_world(w, pf, wf, nw, dw);
  int cnt = 0;
  for (int v = w->part_vert_begin[pv]; v < w->part_vert_begin[pv + 1]; ++v) {
    double x[3];
    apply(wv, w->vert + 3 * v, x);
    int face = 0, neg = 0;
    double best = 0.0;
    for (int f = 0; f < nf; ++f) {
      double s = dw[f] - dot3(x, nw + 3 * f);
      if (f == 0 || s < best) { best = s; face = f; }
      neg += (s < 0.0);
    }
    if (neg == 0 || (neg == 1 && best >= -margin)) {
      if (cnt < cap) {
        contact_t *c = &out[cnt];
        c->a = a; c->b = b;
        memcpy(c->p, x, 24);
        for (int i = 0; i < 3; ++i) c->n[i] = negate ? -nw[3 * face + i] : nw[3 * face + i];
        c->depth = best;
      }
      ++cnt;
    }
  }
  return cnt;
}

/* geometry.py:602-630 (Ericson) */
static void closest_on_triangle(const double *p, const double *a, const double *b, const double *c, double *o) {
  double ab[3], ac[3], ap[3], bp[3], cp[3];
  for (int i = 0; i < 3; ++i) { ab[i] = b[i] - a[i]; ac[i] = c[i] - a[i]; ap[i] = p[i] - a[i]; }
  double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
  if (d1 <= 0 && d2 <= 0) { memcpy(o, a, 24); return; }
  for (int i = 0; i < 3; ++i) bp[i] = p[i] - b[i];
  double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
  if (d3 >= 0 && d4 <= d3) { memcpy(o, b, 24); return; }
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) {
    double t = d1 / (d1 - d3);
    for (int i = 0; i < 3; ++i) o[i] = a[i] + ab[i] * t;
    return;
  }
  for (int i = 0; i < 3; ++i) cp[i] = p[i] - c[i];
  double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
  if (d6 >= 0 && d5 <= d6) { memcpy(o, c, 24); return; }
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) {
    double t = d2 / (d2 - d6);
    for (int i = 0; i < 3; ++i) o[i] = a[i] + ac[i] * t;
    return;
  }
  double va = d3 * d6 - d5 * d4;
  if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0) {
    double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    for (int i = 0; i < 3; ++i) o[i] = b[i] + (c[i] - b[i]) * t;
    return;
  }
  double den = va + vb + vc, v = vb / den, ww = vc / den;
  for (int i = 0; i < 3; ++i) o[i] = a[i] + ab[i] * v + ac[i] * ww;
}

/* geometry.py:579-599 (convex primitive only) */
static void closest_on_convex(const orc_world *w, int p, const pose_t *wp, const double *pt, double *o) {
  if (w->part_kind[p] == RS_BOX) {
    const double *h = w->part_param + 3 * p;
    double d[3], l[3];
    for (int i = 0; i < 3; ++i) d[i] = pt[i] - wp->p[i];
    mattvec(wp->R, d, l);
    for (int i = 0; i < 3; ++i) l[i] = l[i] < -h[i] ? -h[i] : (l[i] > h[i] ? h[i] : l[i]);
    apply(wp, l, o);
    return;
  }
  int v0 = w->part_vert_begin[p];
  double best = 0.0;
  int first = 1;
  for (int t = w->part_tri_begin[p]; t < w->part_tri_begin[p + 1]; ++t) {
    double A[3], B[3], C[3], q[3];
    apply(wp, w->vert + 3 * (v0 + w->tri[3 * t]), A);
    apply(wp, w->vert + 3 * (v0 + w->tri[3 * t + 1]), B);
    apply(wp, w->vert + 3 * (v0 + w->tri[3 * t + 2]), C);
    closest_on_triangle(pt, A, B, C, q);
    double e[3] = {pt[0] - q[0], pt[1] - q[1], pt[2] - q[2]}, d2 = dot3(e, e);
    if (first || d2 < best) { best = d2; memcpy(o, q, 24); first = 0; }
  }
}

/* geometry.py:633-653 */
static int sphere_convex(const orc_world *w, int ps, const pose_t *ws, int pc, const pose_t *wc, int flip,
                         double margin, int a, int b, contact_t *out, int cap) {
  double r = w->part_param[3 * ps];
  const double *c = ws->p;
  double nw[64 * 3], dw[64];
  int nf = w->part_facet_begin[pc + 1] - w->part_facet_begin[pc];
  planes_world(w, pc, wc, nw, dw);
  int inside = 1, f = 0;
  double best = 0.0;
  for (int k = 0; k < nf; ++k) {
    double s = dw[k] - dot3(nw + 3 * k, c);
    if (s < 0.0) inside = 0;
    if (k == 0 || s < best) { best = s; f = k; }
  }
  double n[3], pt[3], depth;
  if (inside) {
    depth = r + best;
    memcpy(n, nw + 3 * f, 24);
    for (int i = 0; i < 3; ++i) pt[i] = c[i] - n[i] * best;
  } else {
    double q[3], d[3];
    closest_on_convex(w, pc, wc, c, q);
    for (int i = 0; i < 3; ++i) d[i] = c[i] - q[i];
    double dist = sqrt(dot3(d, d));
    depth = r - dist;
    if (depth <= -margin) return 0;
    if (dist > 0) for (int i = 0; i < 3; ++i) n[i] = d[i] / dist;
    else { n[0] = 0; n[1] = 0; n[2] = 1; }
    memcpy(pt, q, 24);
  }
  if (flip) for (int i = 0; i < 3; ++i) n[i] = -n[i];
  if (cap > 0) {
    out->a = a; out->b = b; memcpy(out->p, pt, 24); memcpy(out->n, n, 24); out->depth = depth;
  }
  return 1;
}

/* geometry.py:656-664 */
static int sphere_sphere(const orc_world *w, int pa, const pose_t *wa, int pb, const pose_t *wb, double margin,
                         int a, int b, contact_t *out, int cap) {
  double ra = w->part_param[3 * pa], rb = w->part_param[3 * pb], d[3], n[3];
  for (int i = 0; i < 3; ++i) d[i] = wa->p[i] - wb->p[i];
  double dist = sqrt(dot3(d, d)), depth = ra + rb - dist;
  if (depth <= -margin) return 0;
  if (dist > 0) for (int i = 0; i < 3; ++i) n[i] = d[i] / dist;
  else { n[0] = 0; n[1] = 0; n[2] = 1; }
  if (cap > 0) {
    out->a = a; out->b = b;
    for (int i = 0; i < 3; ++i) out->p[i] = wb->p[i] + n[i] * rb;
    memcpy(out->n, n, 24); out->depth = depth;
  }
  return 1;
}

/* geometry.py:701-716 parts_contacts + :667-698 convex_contacts */
static int pair_contacts(const orc_world *w, const ostate *st, int a, int b, double margin, contact_t *out, int cap) {
  pose_t pa, pb, wa, wb;
  body_pose(st, a, &pa);
  body_pose(st, b, &pb);
  int n = 0;
  for (int i = w->body_part_begin[a]; i < w->body_part_begin[a + 1]; ++i) {
    double loa[3], hia[3];
    part_world(w, &pa, i, &wa);
    prim_aabb(w, i, &wa, loa, hia);
    for (int j = w->body_part_begin[b]; j < w->body_part_begin[b + 1]; ++j) {
      double lob[3], hib[3];
      part_world(w, &pb, j, &wb);
      prim_aabb(w, j, &wb, lob, hib);
      int sep = 0;
      for (int k = 0; k < 3; ++k) sep |= (loa[k] > hib[k] + margin) || (lob[k] > hia[k] + margin);
      if (sep) continue;
      int ka = w->part_kind[i], kb = w->part_kind[j];
      int room = cap - n > 0 ? cap - n : 0;
      if (ka == RS_SPHERE && kb == RS_SPHERE)
        n += sphere_sphere(w, i, &wa, j, &wb, margin, a, b, out + n, room);
      else if (ka == RS_SPHERE)
        n += sphere_convex(w, i, &wa, j, &wb, 0, margin, a, b, out + n, room);
      else if (kb == RS_SPHERE)
        n += sphere_convex(w, j, &wb, i, &wa, 1, margin, a, b, out + n, room);
      else {
        n += vertices_in_convex(w, i, &wa, j, &wb, margin, 0, a, b, out + n, room);
        room = cap - n > 0 ? cap - n : 0;
        n += vertices_in_convex(w, j, &wb, i, &wa, margin, 1, a, b, out + n, room);
      }
    }
  }
  return n;
}

/* ---------------------------------------------------------------- solver */

typedef struct {
  int a, b, ja, jb;             /* joint index or -1 */
  double n[3], t1[3], t2[3], ra[3], rb[3];
  double k, mu, ima, imb, Ia[9], Ib[9];
  double jaca[3], jacb[3], jia, jib;
  double point[3], depth;
  double lam, lt1, lt2, vn_pre, target;
  int friction_on;
} row_t;

typedef struct {
  double v[MAXB][6];
  int have[MAXB];
  double jdv[MAXJ];
} velset_t;

static void rel_vel(const row_t *r, const velset_t *vs, double *o) {
  const double *va = vs->v[r->a], *vb = vs->v[r->b];
  double ax = va[0] + va[4] * r->ra[2] - va[5] * r->ra[1];
  double ay = va[1] + va[5] * r->ra[0] - va[3] * r->ra[2];
  double az = va[2] + va[3] * r->ra[1] - va[4] * r->ra[0];
  double bx = vb[0] + vb[4] * r->rb[2] - vb[5] * r->rb[1];
  double by = vb[1] + vb[5] * r->rb[0] - vb[3] * r->rb[2];
  double bz = vb[2] + vb[3] * r->rb[1] - vb[4] * r->rb[0];
  if (r->ja >= 0) {
    double dv = vs->jdv[r->ja];
    ax += r->jaca[0] * dv; ay += r->jaca[1] * dv; az += r->jaca[2] * dv;
  }
  if (r->jb >= 0) {
    double dv = vs->jdv[r->jb];
    bx += r->jacb[0] * dv; by += r->jacb[1] * dv; bz += r->jacb[2] * dv;
  }
  o[0] = ax - bx; o[1] = ay - by; o[2] = az - bz;
}
static double rel_normal_vel(const row_t *r, const velset_t *vs) {
  double v[3];
  rel_vel(r, vs, v);
  return v[0] * r->n[0] + v[1] * r->n[1] + v[2] * r->n[2];
}
/* physics.py:1257-1291 */
static void apply_impulse(const row_t *r, velset_t *vs, double ix, double iy, double iz) {
  if (r->ima > 0.0) {
    double *va = vs->v[r->a], m = r->ima;
    va[0] += ix * m; va[1] += iy * m; va[2] += iz * m;
    double tx = r->ra[1] * iz - r->ra[2] * iy, ty = r->ra[2] * ix - r->ra[0] * iz, tz = r->ra[0] * iy - r->ra[1] * ix;
    const double *I = r->Ia;
    va[3] += I[0] * tx + I[1] * ty + I[2] * tz;
    va[4] += I[3] * tx + I[4] * ty + I[5] * tz;
    va[5] += I[6] * tx + I[7] * ty + I[8] * tz;
  }
  if (r->imb > 0.0) {
    double *vb = vs->v[r->b], m = r->imb;
    vb[0] -= ix * m; vb[1] -= iy * m; vb[2] -= iz * m;
    double tx = r->rb[1] * iz - r->rb[2] * iy, ty = r->rb[2] * ix - r->rb[0] * iz, tz = r->rb[0] * iy - r->rb[1] * ix;
    const double *I = r->Ib;
    vb[3] -= I[0] * tx + I[1] * ty + I[2] * tz;
    vb[4] -= I[3] * tx + I[4] * ty + I[5] * tz;
    vb[5] -= I[6] * tx + I[7] * ty + I[8] * tz;
  }
  if (r->ja >= 0) vs->jdv[r->ja] += (r->jaca[0] * ix + r->jaca[1] * iy + r->jaca[2] * iz) * r->jia;
  if (r->jb >= 0) vs->jdv[r->jb] -= (r->jacb[0] * ix + r->jacb[1] * iy + r->jacb[2] * iz) * r->jib;
}
/* physics.py:1309-1326 */
static void solve_friction(row_t *r, velset_t *vs) {
  if (r->k <= 0.0 || !r->friction_on) return;
  double max_t = r->mu * r->lam;
  for (int which = 0; which < 2; ++which) {
    const double *t = which ? r->t2 : r->t1;
    double *acc = which ? &r->lt2 : &r->lt1;
    double v[3];
    rel_vel(r, vs, v);
    double vt = v[0] * t[0] + v[1] * t[1] + v[2] * t[2];
    double lt = -vt / r->k, nt = *acc + lt;
    if (nt > max_t) nt = max_t;
    else if (nt < -max_t) nt = -max_t;
    lt = nt - *acc;
    *acc = nt;
    if (lt != 0.0) apply_impulse(r, vs, t[0] * lt, t[1] * lt, t[2] * lt);
  }
}
/* physics.py:1293-1307 */
static void solve_row(row_t *r, velset_t *vs) {
  if (r->k <= 0.0) return;
  double vn = rel_normal_vel(r, vs);
  double lam = -(vn - r->target) / r->k, tot = r->lam + lam;
  if (tot < 0.0) tot = 0.0;
  lam = tot - r->lam;
  r->lam = tot;
  if (lam != 0.0) apply_impulse(r, vs, r->n[0] * lam, r->n[1] * lam, r->n[2] * lam);
  solve_friction(r, vs);
}

/* Jacobi eigensolver for a symmetric m x m matrix (row-major, m <= 32) in
 * round-robin ("parallel") ordering: each sweep is m'-1 rounds (m' = m
 * rounded up to even) of m'/2 disjoint rotations, all computed from the
 * matrix at the start of the round, then applied as one column pass and one
 * row pass.  The CUDA block solver executes exactly these per-element
 * operations one element per lane, so the two agree bit for bit.  The pair
 * schedule is the circle method: in round r, (n-1, r) and
 * ((r+k) mod (n-1), (r-k+n-1) mod (n-1)) for k = 1..n/2-1. */
void orc_jacobi_pair(int n, int r, int k, int *p, int *q) {
  int a, b;
  if (k == 0) { a = n - 1; b = r; }
  else { a = (r + k) % (n - 1); b = (r - k + n - 1) % (n - 1); }
  *p = a < b ? a : b;
  *q = a < b ? b : a;
}

#ifdef ORC_PROFILE
/* solver work log for tools/solver_profile.py (not built by default) */
typedef struct { int sub, it, g, m, na, mask, sweeps, asi; } orc_prof_rec;
static orc_prof_rec g_prof[1 << 20];
static int g_nprof, g_prof_sub, g_prof_it, g_prof_g, g_prof_m, g_prof_mask, g_prof_asi, g_last_sweeps;
int orc_profile_take(int *out, int cap) {
  int n = g_nprof < cap ? g_nprof : cap;
  memcpy(out, g_prof, sizeof(orc_prof_rec) * n);
  g_nprof = 0;
  return n;
}
#define PROF_SWEEPS(s) (g_last_sweeps = (s))
#else
#define PROF_SWEEPS(s) ((void)0)
#endif

static void sym_eig(int m, double *A, double *V, double *ev) {
  const int n = m + (m & 1);
  double cs[16], sn[16];
  int pp[16], qq[16];
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) V[i * m + j] = (i == j);
  for (int sweep = 0; sweep < 64 && m > 1; ++sweep) {
    /* Frobenius norms as per-row partial sums, rows added in order (the GPU
       computes one row per lane) */
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < m; ++i) {
      double ro = 0.0, rt = 0.0;
      for (int j = 0; j < m; ++j) {
        double a2 = A[i * m + j] * A[i * m + j];
        rt += a2;
        if (i != j) ro += a2;
      }
      off += ro;
      tot += rt;
    }
    PROF_SWEEPS(sweep);
    if (off <= 1e-30 * tot || off == 0.0) break; /* off-diagonal <= 1e-15 of the Frobenius norm */
    PROF_SWEEPS(sweep + 1);
    for (int r = 0; r < n - 1; ++r) {
      for (int k = 0; k < n / 2; ++k) {
        int p, q;
        orc_jacobi_pair(n, r, k, &p, &q);
        pp[k] = p; qq[k] = q;
        cs[k] = 1.0; sn[k] = 0.0;
        if (q >= m) continue; /* padding index */
        double apq = A[p * m + q];
        if (apq == 0.0) continue;
        double app = A[p * m + p], aqq = A[q * m + q];
        /* t = sgn(theta) / (|theta| + sqrt(theta^2 + 1)), theta = a / b, and
           c = 1 / sqrt(t^2 + 1), multiplied through by |b| */
        double a = aqq - app, b = 2.0 * apq;
        double num = a > 0.0 ? b : (a < 0.0 ? -b : fabs(b));
        double den = fabs(a) + sqrt(a * a + b * b);
        double t = num / den;
        cs[k] = den / sqrt(den * den + b * b);
        sn[k] = t * cs[k];
      }
      /* column pass (A and V) */
      for (int k = 0; k < n / 2; ++k) {
        int p = pp[k], q = qq[k];
        if (q >= m || sn[k] == 0.0) continue;
        for (int i = 0; i < m; ++i) {
          double aip = A[i * m + p], aiq = A[i * m + q];
          A[i * m + p] = cs[k] * aip - sn[k] * aiq;
          A[i * m + q] = sn[k] * aip + cs[k] * aiq;
          double vip = V[i * m + p], viq = V[i * m + q];
          V[i * m + p] = cs[k] * vip - sn[k] * viq;
          V[i * m + q] = sn[k] * vip + cs[k] * viq;
        }
      }
      /* row pass */
      for (int k = 0; k < n / 2; ++k) {
        int p = pp[k], q = qq[k];
        if (q >= m || sn[k] == 0.0) continue;
        for (int j = 0; j < m; ++j) {
          double apj = A[p * m + j], aqj = A[q * m + j];
          A[p * m + j] = cs[k] * apj - sn[k] * aqj;
          A[q * m + j] = sn[k] * apj + cs[k] * aqj;
        }
      }
    }
  }
  for (int i = 0; i < m; ++i) ev[i] = A[i * m + i];
}

/* minimum-norm least squares for a symmetric PSD matrix with LAPACK gelsd's
 * cutoff s_i <= rcond * s_max -> 0 (physics.py:782, np.linalg.lstsq) */
static void pinv_solve(int m, const double *A, const double *b, double rcond, double *x) {
  double W[32 * 32], V[32 * 32], ev[32];
  memcpy(W, A, sizeof(double) * m * m);
  sym_eig(m, W, V, ev);
  double smax = 0.0;
  for (int i = 0; i < m; ++i) smax = fmax(smax, fabs(ev[i]));
  for (int i = 0; i < m; ++i) x[i] = 0.0;
  for (int k = 0; k < m; ++k) {
    if (fabs(ev[k]) <= rcond * smax) continue;
    double c = 0.0;
    for (int i = 0; i < m; ++i) c += V[i * m + k] * b[i];
    c /= ev[k];
    for (int i = 0; i < m; ++i) x[i] += c * V[i * m + k];
  }
}

/* physics.py:760-816 */
static void solve_block(row_t *rows, int first, int m, const double *K, velset_t *vs) {
  double cur[32], q[32], lam[32], wv[32], sub[32 * 32], rhs[32], sol[32];
  int active[32], na = 0;
  for (int i = 0; i < m; ++i) {
    row_t *r = &rows[first + i];
    cur[i] = r->lam;
    wv[i] = rel_normal_vel(r, vs) - r->target; /* resid */
  }
  /* w(lam) = K lam + q with q chosen so w(cur) = resid */
  for (int i = 0; i < m; ++i) {
    double s = 0.0;
    for (int j = 0; j < m; ++j) s += K[i * m + j] * cur[j];
    q[i] = wv[i] - s;
  }
  for (int i = 0; i < m; ++i)
    if (cur[i] > 0.0 || wv[i] < 0.0) active[na++] = i;
  int converged = 0;
  for (int it = 0; it < 4 * m + 4; ++it) {
    for (int i = 0; i < m; ++i) lam[i] = 0.0;
    if (na) {
      for (int i = 0; i < na; ++i) {
        for (int j = 0; j < na; ++j) sub[i * na + j] = K[active[i] * m + active[j]];
        rhs[i] = -q[active[i]];
      }
      pinv_solve(na, sub, rhs, 1e-8, sol);
      for (int i = 0; i < na; ++i) lam[active[i]] = sol[i];
#ifdef ORC_PROFILE
      if (g_nprof < (1 << 20)) {
        int mask = 0;
        for (int i = 0; i < na; ++i) mask |= 1 << active[i];
        orc_prof_rec r = {g_prof_sub, g_prof_it, g_prof_g, m, na, mask, g_last_sweeps, it};
        g_prof[g_nprof++] = r;
      }
#endif
    }
    int worst = -1;
    for (int i = 0; i < na; ++i) {
      int ii = active[i];
      if (lam[ii] < -1e-10 && (worst < 0 || lam[ii] < lam[worst] || (lam[ii] == lam[worst] && ii < worst))) worst = ii;
    }
    if (worst >= 0) {
      int k = 0;
      for (int i = 0; i < na; ++i) if (active[i] != worst) active[k++] = active[i];
      na = k;
      continue;
    }
    worst = -1;
    for (int i = 0; i < m; ++i) {
      int in = 0;
      for (int j = 0; j < na; ++j) in |= (active[j] == i);
      if (in) continue;
      double wi = 0.0;
      for (int j = 0; j < m; ++j) wi += K[i * m + j] * lam[j];
      wi += q[i];
      wv[i] = wi;
      if (wi < -1e-10 && (worst < 0 || wi < wv[worst] || (wi == wv[worst] && i < worst))) worst = i;
    }
    if (worst >= 0) {
      int k = na;
      while (k > 0 && active[k - 1] > worst) { active[k] = active[k - 1]; --k; }
      active[k] = worst;
      ++na;
      continue;
    }
    converged = 1;
    break;
  }
  if (!converged) {
    for (int i = 0; i < m; ++i) solve_row(&rows[first + i], vs);
    return;
  }
  for (int i = 0; i < m; ++i) {
    row_t *r = &rows[first + i];
    double l = lam[i] > 0.0 ? lam[i] : 0.0;
    double d = l - r->lam;
    r->lam = l;
    if (d != 0.0) apply_impulse(r, vs, r->n[0] * d, r->n[1] * d, r->n[2] * d);
  }
  for (int i = 0; i < m; ++i) solve_friction(&rows[first + i], vs);
}

/* physics.py:721-758 */
static void block_matrix(const row_t *rows, int first, int m, double *K) {
  const row_t *r0 = &rows[first];
  double la[32][3], lb[32][3];
  for (int i = 0; i < m; ++i) {
    cross(rows[first + i].ra, rows[first + i].n, la[i]);
    cross(rows[first + i].rb, rows[first + i].n, lb[i]);
  }
  for (int i = 0; i < m; ++i)
    for (int j = i; j < m; ++j) {
      const row_t *ri = &rows[first + i], *rj = &rows[first + j];
      double val = (r0->ima + r0->imb) * dot3(ri->n, rj->n);
      if (r0->ima > 0.0) { double t[3]; matvec(r0->Ia, la[j], t); val += dot3(la[i], t); }
      if (r0->imb > 0.0) { double t[3]; matvec(r0->Ib, lb[j], t); val += dot3(lb[i], t); }
      if (ri->ja >= 0 && rj->ja >= 0 && ri->ja == rj->ja)
        val += dot3(ri->jaca, ri->n) * dot3(rj->jaca, rj->n) * ri->jia;
      if (ri->jb >= 0 && rj->jb >= 0 && ri->jb == rj->jb)
        val += dot3(ri->jacb, ri->n) * dot3(rj->jacb, rj->n) * ri->jib;
      K[i * m + j] = val;
      K[j * m + i] = val;
    }
  for (int i = 0; i < m; ++i) K[i * m + i] += 1e-9;
}

/* physics.py:1329-1336 */
static void tangents(const double *n, double *t1, double *t2) {
  double ref[3] = {0, 0, 0};
  if (fabs(n[0]) < 0.9) ref[0] = 1.0; else ref[1] = 1.0;
  cross(n, ref, t1);
  double l = sqrt(dot3(t1, t1));
  for (int i = 0; i < 3; ++i) t1[i] /= l;
  cross(n, t1, t2);
  l = sqrt(dot3(t2, t2));
  for (int i = 0; i < 3; ++i) t2[i] /= l;
}

/* physics.py:818-825 */
static int solver_dynamic(const orc_world *w, const ostate *st, int b) {
  return w->body_kind[b] == RS_DYNAMIC && !st->asleep[b] && b != st->held;
}
static void body_solver_data(const orc_world *w, const ostate *st, int b, double *im, double *Iw, double *com) {
  pose_t p;
  body_pose(st, b, &p);
  apply(&p, w->com + 3 * b, com);
  if (solver_dynamic(w, st, b)) {
    double T[9], Rt[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) Rt[3 * i + j] = p.R[3 * j + i];
    matmul(p.R, w->inv_inertia + 9 * b, T);
    matmul(T, Rt, Iw);
    *im = w->inv_mass[b];
  } else {
    *im = 0.0;
    memset(Iw, 0, 72);
  }
}
/* physics.py:827-844 */
static int joint_jacobian(const orc_world *w, const ostate *st, int b, const double *pt, double *jac, double *inv_i) {
  int ji = w->body_joint[b];
  if (ji < 0 || st->held_joint == ji) return -1;
  pose_t parent, origin, jf;
  body_pose(st, w->joint_parent[ji], &parent);
  pose12(w->joint_origin + 12 * ji, &origin);
  compose(&parent, &origin, &jf);
  double ax[3];
  matvec(jf.R, w->joint_axis + 3 * ji, ax);
  if (w->joint_type[ji] == RS_PRISMATIC) {
    memcpy(jac, ax, 24);
    *inv_i = 1.0 / w->cfg.joint_inertia_prismatic;
  } else {
    double d[3] = {pt[0] - jf.p[0], pt[1] - jf.p[1], pt[2] - jf.p[2]};
    cross(ax, d, jac);
    *inv_i = 1.0 / w->cfg.joint_inertia_revolute;
  }
  return ji;
}

/* ---------------------------------------------------------------- trace */

typedef struct {
  int32_t cap_pairs, cap_contacts, cap_events;
  int32_t n_pairs, n_contacts, n_events;
  int32_t *pairs;       /* [cap][3]: substep, a, b */
  double *contacts;     /* [cap][10]: substep, a, b, p, n, depth */
  double *events;       /* [cap][7]: a, b, impulse, force, p */
  int64_t counters[3];  /* narrowphase_tests, skipped_sleeping_pairs, wakes (this call) */
} orc_trace;

static void wake(const orc_world *w, ostate *st, int b, orc_trace *tr) {
  if (w->body_kind[b] != RS_DYNAMIC) return;
  if (st->asleep[b] && tr) tr->counters[2]++;
  st->asleep[b] = 0;
  st->sleep_counter[b] = 0;
  st->rider_joint[b] = -1;
}

/* physics.py:498-571 */
static int broadphase(const orc_world *w, ostate *st, int (*pairs)[2], orc_trace *tr, int sub) {
  int nb = w->nb;
  double lo[MAXB][3], hi[MAXB][3];
  for (int b = 0; b < nb; ++b) {
    body_aabb(w, st, b, lo[b], hi[b]);
    if (w->body_kind[b] == RS_KINEMATIC)
      for (int i = 0; i < 3; ++i) { lo[b][i] -= w->cfg.wake_margin; hi[b][i] += w->cfg.wake_margin; }
  }
  int n = 0;
  for (int a = 0; a < nb; ++a)
    for (int b = a + 1; b < nb; ++b) {
      /* SAP on x with (lo.x, id) order + inclusive y/z == inclusive 3-axis overlap */
      int ov = lo[a][0] <= hi[b][0] && lo[b][0] <= hi[a][0] && lo[b][1] <= hi[a][1] && lo[a][1] <= hi[b][1] &&
               lo[b][2] <= hi[a][2] && lo[a][2] <= hi[b][2];
      if (!ov) continue;
      int ka = w->body_kind[a], kb = w->body_kind[b];
      int ga = w->body_group[a], gb = w->body_group[b];
      if (ga != RS_NO_GROUP && ga == gb) continue;
      int dyn_a = ka == RS_DYNAMIC, dyn_b = kb == RS_DYNAMIC, kin_a = ka == RS_KINEMATIC, kin_b = kb == RS_KINEMATIC;
      int adm = 0;
      if (!dyn_a && !dyn_b) {
        if (ka == RS_STATIC && kb == RS_STATIC) continue;
        int robot = w->body_robot[a] || w->body_robot[b] || a == st->held || b == st->held;
        int jointed = w->body_joint[a] >= 0 || w->body_joint[b] >= 0;
        adm = robot || jointed;
      } else {
        int sa = dyn_a && st->asleep[a], sb = dyn_b && st->asleep[b];
        if (sa && sb) { if (tr) tr->counters[1]++; continue; }
        if ((sa && kb == RS_STATIC) || (sb && ka == RS_STATIC)) { if (tr) tr->counters[1]++; continue; }
        if (sa && kin_b && w->body_joint[b] >= 0 && st->rider_joint[a] == w->body_joint[b]) continue;
        if (sb && kin_a && w->body_joint[a] >= 0 && st->rider_joint[b] == w->body_joint[a]) continue;
        int rkb = kin_b && (w->body_robot[b] || b == st->held);
        int rka = kin_a && (w->body_robot[a] || a == st->held);
        if (sa && rkb) wake(w, st, a, tr);
        if (sb && rka) wake(w, st, b, tr);
        adm = 1;
      }
      if (!adm) continue;
      if (n < MAXPAIRS) { pairs[n][0] = a; pairs[n][1] = b; }
      ++n;
      if (tr) {
        if (tr->n_pairs < tr->cap_pairs) {
          int32_t *p = tr->pairs + 3 * tr->n_pairs;
          p[0] = sub; p[1] = a; p[2] = b;
        }
        tr->n_pairs++;
      }
    }
  return n;
}

/* ---------------------------------------------------------------- substep */

typedef struct {
  contact_t c[MAXROWS];
  int nc;
  row_t rows[MAXROWS];
  double budget[MAXJ];
} scratch_t;

static int awake_dynamic(const orc_world *w, const ostate *st, int b) {
  return w->body_kind[b] == RS_DYNAMIC && !st->asleep[b] && b != st->held;
}

/* physics.py:657-701 */
static int substep(const orc_world *w, ostate *st, const double *arm, const double *basecmd, double dt,
                   scratch_t *S, orc_trace *tr, int sub) {
  const rs_physics_config *cfg = &w->cfg;
  int nb = w->nb, nsj = w->nsj;
#ifdef ORC_PROFILE
  g_prof_sub = sub;
#endif
  if (!cfg->sleeping_enabled)
    for (int b = 0; b < nb; ++b)
      if (w->body_kind[b] == RS_DYNAMIC && st->asleep[b]) {
        st->asleep[b] = 0; st->sleep_counter[b] = 0; st->rider_joint[b] = -1;
      }
  if (arm) {
    double nbp[3];
    orc_move_base(w, st->base, basecmd[0], basecmd[1], dt, nbp);
    memcpy(st->base, nbp, 24);
    /* _drive_arm physics.py:608-621 */
    for (int i = 0; i < w->narm; ++i) {
      double q = st->joints[nsj + i], err = arm[i] - q, vdes = cfg->kp * err / dt, v;
      if (cfg->impulse_cap_per_control_step) {
        double cap = S->budget[i];
        v = vdes < -cap ? -cap : (vdes > cap ? cap : vdes);
        S->budget[i] = cap - fabs(v);
      } else {
        double cap = cfg->motor_impulse_cap;
        v = vdes < -cap ? -cap : (vdes > cap ? cap : vdes);
      }
      double nq = q + v * dt, lo = w->arm_limits[2 * i], hi = w->arm_limits[2 * i + 1];
      nq = nq < lo ? lo : (nq > hi ? hi : nq);
      st->joints[nsj + i] = nq;
    }
    update_robot_links(w, st, dt);
  }
  int dragged = -1;
  if (st->held_joint >= 0) {
    /* physics.py:623-655 */
    int ji = st->held_joint;
    dragged = ji;
    pose_t parent, origin, jf, ee;
    body_pose(st, w->joint_parent[ji], &parent);
    pose12(w->joint_origin + 12 * ji, &origin);
    compose(&parent, &origin, &jf);
    ee_pose(w, st, &ee);
    double ax[3], qn;
    matvec(jf.R, w->joint_axis + 3 * ji, ax);
    int skip = 0;
    if (w->joint_type[ji] == RS_PRISMATIC) {
      double d[3] = {ee.p[0] - st->grab_ee[0], ee.p[1] - st->grab_ee[1], ee.p[2] - st->grab_ee[2]};
      qn = st->grab_q + dot3(ax, d);
    } else {
      double ref[3], cur[3], cr[3];
      for (int i = 0; i < 3; ++i) { ref[i] = st->grab_ee[i] - jf.p[i]; cur[i] = ee.p[i] - jf.p[i]; }
      double pr = dot3(ax, ref), pc = dot3(ax, cur);
      for (int i = 0; i < 3; ++i) { ref[i] -= ax[i] * pr; cur[i] -= ax[i] * pc; }
      double nr = sqrt(dot3(ref, ref)), nc = sqrt(dot3(cur, cur));
      if (nr < 1e-9 || nc < 1e-9) {
        skip = 1;
        qn = 0.0;
      } else {
        double ca = dot3(ref, cur) / (nr * nc);
        ca = ca < -1.0 ? -1.0 : (ca > 1.0 ? 1.0 : ca);
        cross(ref, cur, cr);
        double sgn = dot3(ax, cr);
        qn = st->grab_q + acos(ca) * (sgn >= 0 ? 1.0 : -1.0);
      }
    }
    if (!skip) {
      double lo = w->joint_limits[2 * ji], hi = w->joint_limits[2 * ji + 1];
      qn = fmin(fmax(qn, lo), hi);
      double old = st->joints[ji];
      if (qn != old) {
        st->joints[ji] = qn;
        st->jvel[ji] = dt > 0 ? (qn - old) / dt : 0.0;
      }
    }
    update_scene_joint_poses(w, st, &ji, 1, dt);
  }
  if (st->held >= 0 && st->held_joint < 0) {
    /* physics.py:671-684 */
    pose_t ee, off, hp;
    ee_pose(w, st, &ee);
    quat_to_mat(st->held_offset + 3, off.R);
    memcpy(off.p, st->held_offset, 24);
    compose(&ee, &off, &hp);
    set_kinematic(st, st->held, &hp, dt, 0);
  }
  /* physics.py:686-695 */
  uint8_t awake_dyn[MAXB];
  for (int b = 0; b < nb; ++b) {
    awake_dyn[b] = (uint8_t)awake_dynamic(w, st, b);
    if (!awake_dyn[b]) continue;
    st->lv[b][2] -= cfg->gravity * dt;
    for (int i = 0; i < 3; ++i) st->lv[b][i] *= cfg->lin_damping;
    for (int i = 0; i < 3; ++i) st->av[b][i] *= cfg->ang_damping;
  }
  static int pairs[MAXPAIRS][2];
  int np = broadphase(w, st, pairs, tr, sub);
  if (np > MAXPAIRS) return RS_FAULT_OVERFLOW << 16;
  /* narrowphase physics.py:703-719: contacts grouped by pair, in pair order */
  int pair_first[MAXPAIRS + 1], pair_n[MAXPAIRS], npc = 0;
  int pa_list[MAXPAIRS][2];
  S->nc = 0;
  for (int k = 0; k < np; ++k) {
    int a = pairs[k][0], b = pairs[k][1];
    if (tr) tr->counters[0]++;
    int n = pair_contacts(w, st, a, b, cfg->contact_margin, S->c + S->nc, MAXROWS - S->nc);
    if (S->nc + n > MAXROWS) return RS_FAULT_OVERFLOW << 16;
    if (!n) continue;
    for (int i = 0; i < 2; ++i) {
      int bb = i ? b : a;
      if (w->body_kind[bb] == RS_DYNAMIC && st->asleep[bb]) wake(w, st, bb, tr);
    }
    if (tr)
      for (int i = 0; i < n; ++i) {
        if (tr->n_contacts < tr->cap_contacts) {
          double *o = tr->contacts + 10 * tr->n_contacts;
          contact_t *c = &S->c[S->nc + i];
          o[0] = sub; o[1] = a; o[2] = b;
          memcpy(o + 3, c->p, 24); memcpy(o + 6, c->n, 24); o[9] = c->depth;
        }
        tr->n_contacts++;
      }
    pair_first[npc] = S->nc; pair_n[npc] = n; pa_list[npc][0] = a; pa_list[npc][1] = b;
    ++npc;
    S->nc += n;
  }
  /* _solve_contacts physics.py:846-960 */
  static velset_t vs;
  memset(&vs, 0, sizeof vs);
  int nrows = S->nc;
  for (int g = 0; g < npc; ++g) {
    int a = pa_list[g][0], b = pa_list[g][1];
    double ima, imb, Ia[9], Ib[9], ca[3], cb[3];
    body_solver_data(w, st, a, &ima, Ia, ca);
    body_solver_data(w, st, b, &imb, Ib, cb);
    double mu = sqrt(w->friction[a] * w->friction[b]);
    double e = fmax(w->restitution[a], w->restitution[b]);
    for (int i = 0; i < 2; ++i) {
      int bb = i ? b : a;
      if (!vs.have[bb]) {
        memcpy(vs.v[bb], st->lv[bb], 24); memcpy(vs.v[bb] + 3, st->av[bb], 24);
        vs.have[bb] = 1;
      }
    }
    for (int i = pair_first[g]; i < pair_first[g] + pair_n[g]; ++i) {
      contact_t *c = &S->c[i];
      row_t *r = &S->rows[i];
      memset(r, 0, sizeof *r);
      r->a = a; r->b = b;
      memcpy(r->n, c->n, 24);
      for (int k = 0; k < 3; ++k) { r->ra[k] = c->p[k] - ca[k]; r->rb[k] = c->p[k] - cb[k]; }
      double k = ima + imb, t[3], u[3], v[3];
      cross(r->ra, r->n, t); matvec(Ia, t, u); cross(u, r->ra, v); k += dot3(r->n, v);
      cross(r->rb, r->n, t); matvec(Ib, t, u); cross(u, r->rb, v); k += dot3(r->n, v);
      r->ja = joint_jacobian(w, st, a, c->p, r->jaca, &r->jia);
      r->jb = joint_jacobian(w, st, b, c->p, r->jacb, &r->jib);
      if (r->ja >= 0) { double jn = dot3(r->jaca, r->n); k += jn * jn * r->jia; }
      if (r->jb >= 0) { double jn = dot3(r->jacb, r->n); k += jn * jn * r->jib; }
      tangents(r->n, r->t1, r->t2);
      r->k = k; r->mu = mu; r->ima = ima; r->imb = imb;
      memcpy(r->Ia, Ia, 72); memcpy(r->Ib, Ib, 72);
      memcpy(r->point, c->p, 24); r->depth = c->depth;
      r->friction_on = 1;
      r->vn_pre = rel_normal_vel(r, &vs);
      double sep = -c->depth > 0.0 ? -c->depth : 0.0;
      if (sep > 0.0) {
        r->target = -sep / dt;
        r->friction_on = 0;
      } else {
        r->target = r->vn_pre < -cfg->restitution_threshold ? -e * r->vn_pre : 0.0;
      }
    }
  }
  if (nrows) {
    static double Ks[MAXPAIRS][32 * 32];
    static int hasK[MAXPAIRS];
    for (int g = 0; g < npc; ++g) {
      int m = pair_n[g];
      hasK[g] = m > 1 && S->rows[pair_first[g]].k > 0.0;
      if (hasK[g]) {
        if (m > 32) return RS_FAULT_OVERFLOW << 16;
        block_matrix(S->rows, pair_first[g], m, Ks[g]);
      }
    }
    for (int it = 0; it < cfg->solver_iterations; ++it)
      for (int g = 0; g < npc; ++g) {
#ifdef ORC_PROFILE
        g_prof_it = it; g_prof_g = g;
#endif
        if (!hasK[g])
          for (int i = pair_first[g]; i < pair_first[g] + pair_n[g]; ++i) solve_row(&S->rows[i], &vs);
        else
          solve_block(S->rows, pair_first[g], pair_n[g], Ks[g], &vs);
      }
    for (int b = 0; b < nb; ++b)
      if (vs.have[b] && solver_dynamic(w, st, b)) {
        memcpy(st->lv[b], vs.v[b], 24);
        memcpy(st->av[b], vs.v[b] + 3, 24);
      }
    for (int i = 0; i < nrows; ++i) {
      row_t *r = &S->rows[i];
      double lam = r->lam;
      if (r->k <= 0.0) lam = fmax(-r->vn_pre, 0.0);
      if (lam <= 0.0) continue;
      double force = lam / dt;
      if (tr) {
        if (tr->n_events < tr->cap_events) {
          double *o = tr->events + 7 * tr->n_events;
          o[0] = r->a; o[1] = r->b; o[2] = lam; o[3] = force; memcpy(o + 4, r->point, 24);
        }
        tr->n_events++;
      }
      if (w->body_robot[r->a] || w->body_robot[r->b] || r->a == st->held || r->b == st->held) st->acc_force += force;
    }
  }
  /* _integrate physics.py:962-1011 */
  double corr[MAXB][3];
  int ccount[MAXB];
  memset(corr, 0, sizeof corr);
  memset(ccount, 0, sizeof ccount);
  for (int g = 0; g < npc; ++g) {
    int a = pa_list[g][0], b = pa_list[g][1];
    double ima = (!st->asleep[a] && a != st->held) ? w->inv_mass[a] : 0.0;
    double imb = (!st->asleep[b] && b != st->held) ? w->inv_mass[b] : 0.0;
    double tot = ima + imb;
    if (tot <= 0.0) continue;
    for (int i = pair_first[g]; i < pair_first[g] + pair_n[g]; ++i) {
      contact_t *c = &S->c[i];
      double push = cfg->correction_factor * fmax(c->depth - cfg->slop, 0.0);
      if (push <= 0.0) continue;
      if (ima > 0.0) {
        double s = push * ima / tot;
        for (int k = 0; k < 3; ++k) corr[a][k] += c->n[k] * s;
        ccount[a]++;
      }
      if (imb > 0.0) {
        double s = push * imb / tot;
        for (int k = 0; k < 3; ++k) corr[b][k] -= c->n[k] * s;
        ccount[b]++;
      }
    }
  }
  for (int b = 0; b < nb; ++b)
    if (ccount[b] > 1) for (int k = 0; k < 3; ++k) corr[b][k] /= ccount[b];
  for (int b = 0; b < nb; ++b) {
    if (!awake_dyn[b]) continue;
    double lin = sqrt(dot3(st->lv[b], st->lv[b])), ang = sqrt(dot3(st->av[b], st->av[b]));
    int below = lin < cfg->sleep_lin_threshold && ang < cfg->sleep_ang_threshold;
    int has_corr = ccount[b] > 0 && dot3(corr[b], corr[b]) >= 1e-14;
    if (below && cfg->sleeping_enabled && !has_corr) {
      st->sleep_counter[b]++;
      if (st->sleep_counter[b] >= cfg->sleep_substeps) {
        st->asleep[b] = 1;
        memset(st->lv[b], 0, 24);
        memset(st->av[b], 0, 24);
      }
      continue;
    }
    st->sleep_counter[b] = 0;
    for (int k = 0; k < 3; ++k) st->pos[b][k] = st->pos[b][k] + st->lv[b][k] * dt;
    if (ang > 0.0) {
      /* geometry.py:110-114 */
      double wq[4] = {0.0, st->av[b][0], st->av[b][1], st->av[b][2]}, d[4], *q = st->quat[b];
      quat_mul(wq, q, d);
      double h = 0.5 * dt;
      for (int k = 0; k < 4; ++k) q[k] = q[k] + h * d[k];
      double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
      for (int k = 0; k < 4; ++k) q[k] /= n;
    }
    if (has_corr) for (int k = 0; k < 3; ++k) st->pos[b][k] += corr[b][k];
  }
  /* _advance_scene_joints physics.py:1013-1035 */
  int moved[MAXJ], nm = 0;
  for (int ji = 0; ji < nsj; ++ji) {
    if (ji == dragged) continue;
    st->jvel[ji] += vs.jdv[ji];
    st->jvel[ji] *= cfg->joint_damping;
    if (fabs(st->jvel[ji]) < 1e-4) { st->jvel[ji] = 0.0; continue; }
    double lo = w->joint_limits[2 * ji], hi = w->joint_limits[2 * ji + 1];
    double q = st->joints[ji] + st->jvel[ji] * dt;
    if (q <= lo) { q = lo; st->jvel[ji] = 0.0; }
    else if (q >= hi) { q = hi; st->jvel[ji] = 0.0; }
    if (q != st->joints[ji]) { st->joints[ji] = q; moved[nm++] = ji; }
  }
  if (nm) update_scene_joint_poses(w, st, moved, nm, dt);
  return 0;
}

static uint32_t check_finite(const orc_world *w, const ostate *st) {
  for (int b = 0; b < w->nb; ++b)
    for (int i = 0; i < 3; ++i) if (!isfinite(st->pos[b][i])) return (RS_FAULT_NONFINITE_POS << 16) | b;
  for (int b = 0; b < w->nb; ++b)
    for (int i = 0; i < 4; ++i) if (!isfinite(st->quat[b][i])) return (RS_FAULT_NONFINITE_QUAT << 16) | b;
  for (int b = 0; b < w->nb; ++b)
    for (int i = 0; i < 3; ++i) if (!isfinite(st->lv[b][i])) return (RS_FAULT_NONFINITE_VEL << 16) | b;
  for (int j = 0; j < st->nj; ++j) if (!isfinite(st->joints[j])) return (RS_FAULT_NONFINITE_JOINT << 16) | j;
  return 0;
}

/* physics.py:575-594.  Returns 0, RS_ERR_* (>0 small), or a fault word with
 * the kind in bits 16.. (also stored in *fault). */
int orc_step(const orc_world *w, const uint8_t *snap_in, uint8_t *snap_out, const double *arm, const double *basecmd,
             double dt, int substeps, orc_trace *tr, uint32_t *fault) {
  static ostate st;
  static scratch_t S;
  if (fault) *fault = 0;
  if (dt <= 0 || substeps < 1) return RS_ERR_ARG;
  int rc = unpack(snap_in, &st, w->nb, w->nsj + w->narm);
  if (rc) return rc;
  uint32_t f = check_finite(w, &st);
  if (f) { if (fault) *fault = f; return 0x7fffffff; }
  if (tr) { tr->n_pairs = tr->n_contacts = tr->n_events = 0; memset(tr->counters, 0, sizeof tr->counters); }
  double dts = dt / substeps;
  for (int i = 0; i < w->narm; ++i) S.budget[i] = w->cfg.motor_impulse_cap;
  for (int s = 0; s < substeps; ++s) {
    int r = substep(w, &st, arm, basecmd, dts, &S, tr, s);
    if (r) { if (fault) *fault = (uint32_t)r; return 0x7fffffff; }
  }
  st.time += dt;
  st.step_index += 1;
  pack(&st, snap_out);
  return 0;
}

/* ---------------------------------------------------------------- settle */

/* geometry.py:262-275 support_local / support_world */
static void support_world(const orc_world *w, int p, const pose_t *wp, const double *d, double *out) {
  double dl[3], s[3];
  mattvec(wp->R, d, dl);
  int k = w->part_kind[p];
  if (k == RS_BOX) {
    const double *h = w->part_param + 3 * p;
    for (int i = 0; i < 3; ++i) s[i] = dl[i] >= 0 ? h[i] : -h[i];
  } else if (k == RS_SPHERE) {
    double r = w->part_param[3 * p], n = sqrt(dot3(dl, dl));
    if (n == 0.0) { s[0] = r; s[1] = 0.0; s[2] = 0.0; }
    else for (int i = 0; i < 3; ++i) s[i] = (r / n) * dl[i];
  } else {
    int best = w->part_vert_begin[p];
    double bv = -INFINITY;
    for (int v = w->part_vert_begin[p]; v < w->part_vert_begin[p + 1]; ++v) {
      double x = dot3(w->vert + 3 * v, dl);
      if (x > bv) { bv = x; best = v; }  /* np.argmax: first maximum */
    }
    for (int i = 0; i < 3; ++i) s[i] = w->vert[3 * best + i];
  }
  matvec(wp->R, s, out);
  for (int i = 0; i < 3; ++i) out[i] += wp->p[i];
}

/* geometry.py:431-467 _closest_triangle over Minkowski points W[idx[0..2]];
 * writes the closest point and the reduced simplex (indices into W) */
static void closest_triangle(double W[][3], const int *idx, double *pt, int *sub, int *nsub) {
  const double *w1 = W[idx[0]], *w2 = W[idx[1]], *w3 = W[idx[2]];
  double ab[3], ac[3], ap[3], bp[3], cp[3];
  for (int i = 0; i < 3; ++i) { ab[i] = w2[i] - w1[i]; ac[i] = w3[i] - w1[i]; ap[i] = -w1[i]; }
  double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
  if (d1 <= 0 && d2 <= 0) { memcpy(pt, w1, 24); sub[0] = idx[0]; *nsub = 1; return; }
  for (int i = 0; i < 3; ++i) bp[i] = -w2[i];
  double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
  if (d3 >= 0 && d4 <= d3) { memcpy(pt, w2, 24); sub[0] = idx[1]; *nsub = 1; return; }
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) {
    double t = d1 != d3 ? d1 / (d1 - d3) : 0.0;
    for (int i = 0; i < 3; ++i) pt[i] = w1[i] + t * ab[i];
    sub[0] = idx[0]; sub[1] = idx[1]; *nsub = 2; return;
  }
  for (int i = 0; i < 3; ++i) cp[i] = -w3[i];
  double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
  if (d6 >= 0 && d5 <= d6) { memcpy(pt, w3, 24); sub[0] = idx[2]; *nsub = 1; return; }
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) {
    double t = d2 != d6 ? d2 / (d2 - d6) : 0.0;
    for (int i = 0; i < 3; ++i) pt[i] = w1[i] + t * ac[i];
    sub[0] = idx[0]; sub[1] = idx[2]; *nsub = 2; return;
  }
  double va = d3 * d6 - d5 * d4;
  if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0) {
    double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    for (int i = 0; i < 3; ++i) pt[i] = w2[i] + t * (w3[i] - w2[i]);
    sub[0] = idx[1]; sub[1] = idx[2]; *nsub = 2; return;
  }
  double denom = va + vb + vc, v = vb / denom, ww = vc / denom;
  for (int i = 0; i < 3; ++i) pt[i] = w1[i] + ab[i] * v + ac[i] * ww;
  sub[0] = idx[0]; sub[1] = idx[1]; sub[2] = idx[2]; *nsub = 3;
}

/* geometry.py:383-428 _closest_simplex; simplex = W[0..n-1], reduced in place.
 * Returns 1 when a tetrahedron contains the origin. */
static int closest_simplex(double W[4][3], int *n, double *pt) {
  int sub[4], ns = 0;
  if (*n == 1) { memcpy(pt, W[0], 24); return 0; }
  if (*n == 2) {
    double d[3];
    for (int i = 0; i < 3; ++i) d[i] = W[1][i] - W[0][i];
    double dd = dot3(d, d), t = dd == 0.0 ? 0.0 : -dot3(W[0], d) / dd;
    if (t <= 0.0) { memcpy(pt, W[0], 24); *n = 1; return 0; }
    if (t >= 1.0) { memcpy(pt, W[1], 24); memcpy(W[0], W[1], 24); *n = 1; return 0; }
    for (int i = 0; i < 3; ++i) pt[i] = W[0][i] + t * d[i];
    return 0;
  }
  if (*n == 3) {
    int idx[3] = {0, 1, 2};
    closest_triangle(W, idx, pt, sub, &ns);
  } else {
    static const int faces[4][4] = {{0, 1, 2, 3}, {0, 1, 3, 2}, {0, 2, 3, 1}, {1, 2, 3, 0}};
    int contained = 1, have = 0;
    double bd2 = 0.0;
    for (int f = 0; f < 4; ++f) {
      const double *a = W[faces[f][0]], *b = W[faces[f][1]], *c = W[faces[f][2]], *o = W[faces[f][3]];
      double ba[3], ca[3], nrm[3], ma[3], oa[3];
      for (int i = 0; i < 3; ++i) { ba[i] = b[i] - a[i]; ca[i] = c[i] - a[i]; ma[i] = -a[i]; oa[i] = o[i] - a[i]; }
      cross(ba, ca, nrm);
      double side_origin = dot3(nrm, ma), side_opp = dot3(nrm, oa);
      if (side_origin * side_opp > 0) continue;
      contained = 0;
      double p2[3];
      int s2[4], n2 = 0;
      closest_triangle(W, faces[f], p2, s2, &n2);
      double d2 = dot3(p2, p2);
      if (!have || d2 < bd2) { have = 1; bd2 = d2; memcpy(pt, p2, 24); memcpy(sub, s2, sizeof s2); ns = n2; }
    }
    if (contained) { pt[0] = pt[1] = pt[2] = 0.0; return 1; }
  }
  double T[4][3];
  for (int k = 0; k < ns; ++k) memcpy(T[k], W[sub[k]], 24);
  for (int k = 0; k < ns; ++k) memcpy(W[k], T[k], 24);
  *n = ns;
  return 0;
}

/* geometry.py:486-525 gjk_distance (distance only; witnesses unused by settle) */
static double gjk_distance(const orc_world *w, int pa, const pose_t *wa, int pb, const pose_t *wb) {
  const double tol = 1e-10;
  double d[3], nd[3], sa[3], sb[3], W[4][3], pt[3];
  for (int i = 0; i < 3; ++i) d[i] = wb->p[i] - wa->p[i];
  if (dot3(d, d) == 0.0) { d[0] = 1.0; d[1] = 0.0; d[2] = 0.0; }
  for (int i = 0; i < 3; ++i) nd[i] = -d[i];
  support_world(w, pa, wa, d, sa);
  support_world(w, pb, wb, nd, sb);
  int n = 1;
  for (int i = 0; i < 3; ++i) { W[0][i] = sa[i] - sb[i]; pt[i] = W[0][i]; }
  double last_d2 = INFINITY;
  for (int it = 0; it < 64; ++it) {
    int contains = closest_simplex(W, &n, pt);
    double d2 = dot3(pt, pt);
    if (contains || d2 < tol) return 0.0;
    if (isfinite(last_d2) && last_d2 - d2 <= tol * fmax(1.0, last_d2)) break;
    last_d2 = d2;
    for (int i = 0; i < 3; ++i) { d[i] = -pt[i]; nd[i] = pt[i]; }
    support_world(w, pa, wa, d, sa);
    support_world(w, pb, wb, nd, sb);
    double wv[3];
    for (int i = 0; i < 3; ++i) wv[i] = sa[i] - sb[i];
    if (dot3(wv, d) - dot3(pt, d) <= tol * fmax(1.0, sqrt(d2))) break;
    memcpy(W[n++], wv, 24);
  }
  return sqrt(dot3(pt, pt));
}

/* geometry.py:528-539 parts_distance */
static double parts_distance(const orc_world *w, const ostate *st, int a, int b) {
  pose_t pa, pb, wa, wb;
  body_pose(st, a, &pa);
  body_pose(st, b, &pb);
  double best = INFINITY;
  for (int i = w->body_part_begin[a]; i < w->body_part_begin[a + 1]; ++i) {
    part_world(w, &pa, i, &wa);
    for (int j = w->body_part_begin[b]; j < w->body_part_begin[b + 1]; ++j) {
      part_world(w, &pb, j, &wb);
      double d = gjk_distance(w, i, &wa, j, &wb);
      if (d < best) best = d;
      if (best == 0.0) return 0.0;
    }
  }
  return best;
}

/* physics.py:1156-1176 _assert_spawn_clearance over the placed bodies
 * (ascending id).  Returns 1 and the first (body, other, clearance) whose
 * clearance is below 1 mm, else 0. */
static int spawn_clearance(const orc_world *w, const ostate *st, uint64_t placed, int *fb, int *fo, double *fd) {
  const double margin = 1e-3;
  for (int b = 0; b < w->nb; ++b) {
    if (!((placed >> b) & 1ull)) continue;
    double la[3], ha[3];
    body_aabb(w, st, b, la, ha);
    for (int o = 0; o < w->nb; ++o) {
      if (o == b || w->body_robot[o]) continue;
      if (st->pos[o][2] > 40.0 / 2) continue; /* parked, not yet placed (PARK_Z / 2) */
      double lb[3], hb[3];
      body_aabb(w, st, o, lb, hb);
      int ov = 1;
      for (int i = 0; i < 3; ++i) ov &= (la[i] - margin <= hb[i]) && (lb[i] - margin <= ha[i]);
      if (!ov) continue;
      double d = parts_distance(w, st, b, o);
      if (d < margin) { *fb = b; *fo = o; *fd = d; return 1; }
    }
  }
  return 0;
}
int orc_spawn_clearance(const orc_world *w, const uint8_t *snap, uint64_t placed, int *body, int *other,
                        double *dist) {
  static ostate st;
  int rc = unpack(snap, &st, w->nb, w->nsj + w->narm);
  if (rc) return -rc;
  return spawn_clearance(w, &st, placed, body, other, dist);
}
double orc_parts_distance(const orc_world *w, const uint8_t *snap, int a, int b) {
  static ostate st;
  if (unpack(snap, &st, w->nb, w->nsj + w->narm)) return NAN;
  return parts_distance(w, &st, a, b);
}

/* physics.py:1113-1154 settle from a spawn state (placements already
 * applied): clearance check, then control steps without targets until every
 * placed body sleeps.  status: 0 settled after *steps, 1 clearance (info =
 * body, other; *value = clearance), 2 a placed body fell below floor_z - 0.5
 * (info[0] = body), 3 still awake after max_steps, 4 physics fault. */
int orc_settle(const orc_world *w, const uint8_t *spawn, uint64_t placed, int max_steps, double floor_z,
               uint8_t *snap_out, int *info, double *value, int *steps) {
  size_t sz = (size_t)orc_snapshot_size(w->nb, w->nsj + w->narm);
  uint8_t *cur = (uint8_t *)malloc(sz), *nxt = (uint8_t *)malloc(sz);
  memcpy(cur, spawn, sz);
  static ostate st;
  int status = 3;
  *steps = 0;
  info[0] = info[1] = -1;
  *value = 0.0;
  unpack(cur, &st, w->nb, w->nsj + w->narm);
  if (spawn_clearance(w, &st, placed, &info[0], &info[1], value)) {
    status = 1;
  } else {
    for (int k = 0; k < max_steps; ++k) {
      uint32_t fault = 0;
      int rc = orc_step(w, cur, nxt, NULL, NULL, 1.0 / 30.0, 4, NULL, &fault);
      if (rc) { status = 4; info[0] = (int)fault; break; }
      memcpy(cur, nxt, sz);
      *steps = k + 1;
      unpack(cur, &st, w->nb, w->nsj + w->narm);
      int fell = -1, awake = 0;
      for (int b = 0; b < w->nb; ++b) {
        if (!((placed >> b) & 1ull)) continue;
        if (fell < 0 && st.pos[b][2] < floor_z - 0.5) fell = b;
        awake |= !st.asleep[b];
      }
      if (fell >= 0) { status = 2; info[0] = fell; break; }
      if (!awake) { status = 0; break; }
    }
  }
  memcpy(snap_out, cur, sz);
  free(cur);
  free(nxt);
  return status;
}

/* forward kinematics through the oracle (tests) */
void orc_link_poses(const orc_world *w, const double *q, const double *base, double *links12, double *ee12) {
  pose_t l[16], e;
  link_poses(w, q, base, l, &e);
  for (int i = 0; i < w->narm; ++i) { memcpy(links12 + 12 * i, l[i].R, 72); memcpy(links12 + 12 * i + 9, l[i].p, 24); }
  memcpy(ee12, e.R, 72); memcpy(ee12 + 9, e.p, 24);
}

/* ---------------------------------------------------------------- render */

/* geometry.py:734-746 for one ray; returns t (INFINITY on miss) and the
 * entering-plane index (-1 when the origin is inside) */
static double ray_convex(const double *nw, const double *dw, int nf, const double *o, const double *d, int *enter_face) {
  double te = -INFINITY, tx = INFINITY;
  int bad = 0, fe = -1;
  for (int f = 0; f < nf; ++f) {
    double s = dot3(d, nw + 3 * f), bb = dw[f] - dot3(o, nw + 3 * f);
    if (s < -1e-12) {
      double r = bb / s;
      if (fe < 0 || r > te) { te = r; fe = f; }
    } else if (s > 1e-12) {
      double r = bb / s;
      if (r < tx) tx = r;
    } else if (bb < 0) {
      bad = 1;
    }
  }
  int hit = te <= tx && tx >= 0.0 && !bad;
  if (!hit) { *enter_face = -1; return INFINITY; }
  if (te >= 0.0) { *enter_face = fe; return te; }
  *enter_face = -1;
  return 0.0;
}
/* geometry.py:749-759 */
static double ray_sphere(const double *c, double r, const double *o, const double *d) {
  double oc[3] = {o[0] - c[0], o[1] - c[1], o[2] - c[2]};
  double b = dot3(oc, d), cc = dot3(oc, oc) - r * r, disc = b * b - cc;
  if (!(disc >= 0)) return INFINITY;
  double sq = sqrt(disc), t0 = -b - sq, t1 = -b + sq;
  return t0 >= 0.0 ? t0 : (t1 >= 0.0 ? 0.0 : INFINITY);
}

void orc_camera_pose(const orc_world *w, const uint8_t *snap, int cam, double *pose12_out) {
  static ostate st;
  unpack(snap, &st, w->nb, w->nsj + w->narm);
  pose_t parent, mount, cp;
  if (w->cam_parent[cam] == 0) base3(st.base, &parent);
  else ee_pose(w, &st, &parent);
  pose12(w->cam_mount + 12 * cam, &mount);
  compose(&parent, &mount, &cp);
  memcpy(pose12_out, cp.R, 72);
  memcpy(pose12_out + 9, cp.p, 24);
}

/* physics.py:1088-1101 Simulator.sphere_cast: nearest proxy hit along a unit
 * ray, bodies in id order, t_b = min over parts of the reference ray
 * primitive, kept if t_b <= max_dist and finite, strict < (lowest id wins
 * ties).  Returns the body id (-1: none; -2: direction not unit length,
 * PhysicsFault) and *t_out. */
int orc_sphere_cast(const orc_world *w, const uint8_t *snap, const double *o, const double *d, double max_dist,
                    double *t_out) {
  static ostate st;
  if (unpack(snap, &st, w->nb, w->nsj + w->narm)) return -3;
  if (fabs(sqrt(dot3(d, d)) - 1.0) > 1e-6) return -2;
  int best = -1;
  double bt = INFINITY;
  double nw[3 * 64], dw[64];
  for (int b = 0; b < w->nb; ++b) {
    pose_t bp, wp;
    body_pose(&st, b, &bp);
    double tb = INFINITY;
    for (int p = w->body_part_begin[b]; p < w->body_part_begin[b + 1]; ++p) {
      part_world(w, &bp, p, &wp);
      double t;
      if (w->part_kind[p] == RS_SPHERE) {
        t = ray_sphere(wp.p, w->part_param[3 * p], o, d);
      } else {
        int f0 = w->part_facet_begin[p], nf = w->part_facet_begin[p + 1] - f0, fe;
        planes_world(w, p, &wp, nw, dw);
        t = ray_convex(nw, dw, nf, o, d, &fe);
      }
      if (t < tb) tb = t;
    }
    if (tb <= max_dist && isfinite(tb) && (best < 0 || tb < bt)) { best = b; bt = tb; }
  }
  *t_out = bt;
  return best;
}

/* Render restatement (pinned in DESIGN.md §5):
 * ray through pixel centre (u+.5, v+.5), camera frame (right, down, view),
 * normalised then rotated to world; per body t_b = min over parts of the
 * reference ray primitive; t* = min_b t_b; id = lowest b with
 * t_b <= t* + tie_eps; t* > far or miss -> depth 0, id -1, rgba 0;
 * else depth = max(t*, near); rgb = colour * (0.3 + 0.7 max(0, -n.d)). */
int orc_render(const orc_world *w, const uint8_t *snap, int cam, const rs_render_config *rc, uint8_t *rgba,
               float *depth, int32_t *ids, double *t_out) {
  static ostate st;
  int r = unpack(snap, &st, w->nb, w->nsj + w->narm);
  if (r) return r;
  double cp[12];
  orc_camera_pose(w, snap, cam, cp);
  pose_t camp;
  pose12(cp, &camp);
  /* world planes of every convex part, sphere centres */
  int np = w->np;
  double *nw = (double *)malloc(sizeof(double) * 3 * (w->nf + 1));
  double *dw = (double *)malloc(sizeof(double) * (w->nf + 1));
  double *sc = (double *)malloc(sizeof(double) * 3 * np);
  for (int b = 0; b < w->nb; ++b) {
    pose_t bp, wp;
    body_pose(&st, b, &bp);
    for (int p = w->body_part_begin[b]; p < w->body_part_begin[b + 1]; ++p) {
      part_world(w, &bp, p, &wp);
      memcpy(sc + 3 * p, wp.p, 24);
      int f0 = w->part_facet_begin[p];
      if (w->part_kind[p] != RS_SPHERE) planes_world(w, p, &wp, nw + 3 * f0, dw + f0);
    }
  }
  int W = rc->width, H = rc->height;
  double f = (W / 2.0) / tan(rc->fov / 2.0);
  double tb[MAXB];
  int fb[MAXB], pbest[MAXB];
  for (int v = 0; v < H; ++v)
    for (int u = 0; u < W; ++u) {
      double dc[3] = {(u + 0.5 - W / 2.0) / f, (v + 0.5 - H / 2.0) / f, 1.0};
      double l = sqrt(dot3(dc, dc));
      for (int i = 0; i < 3; ++i) dc[i] /= l;
      double d[3];
      matvec(camp.R, dc, d);
      const double *o = camp.p;
      double tmin = INFINITY;
      for (int b = 0; b < w->nb; ++b) {
        tb[b] = INFINITY; fb[b] = -1; pbest[b] = -1;
        for (int p = w->body_part_begin[b]; p < w->body_part_begin[b + 1]; ++p) {
          double t;
          int fe = -1;
          if (w->part_kind[p] == RS_SPHERE) t = ray_sphere(sc + 3 * p, w->part_param[3 * p], o, d);
          else {
            int f0 = w->part_facet_begin[p];
            t = ray_convex(nw + 3 * f0, dw + f0, w->part_facet_begin[p + 1] - f0, o, d, &fe);
            if (fe >= 0) fe += f0;
          }
          if (t < tb[b]) { tb[b] = t; fb[b] = fe; pbest[b] = p; }
        }
        if (tb[b] < tmin) tmin = tb[b];
      }
      int idx = v * W + u, id = -1;
      if (isfinite(tmin) && tmin <= rc->zfar) {
        for (int b = 0; b < w->nb; ++b) if (tb[b] <= tmin + rc->tie_eps) { id = b; break; }
      }
      if (t_out) t_out[idx] = tmin;
      if (id < 0) {
        if (depth) depth[idx] = 0.0f;
        if (ids) ids[idx] = -1;
        if (rgba) memset(rgba + 4 * idx, 0, 4);
        continue;
      }
      if (depth) depth[idx] = (float)(tmin < rc->znear ? rc->znear : tmin);
      if (ids) ids[idx] = id;
      if (rgba) {
        double cosv = 0.0;
        int p = pbest[id];
        if (w->part_kind[p] == RS_SPHERE) {
          double t = tb[id];
          if (t > 0.0) {
            double n[3];
            for (int i = 0; i < 3; ++i) n[i] = (o[i] + t * d[i] - sc[3 * p + i]) / w->part_param[3 * p];
            cosv = -dot3(n, d);
          }
        } else if (fb[id] >= 0) {
          cosv = -dot3(nw + 3 * fb[id], d);
        }
        float shade = 0.3f + 0.7f * (float)(cosv > 0.0 ? cosv : 0.0);
        for (int i = 0; i < 3; ++i) {
          float c = 255.0f * w->color[3 * id + i] * shade + 0.5f;
          rgba[4 * idx + i] = (uint8_t)(c > 255.0f ? 255.0f : c);
        }
        rgba[4 * idx + 3] = 255;
      }
    }
  free(nw); free(dw); free(sc);
  return 0;
}

/* ------------------------------------------------------------------ IK */

/* LAPACK dgesv-style solve (partial pivoting, first max) of the 3x3 system
 * A X = B with nrhs columns (B row-major [3][nrhs]); np.linalg.solve. */
static void solve3(const double *A_in, double *B, int nrhs) {
  double A[9];
  int piv[3];
  memcpy(A, A_in, sizeof A);
  for (int j = 0; j < 3; ++j) {
    int p = j;
    for (int i = j + 1; i < 3; ++i) if (fabs(A[3 * i + j]) > fabs(A[3 * p + j])) p = i;
    piv[j] = p;
    if (p != j) for (int k = 0; k < 3; ++k) { double t = A[3 * j + k]; A[3 * j + k] = A[3 * p + k]; A[3 * p + k] = t; }
    double r = 1.0 / A[3 * j + j];
    for (int i = j + 1; i < 3; ++i) A[3 * i + j] *= r;
    for (int i = j + 1; i < 3; ++i)
      for (int k = j + 1; k < 3; ++k) A[3 * i + k] -= A[3 * i + j] * A[3 * j + k];
  }
  for (int c = 0; c < nrhs; ++c) {
    double x[3];
    for (int i = 0; i < 3; ++i) x[i] = B[i * nrhs + c];
    for (int j = 0; j < 3; ++j) if (piv[j] != j) { double t = x[j]; x[j] = x[piv[j]]; x[piv[j]] = t; }
    for (int i = 1; i < 3; ++i) for (int k = 0; k < i; ++k) x[i] -= A[3 * i + k] * x[k];
    for (int i = 2; i >= 0; --i) {
      for (int k = i + 1; k < 3; ++k) x[i] -= A[3 * i + k] * x[k];
      x[i] /= A[3 * i + i];
    }
    for (int i = 0; i < 3; ++i) B[i * nrhs + c] = x[i];
  }
}

/* robot.py:199-221 one damped-least-squares attempt; returns 1 on success */
static int dls_attempt(const orc_world *w, const double *target, const double *seed, double *q_out) {
  const int n = w->narm;
  const double tol = 5e-3, lam2 = 0.05 * 0.05, zero3[3] = {0, 0, 0};
  double q[16], lo[16], hi[16], mid[16];
  for (int i = 0; i < n; ++i) {
    lo[i] = w->arm_limits[2 * i]; hi[i] = w->arm_limits[2 * i + 1];
    mid[i] = 0.5 * (lo[i] + hi[i]);
    q[i] = seed[i] < lo[i] ? lo[i] : (seed[i] > hi[i] ? hi[i] : seed[i]);
  }
  pose_t links[16], ee;
  for (int it = 0; it <= 100; ++it) {
    link_poses(w, q, zero3, links, &ee);
    double err[3] = {target[0] - ee.p[0], target[1] - ee.p[1], target[2] - ee.p[2]};
    if (sqrt(dot3(err, err)) < tol) { memcpy(q_out, q, 8 * n); return 1; }
    if (it == 100) break;
    double J[3 * 16], JT_sol[3 * 16], jjt[9];
    for (int i = 0; i < n; ++i) {
      double ax[3], d[3], c[3];
      matvec(links[i].R, w->arm_axis + 3 * i, ax);
      for (int k = 0; k < 3; ++k) d[k] = ee.p[k] - links[i].p[k];
      cross(ax, d, c);
      for (int k = 0; k < 3; ++k) J[k * n + i] = c[k];
    }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += J[a * n + i] * J[b * n + i];
        jjt[3 * a + b] = s + (a == b ? lam2 : 0.0);
      }
    double y[3] = {err[0], err[1], err[2]};
    solve3(jjt, y, 1);
    memcpy(JT_sol, J, sizeof(double) * 3 * n);
    solve3(jjt, JT_sol, n);  /* solve(jjt, J): [3][n] */
    double dq[16], r[16];
    for (int i = 0; i < n; ++i) dq[i] = J[0 * n + i] * y[0] + J[1 * n + i] * y[1] + J[2 * n + i] * y[2];
    for (int i = 0; i < n; ++i) r[i] = mid[i] - q[i];
    for (int i = 0; i < n; ++i) {
      /* (I - J^T solve(jjt, J)) (mid - q), row i */
      double s = 0.0;
      for (int j = 0; j < n; ++j) {
        double pij = J[0 * n + i] * JT_sol[0 * n + j] + J[1 * n + i] * JT_sol[1 * n + j] + J[2 * n + i] * JT_sol[2 * n + j];
        s += ((i == j ? 1.0 : 0.0) - pij) * r[j];
      }
      dq[i] += 0.1 * s;
    }
    double step = 0.0;
    for (int i = 0; i < n; ++i) step += dq[i] * dq[i];
    step = sqrt(step);
    if (step > 0.5) for (int i = 0; i < n; ++i) dq[i] *= 0.5 / step;
    for (int i = 0; i < n; ++i) {
      double v = q[i] + dq[i];
      q[i] = v < lo[i] ? lo[i] : (v > hi[i] ? hi[i] : v);
    }
  }
  return 0;
}

static const double RESTART[11][7] = {
    {0.0, 0.25, 0.0, -0.35, 0.0, 0.3, 0.0},       {0.3, -0.2, 0.2, 0.3, -0.2, -0.3, 0.2},
    {-0.3, 0.3, -0.25, -0.3, 0.25, 0.35, -0.2},   {0.15, 0.4, 0.3, 0.4, 0.3, -0.4, 0.3},
    {-0.15, -0.35, -0.3, 0.45, -0.35, 0.4, -0.3}, {0.45, 0.1, 0.45, -0.45, 0.4, -0.1, 0.45},
    {-0.45, -0.1, -0.45, 0.2, 0.45, 0.15, -0.45}, {0.6, 0.85, -0.8, -0.2, 0.7, 0.0, -0.3},
    {-0.6, 0.85, 0.8, -0.2, -0.7, 0.0, 0.3},      {0.85, 0.9, -0.55, 0.3, 0.75, -0.25, 0.0},
    {-0.85, 0.9, 0.55, 0.3, -0.75, 0.25, 0.0}};
static const double WEYL[7] = {0.618034, 0.754878, 0.569840, 0.380110, 0.245122, 0.119409, 0.059683};

/* robot.py:240-279 solve_ik; returns the attempt index that succeeded
 * (0 = seed, 1..11 restarts, 12..35 Weyl spray) or -1 (NoSolution). */
int orc_solve_ik(const orc_world *w, const double *target, const double *seed, double *q_out) {
  const int n = w->narm;
  /* reach check: shoulder = joint 0 offset; max reach = sum |offset_1..| + |gripper| */
  double reach = 0.0;
  for (int i = 1; i < n; ++i) reach += sqrt(dot3(w->arm_offset + 3 * i, w->arm_offset + 3 * i));
  reach += sqrt(dot3(w->gripper, w->gripper));
  double d[3] = {target[0] - w->arm_offset[0], target[1] - w->arm_offset[1], target[2] - w->arm_offset[2]};
  if (sqrt(dot3(d, d)) > reach + 5e-3) return -1;
  if (dls_attempt(w, target, seed, q_out)) return 0;
  double lo[16], hi[16], mid[16], span[16], s[16];
  for (int i = 0; i < n; ++i) {
    lo[i] = w->arm_limits[2 * i]; hi[i] = w->arm_limits[2 * i + 1];
    mid[i] = 0.5 * (lo[i] + hi[i]); span[i] = hi[i] - lo[i];
  }
  for (int r = 0; r < 11; ++r) {
    for (int i = 0; i < n; ++i) s[i] = mid[i] + RESTART[r][i] * span[i] * 0.5;
    if (dls_attempt(w, target, s, q_out)) return 1 + r;
  }
  double u[16];
  for (int i = 0; i < n; ++i) u[i] = 0.5;
  for (int r = 0; r < 24; ++r) {
    for (int i = 0; i < n; ++i) { u[i] = fmod(u[i] + WEYL[i], 1.0); s[i] = lo[i] + u[i] * span[i]; }
    if (dls_attempt(w, target, s, q_out)) return 12 + r;
  }
  return -1;
}

/* robot.py:293-313 apply_arm_action: clamp, FK (base frame), IK; on failure
 * the targets are the current joints.  Returns 1 on IK failure. */
int orc_apply_arm_action(const orc_world *w, const double *q, const double *delta, double *targets) {
  const int n = w->narm;
  double dl[3] = {delta[0], delta[1], delta[2]};
  double nd = sqrt(dot3(dl, dl));
  if (nd > 0.015) for (int k = 0; k < 3; ++k) dl[k] = dl[k] * (0.015 / nd);
  const double zero3[3] = {0, 0, 0};
  pose_t ee;
  link_poses(w, q, zero3, NULL, &ee);
  double target[3] = {ee.p[0] + dl[0], ee.p[1] + dl[1], ee.p[2] + dl[2]};
  if (orc_solve_ik(w, target, q, targets) >= 0) return 0;
  memcpy(targets, q, 8 * n);
  return 1;
}

/* ------------------------------------------------------------------ grasp
 * The env pipeline's grasp phase between control steps: robot.py:323-346
 * grasp_rule over physics.py:1039-1053 grasp_candidates, then
 * physics.py:1055-1079 apply_grasp.  holding = state.held >= 0 (an object or
 * a handle).  out[4] = (kind 0 none / 1 snap / 2 release, body, scene-joint
 * index of a handle snap or -1, wakes counted by Simulator.wake). */
int orc_grasp(const orc_world *w, const uint8_t *snap_in, double gripper, uint8_t *snap_out, int32_t *out) {
  static ostate st;
  int r = unpack(snap_in, &st, w->nb, w->nsj + w->narm);
  if (r) return r;
  out[0] = 0; out[1] = -1; out[2] = -1; out[3] = 0;
  const int holding = st.held >= 0;
  if (gripper > 0 && !holding) {
    pose_t ee;
    ee_pose(w, &st, &ee);
    double best_d = 0.0;
    int best_b = -1, best_j = -1;
    /* candidates: clutter COMs (id order, the held body skipped), then handles */
    for (int c = 0; c < w->nclutter; ++c) {
      int b = w->clutter[c];
      if (b == st.held) continue;
      pose_t bp;
      double com[3], e[3];
      body_pose(&st, b, &bp);
      apply(&bp, w->com + 3 * b, com);
      for (int i = 0; i < 3; ++i) e[i] = ee.p[i] - com[i];
      double d = sqrt(dot3(e, e));
      /* near.sort(key=(d, body)); near[0] */
      if (d <= 0.15 && (best_b < 0 || d < best_d || (d == best_d && b < best_b))) { best_d = d; best_b = b; best_j = -1; }
    }
    for (int ji = 0; ji < w->nsj; ++ji) {
      pose_t child;
      double h[3], e[3];
      joint_child_pose(w, &st, ji, st.joints[ji], &child);  /* scene.py:439-440 handle_world */
      apply(&child, w->joint_handle + 3 * ji, h);
      for (int i = 0; i < 3; ++i) e[i] = ee.p[i] - h[i];
      double d = sqrt(dot3(e, e));
      int b = w->joint_body[ji];
      if (d <= 0.15 && (best_b < 0 || d < best_d || (d == best_d && b < best_b))) { best_d = d; best_b = b; best_j = ji; }
    }
    if (best_b >= 0) {
      out[0] = 1; out[1] = best_b; out[2] = best_j;
      if (best_j >= 0) {
        st.held_joint = best_j;
        st.held = best_b;
        st.grab_q = st.joints[best_j];
        memcpy(st.grab_ee, ee.p, 24);
      } else {
        orc_trace tr;
        memset(&tr, 0, sizeof tr);
        wake(w, &st, best_b, &tr);
        out[3] = (int32_t)tr.counters[2];
        pose_t inv, bp, rel;
        inverse(&ee, &inv);
        body_pose(&st, best_b, &bp);
        compose(&inv, &bp, &rel);
        st.held = best_b;
        memcpy(st.held_offset, rel.p, 24);
        mat_to_quat(rel.R, st.held_offset + 3);
        memset(st.lv[best_b], 0, 24);
        memset(st.av[best_b], 0, 24);
      }
    }
  } else if (gripper < 0 && holding) {
    out[0] = 2;
    if (st.held >= 0 && st.held_joint < 0) {
      st.asleep[st.held] = 0;
      st.sleep_counter[st.held] = 0;
    }
    st.held = -1;
    st.held_joint = -1;
  }
  pack(&st, snap_out);
  return 0;
}
