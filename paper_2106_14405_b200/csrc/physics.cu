// physics.cu -- fused 1/30 s control step (all substeps) for a batch of envs.
//
// One warp owns one environment for the whole control step: it stages the
// env's state slab into shared memory, runs every substep of
// Simulator.step_physics (physics.py:575-1035) there, and writes the slab
// back once.  Work inside a substep is spread over the warp's lanes where
// the reference's semantics allow it and kept on one lane where they are
// order-dependent:
//
//   kinematics      lanes per joint/body; FK chain on lane 0 (robot.py:161)
//   AABBs           lanes per body (geometry.py:278-296)
//   overlap tests   lanes per pair, ballot-compacted in sorted (a, b) order
//                   (== SAP on x + inclusive y/z, physics.py:498-526)
//   admission       lane 0, sorted order (wakes mutate `asleep` mid-walk,
//                   physics.py:528-571)
//   narrowphase     lanes per vertex / facet, ballot-compacted in vertex
//                   order (geometry.py:564-576, :667-716)
//   row build       lanes per contact; block matrices lanes per entry
//   GS sweeps       lane 0 (Gauss-Seidel order is the algorithm,
//                   physics.py:915-937); block LCP with a Jacobi
//                   pseudo-inverse matching lstsq(rcond=1e-8) (:760-816)
//   integrate       lanes per body; per-body correction sums in contact
//                   order (physics.py:962-1011)
//
// Float64 throughout, every sum and product in the oracle's order; the unit is
// built with FMA contraction, so continuous values may differ from the scalar
// C oracle in the last bits (states within 1e-12) while every discrete output
// (pair lists, contact counts, sleep flags, counters) stays bit-exact against
// the oracle and the reference goldens (tests/test_gpu*.py).
#include <cuda_runtime.h>

#include <cub/block/block_scan.cuh>

#include <atomic>
#include <cmath>
#include <cstdint>

#include "device.cuh"
#include "navgrid.cuh"
#include "se3.cuh"

namespace rsim {

// envs (warps) per step_kernel CTA.  One: a CTA lives only as long as its env,
// and with <= 16.5 KB of shared memory per warp three of them fit the slot a
// finished render CTA frees (16 K registers, 53.7 KB) in the interleaved step
// (measured, 2048 envs: 1 env/CTA at 16.6 KB +1.7 % bench, +5 % Interact over
// 2 envs/CTA at 19.7 KB; 3 envs/CTA at 19.7 KB -2 %)
#ifndef RSIM_WARPS_PER_BLOCK
#define RSIM_WARPS_PER_BLOCK 1
#endif
constexpr int kWarpsPerBlock = RSIM_WARPS_PER_BLOCK;
constexpr int kStepMinBlocks = kWarpsPerBlock == 1 ? 10 : (kWarpsPerBlock == 2 ? 5 : (kWarpsPerBlock == 3 ? 4 : 3));
constexpr int kMaxCand = 1024;
constexpr int kMaxAdm = 256;
constexpr int kMaxContacts = 512;  // rows per substep (HBM scratch); 2.8x the 26-object pile's 185
constexpr int kMaxGroups = 96;
constexpr int kMaxBlockRows = 32;
constexpr int kRowD = 44;  // doubles per solver row in global scratch
constexpr int kEigSlots = 16;  // cached eigendecompositions per block (LRU over active sets)
constexpr int kPairD = 31 + 2 * kEigSlots;  // doubles per contact group (pair) in global scratch
constexpr int kKCap = 8192;  // Sigma m^2 of the block matrices of one substep (<= 32 * 256)
constexpr int kMaxPartsCache = 128;
constexpr int kStageD = 13 * kMaxBodies + 2 * kMaxJoints + 16;  // most doubles of a staged slab (StateLayout::stage)

// ---- row field offsets (doubles) ------------------------------------------
enum {
  RN = 0, RT1 = 3, RT2 = 6, RRA = 9, RRB = 12, RK = 15, RMU = 16, RIMA = 17, RIMB = 18, RJACA = 19, RJACB = 22,
  RJIA = 25, RJIB = 26, RLAM = 27, RLT1 = 28, RLT2 = 29, RVN = 30, RTGT = 31, RFRIC = 32, RJA = 33, RJB = 34,
  RA = 35, RB = 36, RPT = 37, RDEPTH = 40, RGRP = 41
};
// ---- pair (group) field offsets --------------------------------------------
// PMASK + s: active set cached in slot s (-1: empty); PSTAMP + s: its last use (PCLK ticks)
enum { PIA = 0, PIB = 9, PCA = 18, PCB = 21, PIMA = 24, PIMB = 25, PMU = 26, PE = 27, PKOFF = 28, PHASK = 29,
       PCLK = 30, PMASK = 31, PSTAMP = 31 + kEigSlots };

// block workspace in shared memory (per warp), m <= kMaxBlockRows
constexpr int kSmemEig = 12;  // eigensolver matrices live in shared memory up to this size
struct BlockWS {
  double cur[kMaxBlockRows], q[kMaxBlockRows], lam[kMaxBlockRows], wv[kMaxBlockRows], rhs[kMaxBlockRows],
      ck[kMaxBlockRows];
  double cs[kMaxBlockRows], sn[kMaxBlockRows];  // rotations (m/2) / row-norm scratch (m)
  int pp[kMaxBlockRows / 2], qq[kMaxBlockRows / 2];
  union {
    struct { double A[kSmemEig * kSmemEig], V[kSmemEig * kSmemEig]; };
    double F[2 * kSmemEig * kSmemEig];  // block_impulse_friction staging (after the LCP)
  };
  int active[kMaxBlockRows];
  int na, converged, slot;
};

struct WarpSmem {
  int32_t si[3 * kMaxBodies + 4];  // asleep, sleep counters, rider joints, held, held joint
  // phase-scoped scratch: FK chain | broadphase AABBs + candidate pairs |
  // narrowphase planes | solver velocities (nothing in it outlives its phase)
  union {
    struct {
      double raa[kMaxArm][9];       // arm joint rotations
      double aoff[kMaxArm + 1][3];  // link offsets, then the gripper offset (staged by lanes)
      double links[kMaxArm][12];    // link poses (R, p), read by the kinematic update
      double ee[12];                // end-effector pose, read by the drag / held follow
    } fk;  // written by forward_kinematics, read before the broadphase
    struct {
      double lo[kMaxBodies][3], hi[kMaxBodies][3];
      uint16_t cand[kMaxCand];  // candidate pairs (a << 8 | b), sorted; read by the admission walk
    } bp;
    struct {
      double planes[2][kMaxFacetsPerPart * 4];
      int off[kMaxAdm];  // first part-pair index of each admitted pair
      int npc[kMaxAdm];  // contacts of each admitted pair
    } np;
    struct { double vel[kMaxBodies][6]; BlockWS ws; } sol;
  } u;
  DevScene sc;  // this env's scene table header (pointers), staged from global
  double jdv[kMaxJoints];
  double budget[kMaxArm];
  uint16_t adm[kMaxAdm];
  int16_t g_a[kMaxGroups], g_b[kMaxGroups], g_first[kMaxGroups], g_n[kMaxGroups];
  int wake_idx[kMaxBodies];  // admission: index of the candidate pair that wakes each body
  unsigned long long cbits[kMaxBodies];  // overlapping pairs (a, b > a) of the last substep, row a
  int cbits_valid;
  int ncand, nadm, nc, ng, fault;
  unsigned long long awake_dyn;
  int moved_mask, dragged, n_active, max_active;
  int64_t ctr[3];
  unsigned kpos[kMaxContacts / 32];  // rows with k > 0, by ballot of the row build (bit i % 32 of word i / 32)
  double sd[2];  // the staged state slab [0, StateLayout::stage): sized at launch (warp_smem_bytes)
};

// shared memory of one env's warp: the fixed part + its staged slab (16-byte multiple)
__host__ __device__ constexpr size_t warp_smem_bytes(int stage) {
  return (sizeof(WarpSmem) - sizeof(double) * 2 + sizeof(double) * (size_t)stage + 15) & ~(size_t)15;
}

static_assert(13 * kMaxBodies + 2 * kMaxJoints + 16 <= kStageD, "state slab prefix must fit the staging buffer");
// the occupancy the launch bounds ask for must fit even a 64-body scene's
// staged slab (228 KB of shared memory per SM, 1 KB reserved per CTA)
static_assert((kWarpsPerBlock == 1 ? 10 : (kWarpsPerBlock == 2 ? 5 : (kWarpsPerBlock == 3 ? 3 : 2))) *
                      (kWarpsPerBlock * warp_smem_bytes(13 * kMaxBodies + 2 * kMaxJoints + 16) + 1024) <=
                  228 * 1024,
              "step_kernel occupancy");

struct Ctx {
  const DevScene *sc;
  const DevBatch *B;
  const rs_physics_config *cfg;
  WarpSmem *S;
  double *rows;   // [row_cap][kRowD]
  double *pairs;  // [kMaxGroups][kPairD]
  double *K;      // [kKCap] block matrices
  double *Vc;     // [kKCap] cached eigenvectors per block
  double *evc;    // [kMaxContacts] cached eigenvalues per block
  double *W;      // [kMaxBlockRows^2] eigensolver workspace
  double *bcache; // [kMaxBodies][14]: pose key (pos bits, quat bits, valid) + body AABB
  double *pcache; // [kMaxPartsCache][18]: world frame (R, p) + AABB of every part, valid for the key pose
  double *ccache; // [kMaxBodies + 1]: candidate pair bit matrix of the last substep + valid flag (bit patterns)
  int env, lane;
  const StateLayout *L;
};

// ------------------------------------------------------------------ access
#define SD(ctx) ((ctx).S->sd)
#define SI(ctx) ((ctx).S->si)
__device__ __forceinline__ double *POS(Ctx &c, int b) { return c.S->sd + c.L->pos + 3 * b; }
__device__ __forceinline__ double *QUAT(Ctx &c, int b) { return c.S->sd + c.L->quat + 4 * b; }
__device__ __forceinline__ double *LV(Ctx &c, int b) { return c.S->sd + c.L->lv + 3 * b; }
__device__ __forceinline__ double *AV(Ctx &c, int b) { return c.S->sd + c.L->av + 3 * b; }
__device__ __forceinline__ int32_t &ASLEEP(Ctx &c, int b) { return c.S->si[c.L->asleep + b]; }
__device__ __forceinline__ int32_t &SLEEPC(Ctx &c, int b) { return c.S->si[c.L->sleep_ctr + b]; }
__device__ __forceinline__ int32_t &RIDER(Ctx &c, int b) { return c.S->si[c.L->rider_joint + b]; }
__device__ __forceinline__ int32_t &HELD(Ctx &c) { return c.S->si[c.L->held]; }
__device__ __forceinline__ int32_t &HELDJ(Ctx &c) { return c.S->si[c.L->held_joint]; }
__device__ __forceinline__ double *JOINTS(Ctx &c) { return c.S->sd + c.L->joints; }
__device__ __forceinline__ double *JVEL(Ctx &c) { return c.S->sd + c.L->jvel; }

__device__ __forceinline__ void body_pose(Ctx &c, int b, Pose &o) {
  quat_to_mat(QUAT(c, b), o.R);
  const double *p = POS(c, b);
  o.p[0] = p[0]; o.p[1] = p[1]; o.p[2] = p[2];
}
__device__ __forceinline__ void body_pose_cached(Ctx &c, int b, Pose &o) { body_pose(c, b, o); }

// write a kinematic pose; 1 if it changed (physics.py:419-433, :441-453)
__device__ int set_kinematic(Ctx &c, int b, const Pose &p, double dt, bool zero_if_same) {
  double q[4];
  mat_to_quat(p.R, q);
  double *pos = POS(c, b), *qu = QUAT(c, b);
  bool same = pos[0] == p.p[0] && pos[1] == p.p[1] && pos[2] == p.p[2] && qu[0] == q[0] && qu[1] == q[1] &&
              qu[2] == q[2] && qu[3] == q[3];
  if (same) {
    if (zero_if_same && dt > 0) {
      double *lv = LV(c, b), *av = AV(c, b);
      lv[0] = lv[1] = lv[2] = 0.0;
      av[0] = av[1] = av[2] = 0.0;
    }
    return 0;
  }
  double op[3] = {pos[0], pos[1], pos[2]}, oq[4] = {qu[0], qu[1], qu[2], qu[3]};
  pos[0] = p.p[0]; pos[1] = p.p[1]; pos[2] = p.p[2];
  qu[0] = q[0]; qu[1] = q[1]; qu[2] = q[2]; qu[3] = q[3];
  if (dt > 0) {
    double *lv = LV(c, b);
    for (int i = 0; i < 3; ++i) lv[i] = (p.p[i] - op[i]) / dt;
    quat_delta_omega(oq, q, dt, AV(c, b));
  }
  return 1;
}

// ---------------------------------------------------------------- kinematics

// FK of the arm chain (robot.py:161-169): lanes compute the joint rotations,
// lane 0 chains them; results in S->u.fk.links / ee.
__device__ void forward_kinematics(Ctx &c) {
  const DevScene &sc = *c.sc;
  if (c.lane <= sc.narm) {  // the chain's constants staged in parallel (no global loads inside it)
    const double *src = c.lane < sc.narm ? sc.arm_offset + 3 * c.lane : sc.gripper;
    for (int k = 0; k < 3; ++k) c.S->u.fk.aoff[c.lane][k] = src[k];
  }
  if (c.lane < sc.narm) axis_angle_mat(sc.arm_axis + 3 * c.lane, JOINTS(c)[sc.nsj + c.lane], c.S->u.fk.raa[c.lane]);
  __syncwarp();
  if (c.lane == 0) {
    Pose t, off, rot;
    base3(c.S->sd + c.L->base, t);
    rot_z(0.0, off.R);
    rot.p[0] = rot.p[1] = rot.p[2] = 0.0;
    for (int i = 0; i < sc.narm; ++i) {
      off.p[0] = c.S->u.fk.aoff[i][0]; off.p[1] = c.S->u.fk.aoff[i][1]; off.p[2] = c.S->u.fk.aoff[i][2];
      compose(t, off, t);
      for (int k = 0; k < 9; ++k) rot.R[k] = c.S->u.fk.raa[i][k];
      compose(t, rot, t);
      for (int k = 0; k < 9; ++k) c.S->u.fk.links[i][k] = t.R[k];
      for (int k = 0; k < 3; ++k) c.S->u.fk.links[i][9 + k] = t.p[k];
    }
    const double *gp = c.S->u.fk.aoff[sc.narm];
    Pose g = {{1, 0, 0, 0, 1, 0, 0, 0, 1}, {gp[0], gp[1], gp[2]}}, e;
    compose(t, g, e);
    for (int k = 0; k < 9; ++k) c.S->u.fk.ee[k] = e.R[k];
    for (int k = 0; k < 3; ++k) c.S->u.fk.ee[9 + k] = e.p[k];
  }
  __syncwarp();
}

// robot.py:349-368 + navgrid.py:55-105
__device__ void move_base(const DevScene &sc, double *base, double lin, double ang, double dt) {
  double x = base[0], y = base[1], yaw = base[2];
  double sy, cy;
  sincos(yaw, &sy, &cy);
  double nx = x + cy * lin * dt, ny = y + sy * lin * dt;
  double nyaw = py_mod(yaw + ang * dt + M_PI, 2.0 * M_PI) - M_PI;
  double p[2];
  nav_nearest_walkable(sc, nx, ny, p);
  base[0] = p[0]; base[1] = p[1]; base[2] = nyaw;
}

__device__ void joint_child_pose(Ctx &c, int ji, double q, Pose &o) {
  const DevScene &sc = *c.sc;
  Pose parent, origin, motion, t;
  body_pose(c, sc.joint_parent[ji], parent);
  pose_load12(sc.joint_origin + 12 * ji, origin);
  compose(parent, origin, t);
  if (sc.joint_type[ji] == RS_REVOLUTE) {
    axis_angle_mat(sc.joint_axis + 3 * ji, q, motion.R);
    motion.p[0] = motion.p[1] = motion.p[2] = 0.0;
  } else {
    const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    for (int k = 0; k < 9; ++k) motion.R[k] = I[k];
    for (int k = 0; k < 3; ++k) motion.p[k] = sc.joint_axis[3 * ji + k] * q;
  }
  compose(t, motion, o);
}

// physics.py:435-467; `mask` = joints to update; warp-collective
__device__ void update_scene_joint_poses(Ctx &c, int mask, double dt) {
  const DevScene &sc = *c.sc;
  if (c.lane == 0) {
    int moved = 0;
    for (int ji = 0; ji < sc.nsj; ++ji) {
      if (!(mask & (1 << ji))) continue;
      Pose p;
      joint_child_pose(c, ji, JOINTS(c)[ji], p);
      if (set_kinematic(c, sc.joint_body[ji], p, dt, false)) moved |= 1 << ji;
    }
    c.S->moved_mask = moved;
  }
  __syncwarp();
  int moved = c.S->moved_mask;
  if (moved) {
    for (int k = c.lane; k < sc.nclutter; k += 32) {
      int b = sc.clutter[k];
      int rj = RIDER(c, b);
      if (rj < 0 || !(moved & (1 << rj)) || !ASLEEP(c, b)) continue;
      Pose part, rel, np_;
      body_pose(c, sc.joint_body[rj], part);
      // rider offsets are constant during a step: read from the input slab in HBM
      const double *ro = c.B->sd + (size_t)c.env * c.L->dbl_size + c.L->rider_off + 7 * b;
      quat_to_mat(ro + 3, rel.R);
      rel.p[0] = ro[0]; rel.p[1] = ro[1]; rel.p[2] = ro[2];
      compose(part, rel, np_);
      double *pos = POS(c, b);
      pos[0] = np_.p[0]; pos[1] = np_.p[1]; pos[2] = np_.p[2];
      mat_to_quat(np_.R, QUAT(c, b));
    }
  }
  __syncwarp();
}

// ------------------------------------------------------------- primitives

__device__ __forceinline__ void part_world(Ctx &c, const Pose &bp, int p, Pose &o) {
  Pose l;
  pose_load12(c.sc->part_local + 12 * p, l);
  compose(bp, l, o);
}
// geometry.py:278-286
__device__ void prim_aabb(Ctx &c, int p, const Pose &wp, double *lo, double *hi) {
  const DevScene &sc = *c.sc;
  int k = sc.part_kind[p];
  if (k == RS_BOX) {
    const double *h = sc.part_param + 3 * p;
    for (int i = 0; i < 3; ++i) {
      double r = fabs(wp.R[3 * i]) * h[0] + fabs(wp.R[3 * i + 1]) * h[1] + fabs(wp.R[3 * i + 2]) * h[2];
      lo[i] = wp.p[i] - r; hi[i] = wp.p[i] + r;
    }
  } else if (k == RS_SPHERE) {
    double r = sc.part_param[3 * p];
    for (int i = 0; i < 3; ++i) { lo[i] = wp.p[i] - r; hi[i] = wp.p[i] + r; }
  } else {
    for (int i = 0; i < 3; ++i) { lo[i] = INFINITY; hi[i] = -INFINITY; }
    for (int v = sc.part_vert_begin[p]; v < sc.part_vert_begin[p + 1]; ++v) {
      double x[3];
      apply(wp, sc.vert + 3 * v, x);
      for (int i = 0; i < 3; ++i) { lo[i] = fmin(lo[i], x[i]); hi[i] = fmax(hi[i], x[i]); }
    }
  }
}

// geometry.py:289-296 parts_aabb (the body AABB = union of its part AABBs)
// with a pose-keyed cache in the env's global scratch: the part world frames
// and AABBs of body b are recomputed only when its position or quaternion
// bits changed (static and sleeping bodies: once), and stay in c.pcache for
// the narrowphase of the same substep.  The cached values are the ones the
// computation would produce (same inputs, same code).
//   bcache[b] = key (pos bits 3, quat bits 4, valid 1) + AABB (lo 3, hi 3)
//   pcache[p] = world frame (R 9, p 3) + AABB (lo 3, hi 3)
__device__ bool body_key_hit(Ctx &c, int b) {
  const double *pos = POS(c, b), *q = QUAT(c, b);
  const double *K = c.bcache + 14 * b;
  const long long *kb = reinterpret_cast<const long long *>(K);
  bool hit = K[7] == 1.0;  // all key words loaded at once (independent loads)
#pragma unroll
  for (int i = 0; i < 3; ++i) hit &= kb[i] == __double_as_longlong(pos[i]);
#pragma unroll
  for (int i = 0; i < 4; ++i) hit &= kb[3 + i] == __double_as_longlong(q[i]);
  return hit;
}

// part p's world frame and AABB from its body's current pose -> pcache.  A
// hull's AABB (a vertex loop) is left to hull_aabb_warp: returns true then.
__device__ bool part_frame_aabb(Ctx &c, int p) {
  Pose bp, wp;
  body_pose(c, c.sc->part_body[p], bp);
  part_world(c, bp, p, wp);
  double *P = c.pcache + 18 * p;
  for (int k = 0; k < 9; ++k) P[k] = wp.R[k];
  for (int i = 0; i < 3; ++i) P[9 + i] = wp.p[i];
  if (c.sc->part_kind[p] == RS_HULL) return true;
  double l[3], h[3];
  prim_aabb(c, p, wp, l, h);
  for (int i = 0; i < 3; ++i) { P[12 + i] = l[i]; P[15 + i] = h[i]; }
  return false;
}

// prim_aabb of hull part q (frame already in pcache), lanes per vertex; the
// min / max reductions are exact, so any order gives the vertex loop's bounds.
// warp-collective.
__device__ void hull_aabb_warp(Ctx &c, int q) {
  const DevScene &sc = *c.sc;
  __syncwarp();
  double *P = c.pcache + 18 * q;
  Pose wp;
  pose_load12(P, wp);
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int v = sc.part_vert_begin[q] + c.lane; v < sc.part_vert_begin[q + 1]; v += 32) {
    double x[3];
    apply(wp, sc.vert + 3 * v, x);
    for (int i = 0; i < 3; ++i) { lo[i] = fmin(lo[i], x[i]); hi[i] = fmax(hi[i], x[i]); }
  }
  for (int o = 16; o; o >>= 1)
    for (int i = 0; i < 3; ++i) {
      lo[i] = fmin(lo[i], __shfl_xor_sync(0xffffffffu, lo[i], o));
      hi[i] = fmax(hi[i], __shfl_xor_sync(0xffffffffu, hi[i], o));
    }
  if (c.lane == 0)
    for (int i = 0; i < 3; ++i) { P[12 + i] = lo[i]; P[15 + i] = hi[i]; }
  __syncwarp();
}

// body b's AABB = union of its parts' (pcache, in part order) -> bcache with the key
__device__ void body_aabb_store(Ctx &c, int b, double *lo, double *hi) {
  const DevScene &sc = *c.sc;
  for (int i = 0; i < 3; ++i) { lo[i] = INFINITY; hi[i] = -INFINITY; }
  for (int p = sc.body_part_begin[b]; p < sc.body_part_begin[b + 1]; ++p) {
    const double *P = c.pcache + 18 * p;
    for (int i = 0; i < 3; ++i) { lo[i] = fmin(lo[i], P[12 + i]); hi[i] = fmax(hi[i], P[15 + i]); }
  }
  const double *pos = POS(c, b), *q = QUAT(c, b);
  double *K = c.bcache + 14 * b;
  for (int i = 0; i < 3; ++i) { K[i] = pos[i]; K[8 + i] = lo[i]; K[11 + i] = hi[i]; }
  for (int i = 0; i < 4; ++i) K[3 + i] = q[i];
  K[7] = 1.0;
}

// world planes of part p into S->planes[slot] (lanes per facet)
__device__ void planes_world(Ctx &c, int p, const Pose &wp, int slot) {
  const DevScene &sc = *c.sc;
  int f0 = sc.part_facet_begin[p], nf = sc.part_facet_begin[p + 1] - f0;
  for (int f = c.lane; f < nf; f += 32) {
    const double *F = sc.facet + 4 * (f0 + f);
    double *o = c.S->u.np.planes[slot] + 4 * f;
    double n[3];
    matvec(wp.R, F, n);
    o[0] = n[0]; o[1] = n[1]; o[2] = n[2];
    o[3] = F[3] + dot3(n, wp.p);
  }
}

// contacts are written straight into their solver rows (global scratch)
__device__ __forceinline__ int add_contact(Ctx &c, int idx, const double *p, const double *n, double depth) {
  if (idx >= kMaxContacts) return 0;
  double *r = c.rows + kRowD * idx;
  for (int i = 0; i < 3; ++i) { r[RPT + i] = p[i]; r[RN + i] = n[i]; }
  r[RDEPTH] = depth;
  return 1;
}

// vertices of part pv (pose wv) against the planes in slot (part pf): geometry.py:564-576, :683-698.
// warp-collective; appends in vertex order; returns the number of contacts.
__device__ int vertices_vs_planes(Ctx &c, int pv, const Pose &wv, int pf, int slot, bool negate, double margin,
                                  int base) {
  const DevScene &sc = *c.sc;
  int v0 = sc.part_vert_begin[pv], nv = sc.part_vert_begin[pv + 1] - v0;
  int nf = sc.part_facet_begin[pf + 1] - sc.part_facet_begin[pf];
  const double *pl = c.S->u.np.planes[slot];
  int total = 0;
  for (int k0 = 0; k0 < nv; k0 += 32) {
    int v = k0 + c.lane;
    bool inside = false;
    double x[3], best = 0.0;
    int face = 0;
    if (v < nv) {
      apply(wv, sc.vert + 3 * (v0 + v), x);
      int neg = 0;
      for (int f = 0; f < nf; ++f) {
        const double *P = pl + 4 * f;
        double s = P[3] - (x[0] * P[0] + x[1] * P[1] + x[2] * P[2]);
        if (f == 0 || s < best) { best = s; face = f; }
        neg += (s < 0.0);
      }
      inside = neg == 0 || (neg == 1 && best >= -margin);
    }
    unsigned m = __ballot_sync(0xffffffffu, inside);
    if (inside) {
      int idx = base + total + __popc(m & ((1u << c.lane) - 1));
      double n[3];
      for (int i = 0; i < 3; ++i) n[i] = negate ? -pl[4 * face + i] : pl[4 * face + i];
      add_contact(c, idx, x, n, best);
    }
    total += __popc(m);
  }
  return total;
}

// geometry.py:602-630
__device__ void closest_on_triangle(const double *p, const double *a, const double *b, const double *cc, double *o) {
  double ab[3], ac[3], ap[3], bp[3], cp[3];
  for (int i = 0; i < 3; ++i) { ab[i] = b[i] - a[i]; ac[i] = cc[i] - a[i]; ap[i] = p[i] - a[i]; }
  double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
  if (d1 <= 0 && d2 <= 0) { for (int i = 0; i < 3; ++i) o[i] = a[i]; return; }
  for (int i = 0; i < 3; ++i) bp[i] = p[i] - b[i];
  double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
  if (d3 >= 0 && d4 <= d3) { for (int i = 0; i < 3; ++i) o[i] = b[i]; return; }
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) {
    double t = d1 / (d1 - d3);
    for (int i = 0; i < 3; ++i) o[i] = a[i] + ab[i] * t;
    return;
  }
  for (int i = 0; i < 3; ++i) cp[i] = p[i] - cc[i];
  double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
  if (d6 >= 0 && d5 <= d6) { for (int i = 0; i < 3; ++i) o[i] = cc[i]; return; }
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) {
    double t = d2 / (d2 - d6);
    for (int i = 0; i < 3; ++i) o[i] = a[i] + ac[i] * t;
    return;
  }
  double va = d3 * d6 - d5 * d4;
  if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0) {
    double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    for (int i = 0; i < 3; ++i) o[i] = b[i] + (cc[i] - b[i]) * t;
    return;
  }
  double den = va + vb + vc, v = vb / den, w = vc / den;
  for (int i = 0; i < 3; ++i) o[i] = a[i] + ab[i] * v + ac[i] * w;
}

// sphere part ps vs convex part pc (planes already in `slot`): geometry.py:633-653. lane 0 only.
__device__ int sphere_convex(Ctx &c, int ps, const Pose &ws, int pc, const Pose &wc, int slot, bool flip,
                             double margin, int idx) {
  const DevScene &sc = *c.sc;
  double r = sc.part_param[3 * ps];
  const double *ctr = ws.p;
  const double *pl = c.S->u.np.planes[slot];
  int nf = sc.part_facet_begin[pc + 1] - sc.part_facet_begin[pc];
  bool inside = true;
  int f = 0;
  double best = 0.0;
  for (int k = 0; k < nf; ++k) {
    double s = pl[4 * k + 3] - dot3(pl + 4 * k, ctr);
    if (s < 0.0) inside = false;
    if (k == 0 || s < best) { best = s; f = k; }
  }
  double n[3], pt[3], depth;
  if (inside) {
    depth = r + best;
    for (int i = 0; i < 3; ++i) { n[i] = pl[4 * f + i]; pt[i] = ctr[i] - n[i] * best; }
  } else {
    double q[3];
    if (sc.part_kind[pc] == RS_BOX) {
      const double *h = sc.part_param + 3 * pc;
      double d[3], l[3];
      for (int i = 0; i < 3; ++i) d[i] = ctr[i] - wc.p[i];
      mattvec(wc.R, d, l);
      for (int i = 0; i < 3; ++i) l[i] = l[i] < -h[i] ? -h[i] : (l[i] > h[i] ? h[i] : l[i]);
      apply(wc, l, q);
    } else {
      int v0 = sc.part_vert_begin[pc];
      double bd = 0.0;
      bool first = true;
      for (int t = sc.part_tri_begin[pc]; t < sc.part_tri_begin[pc + 1]; ++t) {
        double A[3], Bv[3], C[3], qq[3];
        apply(wc, sc.vert + 3 * (v0 + sc.tri[3 * t]), A);
        apply(wc, sc.vert + 3 * (v0 + sc.tri[3 * t + 1]), Bv);
        apply(wc, sc.vert + 3 * (v0 + sc.tri[3 * t + 2]), C);
        closest_on_triangle(ctr, A, Bv, C, qq);
        double e[3] = {ctr[0] - qq[0], ctr[1] - qq[1], ctr[2] - qq[2]}, d2 = dot3(e, e);
        if (first || d2 < bd) { bd = d2; q[0] = qq[0]; q[1] = qq[1]; q[2] = qq[2]; first = false; }
      }
    }
    double d[3] = {ctr[0] - q[0], ctr[1] - q[1], ctr[2] - q[2]};
    double dist = sqrt(dot3(d, d));
    depth = r - dist;
    if (depth <= -margin) return 0;
    if (dist > 0) for (int i = 0; i < 3; ++i) n[i] = d[i] / dist;
    else { n[0] = 0; n[1] = 0; n[2] = 1; }
    pt[0] = q[0]; pt[1] = q[1]; pt[2] = q[2];
  }
  if (flip) for (int i = 0; i < 3; ++i) n[i] = -n[i];
  add_contact(c, idx, pt, n, depth);
  return 1;
}

__device__ int sphere_sphere(Ctx &c, int pa, const Pose &wa, int pb, const Pose &wb, double margin, int idx) {
  const DevScene &sc = *c.sc;
  double ra = sc.part_param[3 * pa], rb = sc.part_param[3 * pb], d[3], n[3];
  for (int i = 0; i < 3; ++i) d[i] = wa.p[i] - wb.p[i];
  double dist = sqrt(dot3(d, d)), depth = ra + rb - dist;
  if (depth <= -margin) return 0;
  if (dist > 0) for (int i = 0; i < 3; ++i) n[i] = d[i] / dist;
  else { n[0] = 0; n[1] = 0; n[2] = 1; }
  double pt[3];
  for (int i = 0; i < 3; ++i) pt[i] = wb.p[i] + n[i] * rb;
  add_contact(c, idx, pt, n, depth);
  return 1;
}

// geometry.py:667-698 convex_contacts for one part pair: i's vertices against
// j's planes, then j's against i's planes (normals negated).  Both plane sets
// are built in one pass (lanes per facet) and, when both vertex sets fit the
// warp together, both vertex passes run in one round (lanes 0..nvi-1: i's
// vertices, then j's) -- one ballot keeps the reference's contact order.
__device__ int convex_pair_contacts(Ctx &c, int i, const Pose &wa, int j, const Pose &wb, double margin, int base) {
  const DevScene &sc = *c.sc;
  const int fi0 = sc.part_facet_begin[i], nfi = sc.part_facet_begin[i + 1] - fi0;
  const int fj0 = sc.part_facet_begin[j], nfj = sc.part_facet_begin[j + 1] - fj0;
  for (int e = c.lane; e < nfj + nfi; e += 32) {  // slot 0: j's planes, slot 1: i's planes (planes_world)
    const bool bj = e < nfj;
    const int f = bj ? e : e - nfj;
    const Pose &wp = bj ? wb : wa;
    const double *F = sc.facet + 4 * ((bj ? fj0 : fi0) + f);
    double *o = c.S->u.np.planes[bj ? 0 : 1] + 4 * f;
    double nrm[3];
    matvec(wp.R, F, nrm);
    o[0] = nrm[0]; o[1] = nrm[1]; o[2] = nrm[2];
    o[3] = F[3] + dot3(nrm, wp.p);
  }
  __syncwarp();
  const int vi0 = sc.part_vert_begin[i], nvi = sc.part_vert_begin[i + 1] - vi0;
  const int vj0 = sc.part_vert_begin[j], nvj = sc.part_vert_begin[j + 1] - vj0;
  int n = 0;
  if (nvi + nvj <= 32) {
    const int v = c.lane;
    bool inside = false, neg_n = false;
    double x[3], best = 0.0;
    const double *pl = nullptr;
    int face = 0;
    if (v < nvi + nvj) {  // vertices_vs_planes for either side
      const bool si = v < nvi;
      neg_n = !si;
      pl = c.S->u.np.planes[si ? 0 : 1];
      const int nf = si ? nfj : nfi;
      apply(si ? wa : wb, sc.vert + 3 * (si ? vi0 + v : vj0 + v - nvi), x);
      int neg = 0;
      for (int f = 0; f < nf; ++f) {
        const double *P = pl + 4 * f;
        double s = P[3] - (x[0] * P[0] + x[1] * P[1] + x[2] * P[2]);
        if (f == 0 || s < best) { best = s; face = f; }
        neg += (s < 0.0);
      }
      inside = neg == 0 || (neg == 1 && best >= -margin);
    }
    const unsigned m = __ballot_sync(0xffffffffu, inside);
    if (inside) {
      double nn[3];
      for (int k = 0; k < 3; ++k) nn[k] = neg_n ? -pl[4 * face + k] : pl[4 * face + k];
      add_contact(c, base + __popc(m & ((1u << c.lane) - 1)), x, nn, best);
    }
    n = __popc(m);
  } else {
    n += vertices_vs_planes(c, i, wa, j, 0, false, margin, base + n);
    n += vertices_vs_planes(c, j, wb, i, 1, true, margin, base + n);
  }
  __syncwarp();
  return n;
}

// geometry.py:701-716 for one part pair (i, j) that passed the margin-AABB
// cull: its contacts, appended at `base`, from the substep's part frames in
// c.pcache ([R(9), p(3), lo(3), hi(3)] per part).  warp-collective.
__device__ int part_pair_contacts(Ctx &c, int i, int j, double margin, int base) {
  const DevScene &sc = *c.sc;
  Pose wa, wb;
  pose_load12(c.pcache + 18 * i, wa);
  pose_load12(c.pcache + 18 * j, wb);
  const int ka = sc.part_kind[i], kb = sc.part_kind[j];
  if (ka == RS_SPHERE && kb == RS_SPHERE) {
    int r = 0;
    if (c.lane == 0) r = sphere_sphere(c, i, wa, j, wb, margin, base);
    return __shfl_sync(0xffffffffu, r, 0);
  }
  if (ka == RS_SPHERE || kb == RS_SPHERE) {
    const bool flip = kb == RS_SPHERE;
    const int ps = flip ? j : i, pc = flip ? i : j;
    const Pose &ws = flip ? wb : wa, &wc = flip ? wa : wb;
    planes_world(c, pc, wc, 0);
    __syncwarp();
    int r = 0;
    if (c.lane == 0) r = sphere_convex(c, ps, ws, pc, wc, 0, flip, margin, base);
    r = __shfl_sync(0xffffffffu, r, 0);
    __syncwarp();
    return r;
  }
  return convex_pair_contacts(c, i, wa, j, wb, margin, base);
}

// phase clocks (rsim_bench_phase_cycles): 0 front, 1 sweeps, 2 eigensolves,
// 3 block LCP iterations, 4 block impulse + friction, 5 scalar rows, 6 back;
// front split: 7 kinematics, 8 AABBs + overlap, 9 admission, 10 narrowphase,
// 11 rows + blocks; 8 split: 12 AABB cache, 13 pair re-tests, 14 candidate emission
constexpr int kPhases = 16;
__device__ __forceinline__ long long phase_now(const Ctx &c) { return c.B->phase_cycles ? clock64() : 0; }
struct PhaseClock {
  long long t0;
  __device__ __forceinline__ explicit PhaseClock(const Ctx &c) { t0 = phase_now(c); }
  __device__ __forceinline__ void add(const Ctx &c, int k) {
    if (c.B->phase_cycles && c.lane == 0) c.B->phase_cycles[kPhases * (size_t)c.env + k] += phase_now(c) - t0;
  }
};

// ------------------------------------------------------------------ solver

__device__ __forceinline__ void row_rel_vel(Ctx &c, const double *r, double *o) {
  const double *va = c.S->u.sol.vel[(int)r[RA]], *vb = c.S->u.sol.vel[(int)r[RB]];
  const double *ra = r + RRA, *rb = r + RRB;
  double ax = va[0] + va[4] * ra[2] - va[5] * ra[1];
  double ay = va[1] + va[5] * ra[0] - va[3] * ra[2];
  double az = va[2] + va[3] * ra[1] - va[4] * ra[0];
  double bx = vb[0] + vb[4] * rb[2] - vb[5] * rb[1];
  double by = vb[1] + vb[5] * rb[0] - vb[3] * rb[2];
  double bz = vb[2] + vb[3] * rb[1] - vb[4] * rb[0];
  int ja = (int)r[RJA], jb = (int)r[RJB];
  if (ja >= 0) {
    double dv = c.S->jdv[ja];
    ax += r[RJACA] * dv; ay += r[RJACA + 1] * dv; az += r[RJACA + 2] * dv;
  }
  if (jb >= 0) {
    double dv = c.S->jdv[jb];
    bx += r[RJACB] * dv; by += r[RJACB + 1] * dv; bz += r[RJACB + 2] * dv;
  }
  o[0] = ax - bx; o[1] = ay - by; o[2] = az - bz;
}
__device__ __forceinline__ double row_vn(Ctx &c, const double *r) {
  double v[3];
  row_rel_vel(c, r, v);
  return v[0] * r[RN] + v[1] * r[RN + 1] + v[2] * r[RN + 2];
}
// physics.py:1257-1291
__device__ void row_apply(Ctx &c, const double *r, double ix, double iy, double iz) {
  const double *pg = c.pairs + kPairD * (int)r[RGRP];
  if (r[RIMA] > 0.0) {
    double *va = c.S->u.sol.vel[(int)r[RA]], m = r[RIMA];
    va[0] += ix * m; va[1] += iy * m; va[2] += iz * m;
    const double *ra = r + RRA;
    double tx = ra[1] * iz - ra[2] * iy, ty = ra[2] * ix - ra[0] * iz, tz = ra[0] * iy - ra[1] * ix;
    const double *I = pg + PIA;
    va[3] += I[0] * tx + I[1] * ty + I[2] * tz;
    va[4] += I[3] * tx + I[4] * ty + I[5] * tz;
    va[5] += I[6] * tx + I[7] * ty + I[8] * tz;
  }
  if (r[RIMB] > 0.0) {
    double *vb = c.S->u.sol.vel[(int)r[RB]], m = r[RIMB];
    vb[0] -= ix * m; vb[1] -= iy * m; vb[2] -= iz * m;
    const double *rb = r + RRB;
    double tx = rb[1] * iz - rb[2] * iy, ty = rb[2] * ix - rb[0] * iz, tz = rb[0] * iy - rb[1] * ix;
    const double *I = pg + PIB;
    vb[3] -= I[0] * tx + I[1] * ty + I[2] * tz;
    vb[4] -= I[3] * tx + I[4] * ty + I[5] * tz;
    vb[5] -= I[6] * tx + I[7] * ty + I[8] * tz;
  }
  int ja = (int)r[RJA], jb = (int)r[RJB];
  if (ja >= 0) c.S->jdv[ja] += (r[RJACA] * ix + r[RJACA + 1] * iy + r[RJACA + 2] * iz) * r[RJIA];
  if (jb >= 0) c.S->jdv[jb] -= (r[RJACB] * ix + r[RJACB + 1] * iy + r[RJACB + 2] * iz) * r[RJIB];
}
// physics.py:1309-1326
__device__ void row_friction(Ctx &c, double *r) {
  if (r[RK] <= 0.0 || r[RFRIC] == 0.0) return;
  double max_t = r[RMU] * r[RLAM];
  for (int w = 0; w < 2; ++w) {
    const double *t = r + (w ? RT2 : RT1);
    double *acc = r + (w ? RLT2 : RLT1);
    double v[3];
    row_rel_vel(c, r, v);
    double vt = v[0] * t[0] + v[1] * t[1] + v[2] * t[2];
    double lt = -vt / r[RK], nt = *acc + lt;
    if (nt > max_t) nt = max_t;
    else if (nt < -max_t) nt = -max_t;
    lt = nt - *acc;
    *acc = nt;
    if (lt != 0.0) row_apply(c, r, t[0] * lt, t[1] * lt, t[2] * lt);
  }
}
// physics.py:1293-1307
__device__ void row_solve(Ctx &c, double *r) {
  if (r[RK] <= 0.0) return;
  double vn = row_vn(c, r);
  double lam = -(vn - r[RTGT]) / r[RK], tot = r[RLAM] + lam;
  if (tot < 0.0) tot = 0.0;
  lam = tot - r[RLAM];
  r[RLAM] = tot;
  if (lam != 0.0) row_apply(c, r, r[RN] * lam, r[RN + 1] * lam, r[RN + 2] * lam);
  row_friction(c, r);
}

// ---------------------------------------------------------------------------
// Block LCP (physics.py:760-816), warp-cooperative.
//
// The reference solves each active sub-block with np.linalg.lstsq(rcond=1e-8)
// (min-norm); for the symmetric PSD K the same solution comes from a
// Jacobi eigendecomposition with the gelsd cutoff s <= rcond * s_max.  The
// oracle runs a serial cyclic Jacobi; here every rotation is still applied
// in the same (p, q) order, but the row / column / eigenvector updates of a
// rotation are spread over the lanes (one element per lane), and every
// reduction keeps the oracle's summation order -- the results are
// bit-identical to the serial code.  K is fixed for the whole substep, so
// the decomposition of K[A, A] is cached per block and active set A: across
// the 16 Gauss-Seidel sweeps the active set repeats and the eigensolve runs
// once per distinct set.

__device__ __forceinline__ void jacobi_pair(int n, int r, int k, int &p, int &q) {
  int a, b;
  if (k == 0) { a = n - 1; b = r; }
  else {  // (r + k) mod (n - 1), (r - k) mod (n - 1) with 0 <= r < n - 1, 0 < k < n / 2
    a = r + k; if (a >= n - 1) a -= n - 1;
    b = r - k + n - 1; if (b >= n - 1) b -= n - 1;
  }
  p = a < b ? a : b;
  q = a < b ? b : a;
}

// A (m x m, row-major, destroyed) -> V (eigenvectors in columns), ev; warp-collective.
// Round-robin Jacobi: m'-1 rounds of m'/2 disjoint rotations per sweep, rotation
// parameters from the matrix at the start of the round (one pair per lane),
// then a column pass and a row pass (one element pair per lane).  Identical
// per-element arithmetic to oracle/rsim_oracle.c sym_eig.
constexpr int kEigCached = 4;  // items per lane with cached indices (half * m <= 128, i.e. m <= 16)
__device__ void sym_eig_warp(int m, double *A, double *V, double *ev, double *cs, double *sn, int *pp, int *qq,
                             int lane) {
  const int n = m + (m & 1), half = n / 2;
  for (int e = lane; e < m * m; e += 32) V[e] = (e / m == e % m);
  // this lane's (rotation, row) items it = lane + 32 t of the column / row
  // passes, fixed for the whole decomposition (no integer division per round)
  int ik[kEigCached], ii[kEigCached];
#pragma unroll
  for (int t = 0; t < kEigCached; ++t) { ik[t] = (lane + 32 * t) / m; ii[t] = (lane + 32 * t) % m; }
  __syncwarp();
  for (int sweep = 0; sweep < 64 && m > 1; ++sweep) {
    // Frobenius norms: row partial sums (lane per row), rows added in order
    if (lane < m) {
      double ro = 0.0, rt = 0.0;
      for (int j = 0; j < m; ++j) {
        double a2 = A[lane * m + j] * A[lane * m + j];
        rt += a2;
        if (lane != j) ro += a2;
      }
      cs[lane] = ro;  // cs/sn double as row-sum scratch
      sn[lane] = rt;
    }
    __syncwarp();
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < m; ++i) { off += cs[i]; tot += sn[i]; }
    __syncwarp();
    if (off <= 1e-30 * tot || off == 0.0) break;  // off-diagonal <= 1e-15 of the Frobenius norm
    for (int r = 0; r < n - 1; ++r) {
      __syncwarp();
      if (lane < half) {
        int p, q;
        jacobi_pair(n, r, lane, p, q);
        double c = 1.0, sv = 0.0;
        if (q < m) {
          const double apq = A[p * m + q];
          if (apq != 0.0) {
            const double app = A[p * m + p], aqq = A[q * m + q];
            // t = sgn(theta) / (|theta| + sqrt(theta^2 + 1)), theta = a / b, and
            // c = 1 / sqrt(t^2 + 1), multiplied through by |b| (fewer dependent
            // divisions / square roots; oracle sym_eig does the same)
            const double a = aqq - app, b = 2.0 * apq;
            const double num = a > 0.0 ? b : (a < 0.0 ? -b : fabs(b));
            const double den = fabs(a) + sqrt(a * a + b * b);
            const double t = num / den;
            c = den / sqrt(den * den + b * b);
            sv = t * c;
          }
        }
        pp[lane] = p; qq[lane] = q; cs[lane] = c; sn[lane] = sv;
      }
      __syncwarp();
      auto col = [&](int k, int i) {  // column pass element: rows i of columns p, q (A and V)
        const int p = pp[k], q = qq[k];
        if (q >= m || sn[k] == 0.0) return;
        const double c = cs[k], sv = sn[k];
        double aip = A[i * m + p], aiq = A[i * m + q];
        A[i * m + p] = c * aip - sv * aiq;
        A[i * m + q] = sv * aip + c * aiq;
        double vip = V[i * m + p], viq = V[i * m + q];
        V[i * m + p] = c * vip - sv * viq;
        V[i * m + q] = sv * vip + c * viq;
      };
      auto row = [&](int k, int j) {  // row pass element: column j of rows p, q
        const int p = pp[k], q = qq[k];
        if (q >= m || sn[k] == 0.0) return;
        const double c = cs[k], sv = sn[k];
        double apj = A[p * m + j], aqj = A[q * m + j];
        A[p * m + j] = c * apj - sv * aqj;
        A[q * m + j] = sv * apj + c * aqj;
      };
#pragma unroll
      for (int t = 0; t < kEigCached; ++t)
        if (lane + 32 * t < half * m) col(ik[t], ii[t]);
      for (int it = lane + 32 * kEigCached; it < half * m; it += 32) col(it / m, it % m);
      __syncwarp();
#pragma unroll
      for (int t = 0; t < kEigCached; ++t)
        if (lane + 32 * t < half * m) row(ik[t], ii[t]);
      for (int it = lane + 32 * kEigCached; it < half * m; it += 32) row(it / m, it % m);
      __syncwarp();
    }
  }
  if (lane < m) ev[lane] = A[lane * m + lane];
  __syncwarp();
}

// physics.py:800-816 after a converged block LCP: apply the normal impulse
// deltas in row order, then one Gauss-Seidel friction pass in row order
// (row_apply / row_friction / row_rel_vel), for a block whose rows touch no
// articulation joint.  The block's rows are staged into shared memory by the
// warp; lane 0 then runs the order-dependent sequence with both bodies'
// velocities and inverse inertias in registers.  Same operations in the same
// order as the generic path.
constexpr int kFastRows = 12;
constexpr int kFastD = 23;  // n, t1, t2, ra, rb, k, mu, fric, lam_old, lt1, lt2, ima, imb
static_assert(kFastRows * kFastD <= 2 * kSmemEig * kSmemEig, "staging area");
__constant__ int kFastSrc[kFastD] = {RN, RN + 1, RN + 2, RT1, RT1 + 1, RT1 + 2, RT2, RT2 + 1, RT2 + 2,
                                     RRA, RRA + 1, RRA + 2, RRB, RRB + 1, RRB + 2, RK, RMU, RFRIC, RLAM,
                                     RLT1, RLT2, RIMA, RIMB};
__device__ void block_impulse_friction(Ctx &c, int g, int first, int m, BlockWS &ws) {
  double *F = ws.F;  // [m][kFastD]
  const int lane = c.lane;
  for (int e = lane; e < m * kFastD; e += 32) {
    const int i = e / kFastD, q = e - i * kFastD;
    const double *r = c.rows + kRowD * (first + i);
    F[e] = r[kFastSrc[q]];
  }
  __syncwarp();
  if (lane == 0) {
    const double *r0 = c.rows + kRowD * first;
    const int a = (int)r0[RA], b = (int)r0[RB];
    const double *pg = c.pairs + kPairD * g;
    double va[6], vb[6], Ia[9], Ib[9];
    for (int k = 0; k < 6; ++k) { va[k] = c.S->u.sol.vel[a][k]; vb[k] = c.S->u.sol.vel[b][k]; }
    for (int k = 0; k < 9; ++k) { Ia[k] = pg[PIA + k]; Ib[k] = pg[PIB + k]; }
    auto apply = [&](const double *f, double ix, double iy, double iz) {  // row_apply
      if (f[21] > 0.0) {
        const double mm = f[21], *ra = f + 9;
        va[0] += ix * mm; va[1] += iy * mm; va[2] += iz * mm;
        double tx = ra[1] * iz - ra[2] * iy, ty = ra[2] * ix - ra[0] * iz, tz = ra[0] * iy - ra[1] * ix;
        va[3] += Ia[0] * tx + Ia[1] * ty + Ia[2] * tz;
        va[4] += Ia[3] * tx + Ia[4] * ty + Ia[5] * tz;
        va[5] += Ia[6] * tx + Ia[7] * ty + Ia[8] * tz;
      }
      if (f[22] > 0.0) {
        const double mm = f[22], *rb = f + 12;
        vb[0] -= ix * mm; vb[1] -= iy * mm; vb[2] -= iz * mm;
        double tx = rb[1] * iz - rb[2] * iy, ty = rb[2] * ix - rb[0] * iz, tz = rb[0] * iy - rb[1] * ix;
        vb[3] -= Ib[0] * tx + Ib[1] * ty + Ib[2] * tz;
        vb[4] -= Ib[3] * tx + Ib[4] * ty + Ib[5] * tz;
        vb[5] -= Ib[6] * tx + Ib[7] * ty + Ib[8] * tz;
      }
    };
    for (int i = 0; i < m; ++i) {  // normal impulse deltas
      double *f = F + kFastD * i;
      const double l = ws.lam[i] > 0.0 ? ws.lam[i] : 0.0;
      const double d = l - f[18];
      f[18] = l;
      c.rows[kRowD * (first + i) + RLAM] = l;
      if (d != 0.0) apply(f, f[0] * d, f[1] * d, f[2] * d);
    }
    for (int i = 0; i < m; ++i) {  // row_friction
      double *f = F + kFastD * i;
      if (f[15] <= 0.0 || f[17] == 0.0) continue;
      const double max_t = f[16] * f[18], *ra = f + 9, *rb = f + 12;
      for (int w = 0; w < 2; ++w) {
        const double *t = f + (w ? 6 : 3);
        double &acc = f[w ? 20 : 19];
        const double ax = va[0] + va[4] * ra[2] - va[5] * ra[1];
        const double ay = va[1] + va[5] * ra[0] - va[3] * ra[2];
        const double az = va[2] + va[3] * ra[1] - va[4] * ra[0];
        const double bx = vb[0] + vb[4] * rb[2] - vb[5] * rb[1];
        const double by = vb[1] + vb[5] * rb[0] - vb[3] * rb[2];
        const double bz = vb[2] + vb[3] * rb[1] - vb[4] * rb[0];
        const double v0 = ax - bx, v1 = ay - by, v2 = az - bz;
        const double vt = v0 * t[0] + v1 * t[1] + v2 * t[2];
        double lt = -vt / f[15], nt = acc + lt;
        if (nt > max_t) nt = max_t;
        else if (nt < -max_t) nt = -max_t;
        lt = nt - acc;
        acc = nt;
        if (lt != 0.0) apply(f, t[0] * lt, t[1] * lt, t[2] * lt);
      }
      double *r = c.rows + kRowD * (first + i);
      r[RLT1] = f[19];
      r[RLT2] = f[20];
    }
    // write back only the velocities this block can change (solver inverse
    // mass > 0): a static / kinematic partner's entry is shared with the
    // blocks other warps solve concurrently (step_kernel_cta) and stays as is
    bool wa = false, wb = false;
    for (int i = 0; i < m; ++i) { wa |= F[kFastD * i + 21] > 0.0; wb |= F[kFastD * i + 22] > 0.0; }
    for (int k = 0; k < 6; ++k) {
      if (wa) c.S->u.sol.vel[a][k] = va[k];
      if (wb) c.S->u.sol.vel[b][k] = vb[k];
    }
  }
  __syncwarp();
}

// physics.py:760-816; warp-collective.  Kc/evc: this block's eigen cache.
__device__ void solve_block(Ctx &c, int g, int first, int m, const double *K, BlockWS &ws, double *W, double *Vc,
                            double *evc) {
  const int lane = c.lane;
  PhaseClock pl(c);
  double *P = c.pairs + kPairD * g;
  if (lane < m) {
    double *r = c.rows + kRowD * (first + lane);
    ws.cur[lane] = r[RLAM];
    ws.wv[lane] = row_vn(c, r) - r[RTGT];
  }
  __syncwarp();
  bool start = false;  // initial active set: rows with lambda > 0 or w < 0, in row order
  if (lane < m) {
    const int i = lane;
    double s = 0.0;
#pragma unroll 4
    for (int j = 0; j < m; ++j) s += K[j * m + i] * ws.cur[j];  // K is stored exactly symmetric: coalesced
    ws.q[i] = ws.wv[i] - s;
    start = ws.cur[i] > 0.0 || ws.wv[i] < 0.0;
  }
  const unsigned am = __ballot_sync(0xffffffffu, start);
  if (start) ws.active[__popc(am & ((1u << lane) - 1))] = lane;
  if (lane == 0) {
    ws.na = __popc(am);
    ws.converged = 0;
  }
  __syncwarp();
  // lexicographic (value, row) minimum over the lanes: the oracle's serial
  // scans ("strictly smaller, or equal with a lower row").  Both callers order
  // rows with lanes, so it is the lowest lane holding the minimum value.  The
  // candidates are finite and < -1e-10 (no NaN, no signed zero) or +inf, so the
  // order-preserving 64-bit key of a double makes the minimum two 32-bit
  // warp reductions (redux.sync) instead of five shuffle rounds
  auto argmin = [&](double v, int r) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned long long key = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mhi = __reduce_min_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_min_sync(0xffffffffu, hi == mhi ? lo : 0xffffffffu);
    const unsigned win = __ballot_sync(0xffffffffu, hi == mhi && lo == mlo);
    return __shfl_sync(0xffffffffu, r, __ffs(win) - 1);
  };
  // the block's decomposition cache directory in registers for the solve
  // (lane s < kEigSlots: slot s's active-set key and last use), written back after it
  double skey = lane < kEigSlots ? P[PMASK + lane] : -2.0, sstamp = lane < kEigSlots ? P[PSTAMP + lane] : INFINITY;
  double clk = P[PCLK];
  for (int it = 0; it < 4 * m + 4; ++it) {
    if (c.B->phase_cycles && lane == 0) c.B->phase_cycles[kPhases * (size_t)c.env + 15] += 1;  // iterations
    const int na = ws.na;
    const int act = lane < na ? ws.active[lane] : -1;  // this lane's active row (active is sorted)
    if (lane < m) ws.lam[lane] = 0.0;
    const unsigned mask = __reduce_or_sync(0xffffffffu, act >= 0 ? 1u << act : 0u);  // the active set
    if (na) {
      if (lane < na) ws.rhs[lane] = -ws.q[act];
      // kEigSlots cached decompositions per block, keyed by the active set
      // (a decomposition is a pure function of K_AA: caching changes no bit);
      // lanes per slot look up, a miss replaces the least recently used slot
      const double key = (double)mask;
      const unsigned hm = __ballot_sync(0xffffffffu, lane < kEigSlots && skey == key);
      int slot = hm ? __ffs(hm) - 1 : -1;
      if (slot < 0) {
        double st = sstamp;
        int sl = lane;
        for (int o = kEigSlots / 2; o; o >>= 1) {
          const double os = __shfl_xor_sync(0xffffffffu, st, o);
          const int ol = __shfl_xor_sync(0xffffffffu, sl, o);
          if (os < st || (os == st && ol < sl)) { st = os; sl = ol; }
        }
        slot = __shfl_sync(0xffffffffu, sl, 0);
        double *A = na <= kSmemEig ? ws.A : W;
        double *Vt = na <= kSmemEig ? ws.V : Vc + slot * m * m;
        for (int e = lane; e < na * na; e += 32) A[e] = K[ws.active[e / na] * m + ws.active[e % na]];
        __syncwarp();
        PhaseClock pe(c);
        sym_eig_warp(na, A, Vt, evc + slot * m, ws.cs, ws.sn, ws.pp, ws.qq, lane);
        pe.add(c, 2);
        if (na <= kSmemEig)
          for (int e = lane; e < na * na; e += 32) Vc[slot * m * m + e] = Vt[e];
        if (lane == slot) skey = key;
      }
      clk += 1.0;
      if (lane == slot) sstamp = clk;
      __syncwarp();
      const double *Vs = Vc + slot * m * m, *es = evc + slot * m;
      // x = sum_k (V_k . b / ev_k) V_k over ev_k > rcond * max|ev| (oracle pinv_solve
      // order; the sums stay sequential, unrolled only to overlap the loads)
      double smax;  // max is exact in any order: non-negative doubles order as their bit patterns
      {
        const unsigned long long b = lane < na ? (unsigned long long)__double_as_longlong(fabs(es[lane])) : 0ull;
        const unsigned mhi = __reduce_max_sync(0xffffffffu, (unsigned)(b >> 32));
        const unsigned mlo = __reduce_max_sync(0xffffffffu, (unsigned)(b >> 32) == mhi ? (unsigned)b : 0u);
        smax = __hiloint2double((int)mhi, (int)mlo);
      }
      bool keep_k = false;
      if (lane < na) {
        const int k = lane;
        double cc = 0.0;
#pragma unroll 4
        for (int i = 0; i < na; ++i) cc += Vs[i * na + k] * ws.rhs[i];
        ws.ck[k] = cc / es[k];
        keep_k = !(fabs(es[k]) <= 1e-8 * smax);  // the pinv cutoff, once per eigenvalue
      }
      const unsigned keep = __ballot_sync(0xffffffffu, keep_k);
      __syncwarp();
      if (lane < na) {
        const int i = lane;
        double x = 0.0;
#pragma unroll 4
        for (int k = 0; k < na; ++k) {
          if (!((keep >> k) & 1u)) continue;
          x += ws.ck[k] * Vs[i * na + k];
        }
        ws.lam[act] = x;
      }
    }
    __syncwarp();
    // drop the most negative lambda (physics.py:790-800; lowest row on ties)
    double lv = INFINITY;
    if (lane < na) {
      const double l = ws.lam[act];
      if (l < -1e-10) lv = l;
    }
    int worst = argmin(lv, lv < INFINITY ? act : 0x7fffffff);
    if (worst != 0x7fffffff) {
      const bool keep = lane < na && act != worst;
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      if (keep) ws.active[__popc(km & ((1u << lane) - 1))] = act;
      if (lane == 0) ws.na = na - 1;
      __syncwarp();
      continue;
    }
    // w = K lam + q on the inactive rows (lane i, oracle order)
    double wv = INFINITY;
    if (lane < m && !((mask >> lane) & 1u)) {
      const int i = lane;
      double wi = 0.0;
#pragma unroll 4
      for (int j = 0; j < m; ++j) wi += K[j * m + i] * ws.lam[j];  // symmetric K: coalesced
      wi += ws.q[i];
      ws.wv[i] = wi;
      if (wi < -1e-10) wv = wi;
    }
    // add the most violated inactive row (lowest row on ties), keeping active sorted
    worst = argmin(wv, wv < INFINITY ? lane : 0x7fffffff);
    if (worst == 0x7fffffff) {
      if (lane == 0) ws.converged = 1;
      __syncwarp();
      break;
    }
    const int below = __popc(__ballot_sync(0xffffffffu, lane < na && act < worst));
    if (lane < na) ws.active[act > worst ? lane + 1 : lane] = act;
    if (lane == 0) { ws.active[below] = worst; ws.na = na + 1; }
    __syncwarp();
  }
  if (lane < kEigSlots) { P[PMASK + lane] = skey; P[PSTAMP + lane] = sstamp; }
  if (lane == 0) P[PCLK] = clk;
  pl.add(c, 3);
  PhaseClock pf(c);
  // register-resident impulse + friction pass for blocks without joint
  // coupling that fit the staging area (A/V of the workspace, free now)
  bool fast = ws.converged && m <= kFastRows;
  if (fast) {
    bool nojoint = true;
    if (lane < m) {
      const double *r = c.rows + kRowD * (first + lane);
      nojoint = r[RJA] < 0.0 && r[RJB] < 0.0;
    }
    fast = __all_sync(0xffffffffu, nojoint);
  }
  if (fast) {
    block_impulse_friction(c, g, first, m, ws);
  } else if (lane == 0) {
    if (!ws.converged) {
      for (int i = 0; i < m; ++i) row_solve(c, c.rows + kRowD * (first + i));
    } else {
      for (int i = 0; i < m; ++i) {
        double *r = c.rows + kRowD * (first + i);
        double l = ws.lam[i] > 0.0 ? ws.lam[i] : 0.0;
        double d = l - r[RLAM];
        r[RLAM] = l;
        if (d != 0.0) row_apply(c, r, r[RN] * d, r[RN + 1] * d, r[RN + 2] * d);
      }
      for (int i = 0; i < m; ++i) row_friction(c, c.rows + kRowD * (first + i));
    }
  }
  __syncwarp();
  pf.add(c, 4);
}

__device__ __forceinline__ bool solver_dynamic(Ctx &c, int b) {
  return c.sc->body_kind[b] == RS_DYNAMIC && !ASLEEP(c, b) && b != HELD(c);
}

// physics.py:827-844
__device__ int joint_jacobian(Ctx &c, int b, const double *pt, double *jac, double &inv_i) {
  const DevScene &sc = *c.sc;
  int ji = sc.body_joint[b];
  if (ji < 0 || HELDJ(c) == ji) return -1;
  Pose parent, origin, jf;
  body_pose_cached(c, sc.joint_parent[ji], parent);
  pose_load12(sc.joint_origin + 12 * ji, origin);
  compose(parent, origin, jf);
  double ax[3];
  matvec(jf.R, sc.joint_axis + 3 * ji, ax);
  if (sc.joint_type[ji] == RS_PRISMATIC) {
    jac[0] = ax[0]; jac[1] = ax[1]; jac[2] = ax[2];
    inv_i = 1.0 / c.cfg->joint_inertia_prismatic;
  } else {
    double d[3] = {pt[0] - jf.p[0], pt[1] - jf.p[1], pt[2] - jf.p[2]};
    cross3(ax, d, jac);
    inv_i = 1.0 / c.cfg->joint_inertia_revolute;
  }
  return ji;
}


__device__ __forceinline__ void wake(Ctx &c, int b) {
  if (c.sc->body_kind[b] != RS_DYNAMIC) return;
  if (ASLEEP(c, b)) c.S->ctr[2]++;
  ASLEEP(c, b) = 0;
  SLEEPC(c, b) = 0;
  RIDER(c, b) = -1;
}

// ------------------------------------------------------------------ substep

__device__ void emit_event(Ctx &c, const double *r, double lam, double force) {
  int k = c.B->event_count[c.env]++;
  if (k < c.B->event_cap) {
    double *o = c.B->events + ((size_t)c.env * c.B->event_cap + k) * 7;
    o[0] = r[RA]; o[1] = r[RB]; o[2] = lam; o[3] = force;
    o[4] = r[RPT]; o[5] = r[RPT + 1]; o[6] = r[RPT + 2];
  }
}

// does group g hold a row with k > 0 (S.kpos of the row build)
__device__ __forceinline__ bool group_has_k(const WarpSmem &S, int g) {
  const int first = S.g_first[g], end = first + S.g_n[g];
  for (int w = first >> 5; w <= (end - 1) >> 5; ++w) {
    unsigned bits = S.kpos[w];
    const int lo = w * 32 > first ? 0 : first - w * 32, hi = (w + 1) * 32 < end ? 32 : end - w * 32;
    bits &= (hi == 32 ? ~0u : (1u << hi) - 1u) & ~((1u << lo) - 1u);
    if (bits) return true;
  }
  return false;
}

// physics.py:657-701; returns false on capacity overflow
// physics.py:657-699 up to the solver set-up (rows, blocks); false on capacity overflow
__device__ bool substep_front(Ctx &c, const double *arm, const double *basecmd, double dt, int sub) {
  PhaseClock pk(c);
  const DevScene &sc = *c.sc;
  const rs_physics_config &cfg = *c.cfg;
  WarpSmem &S = *c.S;
  const int lane = c.lane, nb = sc.nb, nsj = sc.nsj;

  if (!cfg.sleeping_enabled) {
    for (int b = lane; b < nb; b += 32)
      if (sc.body_kind[b] == RS_DYNAMIC && ASLEEP(c, b)) { ASLEEP(c, b) = 0; SLEEPC(c, b) = 0; RIDER(c, b) = -1; }
    __syncwarp();
  }
  bool need_fk = arm != nullptr || HELDJ(c) >= 0 || HELD(c) >= 0;
  if (arm) {
    if (lane == 0) move_base(sc, S.sd + c.L->base, basecmd[0], basecmd[1], dt);
    if (lane < sc.narm) {  // _drive_arm physics.py:608-621
      double q = JOINTS(c)[nsj + lane], err = arm[lane] - q, vdes = cfg.kp * err / dt, v;
      double cap = cfg.impulse_cap_per_control_step ? S.budget[lane] : cfg.motor_impulse_cap;
      v = vdes < -cap ? -cap : (vdes > cap ? cap : vdes);
      if (cfg.impulse_cap_per_control_step) S.budget[lane] = cap - fabs(v);
      double nq = q + v * dt, lo = sc.arm_limits[2 * lane], hi = sc.arm_limits[2 * lane + 1];
      JOINTS(c)[nsj + lane] = nq < lo ? lo : (nq > hi ? hi : nq);
    }
    __syncwarp();
  }
  if (need_fk) forward_kinematics(c);
  if (arm) {
    if (lane <= sc.narm) {
      Pose p;
      if (lane == 0) {
        base3(S.sd + c.L->base, p);
      } else {
        pose_load12(S.u.fk.links[lane - 1], p);
      }
      set_kinematic(c, sc.robot_base + lane, p, dt, true);
    }
    __syncwarp();
  }
  int dragged = HELDJ(c);
  if (lane == 0) S.dragged = dragged;
  if (dragged >= 0) {
    if (lane == 0) {  // physics.py:623-655
      int ji = dragged;
      Pose parent, origin, jf;
      body_pose(c, sc.joint_parent[ji], parent);
      pose_load12(sc.joint_origin + 12 * ji, origin);
      compose(parent, origin, jf);
      const double *ee = S.u.fk.ee + 9;
      double ax[3], qn = 0.0;
      matvec(jf.R, sc.joint_axis + 3 * ji, ax);
      bool skip = false;
      const double *ge = S.sd + c.L->grab_ee;
      double grab_q = S.sd[c.L->grab_q];
      if (sc.joint_type[ji] == RS_PRISMATIC) {
        double d[3] = {ee[0] - ge[0], ee[1] - ge[1], ee[2] - ge[2]};
        qn = grab_q + dot3(ax, d);
      } else {
        double ref[3], cur[3], cr[3];
        for (int i = 0; i < 3; ++i) { ref[i] = ge[i] - jf.p[i]; cur[i] = ee[i] - jf.p[i]; }
        double pr = dot3(ax, ref), pc = dot3(ax, cur);
        for (int i = 0; i < 3; ++i) { ref[i] -= ax[i] * pr; cur[i] -= ax[i] * pc; }
        double nr = sqrt(dot3(ref, ref)), nc = sqrt(dot3(cur, cur));
        if (nr < 1e-9 || nc < 1e-9) {
          skip = true;
        } else {
          double ca = dot3(ref, cur) / (nr * nc);
          ca = ca < -1.0 ? -1.0 : (ca > 1.0 ? 1.0 : ca);
          cross3(ref, cur, cr);
          double sgn = dot3(ax, cr);
          qn = grab_q + acos(ca) * (sgn >= 0 ? 1.0 : -1.0);
        }
      }
      if (!skip) {
        double lo = sc.joint_limits[2 * ji], hi = sc.joint_limits[2 * ji + 1];
        qn = fmin(fmax(qn, lo), hi);
        double old = JOINTS(c)[ji];
        if (qn != old) {
          JOINTS(c)[ji] = qn;
          JVEL(c)[ji] = dt > 0 ? (qn - old) / dt : 0.0;
        }
      }
    }
    __syncwarp();
    update_scene_joint_poses(c, 1 << dragged, dt);
  }
  if (HELD(c) >= 0 && HELDJ(c) < 0) {
    if (lane == 0) {  // physics.py:671-684
      Pose ee, off, hp;
      pose_load12(S.u.fk.ee, ee);
      const double *ho = S.sd + c.L->held_off;
      quat_to_mat(ho + 3, off.R);
      off.p[0] = ho[0]; off.p[1] = ho[1]; off.p[2] = ho[2];
      compose(ee, off, hp);
      set_kinematic(c, HELD(c), hp, dt, false);
    }
    __syncwarp();
  }
  // gravity + damping on awake dynamics; awake_dyn fixed here (physics.py:686-695)
  {
    unsigned long long mine = 0ull;
    for (int b = lane; b < nb; b += 32) {
      if (sc.body_kind[b] != RS_DYNAMIC || ASLEEP(c, b) || b == HELD(c)) continue;
      mine |= 1ull << b;
      double *lv = LV(c, b), *av = AV(c, b);
      lv[2] -= cfg.gravity * dt;
      for (int i = 0; i < 3; ++i) lv[i] *= cfg.lin_damping;
      for (int i = 0; i < 3; ++i) av[i] *= cfg.ang_damping;
    }
    unsigned lo32 = __reduce_or_sync(0xffffffffu, (unsigned)(mine & 0xffffffffu));
    unsigned hi32 = __reduce_or_sync(0xffffffffu, (unsigned)(mine >> 32));
    S.awake_dyn = ((unsigned long long)hi32 << 32) | lo32;
  }
  __syncwarp();

  pk.add(c, 7);
  PhaseClock pb(c);
  // ---- broadphase: AABBs through the pose-keyed cache (body_key_hit,
  // part_frame_aabb, body_aabb_store): only bodies that moved are recomputed;
  // `changed` = those
  PhaseClock pb1(c);
  // key check lanes per body (hits: the cached AABB); the parts of the moved
  // bodies recomputed lanes per part; their body AABBs (unions) lanes per body
  auto bp_store = [&](int b, const double *lo, const double *hi) {
    const bool kin = sc.body_kind[b] == RS_KINEMATIC;
    for (int i = 0; i < 3; ++i) {
      S.u.bp.lo[b][i] = kin ? lo[i] - cfg.wake_margin : lo[i];
      S.u.bp.hi[b][i] = kin ? hi[i] + cfg.wake_margin : hi[i];
    }
  };
  unsigned long long changed = 0ull;
  for (int b0 = 0; b0 < nb; b0 += 32) {
    const int b = b0 + lane;
    bool miss = false;
    if (b < nb) {
      miss = !body_key_hit(c, b);
      if (!miss) bp_store(b, c.bcache + 14 * b + 8, c.bcache + 14 * b + 11);
    }
    changed |= (unsigned long long)__ballot_sync(0xffffffffu, miss) << b0;
  }
  if (changed) {
    const int np = sc.np;
    for (int p0 = 0; p0 < np; p0 += 32) {
      const int p = p0 + lane;
      const bool hull = p < np && ((changed >> sc.part_body[p]) & 1ull) && part_frame_aabb(c, p);
      for (unsigned m = __ballot_sync(0xffffffffu, hull); m; m &= m - 1) hull_aabb_warp(c, p0 + __ffs(m) - 1);
    }
    __syncwarp();
    for (int b = lane; b < nb; b += 32)
      if ((changed >> b) & 1ull) {
        double lo[3], hi[3];
        body_aabb_store(c, b, lo, hi);
        bp_store(b, lo, hi);
      }
  }
  if (!S.cbits_valid) changed = nb == 64 ? ~0ull : ((1ull << nb) - 1ull);
  __syncwarp();
  pb1.add(c, 12);
  PhaseClock pb2(c);
  // ---- overlap candidates (inclusive AABB overlap, not static-static, not
  //      the same no-collide group) kept as a bit matrix across substeps: a
  //      pair of unchanged bodies keeps its bit; the rows / columns of the
  //      changed bodies are re-tested (lanes per partner), then the matrix is
  //      emitted in sorted (a, b) order -- the reference's SAP order
  int ncand = 0;
  bool overflow = false;
  {
    for (int a = lane; a < nb; a += 32) S.cbits[a] = ((changed >> a) & 1ull) ? 0ull : (S.cbits[a] & ~changed);
    __syncwarp();
    // lane l keeps partner y = l (AABB, kind, group) in registers and re-reads
    // partner l + 32's AABB from shared memory in the loop (both in registers
    // were spilled to local memory at the 168-register budget; both from shared
    // memory measured slower: bench physics alone 0.585 vs 0.592 (HEAD) vs
    // 0.607 ms); the changed body's data is a shared-memory broadcast.  The
    // predicate is symmetric in (a, b), so the partner order does not matter.
    double yl0[3], yh0[3];
    int yk0 = 0, yg0 = 0, yk1 = 0, yg1 = 0;
    if (changed) {
      if (lane < nb) {
        for (int i = 0; i < 3; ++i) { yl0[i] = S.u.bp.lo[lane][i]; yh0[i] = S.u.bp.hi[lane][i]; }
        yk0 = sc.body_kind[lane]; yg0 = sc.body_group[lane];
      }
      if (lane + 32 < nb) { yk1 = sc.body_kind[lane + 32]; yg1 = sc.body_group[lane + 32]; }
    }
    for (unsigned long long rest = changed; rest; rest &= rest - 1) {
      const int cb = __ffsll((long long)rest) - 1;
      const int kc = __shfl_sync(0xffffffffu, cb < 32 ? yk0 : yk1, cb & 31);  // lane cb % 32 holds body cb's
      const int gc = __shfl_sync(0xffffffffu, cb < 32 ? yg0 : yg1, cb & 31);
      const double cl0 = S.u.bp.lo[cb][0], cl1 = S.u.bp.lo[cb][1], cl2 = S.u.bp.lo[cb][2];
      const double ch0 = S.u.bp.hi[cb][0], ch1 = S.u.bp.hi[cb][1], ch2 = S.u.bp.hi[cb][2];
      auto test = [&](int y, const double (&l)[3], const double (&h)[3], int ky, int gy) {
        // pairs (cb, y > cb); pairs (y < cb, cb) once: only from an unchanged y
        if (y >= nb || y == cb || (y < cb && ((changed >> y) & 1ull))) return false;
        return !(kc == RS_STATIC && ky == RS_STATIC) && !(gc != RS_NO_GROUP && gc == gy) && cl0 <= h[0] &&
               l[0] <= ch0 && l[1] <= ch1 && cl1 <= h[1] && l[2] <= ch2 && cl2 <= h[2];
      };
      const bool ov0 = test(lane, yl0, yh0, yk0, yg0);
      bool ov1 = false;
      if (nb > 32 && lane + 32 < nb) {
        const volatile double *vl = S.u.bp.lo[lane + 32], *vh = S.u.bp.hi[lane + 32];
        const double yl1[3] = {vl[0], vl[1], vl[2]}, yh1[3] = {vh[0], vh[1], vh[2]};
        ov1 = test(lane + 32, yl1, yh1, yk1, yg1);
      }
      if (ov0 && lane < cb) S.cbits[lane] |= 1ull << cb;  // lane y owns row y
      if (ov1 && lane + 32 < cb) S.cbits[lane + 32] |= 1ull << cb;
      const unsigned long long row = (unsigned long long)__ballot_sync(0xffffffffu, ov0 && lane > cb) |
                                     ((unsigned long long)__ballot_sync(0xffffffffu, ov1 && lane + 32 > cb) << 32);
      __syncwarp();
      if (lane == 0) S.cbits[cb] |= row;
      __syncwarp();
    }
    pb2.add(c, 13);
    PhaseClock pb3(c);
    // emit the pairs in (a, b) order: row offsets by a prefix sum over the
    // rows (lanes per row; kept in S.wake_idx, scratch until the admission
    // walk), then lanes per output pair: its row by binary search over the
    // offsets, its partner as the j-th set bit of the row (rank select)
    int *const roff = S.wake_idx;
    for (int a0 = 0; a0 < nb; a0 += 32) {
      const int a = a0 + lane;
      const int cnt = a < nb ? __popcll(S.cbits[a]) : 0;
      int incl = cnt;
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
      }
      if (a < nb) roff[a] = ncand + incl - cnt;
      ncand += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    const int nemit = ncand < kMaxCand ? ncand : kMaxCand;
    for (int k = lane; k < nemit; k += 32) {
      int lo = 0, hi = nb - 1;  // the row owning k: last a with roff[a] <= k
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (roff[mid] <= k) lo = mid; else hi = mid - 1;
      }
      const unsigned long long row = S.cbits[lo];
      int j = k - roff[lo];  // rank of the partner bit within the row
      unsigned m = (unsigned)row;
      int pos = 0;
      const int nlo = __popc(m);
      if (j >= nlo) { j -= nlo; m = (unsigned)(row >> 32); pos = 32; }
      for (int w = 16; w; w >>= 1) {
        const int cw = __popc(m & ((1u << w) - 1u));
        if (j >= cw) { j -= cw; m >>= w; pos += w; }
      }
      S.u.bp.cand[k] = (uint16_t)((lo << 8) | pos);
    }
    if (lane == 0) S.cbits_valid = 1;
    pb3.add(c, 14);
  }
  if (ncand > kMaxCand) { overflow = true; if (lane == 0) S.fault = RS_OVF_CANDIDATES; }
  __syncwarp();
  pb.add(c, 8);
  PhaseClock pa(c);
  // ---- admission walk (physics.py:528-571), lanes per candidate.  The walk is
  // sequential in the reference only through wakes: a sleeping dynamic body x
  // paired with a robot/held kinematic body is woken when that pair is
  // reached, and every later pair sees x awake.  So x's state at candidate k
  // is "asleep" iff it slept at the start and k <= wake_idx[x], the index of
  // the first such waker pair -- computed first (atomicMin), then every
  // candidate is decided independently and compacted in order.
  if (!overflow) {
    const int held = HELD(c);
    for (int b = lane; b < nb; b += 32) S.wake_idx[b] = 1 << 30;
    __syncwarp();
    for (int k = lane; k < ncand; k += 32) {
      const int a = S.u.bp.cand[k] >> 8, b = S.u.bp.cand[k] & 0xff;
      const int ka = sc.body_kind[a], kb = sc.body_kind[b];
      // x asleep-dynamic at the start, the other kinematic robot/held, not x's rider joint
      if (ka == RS_DYNAMIC && ASLEEP(c, a) && kb == RS_KINEMATIC && (sc.body_robot[b] || b == held) &&
          !(sc.body_joint[b] >= 0 && RIDER(c, a) == sc.body_joint[b]))
        atomicMin(&S.wake_idx[a], k);
      if (kb == RS_DYNAMIC && ASLEEP(c, b) && ka == RS_KINEMATIC && (sc.body_robot[a] || a == held) &&
          !(sc.body_joint[a] >= 0 && RIDER(c, b) == sc.body_joint[a]))
        atomicMin(&S.wake_idx[b], k);
    }
    __syncwarp();
    int nadm = 0, nskip = 0;
    for (int k0 = 0; k0 < ncand; k0 += 32) {
      const int k = k0 + lane;
      bool adm = false, skip = false;
      if (k < ncand) {
        const int a = S.u.bp.cand[k] >> 8, b = S.u.bp.cand[k] & 0xff;
        const int ka = sc.body_kind[a], kb = sc.body_kind[b];
        const bool dyn_a = ka == RS_DYNAMIC, dyn_b = kb == RS_DYNAMIC, kin_a = ka == RS_KINEMATIC,
                   kin_b = kb == RS_KINEMATIC;
        if (!dyn_a && !dyn_b) {
          const bool robot = sc.body_robot[a] || sc.body_robot[b] || a == held || b == held;
          adm = robot || sc.body_joint[a] >= 0 || sc.body_joint[b] >= 0;
        } else {
          const bool sa = dyn_a && ASLEEP(c, a) && k <= S.wake_idx[a];
          const bool sb = dyn_b && ASLEEP(c, b) && k <= S.wake_idx[b];
          if ((sa && sb) || (sa && kb == RS_STATIC) || (sb && ka == RS_STATIC)) {
            skip = true;  // skipped_sleeping_pairs
          } else if ((sa && kin_b && sc.body_joint[b] >= 0 && RIDER(c, a) == sc.body_joint[b]) ||
                     (sb && kin_a && sc.body_joint[a] >= 0 && RIDER(c, b) == sc.body_joint[a])) {
            adm = false;  // a sleeping rider ignores its container
          } else {
            adm = true;
          }
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, adm);
      if (adm) {
        const int idx = nadm + __popc(m & ((1u << lane) - 1));
        if (idx < kMaxAdm) S.adm[idx] = S.u.bp.cand[k];
      }
      nadm += __popc(m);
      nskip += __popc(__ballot_sync(0xffffffffu, skip));
    }
    __syncwarp();
    int nwake = 0;  // wake() on each woken body (dynamic and asleep at the start by construction)
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int b = b0 + lane;
      const bool w = b < nb && S.wake_idx[b] < (1 << 30);
      if (w) { ASLEEP(c, b) = 0; SLEEPC(c, b) = 0; RIDER(c, b) = -1; }
      nwake += __popc(__ballot_sync(0xffffffffu, w));
    }
    if (lane == 0) {
      S.nadm = nadm;
      S.ctr[1] += nskip;
      S.ctr[2] += nwake;
    }
  }
  __syncwarp();
  if (overflow || S.nadm > kMaxAdm) {
    if (lane == 0 && !overflow) S.fault = RS_OVF_ADMITTED;
    return false;
  }

  pa.add(c, 9);
  PhaseClock pn(c);
  // ---- narrowphase (physics.py:703-719).  The part pairs of all admitted
  // pairs form one index space (pair k owns [off_k, off_k + na_k nb_k),
  // ii-major like the reference's part loops, geometry.py:701-716); the
  // margin-AABB cull runs over it 32 part pairs at a time and the survivors
  // are visited in index order -- the reference's pair order, then part
  // order -- each appending its contacts.  Then, lanes per pair in order:
  // the pair trace, the contact groups and the wakes of pairs with contacts
  // (wake() of a body is idempotent, so their order does not matter).
  const int nadm = S.nadm;
  int *const off = S.u.np.off, *const npc = S.u.np.npc;
  const double margin = cfg.contact_margin;
  int tot = 0;
  for (int k0 = 0; k0 < nadm; k0 += 32) {
    const int k = k0 + lane;
    int cnt = 0;
    if (k < nadm) {
      const int a = S.adm[k] >> 8, b = S.adm[k] & 0xff;
      cnt = (sc.body_part_begin[a + 1] - sc.body_part_begin[a]) * (sc.body_part_begin[b + 1] - sc.body_part_begin[b]);
      npc[k] = 0;
    }
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (k < nadm) off[k] = tot + incl - cnt;
    tot += __shfl_sync(0xffffffffu, incl, 31);
  }
  __syncwarp();
  int nct = 0;
  for (int e0 = 0; e0 < tot; e0 += 32) {
    const int e = e0 + lane;
    bool live = false;
    int k = 0, pi = 0, pj = 0;
    if (e < tot) {
      int lo = 0, hi = nadm - 1;  // the pair owning e: last k with off[k] <= e
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= e) lo = mid; else hi = mid - 1;
      }
      k = lo;
      const int a = S.adm[k] >> 8, b = S.adm[k] & 0xff;
      const int b0 = sc.body_part_begin[b], nbp = sc.body_part_begin[b + 1] - b0;
      const int r = e - off[k], ii = r / nbp;
      pi = sc.body_part_begin[a] + ii;
      pj = b0 + (r - ii * nbp);
      const double *la = c.pcache + 18 * pi + 12, *ha = la + 3, *lb = c.pcache + 18 * pj + 12, *hb = lb + 3;
      bool sep = false;
      for (int x = 0; x < 3; ++x) sep |= (la[x] > hb[x] + margin) || (lb[x] > ha[x] + margin);
      live = !sep;
    }
    for (unsigned m = __ballot_sync(0xffffffffu, live); m; m &= m - 1) {
      const int src = __ffs(m) - 1;
      const int kk = __shfl_sync(0xffffffffu, k, src);
      const int n = part_pair_contacts(c, __shfl_sync(0xffffffffu, pi, src), __shfl_sync(0xffffffffu, pj, src),
                                       margin, nct);
      nct += n;
      if (lane == 0) npc[kk] += n;
      __syncwarp();
    }
  }
  __syncwarp();
  const bool tr = c.B->trace_pairs && sub < c.B->trace_sub;
  int ngp = 0, cfirst = 0;
  unsigned long long wmask = 0ull;
  for (int k0 = 0; k0 < nadm; k0 += 32) {
    const int k = k0 + lane;
    const int a = k < nadm ? S.adm[k] >> 8 : 0, b = k < nadm ? S.adm[k] & 0xff : 0;
    const int n = k < nadm ? npc[k] : 0;
    if (tr && k < nadm && k < c.B->trace_cap) {
      int32_t *o = c.B->trace_pairs + (((size_t)c.env * c.B->trace_sub + sub) * c.B->trace_cap + k) * 3;
      o[0] = a; o[1] = b; o[2] = n;
    }
    const unsigned hm = __ballot_sync(0xffffffffu, n > 0);
    int incl = n;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (n > 0) {
      const int g = ngp + __popc(hm & ((1u << lane) - 1));
      if (g < kMaxGroups) { S.g_a[g] = a; S.g_b[g] = b; S.g_first[g] = cfirst + incl - n; S.g_n[g] = n; }
      wmask |= (1ull << a) | (1ull << b);
    }
    ngp += __popc(hm);
    cfirst += __shfl_sync(0xffffffffu, incl, 31);
  }
  wmask = ((unsigned long long)__reduce_or_sync(0xffffffffu, (unsigned)(wmask >> 32)) << 32) |
          __reduce_or_sync(0xffffffffu, (unsigned)(wmask & 0xffffffffu));
  int nwoken = 0;
  for (int b0 = 0; b0 < nb; b0 += 32) {
    const int b = b0 + lane;
    const bool w = b < nb && ((wmask >> b) & 1ull) && sc.body_kind[b] == RS_DYNAMIC && ASLEEP(c, b);
    if (w) { ASLEEP(c, b) = 0; SLEEPC(c, b) = 0; RIDER(c, b) = -1; }  // wake()
    nwoken += __popc(__ballot_sync(0xffffffffu, w));
  }
  if (lane == 0) {
    S.ctr[0] += nadm;
    S.ctr[2] += nwoken;
    S.nc = nct;
    S.ng = ngp;
    if (tr) c.B->trace_count[(size_t)c.env * c.B->trace_sub + sub] = nadm;
  }
  __syncwarp();
  if (nct > kMaxContacts || ngp > kMaxGroups) {
    if (lane == 0) S.fault = nct > kMaxContacts ? RS_OVF_CONTACTS : RS_OVF_GROUPS;
    return false;
  }
  const int nc = S.nc, ng = S.ng;

  pn.add(c, 10);
  PhaseClock pr(c);
  // ---- solver (physics.py:846-960)
  for (int b = lane; b < nb; b += 32) {
    const double *lv = LV(c, b), *av = AV(c, b);
    for (int i = 0; i < 3; ++i) { S.u.sol.vel[b][i] = lv[i]; S.u.sol.vel[b][3 + i] = av[i]; }
  }
  for (int j = lane; j < kMaxJoints; j += 32) S.jdv[j] = 0.0;
  // per-pair solver data (lanes per group)
  for (int g = lane; g < ng; g += 32) {
    double *P = c.pairs + kPairD * g;
    for (int side = 0; side < 2; ++side) {
      int bb = side ? S.g_b[g] : S.g_a[g];
      Pose bp;
      body_pose_cached(c, bb, bp);
      apply(bp, sc.com + 3 * bb, P + (side ? PCB : PCA));
      double *I = P + (side ? PIB : PIA);
      if (solver_dynamic(c, bb)) {
        double T[9], Rt[9];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) Rt[3 * i + j] = bp.R[3 * j + i];
        matmul(bp.R, sc.inv_inertia + 9 * bb, T);
        matmul(T, Rt, I);
        P[side ? PIMB : PIMA] = sc.inv_mass[bb];
      } else {
        for (int i = 0; i < 9; ++i) I[i] = 0.0;
        P[side ? PIMB : PIMA] = 0.0;
      }
    }
    int a = S.g_a[g], b = S.g_b[g];
    P[PMU] = sqrt(sc.friction[a] * sc.friction[b]);
    P[PE] = fmax(sc.restitution[a], sc.restitution[b]);
  }
  __syncwarp();
  // rows (lanes per contact, over all groups at once; the groups partition
  // the contacts in order: g_first ascending)
  for (int c0 = 0; c0 < nc; c0 += 32) {
    const int ci = c0 + lane;
    bool kpos = false;
    if (ci < nc) {
      int g = 0;
      while (g + 1 < ng && S.g_first[g + 1] <= ci) ++g;
      const double *P = c.pairs + kPairD * g;
      double *r = c.rows + kRowD * ci;
      const double *n = r + RN, *pt = r + RPT;
      r[RA] = S.g_a[g]; r[RB] = S.g_b[g]; r[RGRP] = g;
      for (int k = 0; k < 3; ++k) {
        r[RRA + k] = pt[k] - P[PCA + k];
        r[RRB + k] = pt[k] - P[PCB + k];
      }
      // (a side with zero inverse mass has a zero inverse inertia: its term is +0)
      double kk = P[PIMA] + P[PIMB], t[3], u[3], v[3];
      if (P[PIMA] > 0.0) { cross3(r + RRA, n, t); matvec(P + PIA, t, u); cross3(u, r + RRA, v); kk += dot3(n, v); }
      if (P[PIMB] > 0.0) { cross3(r + RRB, n, t); matvec(P + PIB, t, u); cross3(u, r + RRB, v); kk += dot3(n, v); }
      double jia = 0.0, jib = 0.0;
      int ja = joint_jacobian(c, S.g_a[g], pt, r + RJACA, jia);
      int jb = joint_jacobian(c, S.g_b[g], pt, r + RJACB, jib);
      r[RJA] = ja; r[RJB] = jb; r[RJIA] = jia; r[RJIB] = jib;
      if (ja >= 0) { double jn = dot3(r + RJACA, n); kk += jn * jn * jia; }
      if (jb >= 0) { double jn = dot3(r + RJACB, n); kk += jn * jn * jib; }
      // tangents physics.py:1329-1336 (read only by friction, which skips k <= 0 rows)
      if (kk > 0.0) {
        double ref[3] = {0.0, 0.0, 0.0};
        if (fabs(n[0]) < 0.9) ref[0] = 1.0; else ref[1] = 1.0;
        double *t1 = r + RT1, *t2 = r + RT2;
        cross3(n, ref, t1);
        double l = sqrt(dot3(t1, t1));
        for (int k = 0; k < 3; ++k) t1[k] /= l;
        cross3(n, t1, t2);
        l = sqrt(dot3(t2, t2));
        for (int k = 0; k < 3; ++k) t2[k] /= l;
      }
      r[RK] = kk; r[RMU] = P[PMU]; r[RIMA] = P[PIMA]; r[RIMB] = P[PIMB];
      kpos = kk > 0.0;
      r[RLAM] = r[RLT1] = r[RLT2] = 0.0;
      double vn = row_vn(c, r);
      r[RVN] = vn;
      double sep = -r[RDEPTH] > 0.0 ? -r[RDEPTH] : 0.0;
      if (sep > 0.0) {
        r[RTGT] = -sep / dt;
        r[RFRIC] = 0.0;
      } else {
        r[RTGT] = vn < -cfg.restitution_threshold ? -P[PE] * vn : 0.0;
        r[RFRIC] = 1.0;
      }
    }
    const unsigned kb = __ballot_sync(0xffffffffu, kpos);
    if (lane == 0) S.kpos[c0 >> 5] = kb;
  }
  __syncwarp();
  {  // groups with a row of k > 0 (the only ones the sweeps change): load metric for scheduling
    int act = 0;
    for (int g = lane; g < ng; g += 32) act += group_has_k(S, g);
    act = __reduce_add_sync(0xffffffffu, act);
    if (lane == 0) S.n_active = act;
  }
  if (nc) {
    // block matrices (physics.py:721-758): lanes per entry
    int koff = 0;
    for (int g = 0; g < ng; ++g) {
      const int first = S.g_first[g], m = S.g_n[g];
      double *P = c.pairs + kPairD * g;
      bool hask = m > 1 && ((S.kpos[first >> 5] >> (first & 31)) & 1u);  // first row's k > 0
      if (hask && (m > kMaxBlockRows || koff + m * m > kKCap)) {
        if (lane == 0) S.fault = m > kMaxBlockRows ? RS_OVF_BLOCK_ROWS : RS_OVF_BLOCK_MATRIX;
        return false;
      }
      if (lane == 0) { P[PHASK] = hask ? 1.0 : 0.0; P[PKOFF] = koff; P[PCLK] = 0.0; }
      if (lane < kEigSlots) { P[PMASK + lane] = -1.0; P[PSTAMP + lane] = 0.0; }
      if (hask) {
        double *K = c.K + koff;
        const double *r0 = c.rows + kRowD * first;
        for (int e = lane; e < m * m; e += 32) {
          int i = e / m, j = e % m;
          if (j < i) continue;
          const double *ri = c.rows + kRowD * (first + i), *rj = c.rows + kRowD * (first + j);
          double val = (r0[RIMA] + r0[RIMB]) * dot3(ri + RN, rj + RN);
          if (r0[RIMA] > 0.0) {
            double li[3], lj[3], t[3];
            cross3(ri + RRA, ri + RN, li); cross3(rj + RRA, rj + RN, lj);
            matvec(P + PIA, lj, t);
            val += dot3(li, t);
          }
          if (r0[RIMB] > 0.0) {
            double li[3], lj[3], t[3];
            cross3(ri + RRB, ri + RN, li); cross3(rj + RRB, rj + RN, lj);
            matvec(P + PIB, lj, t);
            val += dot3(li, t);
          }
          if (ri[RJA] >= 0 && rj[RJA] >= 0 && ri[RJA] == rj[RJA])
            val += dot3(ri + RJACA, ri + RN) * dot3(rj + RJACA, rj + RN) * ri[RJIA];
          if (ri[RJB] >= 0 && rj[RJB] >= 0 && ri[RJB] == rj[RJB])
            val += dot3(ri + RJACB, ri + RN) * dot3(rj + RJACB, rj + RN) * ri[RJIB];
          if (i == j) val += 1e-9;
          K[i * m + j] = val;
          K[j * m + i] = val;
        }
        koff += m * m;
      }
    }
    __syncwarp();
  }
  __syncwarp();
  pr.add(c, 11);
  return true;
}

// Gauss-Seidel sweeps, single warp (physics.py:915-937)
__device__ void substep_sweeps(Ctx &c) {
  const rs_physics_config &cfg = *c.cfg;
  WarpSmem &S = *c.S;
  const int lane = c.lane, nc = S.nc, ng = S.ng;
  if (!nc) return;
    // blocks in sorted pair order (physics.py:931-937).
    // Rows with k <= 0 are no-ops in the reference (physics.py:1294): when
    // every row is such, the sweeps change nothing and are skipped.
    if (S.n_active > 0) {  // some row has k > 0
      for (int it = 0; it < cfg.solver_iterations; ++it)
        for (int g = 0; g < ng; ++g) {
          const int first = S.g_first[g], m = S.g_n[g];
          const double *P = c.pairs + kPairD * g;
          if (P[PHASK] == 0.0) {
            PhaseClock pr(c);
            if (lane == 0)
              for (int i = 0; i < m; ++i) row_solve(c, c.rows + kRowD * (first + i));
            __syncwarp();
            pr.add(c, 5);
          } else {
            const int koff = (int)P[PKOFF];
            solve_block(c, g, first, m, c.K + koff, S.u.sol.ws, c.W, c.Vc + kEigSlots * koff, c.evc + kEigSlots * first);
          }
        }
    }
    __syncwarp();
}

// physics.py:939-1035: velocity write-back, events, integration, joints
__device__ void substep_back(Ctx &c, double dt) {
  const DevScene &sc = *c.sc;
  const rs_physics_config &cfg = *c.cfg;
  WarpSmem &S = *c.S;
  const int lane = c.lane, nb = sc.nb, nsj = sc.nsj, nc = S.nc, ng = S.ng, dragged = S.dragged;
  if (nc) {
    for (int b = lane; b < nb; b += 32)
      if (solver_dynamic(c, b)) {
        double *lv = LV(c, b), *av = AV(c, b);
        for (int i = 0; i < 3; ++i) { lv[i] = S.u.sol.vel[b][i]; av[i] = S.u.sol.vel[b][3 + i]; }
      }
    // events + force tally in row order: each row's impulse lanes-parallel,
    // then lane 0 visits the rows that register one, in order
    const int held = HELD(c);
    double acc = lane == 0 ? S.sd[c.L->acc] : 0.0;  // lane 0 owns the tally
    for (int i0 = 0; i0 < nc; i0 += 32) {
      double lam = 0.0;
      if (i0 + lane < nc) {
        const double *r = c.rows + kRowD * (i0 + lane);
        lam = r[RLAM];
        if (r[RK] <= 0.0) lam = fmax(-r[RVN], 0.0);
      }
      for (unsigned m = __ballot_sync(0xffffffffu, i0 + lane < nc && !(lam <= 0.0)); m; m &= m - 1) {
        const int src = __ffs(m) - 1;
        const double l = __shfl_sync(0xffffffffu, lam, src);
        if (lane == 0) {
          const double *r = c.rows + kRowD * (i0 + src);
          const double force = l / dt;
          emit_event(c, r, l, force);
          const int a = (int)r[RA], b = (int)r[RB];
          if (sc.body_robot[a] || sc.body_robot[b] || a == held || b == held) acc += force;
        }
      }
    }
    if (lane == 0) S.sd[c.L->acc] = acc;
    __syncwarp();
  }

  // ---- integrate (physics.py:962-1011): lanes per body.  The corrections
  // read every body's sleep flag as it was before this loop (the reference
  // computes all of them first): a snapshot of the flags, because a lane may
  // put its body to sleep while another lane (or its own second round, body
  // b + 32) is still summing the corrections of a contact with it.
  {
    const int held = HELD(c);
    unsigned long long asleep0 = 0ull;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const unsigned m = __ballot_sync(0xffffffffu, b0 + lane < nb && ASLEEP(c, b0 + lane));
      asleep0 |= (unsigned long long)m << b0;
    }
    __syncwarp();
    for (int b = lane; b < nb; b += 32) {
      if (!((S.awake_dyn >> b) & 1ull)) continue;
      double corr[3] = {0.0, 0.0, 0.0};
      int cnt = 0;
      for (int g = 0; g < ng; ++g) {
        int a = S.g_a[g], bb = S.g_b[g];
        if (a != b && bb != b) continue;
        double ima = (!((asleep0 >> a) & 1ull) && a != held) ? sc.inv_mass[a] : 0.0;
        double imb = (!((asleep0 >> bb) & 1ull) && bb != held) ? sc.inv_mass[bb] : 0.0;
        double tot = ima + imb;
        if (tot <= 0.0) continue;
        for (int i = S.g_first[g]; i < S.g_first[g] + S.g_n[g]; ++i) {
          const double *r = c.rows + kRowD * i;
          double push = cfg.correction_factor * fmax(r[RDEPTH] - cfg.slop, 0.0);
          if (push <= 0.0) continue;
          if (a == b && ima > 0.0) {
            double s = push * ima / tot;
            for (int k = 0; k < 3; ++k) corr[k] += r[RN + k] * s;
            cnt++;
          }
          if (bb == b && imb > 0.0) {
            double s = push * imb / tot;
            for (int k = 0; k < 3; ++k) corr[k] -= r[RN + k] * s;
            cnt++;
          }
        }
      }
      if (cnt > 1) for (int k = 0; k < 3; ++k) corr[k] /= cnt;
      double *lv = LV(c, b), *av = AV(c, b);
      double lin = sqrt(dot3(lv, lv)), ang = sqrt(dot3(av, av));
      bool below = lin < cfg.sleep_lin_threshold && ang < cfg.sleep_ang_threshold;
      bool has_corr = cnt > 0 && dot3(corr, corr) >= 1e-14;
      if (below && cfg.sleeping_enabled && !has_corr) {
        SLEEPC(c, b)++;
        if (SLEEPC(c, b) >= cfg.sleep_substeps) {
          ASLEEP(c, b) = 1;
          lv[0] = lv[1] = lv[2] = 0.0;
          av[0] = av[1] = av[2] = 0.0;
        }
        continue;
      }
      SLEEPC(c, b) = 0;
      double *pos = POS(c, b);
      for (int k = 0; k < 3; ++k) pos[k] = pos[k] + lv[k] * dt;
      if (ang > 0.0) {  // geometry.py:110-114
        double wq[4] = {0.0, av[0], av[1], av[2]}, d[4], *q = QUAT(c, b);
        quat_mul(wq, q, d);
        double h = 0.5 * dt;
        for (int k = 0; k < 4; ++k) q[k] = q[k] + h * d[k];
        double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        for (int k = 0; k < 4; ++k) q[k] /= n;
      }
      if (has_corr) for (int k = 0; k < 3; ++k) pos[k] += corr[k];
    }
    __syncwarp();
  }
  // ---- scene joints (physics.py:1013-1035)
  if (lane == 0) {
    int moved = 0;
    for (int ji = 0; ji < nsj; ++ji) {
      if (ji == dragged) continue;
      double *jv = JVEL(c) + ji;
      *jv += S.jdv[ji];
      *jv *= cfg.joint_damping;
      if (fabs(*jv) < 1e-4) { *jv = 0.0; continue; }
      double lo = sc.joint_limits[2 * ji], hi = sc.joint_limits[2 * ji + 1];
      double q = JOINTS(c)[ji] + *jv * dt;
      if (q <= lo) { q = lo; *jv = 0.0; }
      else if (q >= hi) { q = hi; *jv = 0.0; }
      if (q != JOINTS(c)[ji]) { JOINTS(c)[ji] = q; moved |= 1 << ji; }
    }
    S.moved_mask = moved;
  }
  __syncwarp();
  int moved = S.moved_mask;
  if (moved) update_scene_joint_poses(c, moved, dt);
}

__device__ bool substep(Ctx &c, const double *arm, const double *basecmd, double dt, int sub) {
  PhaseClock p0(c);
  if (!substep_front(c, arm, basecmd, dt, sub)) return false;
  p0.add(c, 0);
  PhaseClock p1(c);
  substep_sweeps(c);
  p1.add(c, 1);
  PhaseClock p2(c);
  substep_back(c, dt);
  p2.add(c, 6);
  return true;
}

// ---------------------------------------------------------------------------
// Contact-heavy envs: one CTA of kHeavyWarps warps per env.  Warp 0 runs every
// phase as in the warp-per-env kernel; the Gauss-Seidel sweeps are run by all
// warps over a wavefront schedule of the contact groups.  Group g depends on
// every earlier group h < g that shares a velocity it writes (a body with
// non-zero solver inverse mass, or a scene joint's joint_dv); groups of one
// level touch disjoint state, so solving them concurrently gives bit-identical
// results to the reference's sequential order (physics.py:931-937).
constexpr int kHeavyWarps = 16;  // the widest CTA (scratch is sized for it)
// batches up to this size run their contact-heavy envs in 16-warp CTAs (8 above)
constexpr int kWideHeavyMaxEnvs = 2048;
// envs with >= this many active contact groups go to the CTA kernel in the next
// step: 3 with the 16-warp CTAs, 2 with the 8-warp ones (measured)
__host__ __device__ inline int heavy_groups(int n_env) { return n_env <= kWideHeavyMaxEnvs ? 3 : 2; }

template <int kW>
struct HeavyShared {
  BlockWS ws[kW - 1];  // block-solver workspaces of warps 1..
  unsigned long long res[kMaxGroups];  // per group: the body velocities it writes
  unsigned resj[kMaxGroups];           // ... and the scene joints' joint_dv
  int16_t level[kMaxGroups];           // wavefront level (-1: no row with k > 0)
  int16_t lvl_order[kMaxGroups];
  int16_t lvl_start[kMaxGroups + 1];
  int nlev, ok;
};

// wavefront levels of the active groups (warp 0, warp-collective): group g's
// level is 1 + the highest level of an earlier active group sharing a written
// velocity (lanes over the earlier groups, max-reduced), 0 if none
template <class HS>
__device__ void build_levels(Ctx &c, HS &H) {
  WarpSmem &S = *c.S;
  const int ng = S.ng, lane = c.lane;
  for (int g = lane; g < ng; g += 32) {
    const bool act = group_has_k(S, g);
    unsigned long long rs = 0ull;
    unsigned rj = 0u;
    if (act) {
      const double *r0 = c.rows + kRowD * S.g_first[g];
      if (r0[RIMA] > 0.0) rs |= 1ull << (int)r0[RA];
      if (r0[RIMB] > 0.0) rs |= 1ull << (int)r0[RB];
      if (r0[RJA] >= 0.0) rj |= 1u << (int)r0[RJA];
      if (r0[RJB] >= 0.0) rj |= 1u << (int)r0[RJB];
    }
    H.res[g] = rs;
    H.resj[g] = rj;
    H.level[g] = act ? 0 : -1;
  }
  __syncwarp();
  int nlev = 0;
  for (int g = 0; g < ng; ++g) {
    if (H.level[g] < 0) continue;
    const unsigned long long rs = H.res[g];
    const unsigned rj = H.resj[g];
    int lv = -1;
    for (int h = lane; h < g; h += 32)
      if (H.level[h] >= 0 && ((H.res[h] & rs) || (H.resj[h] & rj)) && H.level[h] > lv) lv = H.level[h];
    lv = __reduce_max_sync(0xffffffffu, lv) + 1;
    __syncwarp();
    if (lane == 0) H.level[g] = (int16_t)lv;
    __syncwarp();
    if (lv + 1 > nlev) nlev = lv + 1;
  }
  if (lane == 0) {  // groups ordered by level, group order within a level (counting sort)
    int count[kMaxGroups + 1];
    for (int l = 0; l <= nlev; ++l) count[l] = 0;
    for (int g = 0; g < ng; ++g)
      if (H.level[g] >= 0) count[H.level[g] + 1]++;
    for (int l = 0; l < nlev; ++l) count[l + 1] += count[l];
    for (int l = 0; l <= nlev; ++l) H.lvl_start[l] = (int16_t)count[l];
    for (int g = 0; g < ng; ++g)
      if (H.level[g] >= 0) H.lvl_order[count[H.level[g]]++] = (int16_t)g;
    H.nlev = nlev;
  }
  __syncwarp();
}

// all warps of the CTA; ends with a CTA barrier
template <int kW>
__device__ void sweeps_cta(Ctx &c, HeavyShared<kW> &H, int warp, BlockWS &ws, double *W) {
  const int iters = c.cfg->solver_iterations, nlev = H.nlev;
  for (int it = 0; it < iters; ++it)
    for (int l = 0; l < nlev; ++l) {
      for (int idx = H.lvl_start[l] + warp; idx < H.lvl_start[l + 1]; idx += kW) {
        const int g = H.lvl_order[idx];
        const int first = c.S->g_first[g], m = c.S->g_n[g];
        const double *P = c.pairs + kPairD * g;
        if (P[PHASK] == 0.0) {
          if (c.lane == 0)
            for (int i = 0; i < m; ++i) row_solve(c, c.rows + kRowD * (first + i));
          __syncwarp();
        } else {
          const int koff = (int)P[PKOFF];
          solve_block(c, g, first, m, c.K + koff, ws, W, c.Vc + kEigSlots * koff, c.evc + kEigSlots * first);
        }
      }
      __syncthreads();
    }
}

__host__ __device__ size_t step_scratch_doubles_per_env(int row_cap);

// a faulted env keeps its input state (the reference raises before mutating)
__device__ void copy_through(const DevBatch &B, int env, int lane) {
  const StateLayout &L = B.L;
  const double *a = B.sd + (size_t)env * L.dbl_size;
  double *b = B.sd_out + (size_t)env * L.dbl_size;
  for (int i = lane; i < L.dbl_size; i += 32) b[i] = a[i];
  const int32_t *x = B.si + (size_t)env * L.int_size;
  int32_t *y = B.si_out + (size_t)env * L.int_size;
  for (int i = lane; i < L.int_size; i += 32) y[i] = x[i];
}

// per-env context over the batch scratch (any warp of the env's CTA)
__device__ void make_ctx(Ctx &c, const DevBatch &B, WarpSmem &S, int env, int lane, int warp) {
  c.sc = &S.sc;
  c.B = &B;
  c.cfg = &B.cfg;
  c.S = &S;
  c.env = env;
  c.lane = lane;
  c.L = &B.L;
  const size_t per_env = step_scratch_doubles_per_env(B.row_cap);
  c.rows = B.row_scratch + per_env * env;
  c.pairs = c.rows + (size_t)B.row_cap * kRowD;
  c.K = c.pairs + kMaxGroups * kPairD;
  c.Vc = c.K + kKCap;
  c.evc = c.Vc + kEigSlots * kKCap;
  c.bcache = c.evc + kEigSlots * kMaxContacts;
  c.pcache = c.bcache + 14 * kMaxBodies;
  c.ccache = c.pcache + 18 * kMaxPartsCache;
  c.W = c.ccache + kMaxBodies + 1 + (size_t)warp * kMaxBlockRows * kMaxBlockRows;
}

// stage scene header + state slab, _check_finite (physics.py:596-606), per-step
// set-up; false if the env faulted (its input state is copied through).  One warp.
__device__ bool env_begin(Ctx &c, const DevBatch &B, int env) {
  WarpSmem &S = *c.S;
  const StateLayout &L = B.L;
  const int lane = c.lane;
  {
    const uint32_t *src = reinterpret_cast<const uint32_t *>(&B.scenes[B.env_scene[env]]);
    uint32_t *dst = reinterpret_cast<uint32_t *>(&S.sc);
    for (int i = lane; i < (int)(sizeof(DevScene) / 4); i += 32) dst[i] = src[i];
  }
  const double *gsd = B.sd + (size_t)env * L.dbl_size;
  const int32_t *gsi = B.si + (size_t)env * L.int_size;
  for (int i = lane; i < L.stage; i += 32) S.sd[i] = gsd[i];
  for (int i = lane; i < L.int_size; i += 32) S.si[i] = gsi[i];
  if (lane < 3) S.ctr[lane] = 0;
  if (lane == 0) { B.event_count[env] = 0; S.fault = 0; S.max_active = 0; }
  __syncwarp();
  const DevScene &sc = *c.sc;
  uint32_t f = 0;
  for (int cls = 0; cls < 4 && !f; ++cls) {
    int n = cls == 3 ? L.nj : sc.nb, best = 1 << 30;
    for (int i = lane; i < n; i += 32) {
      bool bad = false;
      if (cls == 0) { const double *p = POS(c, i); bad = !isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2]); }
      if (cls == 1) { const double *q = QUAT(c, i); bad = !isfinite(q[0]) || !isfinite(q[1]) || !isfinite(q[2]) || !isfinite(q[3]); }
      if (cls == 2) { const double *v = LV(c, i); bad = !isfinite(v[0]) || !isfinite(v[1]) || !isfinite(v[2]); }
      if (cls == 3) bad = !isfinite(JOINTS(c)[i]);
      if (bad && i < best) best = i;
    }
    best = __reduce_min_sync(0xffffffffu, best);
    if (best < (1 << 30)) f = ((uint32_t)(cls + 1) << 16) | (uint32_t)best;
  }
  if (f) {
    if (lane == 0) B.fault[env] = f;
    copy_through(B, env, lane);
    return false;
  }
  if (lane < kMaxArm) S.budget[lane] = B.cfg.motor_impulse_cap;
  {  // candidate bit matrix of the last completed step (invalid until env_end stores it again)
    const unsigned long long *cg = reinterpret_cast<const unsigned long long *>(c.ccache);
    const bool valid = cg[kMaxBodies] == 1ull;
    for (int b = lane; b < kMaxBodies; b += 32) S.cbits[b] = valid ? cg[b] : 0ull;
    __syncwarp();
    if (lane == 0) {
      S.cbits_valid = valid;
      reinterpret_cast<unsigned long long *>(c.ccache)[kMaxBodies] = 0ull;
    }
  }
  __syncwarp();
  return true;
}

// time / step index / counters, write the successor slab (physics.py:592-594). One warp.
__device__ void env_end(Ctx &c, const DevBatch &B, int env, double dt, bool ok, uint8_t *heavy_out) {
  WarpSmem &S = *c.S;
  const StateLayout &L = B.L;
  const int lane = c.lane;
  // the step's most active contact groups (saturating byte): >= heavy_groups ->
  // the CTA kernel next step; >= 1 -> early in a busy-first dispatch order
  if (lane == 0 && heavy_out) heavy_out[env] = (uint8_t)(S.max_active < 255 ? S.max_active : 255);
  if (!ok) {
    if (lane == 0) B.fault[env] = ((uint32_t)RS_FAULT_OVERFLOW << 16) | (uint32_t)S.fault;
    copy_through(B, env, lane);
    return;
  }
  if (lane == 0) {
    S.sd[L.time] += dt;
    B.step_index[env] += 1;
    B.fault[env] = 0;
    for (int i = 0; i < 3; ++i) B.counters[3 * env + i] += S.ctr[i];
  }
  {
    unsigned long long *cg = reinterpret_cast<unsigned long long *>(c.ccache);
    for (int b = lane; b < kMaxBodies; b += 32) cg[b] = S.cbits[b];
    __syncwarp();
    if (lane == 0) cg[kMaxBodies] = S.cbits_valid ? 1ull : 0ull;
  }
  __syncwarp();
  double *wsd = B.sd_out + (size_t)env * L.dbl_size;
  int32_t *wsi = B.si_out + (size_t)env * L.int_size;
  for (int i = lane; i < L.stage; i += 32) wsd[i] = S.sd[i];
  const double *rsd = B.sd + (size_t)env * L.dbl_size;  // rider offsets: unchanged by the step
  for (int i = L.stage + lane; i < L.dbl_size; i += 32) wsd[i] = rsd[i];
  for (int i = lane; i < L.int_size; i += 32) wsi[i] = S.si[i];
}

// warp per env (envs not flagged heavy by the previous step)
// kClass: 0 every non-heavy env; 1 the quiet ones (no active contact group in
// the previous step); 2 the busy ones (1 <= groups < heavy_groups), compiled
// for 4 CTAs per SM -- 255 registers, no spills, lower latency for the envs
// whose contact work sets the step's tail, while the many quiet envs keep the
// 5-CTA footprint that co-resides with the render
template <int kClass>
__global__ void __launch_bounds__(32 * kWarpsPerBlock, kClass == 2 ? 4 : kStepMinBlocks) step_kernel(DevBatch B, const double *arm_targets,
                                                                   const double *base_cmd, int base_stride,
                                                                   const uint8_t *has_targets, double dt,
                                                                   int substeps, const uint8_t *heavy_in,
                                                                   uint8_t *heavy_out) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const size_t stride = warp_smem_bytes(B.L.stage);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = blockIdx.x * kWarpsPerBlock + warp;
  if (slot >= B.n_env) return;
  const int env = B.env_order ? B.env_order[slot] : slot;
  if (heavy_in && heavy_in[env] >= heavy_groups(B.n_env)) return;
  if (kClass == 1 && heavy_in[env] != 0) return;
  if (kClass == 2 && heavy_in[env] == 0) return;
  if (B.env_active && !B.env_active[env]) {  // not stepping (rs_settle): state copied through
    copy_through(B, env, lane);
    if (lane == 0 && heavy_out) heavy_out[env] = 0;
    return;
  }
  const long long t_begin = B.env_cycles ? clock64() : 0;
  WarpSmem &S = *reinterpret_cast<WarpSmem *>(dsm + stride * warp);
  Ctx c;
  make_ctx(c, B, S, env, lane, 0);
  if (!env_begin(c, B, env)) return;
  const DevScene &sc = *c.sc;
  const bool ht = has_targets == nullptr || has_targets[env];
  const double *arm = ht ? arm_targets + (size_t)env * sc.narm : nullptr;
  const double *bc = base_cmd + (size_t)env * base_stride;
  const double dts = dt / substeps;
  bool ok = true;
  for (int s = 0; s < substeps && ok; ++s) {
    ok = substep(c, arm, bc, dts, s);
    if (lane == 0 && S.n_active > S.max_active) S.max_active = S.n_active;
  }
  __syncwarp();
  env_end(c, B, env, dt, ok, heavy_out);
  if (B.env_cycles && lane == 0) B.env_cycles[env] = clock64() - t_begin;
}

// CTA of kW warps per env (envs flagged heavy by the previous step)
template <int kW>
__global__ void __launch_bounds__(32 * kW) step_kernel_cta(DevBatch B, const double *arm_targets,
                                                                   const double *base_cmd, int base_stride,
                                                                   const uint8_t *has_targets, double dt,
                                                                   int substeps, const uint8_t *heavy_in,
                                                                   uint8_t *heavy_out) {
  extern __shared__ __align__(16) unsigned char dsm[];
  WarpSmem &S = *reinterpret_cast<WarpSmem *>(dsm);
  HeavyShared<kW> &H = *reinterpret_cast<HeavyShared<kW> *>(dsm + warp_smem_bytes(B.L.stage));
  const int env = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (heavy_in[env] < heavy_groups(B.n_env)) return;
  if (B.env_active && !B.env_active[env]) {
    if (threadIdx.x < 32) copy_through(B, env, threadIdx.x);
    if (threadIdx.x == 0) heavy_out[env] = 0;
    return;
  }
  const long long t_begin = B.env_cycles ? clock64() : 0;
  Ctx c;
  make_ctx(c, B, S, env, lane, warp);
  if (warp == 0) {
    bool ok = env_begin(c, B, env);
    if (lane == 0) H.ok = ok;
  }
  __syncthreads();
  const bool ok0 = H.ok;
  __syncthreads();  // every warp has read H.ok before warp 0 rewrites it in the substep loop
  if (!ok0) return;
  const DevScene &sc = *c.sc;
  const bool ht = has_targets == nullptr || has_targets[env];
  const double *arm = ht ? arm_targets + (size_t)env * sc.narm : nullptr;
  const double *bc = base_cmd + (size_t)env * base_stride;
  const double dts = dt / substeps;
  BlockWS &ws = warp == 0 ? S.u.sol.ws : H.ws[warp - 1];
  bool ok = true;
  for (int s = 0; s < substeps; ++s) {
    if (warp == 0) {
      const bool f = substep_front(c, arm, bc, dts, s);
      if (lane == 0) {
        H.ok = f;
        if (S.n_active > S.max_active) S.max_active = S.n_active;
      }
      if (f) build_levels(c, H);
    }
    __syncthreads();
    ok = H.ok;
    if (!ok) break;
    sweeps_cta(c, H, warp, ws, c.W);
    if (warp == 0) substep_back(c, dts);
    __syncthreads();
  }
  if (warp == 0) env_end(c, B, env, dt, ok, heavy_out);
  if (B.env_cycles && threadIdx.x == 0) B.env_cycles[env] = -(clock64() - t_begin);  // negative: CTA kernel
}

__host__ __device__ size_t step_scratch_doubles_per_env(int row_cap) {
  return (size_t)row_cap * kRowD + kMaxGroups * kPairD + (1 + kEigSlots) * kKCap + kEigSlots * kMaxContacts +
         14 * kMaxBodies +
         18 * kMaxPartsCache + kMaxBodies + 1 +
         (size_t)kHeavyWarps * kMaxBlockRows * kMaxBlockRows;
}
int step_row_cap() { return kMaxContacts; }

// Busy-first dispatch order of the warp-per-env kernel (rs_set_env_order,
// policy 1): a stable partition of the scene-sorted order into envs that had
// active contact groups last step (1 <= groups < heavy_groups: this kernel's
// latency tail) first, then the quiet ones, then the CTA kernel's heavy envs
// (they exit at once).  With more envs than resident warps, the expensive
// envs then start in the first wave instead of wherever their index falls.
// The envs are independent: the order changes no result.
constexpr int kOrderThreads = 1024;
__global__ void __launch_bounds__(kOrderThreads) env_order_kernel(int n, int thr, const int32_t *scene_order,
                                                                  const uint8_t *heavy_in, int32_t *out) {
  // one CTA: each thread takes a contiguous run of the scene order, counts its
  // envs per bucket (3 x 21-bit fields of one 64-bit word), one block-wide
  // exclusive scan gives every run its output offsets, then the runs are written
  using Scan = cub::BlockScan<unsigned long long, kOrderThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long total;
  const int per = (n + kOrderThreads - 1) / kOrderThreads, i0 = threadIdx.x * per, i1 = min(n, i0 + per);
  auto bucket = [&](int e) {
    const int v = heavy_in[e];
    return v >= thr ? 2 : (v >= 1 ? 0 : 1);
  };
  unsigned long long mine = 0ull;
  for (int i = i0; i < i1; ++i) mine += 1ull << (21 * bucket(scene_order[i]));
  unsigned long long before;
  Scan(tmp).ExclusiveSum(mine, before);
  if (threadIdx.x == kOrderThreads - 1) total = before + mine;
  __syncthreads();
  const unsigned long long m = (1ull << 21) - 1ull, t = total;
  const int c0 = (int)(t & m), c1 = (int)((t >> 21) & m);
  int off[3] = {(int)(before & m), c0 + (int)((before >> 21) & m), c0 + c1 + (int)((before >> 42) & m)};
  for (int i = i0; i < i1; ++i) {
    const int e = scene_order[i];
    out[off[bucket(e)]++] = e;
  }
}

cudaError_t launch_env_order(const DevBatch &B, const int32_t *scene_order, const uint8_t *heavy_in, int32_t *out,
                             cudaStream_t stream) {
  env_order_kernel<<<1, kOrderThreads, 0, stream>>>(B.n_env, heavy_groups(B.n_env), scene_order, heavy_in, out);
  return cudaGetLastError();
}

cudaError_t launch_step(const DevBatch &B, const double *arm, const double *base_cmd, int base_stride,
                        const uint8_t *has_targets, double dt, int substeps, cudaStream_t stream,
                        const uint8_t *heavy_in, uint8_t *heavy_out, cudaStream_t side, cudaEvent_t fork,
                        cudaEvent_t join, int force_width, cudaStream_t side2, cudaEvent_t join2) {
  // kernel attributes are per device context: configure each device once
  static std::atomic<unsigned long long> configured{0ull};
  const size_t ws0 = warp_smem_bytes(B.L.stage), wsmax = warp_smem_bytes(kStageD);
  const size_t smem = ws0 * kWarpsPerBlock;
  const size_t smem16 = ws0 + sizeof(HeavyShared<16>), smem8 = ws0 + sizeof(HeavyShared<8>);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (!(configured.load() >> dev & 1ull)) {
    // sized for the largest staged slab any batch can have
    e = cudaFuncSetAttribute(step_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(wsmax * kWarpsPerBlock));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(step_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(wsmax * kWarpsPerBlock));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(step_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(wsmax * kWarpsPerBlock));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(step_kernel_cta<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(wsmax + sizeof(HeavyShared<16>)));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(step_kernel_cta<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(wsmax + sizeof(HeavyShared<8>)));
    if (e != cudaSuccess) return e;
    configured.fetch_or(1ull << dev);
  }
  if (heavy_in && side) {
    // contact-heavy envs (flagged by the previous step) on a second stream, first
    cudaEventRecord(fork, stream);
    cudaStreamWaitEvent(side, fork, 0);
    // 16 warps per heavy env for batches up to 2048 envs; 8 for larger ones,
    // whose many heavy envs would crowd the SMs with mostly idle warps
    // (measured: bench 2048 envs +2 % with 16; configs[2] 4096 envs Interact
    // 568 k with 8 vs 500 k with 16)
    if (force_width ? force_width == 16 : B.n_env <= kWideHeavyMaxEnvs)
      step_kernel_cta<16><<<B.n_env, 32 * 16, smem16, side>>>(B, arm, base_cmd, base_stride, has_targets, dt,
                                                              substeps, heavy_in, heavy_out);
    else
      step_kernel_cta<8><<<B.n_env, 32 * 8, smem8, side>>>(B, arm, base_cmd, base_stride, has_targets, dt,
                                                           substeps, heavy_in, heavy_out);
    cudaEventRecord(join, side);
  }
  dim3 grid((B.n_env + kWarpsPerBlock - 1) / kWarpsPerBlock);
  if (heavy_in && side && side2) {  // busy envs on their own stream, quiet ones here (concurrently)
    cudaStreamWaitEvent(side2, fork, 0);
    step_kernel<2><<<grid, 32 * kWarpsPerBlock, smem, side2>>>(B, arm, base_cmd, base_stride, has_targets, dt,
                                                              substeps, heavy_in, heavy_out);
    cudaEventRecord(join2, side2);
    step_kernel<1><<<grid, 32 * kWarpsPerBlock, smem, stream>>>(B, arm, base_cmd, base_stride, has_targets, dt,
                                                               substeps, heavy_in, heavy_out);
    cudaStreamWaitEvent(stream, join2, 0);
  } else {
    step_kernel<0><<<grid, 32 * kWarpsPerBlock, smem, stream>>>(B, arm, base_cmd, base_stride, has_targets, dt,
                                                               substeps, heavy_in && side ? heavy_in : nullptr, heavy_out);
  }
  if (heavy_in && side) cudaStreamWaitEvent(stream, join, 0);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ grasp
// robot.py:323-346 grasp_rule + physics.py:1039-1079 grasp_candidates /
// apply_grasp; one thread per env, between control steps.
__global__ void grasp_kernel(DevBatch B, const double *gripper, int stride) {
  const int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env >= B.n_env) return;
  const DevScene &sc = B.scenes[B.env_scene[env]];
  const StateLayout &L = B.L;
  double *sd = B.sd + (size_t)env * L.dbl_size;
  int32_t *si = B.si + (size_t)env * L.int_size;
  const double g = gripper[(size_t)stride * env];
  const bool holding = si[L.held] >= 0;
  if (g < 0 && holding) {
    int h = si[L.held];
    if (si[L.held_joint] < 0) { si[L.asleep + h] = 0; si[L.sleep_ctr + h] = 0; }
    si[L.held] = -1;
    si[L.held_joint] = -1;
    return;
  }
  if (!(g > 0) || holding) return;
  // end-effector pose (robot.py:161-169)
  Pose t, off, rot, ee;
  base3(sd + L.base, t);
  rot_z(0.0, off.R);
  rot.p[0] = rot.p[1] = rot.p[2] = 0.0;
  for (int i = 0; i < sc.narm; ++i) {
    off.p[0] = sc.arm_offset[3 * i]; off.p[1] = sc.arm_offset[3 * i + 1]; off.p[2] = sc.arm_offset[3 * i + 2];
    compose(t, off, t);
    axis_angle_mat(sc.arm_axis + 3 * i, sd[L.joints + sc.nsj + i], rot.R);
    compose(t, rot, t);
  }
  Pose gp = {{1, 0, 0, 0, 1, 0, 0, 0, 1}, {sc.gripper[0], sc.gripper[1], sc.gripper[2]}};
  compose(t, gp, ee);
  double best_d = 0.0;
  int best_b = -1, best_j = -1;
  auto consider = [&](double d, int body, int joint) {
    if (!(d <= 0.15)) return;
    if (best_b < 0 || d < best_d || (d == best_d && body < best_b)) { best_d = d; best_b = body; best_j = joint; }
  };
  for (int k = 0; k < sc.nclutter; ++k) {
    int b = sc.clutter[k];
    if (b == si[L.held]) continue;
    Pose bp;
    quat_to_mat(sd + L.quat + 4 * b, bp.R);
    bp.p[0] = sd[L.pos + 3 * b]; bp.p[1] = sd[L.pos + 3 * b + 1]; bp.p[2] = sd[L.pos + 3 * b + 2];
    double com[3], e[3];
    apply(bp, sc.com + 3 * b, com);
    for (int i = 0; i < 3; ++i) e[i] = ee.p[i] - com[i];
    consider(sqrt(dot3(e, e)), b, -1);
  }
  for (int ji = 0; ji < sc.nsj; ++ji) {
    Pose parent, origin, motion, tt, child;
    int pb = sc.joint_parent[ji];
    quat_to_mat(sd + L.quat + 4 * pb, parent.R);
    parent.p[0] = sd[L.pos + 3 * pb]; parent.p[1] = sd[L.pos + 3 * pb + 1]; parent.p[2] = sd[L.pos + 3 * pb + 2];
    pose_load12(sc.joint_origin + 12 * ji, origin);
    compose(parent, origin, tt);
    double q = sd[L.joints + ji];
    if (sc.joint_type[ji] == RS_REVOLUTE) {
      axis_angle_mat(sc.joint_axis + 3 * ji, q, motion.R);
      motion.p[0] = motion.p[1] = motion.p[2] = 0.0;
    } else {
      const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
      for (int k = 0; k < 9; ++k) motion.R[k] = I[k];
      for (int k = 0; k < 3; ++k) motion.p[k] = sc.joint_axis[3 * ji + k] * q;
    }
    compose(tt, motion, child);
    double h[3], e[3];
    apply(child, sc.joint_handle + 3 * ji, h);
    for (int i = 0; i < 3; ++i) e[i] = ee.p[i] - h[i];
    consider(sqrt(dot3(e, e)), sc.joint_body[ji], ji);
  }
  if (best_b < 0) return;
  if (best_j >= 0) {
    si[L.held_joint] = best_j;
    si[L.held] = best_b;
    sd[L.grab_q] = sd[L.joints + best_j];
    for (int i = 0; i < 3; ++i) sd[L.grab_ee + i] = ee.p[i];
    return;
  }
  const int b = best_b;
  if (si[L.asleep + b]) B.counters[3 * env + 2] += 1;  // wake() physics.py:471-478
  si[L.asleep + b] = 0;
  si[L.sleep_ctr + b] = 0;
  si[L.rider_joint + b] = -1;
  Pose inv, bp, rel;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) inv.R[3 * i + j] = ee.R[3 * j + i];
  matvec(inv.R, ee.p, inv.p);
  for (int i = 0; i < 3; ++i) inv.p[i] = -inv.p[i];
  quat_to_mat(sd + L.quat + 4 * b, bp.R);
  bp.p[0] = sd[L.pos + 3 * b]; bp.p[1] = sd[L.pos + 3 * b + 1]; bp.p[2] = sd[L.pos + 3 * b + 2];
  compose(inv, bp, rel);
  si[L.held] = b;
  for (int i = 0; i < 3; ++i) sd[L.held_off + i] = rel.p[i];
  mat_to_quat(rel.R, sd + L.held_off + 3);
  for (int i = 0; i < 3; ++i) { sd[L.lv + 3 * b + i] = 0.0; sd[L.av + 3 * b + i] = 0.0; }
}

__global__ void stats_kernel(DevBatch B, double *out) {
  const int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env >= B.n_env) return;
  const StateLayout &L = B.L;
  const int32_t *si = B.si + (size_t)env * L.int_size;
  int asleep = 0;
  for (int b = 0; b < L.nb; ++b) asleep += si[L.asleep + b];
  out[4 * env + 0] = B.sd[(size_t)env * L.dbl_size + L.acc];
  out[4 * env + 1] = (double)B.fault[env];
  out[4 * env + 2] = (double)B.event_count[env];
  out[4 * env + 3] = (double)asleep;
}

cudaError_t launch_grasp(const DevBatch &B, const double *gripper, int stride, cudaStream_t stream) {
  grasp_kernel<<<(B.n_env + 127) / 128, 128, 0, stream>>>(B, gripper, stride);
  return cudaGetLastError();
}

cudaError_t launch_stats(const DevBatch &B, double *out, cudaStream_t stream) {
  stats_kernel<<<(B.n_env + 255) / 256, 256, 0, stream>>>(B, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ IK
// robot.py:185-313 apply_arm_action -> solve_ik -> _dls_attempt, batched.
// One warp per env: lane 0 runs the attempt from the current joints; if it
// fails, the 11 restart seeds and the 24 Weyl-spray seeds run one per lane
// and the lowest-index success wins (= the reference's sequential order).
// Same operation order as oracle/rsim_oracle.c.

__device__ void ik_link_poses(const DevScene &sc, const double *q, Pose *links, Pose &ee) {
  Pose t, off, rot;
  const double zero3[3] = {0.0, 0.0, 0.0};
  base3(zero3, t);
  rot_z(0.0, off.R);
  rot.p[0] = rot.p[1] = rot.p[2] = 0.0;
  for (int i = 0; i < sc.narm; ++i) {
    off.p[0] = sc.arm_offset[3 * i]; off.p[1] = sc.arm_offset[3 * i + 1]; off.p[2] = sc.arm_offset[3 * i + 2];
    compose(t, off, t);
    axis_angle_mat(sc.arm_axis + 3 * i, q[i], rot.R);
    compose(t, rot, t);
    if (links) links[i] = t;
  }
  Pose g = {{1, 0, 0, 0, 1, 0, 0, 0, 1}, {sc.gripper[0], sc.gripper[1], sc.gripper[2]}};
  compose(t, g, ee);
}

// SPEC.md:247-249 Observation proprioception (PAPER §5.1: "arm joint angles
// (7-dim), end-effector position (3-dim), and base-egomotion (6-dim)") and
// goal vectors, from the batch's current state; thread per env.  out[e]:
// [0,7) arm joints, [7,10) EE position in the robot frame (FK from the base,
// robot.py:161-169), [10,16) base egomotion since base_prev[e] in the previous
// robot frame (dx, dy, dz = 0, droll = 0, dpitch = 0, dyaw wrapped to
// [-pi, pi)), [16, 16 + 3 K) goal vectors (world goals in the robot frame).
__global__ void proprio_kernel(DevBatch B, const double *base_prev, const double *goals, int n_goals, double *out,
                               double *base_out) {
  const int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env >= B.n_env) return;
  const DevScene &sc = B.scenes[B.env_scene[env]];
  const StateLayout &L = B.L;
  const double *sd = B.sd + (size_t)env * L.dbl_size;
  const int stride = 16 + 3 * n_goals;
  double *o = out + (size_t)env * stride;
  const double *q = sd + L.joints + sc.nsj, *base = sd + L.base;
  for (int i = 0; i < 7; ++i) o[i] = i < sc.narm ? q[i] : 0.0;
  Pose ee;
  ik_link_poses(sc, q, nullptr, ee);
  for (int i = 0; i < 3; ++i) o[7 + i] = ee.p[i];
  for (int i = 0; i < 6; ++i) o[10 + i] = 0.0;
  if (base_prev) {
    const double *bp = base_prev + 3 * env, c = cos(bp[2]), s = sin(bp[2]);
    const double dx = base[0] - bp[0], dy = base[1] - bp[1];
    o[10] = c * dx + s * dy;
    o[11] = -s * dx + c * dy;
    o[15] = py_mod(base[2] - bp[2] + M_PI, 2.0 * M_PI) - M_PI;
  }
  const double c = cos(base[2]), s = sin(base[2]);
  for (int k = 0; k < n_goals; ++k) {
    const double *g = goals + ((size_t)env * n_goals + k) * 3;
    const double gx = g[0] - base[0], gy = g[1] - base[1];
    o[16 + 3 * k] = c * gx + s * gy;
    o[17 + 3 * k] = -s * gx + c * gy;
    o[18 + 3 * k] = g[2];
  }
  if (base_out)
    for (int i = 0; i < 3; ++i) base_out[3 * env + i] = base[i];
}

cudaError_t launch_proprio(const DevBatch &B, const double *base_prev, const double *goals, int n_goals, double *out,
                           double *base_out, cudaStream_t stream) {
  proprio_kernel<<<(B.n_env + 127) / 128, 128, 0, stream>>>(B, base_prev, goals, n_goals, out, base_out);
  return cudaGetLastError();
}

__device__ void ik_solve3(const double *A_in, double *B, int nrhs) {
  double A[9];
  int piv[3];
  for (int i = 0; i < 9; ++i) A[i] = A_in[i];
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

// FK for the IK loop: rotated joint axes, link origins and the EE position
// (the values arm_jacobian reads, robot.py:185-192), without storing poses.
__device__ void ik_fk(const DevScene &sc, const double *q, double (*ax)[3], double (*lp)[3], double *ee) {
  Pose t, off, rot;
  const double zero3[3] = {0.0, 0.0, 0.0};
  base3(zero3, t);
  rot_z(0.0, off.R);
  rot.p[0] = rot.p[1] = rot.p[2] = 0.0;
  for (int i = 0; i < sc.narm; ++i) {
    off.p[0] = sc.arm_offset[3 * i]; off.p[1] = sc.arm_offset[3 * i + 1]; off.p[2] = sc.arm_offset[3 * i + 2];
    compose(t, off, t);
    axis_angle_mat(sc.arm_axis + 3 * i, q[i], rot.R);
    compose(t, rot, t);
    if (ax) {
      matvec(t.R, sc.arm_axis + 3 * i, ax[i]);
      lp[i][0] = t.p[0]; lp[i][1] = t.p[1]; lp[i][2] = t.p[2];
    }
  }
  Pose g = {{1, 0, 0, 0, 1, 0, 0, 0, 1}, {sc.gripper[0], sc.gripper[1], sc.gripper[2]}}, e;
  compose(t, g, e);
  ee[0] = e.p[0]; ee[1] = e.p[1]; ee[2] = e.p[2];
}

// robot.py:199-221; one thread
__device__ bool ik_dls_attempt(const DevScene &sc, const double *target, const double *seed, double *q_out) {
  const int n = sc.narm;
  const double tol = 5e-3, lam2 = 0.05 * 0.05;
  double q[kMaxArm], lo[kMaxArm], hi[kMaxArm], mid[kMaxArm];
  for (int i = 0; i < n; ++i) {
    lo[i] = sc.arm_limits[2 * i]; hi[i] = sc.arm_limits[2 * i + 1];
    mid[i] = 0.5 * (lo[i] + hi[i]);
    q[i] = seed[i] < lo[i] ? lo[i] : (seed[i] > hi[i] ? hi[i] : seed[i]);
  }
  double ax[kMaxArm][3], lp[kMaxArm][3], ee[3];
  for (int it = 0; it <= 100; ++it) {
    ik_fk(sc, q, ax, lp, ee);
    double err[3] = {target[0] - ee[0], target[1] - ee[1], target[2] - ee[2]};
    if (sqrt(dot3(err, err)) < tol) {
      for (int i = 0; i < n; ++i) q_out[i] = q[i];
      return true;
    }
    if (it == 100) break;
    double J[3 * kMaxArm], JS[3 * kMaxArm], jjt[9];
    for (int i = 0; i < n; ++i) {
      double d[3], cc[3];
      for (int k = 0; k < 3; ++k) d[k] = ee[k] - lp[i][k];
      cross3(ax[i], d, cc);
      for (int k = 0; k < 3; ++k) J[k * n + i] = cc[k];
    }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double sacc = 0.0;
        for (int i = 0; i < n; ++i) sacc += J[a * n + i] * J[b * n + i];
        jjt[3 * a + b] = sacc + (a == b ? lam2 : 0.0);
      }
    double y[3] = {err[0], err[1], err[2]};
    ik_solve3(jjt, y, 1);
    for (int i = 0; i < 3 * n; ++i) JS[i] = J[i];
    ik_solve3(jjt, JS, n);
    double dq[kMaxArm], r[kMaxArm];
    for (int i = 0; i < n; ++i) dq[i] = J[0 * n + i] * y[0] + J[1 * n + i] * y[1] + J[2 * n + i] * y[2];
    for (int i = 0; i < n; ++i) r[i] = mid[i] - q[i];
    for (int i = 0; i < n; ++i) {
      double sacc = 0.0;
      for (int jj = 0; jj < n; ++jj) {
        double pij = J[0 * n + i] * JS[0 * n + jj] + J[1 * n + i] * JS[1 * n + jj] + J[2 * n + i] * JS[2 * n + jj];
        sacc += ((i == jj ? 1.0 : 0.0) - pij) * r[jj];
      }
      dq[i] += 0.1 * sacc;
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
  return false;
}

__constant__ double kRestart[11][7] = {
    {0.0, 0.25, 0.0, -0.35, 0.0, 0.3, 0.0},       {0.3, -0.2, 0.2, 0.3, -0.2, -0.3, 0.2},
    {-0.3, 0.3, -0.25, -0.3, 0.25, 0.35, -0.2},   {0.15, 0.4, 0.3, 0.4, 0.3, -0.4, 0.3},
    {-0.15, -0.35, -0.3, 0.45, -0.35, 0.4, -0.3}, {0.45, 0.1, 0.45, -0.45, 0.4, -0.1, 0.45},
    {-0.45, -0.1, -0.45, 0.2, 0.45, 0.15, -0.45}, {0.6, 0.85, -0.8, -0.2, 0.7, 0.0, -0.3},
    {-0.6, 0.85, 0.8, -0.2, -0.7, 0.0, 0.3},      {0.85, 0.9, -0.55, 0.3, 0.75, -0.25, 0.0},
    {-0.85, 0.9, 0.55, 0.3, -0.75, 0.25, 0.0}};
__constant__ double kWeyl[7] = {0.618034, 0.754878, 0.569840, 0.380110, 0.245122, 0.119409, 0.059683};

// seed of attempt a (0 = current joints, 1..11 restarts, 12..35 Weyl spray)
__device__ void ik_seed(const DevScene &sc, int a, const double *q0, double *seed) {
  const int n = sc.narm;
  if (a == 0) { for (int i = 0; i < n; ++i) seed[i] = q0[i]; return; }
  for (int i = 0; i < n; ++i) {
    const double lo = sc.arm_limits[2 * i], hi = sc.arm_limits[2 * i + 1];
    const double mid = 0.5 * (lo + hi), span = hi - lo;
    if (a <= 11) {
      seed[i] = mid + kRestart[a - 1][i] * span * 0.5;
    } else {
      double u = 0.5;
      for (int r = 0; r <= a - 12; ++r) u = fmod(u + kWeyl[i], 1.0);
      seed[i] = lo + u * span;
    }
  }
}

// phase 1: one thread per env -- clamp, target, reach check, attempt 0 from the
// current joints (robot.py:293-313, :256-262).  status: 0 done, 1 IK failure
// (targets = current joints), 2 attempt 0 failed -> phase 2.
__global__ void __launch_bounds__(128) ik_first_kernel(DevBatch B, const double *delta, int stride, double *targets,
                                                       double *tgt_scratch, int32_t *status) {
  const int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env >= B.n_env) return;
  const DevScene &sc = B.scenes[B.env_scene[env]];
  const StateLayout &L = B.L;
  const double *sd = B.sd + (size_t)env * L.dbl_size;
  const int n = sc.narm;
  double q0[kMaxArm], target[3], ee[3];
  for (int i = 0; i < n; ++i) q0[i] = sd[L.joints + sc.nsj + i];
  double dl[3] = {delta[(size_t)stride * env], delta[(size_t)stride * env + 1], delta[(size_t)stride * env + 2]};
  double nd = sqrt(dot3(dl, dl));
  if (nd > 0.015) for (int k = 0; k < 3; ++k) dl[k] = dl[k] * (0.015 / nd);
  ik_fk(sc, q0, nullptr, nullptr, ee);
  for (int k = 0; k < 3; ++k) target[k] = ee[k] + dl[k];
  for (int k = 0; k < 3; ++k) tgt_scratch[3 * env + k] = target[k];
  double reach = 0.0;
  for (int i = 1; i < n; ++i) reach += sqrt(dot3(sc.arm_offset + 3 * i, sc.arm_offset + 3 * i));
  reach += sqrt(dot3(sc.gripper, sc.gripper));
  double dd[3] = {target[0] - sc.arm_offset[0], target[1] - sc.arm_offset[1], target[2] - sc.arm_offset[2]};
  double q[kMaxArm];
  int st = 1;
  if (!(sqrt(dot3(dd, dd)) > reach + 5e-3)) st = ik_dls_attempt(sc, target, q0, q) ? 0 : 2;
  for (int i = 0; i < n; ++i) targets[(size_t)env * n + i] = st == 0 ? q[i] : q0[i];
  status[env] = st;
}

// phase 2 (rare): one warp per env whose first attempt failed -- the 11 restart
// seeds and 24 Weyl-spray seeds one per lane, lowest-index success wins.
__global__ void __launch_bounds__(128) ik_fallback_kernel(DevBatch B, double *targets, const double *tgt_scratch,
                                                          int32_t *status, int32_t *failed) {
  const int env = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (env >= B.n_env) return;
  const int st = status[env];
  if (st != 2) {
    if (lane == 0 && failed) failed[env] = st;
    return;
  }
  const DevScene &sc = B.scenes[B.env_scene[env]];
  const StateLayout &L = B.L;
  const double *sd = B.sd + (size_t)env * L.dbl_size;
  const int n = sc.narm;
  double q0[kMaxArm], q[kMaxArm], seed[kMaxArm];
  for (int i = 0; i < n; ++i) q0[i] = sd[L.joints + sc.nsj + i];
  const double target[3] = {tgt_scratch[3 * env], tgt_scratch[3 * env + 1], tgt_scratch[3 * env + 2]};
  int win = -1;
  for (int base = 1; base < 36 && win < 0; base += 32) {
    const int a = base + lane;
    bool oka = false;
    if (a < 36) {
      ik_seed(sc, a, q0, seed);
      oka = ik_dls_attempt(sc, target, seed, q);
    }
    unsigned m = __ballot_sync(0xffffffffu, oka);
    if (m) win = base + __ffs(m) - 1;
  }
  const int src = win < 0 ? 0 : (win - 1) % 32;
  for (int i = 0; i < n; ++i) {
    double v = __shfl_sync(0xffffffffu, q[i], src);
    if (lane == 0) targets[(size_t)env * n + i] = win < 0 ? q0[i] : v;
  }
  if (lane == 0 && failed) failed[env] = win < 0 ? 1 : 0;
}

cudaError_t launch_ik(const DevBatch &B, const double *delta, int stride, double *targets, int32_t *failed,
                      double *scratch, cudaStream_t stream) {
  // scratch: [n_env] status (int32, stored in doubles) + [n_env][3] targets
  int32_t *status = reinterpret_cast<int32_t *>(scratch);
  double *tgt = scratch + (B.n_env + 1) / 2 + 1;
  ik_first_kernel<<<(B.n_env + 127) / 128, 128, 0, stream>>>(B, delta, stride, targets, tgt, status);
  ik_fallback_kernel<<<(B.n_env + 3) / 4, 128, 0, stream>>>(B, targets, tgt, status, failed);
  return cudaGetLastError();
}

}  // namespace rsim
