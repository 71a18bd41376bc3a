// device.cuh -- device-side data layout of the batched simulator.
//
// Static scene tables (one set per layout variant, shared by every env of
// that layout, ~30 KB, L1/L2 resident) and the per-env state slab.
//
// Per-env state is one contiguous slab of doubles + one of int32 per env
// ([E][SLAB]): a warp that owns an env stages its slab into shared memory
// with coalesced loads, runs all substeps there, and writes it back once.
// Field order inside the slab (offsets from StateLayout) mirrors the
// reference WorldState (physics.py:93-124); the host/ABI converts to and
// from the reference's snapshot bytes.
#pragma once
#include <cstdint>

#include "../../include/rsim.h"

namespace rsim {

constexpr int kMaxBodies = 64;   // 42 in the benchmark world (64-bit body masks)
constexpr int kMaxJoints = 16;   // 4 scene + 7 arm
constexpr int kMaxArm = 8;
constexpr int kMaxFacetsPerPart = 48;
constexpr int kMaxFacets = 2048;  // per scene (render stages every world plane in shared memory)

struct DevScene {
  int nb, np, nf, nv, nt, nsj, narm, robot_base, nclutter;
  // bodies
  const int32_t *body_kind, *body_robot, *body_group, *body_joint, *body_part_begin;
  const double *inv_mass, *com, *inv_inertia, *friction, *restitution;
  const float *color;
  // parts
  const int32_t *part_body, *part_kind, *part_facet_begin, *part_vert_begin, *part_tri_begin;
  const double *part_local, *part_param;
  const double *part_bound;  // local bounding sphere radius about the part origin
  const double *facet, *vert;
  const int32_t *tri;
  // joints
  const int32_t *joint_type, *joint_body, *joint_parent;
  const double *joint_axis, *joint_origin, *joint_limits, *joint_handle;
  const double *arm_offset, *arm_axis, *arm_limits;
  double gripper[3];
  int ncam;
  const int32_t *cam_parent;
  const double *cam_mount;
  int nav_nx, nav_ny;
  double nav_origin[2], nav_cell;
  const uint8_t *nav;
  const int32_t *clutter;  // clutter body ids (dynamic, after the robot)
  // optional triangle-soup representation (rs_scene_set_mesh)
  int n_tri, n_nodes;
  const double *mtri;            // [n_tri][9]: v0, e1, e2 in the part frame
  const float *node_lo, *node_hi;  // [n_nodes][3]
  const int32_t *node_meta;      // [n_nodes][2]: leaf (first, count) | internal (right, -1)
  const float4 *node4;           // [n_nodes][2]: (lo.xyz, meta.x bits), (hi.xyz, meta.y bits) -- 2 x 16 B per node
  const int32_t *part_node_begin;  // [np + 1] BVH root per part
  const double *mesh_bound;      // [np] bounding radius of the part's mesh
};

// offsets (in doubles / int32s) inside one env's slabs
struct StateLayout {
  int nb, nj;
  // doubles; [0, stage) is what the step kernel stages in shared memory (the
  // rider offsets after it are constant during a step and stay in HBM)
  int pos, quat, lv, av, joints, jvel, base, held_off, grab_ee, grab_q, acc, time, stage, rider_off, dbl_size;
  // int32
  int asleep, sleep_ctr, rider_joint, held, held_joint, int_size;

  __host__ __device__ static StateLayout make(int nb, int nj) {
    StateLayout L;
    L.nb = nb; L.nj = nj;
    int o = 0;
    L.pos = o; o += 3 * nb;
    L.quat = o; o += 4 * nb;
    L.lv = o; o += 3 * nb;
    L.av = o; o += 3 * nb;
    L.joints = o; o += nj;
    L.jvel = o; o += nj;
    L.base = o; o += 3;
    L.held_off = o; o += 7;
    L.grab_ee = o; o += 3;
    L.grab_q = o; o += 1;
    L.acc = o; o += 1;
    L.time = o; o += 1;
    L.stage = o;
    L.rider_off = o; o += 7 * nb;
    L.dbl_size = (o + 3) & ~3;  // 32-byte multiple
    int i = 0;
    L.asleep = i; i += nb;
    L.sleep_ctr = i; i += nb;
    L.rider_joint = i; i += nb;
    L.held = i; i += 1;
    L.held_joint = i; i += 1;
    L.int_size = (i + 3) & ~3;
    return L;
  }
};

struct DevBatch {
  int n_env, nb, nj;
  int max_nf;          // most facets of any scene in the batch (render smem sizing)
  StateLayout L;
  double *sd;          // [E][L.dbl_size]  current state s_t (read)
  int32_t *si;         // [E][L.int_size]
  double *sd_out;      // successor s_{t+1} written by the step kernel (ping-pong buffer)
  int32_t *si_out;
  int64_t *step_index; // [E]
  const DevScene *scenes;  // device array
  const int32_t *env_scene;
  const int32_t *env_order;  // envs sorted by scene (stable): the warp-per-env step kernel's order, so
                             // co-resident warps share their scene tables in L1
  rs_physics_config cfg;
  rs_render_config rcfg;
  uint32_t *fault;
  int32_t *event_count;
  double *events;
  int64_t *counters;
  int event_cap;
  // per-env global scratch for the solver (rows), sized at batch creation
  double *row_scratch;
  int row_cap;
  // optional parity trace (rs_set_trace)
  int32_t *trace_pairs, *trace_count;
  int trace_cap, trace_sub;
  // render tables (render_tables_kernel): unit camera-frame ray per pixel, tile frustum planes
  const double *ray_dir, *tile_frustum;
  // optional per-env step mask (rs_settle): envs with env_active[e] == 0 are copied through unchanged
  const uint8_t *env_active;
  // optional per-env step latency probe (rsim_bench_env_cycles): SM clock cycles of the last step
  long long *env_cycles;
  // optional per-env phase clock accumulators [E][8] (rsim_bench_phase_cycles)
  long long *phase_cycles;
};

}  // namespace rsim
