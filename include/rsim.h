/*
 * rsim.h -- C ABI of the B200 batched rearrangement-simulator step.
 *
 * This is the drop-in boundary for the reference's hot path
 * (SURVEY.md §8b).  The reference's operator API is the Python class
 * `rearrange_sim.physics.Simulator` plus the (specified but unshipped)
 * sensors/pipeline modules; every entry point below replaces one of them,
 * with a leading environment dimension added:
 *
 *   rs_scene_create   <- Simulator.__init__ body tables       physics.py:257-330
 *                        (+ scene.load_scene tables             scene.py:475-588)
 *   rs_batch_create   <- one Simulator per env + PhysicsConfig physics.py:54-74
 *   rs_set_state      <- WorldState.from_bytes                 physics.py:166-203
 *   rs_get_state      <- WorldState.to_bytes                   physics.py:147-164
 *   rs_step           <- Simulator.step_physics                physics.py:575-594
 *   rs_render         <- sensors.render_depth (SPEC only)
 *                        restated over geometry.parts_ray_hits geometry.py:772-776
 *   rs_step_host      <- pipeline.step (SPEC only)
 *                        physics + render with host buffers
 *   rs_env_step[_host]<- pipeline.step with ArmAction/BaseAction SPEC.md:316, robot.py:84-104
 *   rs_grasp          <- grasp_rule + apply_grasp              robot.py:323-346, physics.py:1039-1079
 *   rs_arm_action     <- apply_arm_action / solve_ik           robot.py:185-313
 *   rs_render_mesh    <- render over AssetDef.visual_mesh      scene.py:63-76
 *   rs_proprio        <- Observation proprioception fields
 *   rs_sphere_cast    <- Simulator.sphere_cast                 physics.py:1088-1101
 *   rs_settle         <- Simulator.settle (+ spawn clearance)  physics.py:1113-1176
 *   rs_nav_fields     <- NavGrid.distance_field                navgrid.py:109-143
 *   rs_nav_geodesic   <- NavGrid.geodesic_distance             navgrid.py:145-148
 *   rs_nav_path       <- NavGrid.shortest_path                 navgrid.py:150-172
 *
 * Conventions:
 *   - every call is stream-ordered on the cudaStream_t passed as `stream`
 *     (NULL = legacy default stream); a batch is owned by one host thread;
 *   - a batch is bound to the CUDA device current at rs_batch_create: every
 *     rs_* call on it runs on that device (and restores the caller's current
 *     device), so `stream` must belong to that device;
 *   - device pointers are caller-allocated and never freed by the library;
 *   - return value 0 = success; non-zero = error code, message in
 *     rs_last_error() (thread-local).  Per-env physics faults (non-finite
 *     state, the reference's PhysicsFault physics.py:596-606) are reported
 *     in the fault word of rs_buffers, not as a return code;
 *   - snapshot buffers are the reference's WorldState byte format.
 */
#ifndef RSIM_H
#define RSIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 1

enum { RS_STATIC = 0, RS_KINEMATIC = 1, RS_DYNAMIC = 2 };
enum { RS_BOX = 0, RS_SPHERE = 1, RS_HULL = 2 };
enum { RS_REVOLUTE = 0, RS_PRISMATIC = 1 };
enum {
  RS_OK = 0,
  RS_ERR_ARG = 1,     /* bad argument / shape */
  RS_ERR_CUDA = 2,    /* CUDA runtime error */
  RS_ERR_SNAPSHOT = 3,/* malformed snapshot (bad magic/version/size) */
  RS_ERR_CAPACITY = 4 /* scene exceeds compiled kernel capacities */
};
/* fault word kinds (high 16 bits; low 16 bits = body or joint index) */
enum {
  RS_FAULT_NONE = 0,
  RS_FAULT_NONFINITE_POS = 1,
  RS_FAULT_NONFINITE_QUAT = 2,
  RS_FAULT_NONFINITE_VEL = 3,
  RS_FAULT_NONFINITE_JOINT = 4,
  RS_FAULT_OVERFLOW = 5 /* a per-substep capacity exceeded: the env keeps its input state;
                          low 16 bits = which one (RS_OVF_*) */
};
/* capacities of one substep of one env (fault word low bits with RS_FAULT_OVERFLOW) */
enum {
  RS_OVF_CANDIDATES = 1,   /* overlapping AABB pairs > 1024 */
  RS_OVF_ADMITTED = 2,     /* admitted pairs > 256 */
  RS_OVF_CONTACTS = 3,     /* contact rows > 512 */
  RS_OVF_GROUPS = 4,       /* touching pairs > 96 */
  RS_OVF_BLOCK_ROWS = 5,   /* contacts of one pair in a block solve > 32 */
  RS_OVF_BLOCK_MATRIX = 6  /* sum of m^2 over the block matrices > 8192 */
};

#define RS_NO_GROUP ((int32_t)0x80000000)

/* Static scene tables of one layout (see paper_2106_14405_b200/compiler.py). */
typedef struct {
  int32_t n_bodies, n_parts, n_facets, n_verts, n_tris;
  int32_t n_scene_joints, n_arm, robot_base;
  /* bodies [n_bodies] */
  const int32_t *body_kind, *body_robot, *body_group, *body_joint;
  const double *body_inv_mass, *body_com /*3*/, *body_inv_inertia /*9*/;
  const double *body_friction, *body_restitution;
  const int32_t *body_part_begin; /* n_bodies + 1 */
  const float *body_color;        /* 3 */
  /* parts [n_parts] */
  const int32_t *part_body, *part_kind;
  const double *part_local; /* 12: row-major R, t */
  const double *part_param; /* 3: box half extents | sphere radius */
  const int32_t *part_facet_begin, *part_vert_begin, *part_tri_begin; /* n_parts + 1 */
  const double *facet; /* 4: n, offset (n.x <= offset inside) */
  const double *vert;  /* 3 */
  const int32_t *tri;  /* 3, part-local vertex indices */
  /* scene joints [n_scene_joints] */
  const int32_t *joint_type, *joint_body, *joint_parent;
  const double *joint_axis /*3*/, *joint_origin /*12*/, *joint_limits /*2*/, *joint_handle /*3*/;
  /* arm chain [n_arm] */
  const double *arm_offset /*3*/, *arm_axis /*3*/, *arm_limits /*2*/;
  double gripper_offset[3];
  /* cameras */
  int32_t n_cameras;
  const int32_t *cam_parent; /* 0 = base, 1 = end effector */
  const double *cam_mount;   /* 12 */
  /* walk grid, x-major [nav_nx][nav_ny] */
  int32_t nav_nx, nav_ny;
  double nav_origin[2], nav_cell;
  const uint8_t *nav_walkable;
} rs_scene_desc;

/* physics.py:54-74 PhysicsConfig, field for field */
typedef struct {
  double gravity;
  int32_t solver_iterations;
  double correction_factor, slop, restitution_threshold, contact_margin;
  double sleep_lin_threshold, sleep_ang_threshold;
  int32_t sleep_substeps;
  double wake_margin, lin_damping, ang_damping, joint_damping;
  double joint_inertia_revolute, joint_inertia_prismatic, kp, motor_impulse_cap;
  int32_t impulse_cap_per_control_step, sleeping_enabled;
} rs_physics_config;

/* pinned sensor conventions */
typedef struct {
  int32_t width, height;
  double fov;      /* radians, horizontal = vertical */
  double znear, zfar;
  double tie_eps;  /* |t_b - t_min| <= tie_eps -> lowest body id */
} rs_render_config;

/* device-side views owned by the batch (valid until rs_batch_destroy) */
typedef struct {
  int32_t n_env, n_bodies, n_joints, event_cap;
  uint32_t *fault;        /* [n_env] */
  int32_t *event_count;   /* [n_env] events of the last rs_step (may exceed cap: overflow) */
  double *events;         /* [n_env][event_cap][7]: a, b, impulse, force, point xyz */
  int64_t *counters;      /* [n_env][3] narrowphase_tests, skipped_sleeping_pairs, wakes (since rs_set_state) */
} rs_buffers;

typedef struct rs_scene rs_scene;
typedef struct rs_batch rs_batch;

int rs_abi_version(void);
const char *rs_last_error(void);
/* bytes of one snapshot for (n_bodies, n_joints) */
int64_t rs_snapshot_size(int32_t n_bodies, int32_t n_joints);

int rs_scene_create(const rs_scene_desc *desc, rs_scene **out);
void rs_scene_destroy(rs_scene *scene);

/* env e simulates scenes[env_scene[e]]; all scenes must share body/joint counts */
int rs_batch_create(rs_scene *const *scenes, int32_t n_scenes, const int32_t *env_scene, int32_t n_env,
                    const rs_physics_config *cfg, const rs_render_config *rcfg, int32_t event_cap,
                    rs_batch **out);
void rs_batch_destroy(rs_batch *batch);
int rs_batch_buffers(rs_batch *batch, rs_buffers *out);

/* host snapshots <-> device state; env_ids NULL = 0..n-1; stride = bytes between snapshots */
int rs_set_state(rs_batch *batch, const uint8_t *snapshots, int64_t stride, const int32_t *env_ids,
                 int32_t n, void *stream);
int rs_get_state(rs_batch *batch, uint8_t *snapshots, int64_t stride, const int32_t *env_ids,
                 int32_t n, void *stream);

/* one control step for every env (device pointers).  The batch keeps two
 * state buffers: rs_step reads s_t and writes s_{t+1} into the other one, so
 * an rs_render of s_t enqueued BEFORE rs_step (on another stream) may run
 * concurrently with it (interleaved physics || render).
 *   arm_targets [n_env][n_arm] f64 joint targets (JointTargets.arm)
 *   base_cmd    [n_env][2] f64 linear, angular velocity (BaseAction)
 *   has_targets [n_env] u8, 0 = targets None (settle mode); NULL = all 1 */
int rs_step(rs_batch *batch, const double *arm_targets, const double *base_cmd, const uint8_t *has_targets,
            double dt, int32_t substeps, void *stream);

/* render cameras in cam_mask for every env into device tensors
 *   rgba [n_env][n_cam_out][H][W][4] u8, depth [..][H][W] f32, ids [..][H][W] i32;
 * n_cam_out = popcount(cam_mask); any output pointer may be NULL. */
int rs_render(rs_batch *batch, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids, void *stream);

/* End-effector action -> joint targets per env (robot.py:293-313
 * apply_arm_action: clamp |delta| to 1.5 cm, damped-least-squares IK with the
 * reference's deterministic restarts, robot.py:199-279).  Device pointers:
 *   delta_ee [n_env][3] f64 (robot base frame), arm_targets [n_env][n_arm] f64 out,
 *   ik_failed [n_env] i32 out (nullable; 1 = NoSolution -> targets = current joints). */
int rs_arm_action(rs_batch *batch, const double *delta_ee, double *arm_targets, int32_t *ik_failed, void *stream);

/* The SPEC env step with the paper's action space (SPEC.md:316-324,
 * PAPER.md §5.1): action [n_env][6] f64 device = (dx, dy, dz EE displacement
 * in the robot base frame, gripper scalar, base linear m/s, base angular
 * rad/s).  Runs rs_arm_action -> rs_step -> rs_grasp on `stream`. */
int rs_env_step(rs_batch *batch, const double *action, double dt, int32_t substeps, void *stream);

/* rs_env_step with a HOST action buffer, the observation o_t = render(s_t)
 * rendered concurrently on an internal stream (observation delay 1,
 * interleaved), and the per-env results of rs_step_host copied back.
 * Returns when the step and h_out_stats are complete (h_action may be
 * reused); the observation tensors complete in `stream` order (`stream` is
 * left waiting on the render), so a consumer on `stream`, or the next call,
 * sees o_t. */
int rs_env_step_host(rs_batch *batch, const double *h_action, double dt, int32_t substeps, uint32_t cam_mask,
                     uint8_t *rgba, float *depth, int32_t *ids, double *h_out_stats, void *stream);

/* grasp transition per env between steps (robot.py:323-346 + physics.py:1055-1079):
 * gripper [n_env] f64 device; scalar > 0 snaps the nearest candidate within 0.15 m,
 * < 0 releases. */
int rs_grasp(rs_batch *batch, const double *gripper, void *stream);

/* End-to-end env step with HOST buffers (pipeline.step restated, SPEC.md:316,
 * default StepConfig: observation_delay = 1, interleave = true):
 * renders o_t = render(s_t) (cam_mask) into the device observation tensors on
 * an internal side stream WHILE copying arm_targets/base_cmd (host) to the
 * device and running rs_step s_t -> s_{t+1} on `stream`; then copies per-env
 * step results back to host: out_stats [n_env][4] = accumulated_contact_force,
 * fault word, event count, sleeping-body count.  Returns when the step and
 * h_out_stats are complete (the host buffers may be reused); it does NOT
 * synchronise `stream`: the observation tensors complete in `stream` order
 * (`stream` is left waiting on the render).  A host reader of rgba/depth/ids
 * must synchronise `stream` first; a reader on another stream must wait on an
 * event recorded on `stream`.  Every later rs_* call on the batch must be
 * issued on `stream` (or after it), since the next step overwrites the state
 * buffer the render reads. */
int rs_step_host(rs_batch *batch, const double *h_arm_targets, const double *h_base_cmd, double dt,
                 int32_t substeps, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids,
                 double *h_out_stats, void *stream);

/* Dispatch order of the warp-per-env step kernel (a scheduling choice; no
 * result depends on it): 0 = envs sorted by scene (default: warps resident on
 * an SM share one layout's tables in L1); 1 = busy first -- each step, the
 * envs that had active contact groups in the previous step go first (still
 * scene-sorted within each group), so with more envs than resident warps the
 * latency tail starts in the first wave.  Measured: physics-only batches of
 * 4096 envs gain from 1; the interleaved 2048-env physics || render step does
 * not. */
int rs_set_env_order(rs_batch *batch, int32_t policy);

/* Per-env results of the current state on `stream`, device out [n_env][4] f64:
 * accumulated_contact_force (physics.py:944-959; the SPEC's StepResult
 * info "accumulated force N"), fault word, event count of the last step,
 * sleeping-body count -- what rs_step_host copies back, for device callers. */
int rs_step_stats(rs_batch *batch, double *out, void *stream);

/* Triangle-soup scene representation (AssetDef.visual_mesh scene.py:63-76,
 * SURVEY.md §8a R3): per part a triangle list in the part frame with a BVH
 * (paper_2106_14405_b200/mesh.py).  Must be attached before rs_batch_create. */
typedef struct {
  int32_t n_parts, n_tris, n_nodes;
  const double *tri;             /* [n_tris][9]: v0, e1 = v1 - v0, e2 = v2 - v0 */
  const float *node_lo, *node_hi; /* [n_nodes][3], rounded outward */
  const int32_t *node_meta;      /* [n_nodes][2]: leaf (first_tri, count) | internal (right child, -1) */
  const int32_t *part_node_begin; /* [n_parts + 1]: BVH root of each part */
  const double *part_bound;      /* [n_parts]: bounding radius of the part mesh about its origin */
} rs_mesh_desc;
int rs_scene_set_mesh(rs_scene *scene, const rs_mesh_desc *mesh);

/* RGBD render against the triangle soups (same outputs and conventions as
 * rs_render; a camera inside a closed mesh sees its exit faces). */
int rs_render_mesh(rs_batch *batch, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids, void *stream);

/* Observation proprioception of the current state (PAPER
 * §5.1): out [n_env][16 + 3 n_goals] = arm joints (7), end-effector position
 * in the robot frame (3), base egomotion since base_prev [n_env][3] (x, y,
 * yaw; NULL = zero) in the previous robot frame (dx, dy, 0, 0, 0, dyaw), and
 * the goal vectors goals [n_env][n_goals][3] (world) in the robot frame;
 * base_out [n_env][3] (optional) receives the current base for the next call.
 * Reads the state a render enqueued at the same point would read (s_t of an
 * interleaved step when enqueued before the step). */
int rs_proprio(rs_batch *batch, const double *base_prev, const double *goals, int32_t n_goals, double *out,
               double *base_out, void *stream);

/* Simulator.sphere_cast (physics.py:1088-1101) for n_queries rays: query q
 * in env env_of_query[q] (NULL: env q), unit direction dirs[q], hits farther
 * than max_dist[q] ignored.  out_body[q] = nearest body (lowest id on ties),
 * -1 for no hit, -2 when the direction is not unit length (the reference's
 * PhysicsFault); out_t[q] its range.  Device pointers, stream-ordered. */
int rs_sphere_cast(rs_batch *batch, const int32_t *env_of_query, const double *origins, const double *dirs,
                   const double *max_dist, int32_t n_queries, int32_t *out_body, double *out_t, void *stream);

/* ---- batched settle (Simulator.settle physics.py:1113-1176)
 * for fast resets.  The caller writes each settling env's spawn state with
 * rs_set_state (placements applied the way settle does: pose set, awake,
 * zero velocity, sleep counter 0, no rider; physics.py:1124-1137).  For the
 * envs with active[e] = 1 (device uint8, cleared as envs finish):
 * _assert_spawn_clearance over the placed bodies (device uint64 bitmask
 * placed[e], checked in ascending body id) with GJK parts_distance, then
 * control steps without targets (dt 1/30, 4 substeps) until every placed
 * body sleeps.  Per env: status 0 settled after steps[e] control steps,
 * 1 clearance < 1 mm (info[e] = body, other; value[e] = clearance), 2 a
 * placed body fell below floor_z - 0.5 (info[e][0] = body), 3 still awake
 * after max_steps (max_time 10 s = 301 steps), 4 physics fault (info[e][0]
 * = fault word).  Envs with active[e] = 0 are not modified.  Synchronises
 * `stream` every 8 steps to stop early. */
int rs_settle(rs_batch *batch, const uint64_t *placed, uint8_t *active, int32_t max_steps, double floor_z,
              int32_t *status, int32_t *info, double *value, int32_t *steps, void *stream);

/* ---- geodesics on the walk grid (navgrid.py:109-172).
 * Every scene of the batch must share the walk-grid shape (rs_nav_shape).
 * Fields are float64 [nx][ny] (x-major, the reference's NavGrid layout),
 * +inf where unreachable; all pointers are device pointers. */
/* grid shape of the batch's scenes; RS_ERR_ARG if they differ */
int rs_nav_shape(rs_batch *batch, int32_t *nx, int32_t *ny);
/* NavGrid.distance_field (navgrid.py:109-143): for goal g (scene
 * scene_of_goal[g], NULL = scene 0) the geodesic distance from every cell to
 * the cell of nearest_walkable(goal_xy[g]) -> fields[g]; goal_cell[g]
 * (optional) = i*ny + j of that cell.  Bit-identical to the reference's
 * Dijkstra (unique fixed point of the relaxation). */
int rs_nav_fields(rs_batch *batch, const int32_t *scene_of_goal, const double *goal_xy, int32_t n_goals,
                  double *fields, int32_t *goal_cell, void *stream);
/* NavGrid.geodesic_distance (navgrid.py:145-148) against precomputed fields:
 * out[q] = fields[field_of_query[q]] at the cell of nearest_walkable(from_xy[q]).
 * from_xy = NULL: query q is env q's robot base (n_queries = n_env, the env's
 * scene); else scene_of_query (NULL = scene 0). */
int rs_nav_geodesic(rs_batch *batch, const double *fields, const int32_t *field_of_query,
                    const int32_t *scene_of_query, const double *from_xy, int32_t n_queries, double *out,
                    void *stream);
/* NavGrid.shortest_path (navgrid.py:150-172): steepest-descent waypoints
 * (cell centres) [n_queries][cap][2] and their count (0 = unreachable,
 * truncated at cap). */
int rs_nav_path(rs_batch *batch, const double *fields, const int32_t *field_of_query, const int32_t *scene_of_query,
                const double *from_xy, int32_t n_queries, int32_t cap, double *waypoints, int32_t *count,
                void *stream);

/* Debug trace for parity tests (not on the hot path): when set, every rs_step
 * records per env and substep the admitted broadphase pairs in sorted order
 * with their narrowphase contact counts:
 *   pairs [n_env][max_substeps][cap][3] = (a, b, n_contacts), count [n_env][max_substeps]
 * (count may exceed cap).  Pass NULL pointers to disable. */
int rs_set_trace(rs_batch *batch, int32_t *pairs, int32_t *count, int32_t cap, int32_t max_substeps);

#ifdef __cplusplus
}
#endif
#endif /* RSIM_H */
