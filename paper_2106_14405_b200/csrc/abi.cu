// abi.cu -- C-ABI implementation (include/rsim.h): scene/batch lifetime,
// snapshot <-> device-slab conversion, launches.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rsim.h"
#include "../../include/rsim_bench.h"
#include "device.cuh"

namespace rsim {
cudaError_t launch_env_order(const DevBatch &B, const int32_t *scene_order, const uint8_t *heavy_in, int32_t *out,
                             cudaStream_t stream);
cudaError_t launch_step(const DevBatch &B, const double *arm, const double *base_cmd, int base_stride,
                        const uint8_t *has_targets, double dt, int substeps, cudaStream_t stream,
                        const uint8_t *heavy_in, uint8_t *heavy_out, cudaStream_t side, cudaEvent_t fork,
                        cudaEvent_t join, int force_width, cudaStream_t side2, cudaEvent_t join2);
cudaError_t launch_render(const DevBatch &B, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids,
                          cudaStream_t stream, unsigned long long *work = nullptr);
cudaError_t launch_render_mesh(const DevBatch &B, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids,
                               cudaStream_t stream, unsigned long long *work = nullptr);
cudaError_t launch_render_tables(const DevBatch &B, cudaStream_t stream);
cudaError_t launch_proprio(const DevBatch &B, const double *base_prev, const double *goals, int n_goals, double *out,
                           double *base_out, cudaStream_t stream);
cudaError_t launch_sphere_cast(const DevBatch &B, const int32_t *env_of_query, const double *origins,
                               const double *dirs, const double *max_dist, int nq, int32_t *out_body, double *out_t,
                               cudaStream_t stream);
cudaError_t launch_settle_clearance(const DevBatch &B, const uint64_t *placed, uint8_t *active, int32_t *status,
                                    int32_t *info, double *value, int32_t *steps, cudaStream_t stream);
cudaError_t launch_settle_check(const DevBatch &B, const uint64_t *placed, uint8_t *active, int32_t *status,
                                int32_t *info, double *value, int32_t *steps, double floor_limit, int step_no,
                                int max_steps, int32_t *n_active, cudaStream_t stream);
cudaError_t launch_nav_fields(const DevBatch &B, int nx, int ny, const int32_t *scene_of_goal, const double *goal_xy,
                              int n_goals, double *fields, int32_t *goal_cell, cudaStream_t stream);
cudaError_t launch_nav_geodesic(const DevBatch &B, int nx, int ny, const double *fields, const int32_t *field_of_query,
                                const int32_t *scene_of_query, const double *from_xy, int nq, double *out,
                                cudaStream_t stream);
cudaError_t launch_nav_path(const DevBatch &B, int nx, int ny, const double *fields, const int32_t *field_of_query,
                            const int32_t *scene_of_query, const double *from_xy, int nq, int cap, double *waypoints,
                            int32_t *count, cudaStream_t stream);
cudaError_t launch_render_exact(const DevBatch &B, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids,
                                cudaStream_t stream, unsigned long long *work = nullptr);
cudaError_t launch_grasp(const DevBatch &B, const double *gripper, int stride, cudaStream_t stream);
cudaError_t launch_ik(const DevBatch &B, const double *delta, int stride, double *targets, int32_t *failed,
                      double *scratch, cudaStream_t stream);
cudaError_t launch_stats(const DevBatch &B, double *out, cudaStream_t stream);
size_t step_scratch_doubles_per_env(int row_cap);
int step_row_cap();
}  // namespace rsim

using namespace rsim;

static thread_local std::string g_err;

static int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}
#define CUDA_TRY(x)                                                                                  \
  do {                                                                                               \
    cudaError_t e_ = (x);                                                                            \
    if (e_ != cudaSuccess) return fail(RS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct rs_scene {
  DevScene d;
  std::vector<void *> allocs;
};

struct rs_batch {
  DevBatch d;
  DevScene *d_scenes = nullptr;
  int32_t *d_env_scene = nullptr;
  int32_t *d_order = nullptr;  // busy-first dispatch order of the warp-per-env step kernel (policy 1)
  int order_policy = 0;        // rs_set_env_order: 0 scene order, 1 busy first
  bool order_pending = false;
  cudaEvent_t ord_fork = nullptr, ord_done = nullptr;
  cudaStream_t phys_busy = nullptr;  // the busy envs' step kernel (a third physics stream)
  cudaEvent_t busy_join = nullptr;
  std::vector<void *> allocs;
  int narm = 0;
  bool has_mesh = false;
  int nav_nx = -1, nav_ny = -1;  // shared walk-grid shape (-1: scenes differ)
  // rs_settle scratch: zero targets, has_targets = 0, active-env counter
  double *d_settle_zero = nullptr;
  uint8_t *d_settle_noct = nullptr;
  int32_t *d_settle_count = nullptr, *h_settle_count = nullptr;
  int n_scenes = 0;
  // ping-pong state buffers: rs_step reads buf[cur] and writes buf[cur ^ 1]
  double *sd_buf[2] = {nullptr, nullptr};
  int32_t *si_buf[2] = {nullptr, nullptr};
  int cur = 0;
  DevBatch view() const {
    DevBatch v = d;
    v.sd = sd_buf[cur]; v.si = si_buf[cur];
    v.sd_out = sd_buf[cur ^ 1]; v.si_out = si_buf[cur ^ 1];
    return v;
  }
  // lazily allocated staging for rs_step_host
  double *h_pin = nullptr, *d_act = nullptr, *d_stats = nullptr, *d_env_act = nullptr, *d_targets = nullptr;
  int32_t *d_ik_failed = nullptr;
  double *d_ik_scratch = nullptr;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // contact-heavy scheduling: per-env flags (ping-pong like the state) and a physics side stream
  uint8_t *heavy[2] = {nullptr, nullptr};
  int force_heavy = 0;  // rsim_bench_force_heavy: 0, or the CTA width every env is stepped with
  cudaStream_t phys_side = nullptr;
  cudaEvent_t ph_fork = nullptr, ph_join = nullptr;
  // host-buffer steps: physics on a high-priority stream next to the render
  cudaStream_t phys_hp = nullptr;
  cudaEvent_t hp_join = nullptr;
  int device = 0;  // the CUDA device current at rs_batch_create; every entry point runs on it
};

// NVTX range per entry point (named after it): the library's calls show up as
// ranges in Nsight Systems / ncu --nvtx timelines; free when no tool is attached
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Entry points run on the batch's device whatever the caller's current
// device is (kernel attributes, streams and buffers are per device), and
// restore the caller's device on return.
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(const rs_batch *b) {
    if (b && cudaGetDevice(&prev) == cudaSuccess && prev != b->device) cudaSetDevice(b->device);
    else prev = -1;
  }
  ~DeviceScope() { if (prev >= 0) cudaSetDevice(prev); }
};

// exported functions take C linkage from their declarations in rsim.h
int rs_abi_version(void) { return RS_ABI_VERSION; }
const char *rs_last_error(void) { return g_err.c_str(); }

int64_t rs_snapshot_size(int32_t nb, int32_t nj) {
  return 16 + 8 * 13 * (int64_t)nb + nb + 8 * nb + 16 * (int64_t)nj + 8 * 13 + 8 * nb + 56 * nb + 40;
}

template <typename T>
static int upload(rs_scene *s, const T *src, size_t n, const T **dst) {
  void *p = nullptr;
  size_t bytes = sizeof(T) * (n ? n : 1);
  CUDA_TRY(cudaMalloc(&p, bytes));
  s->allocs.push_back(p);
  if (n) CUDA_TRY(cudaMemcpy(p, src, sizeof(T) * n, cudaMemcpyHostToDevice));
  *dst = static_cast<const T *>(p);
  return 0;
}

int rs_scene_create(const rs_scene_desc *D, rs_scene **out) {
  if (!D || !out) return fail(RS_ERR_ARG, "null argument");
  const int nb = D->n_bodies, np = D->n_parts, nf = D->n_facets, nj = D->n_scene_joints + D->n_arm;
  if (nb > kMaxBodies || nj > kMaxJoints || D->n_arm > kMaxArm || np > 128 || nf > kMaxFacets ||
      D->n_scene_joints > 30)
    return fail(RS_ERR_CAPACITY, "scene exceeds compiled capacities (bodies<=64, joints<=16, parts<=128, facets<=2048)");
  for (int p = 0; p < np; ++p)
    if (D->part_facet_begin[p + 1] - D->part_facet_begin[p] > kMaxFacetsPerPart)
      return fail(RS_ERR_CAPACITY, "part with more than 48 facets");
  for (int b = 0; b < nb; ++b)
    if (D->body_part_begin[b + 1] - D->body_part_begin[b] > 8)
      return fail(RS_ERR_CAPACITY, "body with more than 8 parts");
  if (D->robot_base < 0 || D->robot_base + D->n_arm >= nb) return fail(RS_ERR_ARG, "robot bodies out of range");
  rs_scene *s = new rs_scene();
  DevScene &d = s->d;
  memset(&d, 0, sizeof d);
  d.nb = nb; d.np = np; d.nf = nf; d.nv = D->n_verts; d.nt = D->n_tris;
  d.nsj = D->n_scene_joints; d.narm = D->n_arm; d.robot_base = D->robot_base;
  // bounding radius of each convex part about its origin
  std::vector<double> bound(np, 0.0);
  for (int p = 0; p < np; ++p) {
    if (D->part_kind[p] == RS_BOX) {
      const double *h = D->part_param + 3 * p;
      bound[p] = sqrt(h[0] * h[0] + h[1] * h[1] + h[2] * h[2]);
    } else if (D->part_kind[p] == RS_HULL) {
      for (int v = D->part_vert_begin[p]; v < D->part_vert_begin[p + 1]; ++v) {
        const double *x = D->vert + 3 * v;
        bound[p] = fmax(bound[p], sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]));
      }
    } else {
      bound[p] = D->part_param[3 * p];
    }
    bound[p] = bound[p] * (1.0 + 1e-12) + 1e-12;
  }
  std::vector<int32_t> clutter;
  for (int b = 0; b < nb; ++b)
    if (D->body_kind[b] == RS_DYNAMIC && b > D->robot_base) clutter.push_back(b);
  d.nclutter = (int)clutter.size();
  int rc = 0;
#define UP(field, src, n) \
  if (!rc) rc = upload(s, src, (size_t)(n), &d.field)
  UP(body_kind, D->body_kind, nb); UP(body_robot, D->body_robot, nb); UP(body_group, D->body_group, nb);
  UP(body_joint, D->body_joint, nb); UP(body_part_begin, D->body_part_begin, nb + 1);
  UP(inv_mass, D->body_inv_mass, nb); UP(com, D->body_com, 3 * nb); UP(inv_inertia, D->body_inv_inertia, 9 * nb);
  UP(friction, D->body_friction, nb); UP(restitution, D->body_restitution, nb); UP(color, D->body_color, 3 * nb);
  UP(part_body, D->part_body, np); UP(part_kind, D->part_kind, np);
  UP(part_facet_begin, D->part_facet_begin, np + 1); UP(part_vert_begin, D->part_vert_begin, np + 1);
  UP(part_tri_begin, D->part_tri_begin, np + 1); UP(part_local, D->part_local, 12 * np);
  UP(part_param, D->part_param, 3 * np); UP(part_bound, bound.data(), np);
  UP(facet, D->facet, 4 * nf); UP(vert, D->vert, 3 * D->n_verts); UP(tri, D->tri, 3 * D->n_tris);
  UP(joint_type, D->joint_type, d.nsj); UP(joint_body, D->joint_body, d.nsj); UP(joint_parent, D->joint_parent, d.nsj);
  UP(joint_axis, D->joint_axis, 3 * d.nsj); UP(joint_origin, D->joint_origin, 12 * d.nsj);
  UP(joint_limits, D->joint_limits, 2 * d.nsj); UP(joint_handle, D->joint_handle, 3 * d.nsj);
  UP(arm_offset, D->arm_offset, 3 * d.narm); UP(arm_axis, D->arm_axis, 3 * d.narm);
  UP(arm_limits, D->arm_limits, 2 * d.narm);
  UP(cam_parent, D->cam_parent, D->n_cameras); UP(cam_mount, D->cam_mount, 12 * D->n_cameras);
  UP(nav, D->nav_walkable, (size_t)D->nav_nx * D->nav_ny);
  UP(clutter, clutter.data(), clutter.size());
#undef UP
  if (rc) {
    rs_scene_destroy(s);
    return rc;
  }
  memcpy(d.gripper, D->gripper_offset, sizeof d.gripper);
  d.ncam = D->n_cameras;
  d.nav_nx = D->nav_nx; d.nav_ny = D->nav_ny;
  d.nav_origin[0] = D->nav_origin[0]; d.nav_origin[1] = D->nav_origin[1]; d.nav_cell = D->nav_cell;
  *out = s;
  return RS_OK;
}

int rs_scene_set_mesh(rs_scene *s, const rs_mesh_desc *M) {
  if (!s || !M) return fail(RS_ERR_ARG, "null argument");
  DevScene &d = s->d;
  if (M->n_parts != d.np) return fail(RS_ERR_ARG, "mesh part count differs from the scene's");
  int rc = 0;
  if (!rc) rc = upload(s, M->tri, (size_t)9 * M->n_tris, &d.mtri);
  if (!rc) rc = upload(s, M->node_lo, (size_t)3 * M->n_nodes, &d.node_lo);
  if (!rc) rc = upload(s, M->node_hi, (size_t)3 * M->n_nodes, &d.node_hi);
  if (!rc) rc = upload(s, M->node_meta, (size_t)2 * M->n_nodes, &d.node_meta);
  if (!rc) rc = upload(s, M->part_node_begin, (size_t)M->n_parts + 1, &d.part_node_begin);
  if (!rc) {  // packed nodes for the render's traversal: one 32-byte record per node
    std::vector<float4> n4(2 * (size_t)(M->n_nodes > 0 ? M->n_nodes : 1));
    for (int n = 0; n < M->n_nodes; ++n) {
      float mx, my;
      memcpy(&mx, &M->node_meta[2 * n], 4);
      memcpy(&my, &M->node_meta[2 * n + 1], 4);
      n4[2 * n] = make_float4(M->node_lo[3 * n], M->node_lo[3 * n + 1], M->node_lo[3 * n + 2], mx);
      n4[2 * n + 1] = make_float4(M->node_hi[3 * n], M->node_hi[3 * n + 1], M->node_hi[3 * n + 2], my);
    }
    rc = upload(s, n4.data(), n4.size(), &d.node4);
  }
  if (!rc) rc = upload(s, M->part_bound, (size_t)M->n_parts, &d.mesh_bound);
  if (rc) return rc;
  d.n_tri = M->n_tris;
  d.n_nodes = M->n_nodes;
  return RS_OK;
}

void rs_scene_destroy(rs_scene *s) {
  if (!s) return;
  for (void *p : s->allocs) cudaFree(p);
  delete s;
}

static int balloc(rs_batch *b, void **p, size_t bytes) {
  CUDA_TRY(cudaMalloc(p, bytes ? bytes : 1));
  b->allocs.push_back(*p);
  CUDA_TRY(cudaMemset(*p, 0, bytes ? bytes : 1));
  return 0;
}

int rs_batch_create(rs_scene *const *scenes, int32_t n_scenes, const int32_t *env_scene, int32_t n_env,
                    const rs_physics_config *cfg, const rs_render_config *rcfg, int32_t event_cap, rs_batch **out) {
  if (!scenes || n_scenes < 1 || n_env < 1 || !cfg || !rcfg || !out || event_cap < 0)
    return fail(RS_ERR_ARG, "bad batch arguments");
  if (n_env >= (1 << 21)) return fail(RS_ERR_CAPACITY, "n_env must be < 2^21 (dispatch order counters)");
  const DevScene &s0 = scenes[0]->d;
  for (int i = 1; i < n_scenes; ++i)
    if (scenes[i]->d.nb != s0.nb || scenes[i]->d.nsj != s0.nsj || scenes[i]->d.narm != s0.narm)
      return fail(RS_ERR_ARG, "all scenes of a batch must share body and joint counts");
  if (env_scene)
    for (int e = 0; e < n_env; ++e)
      if (env_scene[e] < 0 || env_scene[e] >= n_scenes) return fail(RS_ERR_ARG, "env_scene index out of range");
  if (rcfg->width % 16 || rcfg->height % 16 || rcfg->width > 128 || rcfg->height > 128 || rcfg->width <= 0 ||
      rcfg->height <= 0)
    return fail(RS_ERR_ARG, "render width/height must be multiples of 16 and <= 128");
  if (cfg->solver_iterations < 0 || cfg->sleep_substeps < 0) return fail(RS_ERR_ARG, "bad physics config");
  rs_batch *b = new rs_batch();
  if (cudaGetDevice(&b->device) != cudaSuccess) b->device = 0;
  DevBatch &d = b->d;
  memset(&d, 0, sizeof d);
  d.n_env = n_env; d.nb = s0.nb; d.nj = s0.nsj + s0.narm;
  d.L = StateLayout::make(d.nb, d.nj);
  d.cfg = *cfg; d.rcfg = *rcfg; d.event_cap = event_cap;
  d.row_cap = step_row_cap();
  b->narm = s0.narm;
  int rc = 0;
  void *p;
#define BA(field, bytes)                          \
  if (!rc) {                                      \
    rc = balloc(b, &p, (bytes));                  \
    d.field = reinterpret_cast<decltype(d.field)>(p); \
  }
  BA(sd, sizeof(double) * d.L.dbl_size * (size_t)n_env);
  BA(si, sizeof(int32_t) * d.L.int_size * (size_t)n_env);
  BA(sd_out, sizeof(double) * d.L.dbl_size * (size_t)n_env);
  BA(si_out, sizeof(int32_t) * d.L.int_size * (size_t)n_env);
  BA(step_index, sizeof(int64_t) * n_env);
  BA(fault, sizeof(uint32_t) * n_env);
  BA(event_count, sizeof(int32_t) * n_env);
  BA(events, sizeof(double) * 7 * (size_t)(event_cap ? event_cap : 1) * n_env);
  BA(counters, sizeof(int64_t) * 3 * n_env);
  BA(ray_dir, sizeof(double) * 3 * (size_t)rcfg->width * rcfg->height);
  BA(tile_frustum, sizeof(double) * 8 * (size_t)(rcfg->width / 16) * (rcfg->height / 16));
  BA(row_scratch, sizeof(double) * step_scratch_doubles_per_env(d.row_cap) * (size_t)n_env);
  if (!rc) rc = balloc(b, &p, 2 * (size_t)n_env), b->heavy[0] = (uint8_t *)p, b->heavy[1] = (uint8_t *)p + n_env;
#undef BA
  if (!rc) rc = balloc(b, &p, sizeof(DevScene) * n_scenes), b->d_scenes = (DevScene *)p;
  if (!rc) rc = balloc(b, &p, sizeof(int32_t) * 2 * (size_t)n_env), b->d_env_scene = (int32_t *)p;
  if (!rc) rc = balloc(b, &p, sizeof(int32_t) * (size_t)n_env), b->d_order = (int32_t *)p;
  if (rc) {
    rs_batch_destroy(b);
    return rc;
  }
  std::vector<DevScene> hs(n_scenes);
  b->has_mesh = true;
  b->n_scenes = n_scenes;
  b->nav_nx = s0.nav_nx; b->nav_ny = s0.nav_ny;
  for (int i = 0; i < n_scenes; ++i) {
    hs[i] = scenes[i]->d;
    if (hs[i].nav_nx != s0.nav_nx || hs[i].nav_ny != s0.nav_ny) b->nav_nx = b->nav_ny = -1;
    d.max_nf = hs[i].nf > d.max_nf ? hs[i].nf : d.max_nf;
    b->has_mesh = b->has_mesh && hs[i].mtri != nullptr;
  }
  std::vector<int32_t> es(n_env, 0);
  if (env_scene) memcpy(es.data(), env_scene, sizeof(int32_t) * n_env);
  cudaError_t e1 = cudaMemcpy(b->d_scenes, hs.data(), sizeof(DevScene) * n_scenes, cudaMemcpyHostToDevice);
  for (int e = 0; e < n_env; ++e) es.push_back(e);  // env_order: envs stably sorted by scene
  std::stable_sort(es.begin() + n_env, es.end(), [&](int32_t x, int32_t y) { return es[x] < es[y]; });
  cudaError_t e2 = cudaMemcpy(b->d_env_scene, es.data(), sizeof(int32_t) * 2 * n_env, cudaMemcpyHostToDevice);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    rs_batch_destroy(b);
    return fail(RS_ERR_CUDA, "batch table upload failed");
  }
  d.scenes = b->d_scenes;
  d.env_scene = b->d_env_scene;
  d.env_order = b->d_env_scene + n_env;
  if (launch_render_tables(d, 0) != cudaSuccess || cudaStreamSynchronize(0) != cudaSuccess) {
    rs_batch_destroy(b);
    return fail(RS_ERR_CUDA, "render table setup failed");
  }
  b->sd_buf[0] = d.sd; b->sd_buf[1] = d.sd_out;
  b->si_buf[0] = d.si; b->si_buf[1] = d.si_out;
  *out = b;
  return RS_OK;
}

void rs_batch_destroy(rs_batch *b) {
  if (!b) return;
  DeviceScope device_scope(b);
  for (void *p : b->allocs) cudaFree(p);
  if (b->h_pin) cudaFreeHost(b->h_pin);
  if (b->d_act) cudaFree(b->d_act);
  if (b->d_stats) cudaFree(b->d_stats);
  if (b->d_env_act) cudaFree(b->d_env_act);
  if (b->d_targets) cudaFree(b->d_targets);
  if (b->d_ik_failed) cudaFree(b->d_ik_failed);
  if (b->d_ik_scratch) cudaFree(b->d_ik_scratch);
  if (b->d_settle_zero) cudaFree(b->d_settle_zero);
  if (b->d_settle_noct) cudaFree(b->d_settle_noct);
  if (b->d_settle_count) cudaFree(b->d_settle_count);
  if (b->h_settle_count) cudaFreeHost(b->h_settle_count);
  if (b->side) cudaStreamDestroy(b->side);
  if (b->phys_side) cudaStreamDestroy(b->phys_side);
  if (b->phys_hp) cudaStreamDestroy(b->phys_hp);
  if (b->hp_join) cudaEventDestroy(b->hp_join);
  if (b->phys_busy) cudaStreamDestroy(b->phys_busy);
  if (b->busy_join) cudaEventDestroy(b->busy_join);
  if (b->ord_fork) cudaEventDestroy(b->ord_fork);
  if (b->ord_done) cudaEventDestroy(b->ord_done);
  if (b->ph_fork) cudaEventDestroy(b->ph_fork);
  if (b->ph_join) cudaEventDestroy(b->ph_join);
  if (b->ev_fork) cudaEventDestroy(b->ev_fork);
  if (b->ev_join) cudaEventDestroy(b->ev_join);
  delete b;
}

int rs_batch_buffers(rs_batch *b, rs_buffers *o) {
  DeviceScope device_scope(b);
  if (!b || !o) return fail(RS_ERR_ARG, "null argument");
  o->n_env = b->d.n_env; o->n_bodies = b->d.nb; o->n_joints = b->d.nj; o->event_cap = b->d.event_cap;
  o->fault = b->d.fault; o->event_count = b->d.event_count; o->events = b->d.events; o->counters = b->d.counters;
  return RS_OK;
}

// snapshot bytes (physics.py:147-203) <-> slab
static int unpack_snapshot(const uint8_t *s, const StateLayout &L, double *sd, int32_t *si, int64_t *step) {
  if (memcmp(s, "RSIM", 4) != 0) return fail(RS_ERR_SNAPSHOT, "bad snapshot magic");
  uint32_t ver, nb, nj;
  memcpy(&ver, s + 4, 4); memcpy(&nb, s + 8, 4); memcpy(&nj, s + 12, 4);
  if (ver != 1) return fail(RS_ERR_SNAPSHOT, "unsupported snapshot version");
  if ((int)nb != L.nb || (int)nj != L.nj) return fail(RS_ERR_SNAPSHOT, "snapshot body/joint count mismatch");
  const uint8_t *p = s + 16;
  auto take = [&](void *dst, size_t n) { memcpy(dst, p, n); p += n; };
  memset(sd, 0, sizeof(double) * L.dbl_size);
  memset(si, 0, sizeof(int32_t) * L.int_size);
  take(sd + L.pos, 24 * nb); take(sd + L.quat, 32 * nb); take(sd + L.lv, 24 * nb); take(sd + L.av, 24 * nb);
  for (uint32_t b = 0; b < nb; ++b) si[L.asleep + b] = p[b] ? 1 : 0;
  p += nb;
  for (uint32_t b = 0; b < nb; ++b) { int64_t v; take(&v, 8); si[L.sleep_ctr + b] = (int32_t)v; }
  take(sd + L.joints, 8 * nj); take(sd + L.jvel, 8 * nj);
  take(sd + L.base, 24); take(sd + L.held_off, 56); take(sd + L.grab_ee, 24);
  for (uint32_t b = 0; b < nb; ++b) { int64_t v; take(&v, 8); si[L.rider_joint + b] = (int32_t)v; }
  take(sd + L.rider_off, 56 * nb);
  int32_t held, held_joint;
  take(&held, 4); take(&held_joint, 4);
  si[L.held] = held; si[L.held_joint] = held_joint;
  take(sd + L.grab_q, 8); take(sd + L.acc, 8); take(sd + L.time, 8); take(step, 8);
  return 0;
}

static void pack_snapshot(const StateLayout &L, const double *sd, const int32_t *si, int64_t step, uint8_t *s) {
  const int nb = L.nb, nj = L.nj;
  memcpy(s, "RSIM", 4);
  uint32_t hdr[3] = {1u, (uint32_t)nb, (uint32_t)nj};
  memcpy(s + 4, hdr, 12);
  uint8_t *p = s + 16;
  auto put = [&](const void *src, size_t n) { memcpy(p, src, n); p += n; };
  put(sd + L.pos, 24 * nb); put(sd + L.quat, 32 * nb); put(sd + L.lv, 24 * nb); put(sd + L.av, 24 * nb);
  for (int b = 0; b < nb; ++b) p[b] = si[L.asleep + b] ? 1 : 0;
  p += nb;
  for (int b = 0; b < nb; ++b) { int64_t v = si[L.sleep_ctr + b]; put(&v, 8); }
  put(sd + L.joints, 8 * nj); put(sd + L.jvel, 8 * nj);
  put(sd + L.base, 24); put(sd + L.held_off, 56); put(sd + L.grab_ee, 24);
  for (int b = 0; b < nb; ++b) { int64_t v = si[L.rider_joint + b]; put(&v, 8); }
  put(sd + L.rider_off, 56 * nb);
  int32_t held = si[L.held], held_joint = si[L.held_joint];
  put(&held, 4); put(&held_joint, 4);
  put(sd + L.grab_q, 8); put(sd + L.acc, 8); put(sd + L.time, 8); put(&step, 8);
}

int rs_set_state(rs_batch *b, const uint8_t *snaps, int64_t stride, const int32_t *env_ids, int32_t n, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !snaps || n < 0) return fail(RS_ERR_ARG, "null argument");
  const DevBatch d = b->view();
  const StateLayout &L = d.L;
  if (stride <= 0) stride = rs_snapshot_size(L.nb, L.nj);
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<double> sd((size_t)L.dbl_size * n);
  std::vector<int32_t> si((size_t)L.int_size * n);
  std::vector<int64_t> step(n);
  for (int i = 0; i < n; ++i) {
    int e = env_ids ? env_ids[i] : i;
    if (e < 0 || e >= d.n_env) return fail(RS_ERR_ARG, "env id out of range");
    int rc = unpack_snapshot(snaps + stride * i, L, sd.data() + (size_t)L.dbl_size * i,
                             si.data() + (size_t)L.int_size * i, &step[i]);
    if (rc) return rc;
  }
  bool contiguous = true;
  for (int i = 0; i < n && contiguous; ++i) contiguous = (env_ids ? env_ids[i] : i) == (env_ids ? env_ids[0] : 0) + i;
  int e0 = n ? (env_ids ? env_ids[0] : 0) : 0;
  std::vector<int64_t> zeros(3, 0);
  if (contiguous && n) {
    CUDA_TRY(cudaMemcpyAsync(d.sd + (size_t)L.dbl_size * e0, sd.data(), sizeof(double) * L.dbl_size * n,
                             cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.si + (size_t)L.int_size * e0, si.data(), sizeof(int32_t) * L.int_size * n,
                             cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.step_index + e0, step.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(d.counters + 3 * (size_t)e0, 0, sizeof(int64_t) * 3 * n, st));
    CUDA_TRY(cudaMemsetAsync(d.fault + e0, 0, sizeof(uint32_t) * n, st));
    CUDA_TRY(cudaMemsetAsync(d.event_count + e0, 0, sizeof(int32_t) * n, st));
  } else {
    for (int i = 0; i < n; ++i) {
      int e = env_ids[i];
      CUDA_TRY(cudaMemcpyAsync(d.sd + (size_t)L.dbl_size * e, sd.data() + (size_t)L.dbl_size * i,
                               sizeof(double) * L.dbl_size, cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(d.si + (size_t)L.int_size * e, si.data() + (size_t)L.int_size * i,
                               sizeof(int32_t) * L.int_size, cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(d.step_index + e, &step[i], sizeof(int64_t), cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemsetAsync(d.counters + 3 * (size_t)e, 0, sizeof(int64_t) * 3, st));
      CUDA_TRY(cudaMemsetAsync(d.fault + e, 0, sizeof(uint32_t), st));
      CUDA_TRY(cudaMemsetAsync(d.event_count + e, 0, sizeof(int32_t), st));
    }
  }
  CUDA_TRY(cudaStreamSynchronize(st));  // host staging goes out of scope
  return RS_OK;
}

int rs_get_state(rs_batch *b, uint8_t *snaps, int64_t stride, const int32_t *env_ids, int32_t n, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !snaps || n < 0) return fail(RS_ERR_ARG, "null argument");
  const DevBatch d = b->view();
  const StateLayout &L = d.L;
  if (stride <= 0) stride = rs_snapshot_size(L.nb, L.nj);
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<double> sd((size_t)L.dbl_size * n);
  std::vector<int32_t> si((size_t)L.int_size * n);
  std::vector<int64_t> step(n);
  for (int i = 0; i < n; ++i) {
    int e = env_ids ? env_ids[i] : i;
    if (e < 0 || e >= d.n_env) return fail(RS_ERR_ARG, "env id out of range");
    CUDA_TRY(cudaMemcpyAsync(sd.data() + (size_t)L.dbl_size * i, d.sd + (size_t)L.dbl_size * e,
                             sizeof(double) * L.dbl_size, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(si.data() + (size_t)L.int_size * i, d.si + (size_t)L.int_size * e,
                             sizeof(int32_t) * L.int_size, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&step[i], d.step_index + e, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int i = 0; i < n; ++i)
    pack_snapshot(L, sd.data() + (size_t)L.dbl_size * i, si.data() + (size_t)L.int_size * i, step[i],
                  snaps + stride * i);
  return RS_OK;
}

static cudaError_t ensure_phys_side(rs_batch *b) {
  if (b->phys_side) return cudaSuccess;
  // highest priority: contact-heavy envs (the step's latency tail) get SMs
  // ahead of queued render CTAs of an interleaved observation render
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaError_t e = cudaStreamCreateWithPriority(&b->phys_side, cudaStreamNonBlocking, hi);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b->ph_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b->ph_join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b->ord_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b->ord_done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&b->phys_busy, cudaStreamNonBlocking, hi);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b->busy_join, cudaEventDisableTiming);
  return e;
}

// policy 1: the step's dispatch order from the previous step's contact
// activity, built on the physics side stream so that it overlaps what `st`
// runs before the step (the IK of rs_env_step); launch_step_b waits for it
static cudaError_t enqueue_env_order(rs_batch *b, cudaStream_t st) {
  cudaError_t e = ensure_phys_side(b);
  if (e != cudaSuccess) return e;
  if (b->force_heavy > 0) {  // debug: every env through the CTA kernel of that width
    if ((e = cudaMemsetAsync(b->heavy[b->cur], 255, (size_t)b->d.n_env, st)) != cudaSuccess) return e;
  }
  if (b->order_policy != 1) return cudaSuccess;
  if ((e = cudaEventRecord(b->ord_fork, st)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(b->phys_side, b->ord_fork, 0)) != cudaSuccess) return e;
  const DevBatch v = b->view();
  if ((e = launch_env_order(v, b->d_env_scene + v.n_env, b->heavy[b->cur], b->d_order, b->phys_side)) != cudaSuccess)
    return e;
  if ((e = cudaEventRecord(b->ord_done, b->phys_side)) != cudaSuccess) return e;
  b->order_pending = true;
  return cudaSuccess;
}

static cudaError_t launch_step_b(rs_batch *b, const double *arm, const double *base_cmd, int base_stride,
                                 const uint8_t *has_targets, double dt, int substeps, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  const bool pre = b->order_pending;  // enqueued by rs_env_step before its IK
  b->order_pending = false;
  if (!pre && (e = enqueue_env_order(b, st)) != cudaSuccess) return e;
  DevBatch v = b->view();
  if (b->order_policy == 1) {
    b->order_pending = false;
    if ((e = cudaStreamWaitEvent(st, b->ord_done, 0)) != cudaSuccess) return e;
    v.env_order = b->d_order;
  }
  // force_heavy == -1 (debug): no CTA kernel, every env on the warp kernel
  return launch_step(v, arm, base_cmd, base_stride, has_targets, dt, substeps, st, b->heavy[b->cur],
                     b->heavy[b->cur ^ 1], b->force_heavy == -1 ? nullptr : b->phys_side, b->ph_fork, b->ph_join,
                     b->force_heavy < -1 ? -b->force_heavy : (b->force_heavy > 0 ? b->force_heavy : 0),
                     b->phys_busy, b->busy_join);
}

int rs_set_env_order(rs_batch *b, int32_t policy) {
  DeviceScope device_scope(b);
  if (!b) return fail(RS_ERR_ARG, "null batch");
  if (policy != 0 && policy != 1) return fail(RS_ERR_ARG, "env order policy must be 0 (scene) or 1 (busy first)");
  b->order_policy = policy;
  return RS_OK;
}

// physics of a host-buffer step runs on a highest-priority stream so that the
// contact-heavy envs (the step's latency tail) get SMs ahead of queued render
// CTAs; `st` joins it at the end
static int ensure_phys_hp(rs_batch *b) {
  if (!b->phys_hp) {
    int lo = 0, hi = 0;
    CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_TRY(cudaStreamCreateWithPriority(&b->phys_hp, cudaStreamNonBlocking, hi));
    CUDA_TRY(cudaEventCreateWithFlags(&b->hp_join, cudaEventDisableTiming));
  }
  return RS_OK;
}

int rs_step(rs_batch *b, const double *arm, const double *base_cmd, const uint8_t *has_targets, double dt,
            int32_t substeps, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b) return fail(RS_ERR_ARG, "null batch");
  if (!(dt > 0) || substeps < 1) return fail(RS_ERR_ARG, "bad step parameters (dt > 0, substeps >= 1)");
  if (!arm || !base_cmd) return fail(RS_ERR_ARG, "arm_targets and base_cmd are required device pointers");
  CUDA_TRY(launch_step_b(b, arm, base_cmd, 2, has_targets, dt, substeps, (cudaStream_t)stream));
  b->cur ^= 1;
  return RS_OK;
}

int rs_render(rs_batch *b, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b) return fail(RS_ERR_ARG, "null batch");
  if (cam_mask >> 2) return fail(RS_ERR_ARG, "camera mask selects a camera the robot does not have");
  CUDA_TRY(launch_render(b->view(), cam_mask, rgba, depth, ids, (cudaStream_t)stream));
  return RS_OK;
}

int rs_render_mesh(rs_batch *b, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b) return fail(RS_ERR_ARG, "null batch");
  if (cam_mask >> 2) return fail(RS_ERR_ARG, "camera mask selects a camera the robot does not have");
  DevBatch v = b->view();
  if (!b->has_mesh) return fail(RS_ERR_ARG, "scene has no mesh (rs_scene_set_mesh before rs_batch_create)");
  CUDA_TRY(launch_render_mesh(v, cam_mask, rgba, depth, ids, (cudaStream_t)stream));
  return RS_OK;
}

static int ensure_ik_scratch(rs_batch *b) {
  if (!b->d_ik_scratch) CUDA_TRY(cudaMalloc(&b->d_ik_scratch, sizeof(double) * ((size_t)b->d.n_env * 4 + 2)));
  return RS_OK;
}

int rs_arm_action(rs_batch *b, const double *delta_ee, double *arm_targets, int32_t *ik_failed, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !delta_ee || !arm_targets) return fail(RS_ERR_ARG, "null argument");
  int rc = ensure_ik_scratch(b);
  if (rc) return rc;
  CUDA_TRY(launch_ik(b->view(), delta_ee, 3, arm_targets, ik_failed, b->d_ik_scratch, (cudaStream_t)stream));
  return RS_OK;
}

int rs_grasp(rs_batch *b, const double *gripper, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !gripper) return fail(RS_ERR_ARG, "null argument");
  CUDA_TRY(launch_grasp(b->view(), gripper, 1, (cudaStream_t)stream));
  return RS_OK;
}

int rs_set_trace(rs_batch *b, int32_t *pairs, int32_t *count, int32_t cap, int32_t max_substeps) {
  DeviceScope device_scope(b);
  if (!b) return fail(RS_ERR_ARG, "null batch");
  if ((pairs == nullptr) != (count == nullptr)) return fail(RS_ERR_ARG, "pairs and count must both be set or NULL");
  b->d.trace_pairs = pairs;
  b->d.trace_count = count;
  b->d.trace_cap = pairs ? cap : 0;
  b->d.trace_sub = pairs ? max_substeps : 0;
  return RS_OK;
}

// stats buffer, render side stream and fork/join events shared by
// rs_step_host and rs_env_step_host; each resource guarded on its own handle
static int ensure_host_step(rs_batch *b) {
  if (!b->d_stats) CUDA_TRY(cudaMalloc(&b->d_stats, sizeof(double) * (size_t)b->d.n_env * 4));
  if (!b->side) CUDA_TRY(cudaStreamCreateWithFlags(&b->side, cudaStreamNonBlocking));
  if (!b->ev_fork) CUDA_TRY(cudaEventCreateWithFlags(&b->ev_fork, cudaEventDisableTiming));
  if (!b->ev_join) CUDA_TRY(cudaEventCreateWithFlags(&b->ev_join, cudaEventDisableTiming));
  return RS_OK;
}

int rs_step_host(rs_batch *b, const double *h_arm, const double *h_base, double dt, int32_t substeps,
                 uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids, double *h_out_stats, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !h_arm || !h_base || !h_out_stats) return fail(RS_ERR_ARG, "null argument");
  const int E = b->d.n_env, na = b->narm;
  cudaStream_t st = (cudaStream_t)stream;
  if (!b->d_act) CUDA_TRY(cudaMalloc(&b->d_act, sizeof(double) * (size_t)E * (na + 2)));
  if (int rc0 = ensure_host_step(b)) return rc0;
  if (int rc0 = ensure_phys_hp(b)) return rc0;
  cudaStream_t hp = b->phys_hp;
  // render o_t = render(s_t) on the side stream, concurrently with the physics
  // s_t -> s_{t+1} on the high-priority stream (ping-pong state buffers;
  // PAPER.md:453-457); the render is enqueued before the step flips the buffers
  CUDA_TRY(cudaEventRecord(b->ev_fork, st));
  if (cam_mask) {
    CUDA_TRY(cudaStreamWaitEvent(b->side, b->ev_fork, 0));
    int rc = rs_render(b, cam_mask, rgba, depth, ids, b->side);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(b->ev_join, b->side));
  }
  CUDA_TRY(cudaStreamWaitEvent(hp, b->ev_fork, 0));
  double *d_arm = b->d_act, *d_base = b->d_act + (size_t)E * na;
  CUDA_TRY(cudaMemcpyAsync(d_arm, h_arm, sizeof(double) * (size_t)E * na, cudaMemcpyHostToDevice, hp));
  CUDA_TRY(cudaMemcpyAsync(d_base, h_base, sizeof(double) * (size_t)E * 2, cudaMemcpyHostToDevice, hp));
  int rc = rs_step(b, d_arm, d_base, nullptr, dt, substeps, hp);
  if (rc) return rc;
  CUDA_TRY(launch_stats(b->view(), b->d_stats, hp));
  CUDA_TRY(cudaMemcpyAsync(h_out_stats, b->d_stats, sizeof(double) * (size_t)E * 4, cudaMemcpyDeviceToHost, hp));
  CUDA_TRY(cudaEventRecord(b->hp_join, hp));
  CUDA_TRY(cudaStreamWaitEvent(st, b->hp_join, 0));
  if (cam_mask) CUDA_TRY(cudaStreamWaitEvent(st, b->ev_join, 0));
  // return once the step and its host results are done; the observation
  // completes in `stream` order (the next call's step waits for it there, so
  // the host can enqueue step t+1 while o_t is still rendering)
  CUDA_TRY(cudaEventSynchronize(b->hp_join));
  return RS_OK;
}

int rs_step_stats(rs_batch *b, double *out, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !out) return fail(RS_ERR_ARG, "null argument");
  CUDA_TRY(launch_stats(b->view(), out, (cudaStream_t)stream));
  return RS_OK;
}

int rsim_bench_render_work_detail(rs_batch *b, uint32_t cam_mask, unsigned long long *d_counters, void *stream) {
  DeviceScope device_scope(b);
  if (!b || !d_counters) return fail(RS_ERR_ARG, "null argument");
  CUDA_TRY(launch_render(b->view(), cam_mask, nullptr, nullptr, nullptr, (cudaStream_t)stream, d_counters));
  return RS_OK;
}

__global__ void work_total_kernel(const unsigned long long *w, unsigned long long *out) {
  *out += w[0] + w[1] + w[2] + w[6];
}

int rsim_bench_render_work(rs_batch *b, uint32_t cam_mask, unsigned long long *d_counter, void *stream) {
  DeviceScope device_scope(b);
  if (!b || !d_counter) return fail(RS_ERR_ARG, "null argument");
  unsigned long long *w = nullptr;
  CUDA_TRY(cudaMalloc(&w, 20 * sizeof(unsigned long long)));
  CUDA_TRY(cudaMemsetAsync(w, 0, 20 * sizeof(unsigned long long), (cudaStream_t)stream));
  CUDA_TRY(launch_render(b->view(), cam_mask, nullptr, nullptr, nullptr, (cudaStream_t)stream, w));
  work_total_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(w, d_counter);
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  cudaFree(w);
  return RS_OK;
}

// ---- observation proprioception
int rs_proprio(rs_batch *b, const double *base_prev, const double *goals, int32_t n_goals, double *out,
               double *base_out, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !out || n_goals < 0 || (n_goals > 0 && !goals)) return fail(RS_ERR_ARG, "bad proprioception arguments");
  CUDA_TRY(launch_proprio(b->view(), base_prev, goals, n_goals, out, base_out, (cudaStream_t)stream));
  return RS_OK;
}

// ---- point queries (physics.py:1088-1101)
int rs_sphere_cast(rs_batch *b, const int32_t *env_of_query, const double *origins, const double *dirs,
                   const double *max_dist, int32_t n_queries, int32_t *out_body, double *out_t, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !origins || !dirs || !max_dist || !out_body || !out_t || n_queries < 0)
    return fail(RS_ERR_ARG, "bad sphere_cast arguments");
  if (!env_of_query && n_queries > b->d.n_env) return fail(RS_ERR_ARG, "env_of_query = NULL needs n_queries <= n_env");
  CUDA_TRY(launch_sphere_cast(b->view(), env_of_query, origins, dirs, max_dist, n_queries, out_body, out_t,
                              (cudaStream_t)stream));
  return RS_OK;
}

// ---- batched settle (physics.py:1113-1176)
int rs_settle(rs_batch *b, const uint64_t *placed, uint8_t *active, int32_t max_steps, double floor_z,
              int32_t *status, int32_t *info, double *value, int32_t *steps, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !placed || !active || !status || !info || !value || !steps || max_steps < 0)
    return fail(RS_ERR_ARG, "bad settle arguments");
  const int E = b->d.n_env;
  cudaStream_t st = (cudaStream_t)stream;
  if (!b->d_settle_zero) {
    CUDA_TRY(cudaMalloc(&b->d_settle_zero, sizeof(double) * (size_t)E * (b->narm > 2 ? b->narm : 2)));
    CUDA_TRY(cudaMemset(b->d_settle_zero, 0, sizeof(double) * (size_t)E * (b->narm > 2 ? b->narm : 2)));
    CUDA_TRY(cudaMalloc(&b->d_settle_noct, E));
    CUDA_TRY(cudaMemset(b->d_settle_noct, 0, E));
    CUDA_TRY(cudaMalloc(&b->d_settle_count, sizeof(int32_t)));
    CUDA_TRY(cudaMallocHost(&b->h_settle_count, sizeof(int32_t)));
  }
  CUDA_TRY(launch_settle_clearance(b->view(), placed, active, status, info, value, steps, st));
  const double floor_limit = floor_z - 0.5;
  int rc = RS_OK;
  for (int k = 1; k <= max_steps; ++k) {
    b->d.env_active = active;  // Simulator.step_physics(state, None) on the envs still settling
    cudaError_t e = launch_step_b(b, b->d_settle_zero, b->d_settle_zero, 2, b->d_settle_noct, 1.0 / 30.0, 4, st);
    b->d.env_active = nullptr;
    if (e != cudaSuccess) { rc = fail(RS_ERR_CUDA, cudaGetErrorString(e)); break; }
    b->cur ^= 1;
    CUDA_TRY(cudaMemsetAsync(b->d_settle_count, 0, sizeof(int32_t), st));
    CUDA_TRY(launch_settle_check(b->view(), placed, active, status, info, value, steps, floor_limit, k, max_steps,
                                 b->d_settle_count, st));
    if (k % 8 == 0 || k == max_steps) {  // stop once every env is done
      CUDA_TRY(cudaMemcpyAsync(b->h_settle_count, b->d_settle_count, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      if (*b->h_settle_count == 0) break;
    }
  }
  return rc;
}

// ---- geodesics (navgrid.py:109-172)
int rs_nav_shape(rs_batch *b, int32_t *nx, int32_t *ny) {
  DeviceScope device_scope(b);
  if (!b || !nx || !ny) return fail(RS_ERR_ARG, "null argument");
  if (b->nav_nx < 0) return fail(RS_ERR_ARG, "the batch's scenes have different walk-grid shapes");
  *nx = b->nav_nx; *ny = b->nav_ny;
  return RS_OK;
}

int rs_nav_fields(rs_batch *b, const int32_t *scene_of_goal, const double *goal_xy, int32_t n_goals, double *fields,
                  int32_t *goal_cell, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !goal_xy || !fields || n_goals < 0) return fail(RS_ERR_ARG, "bad nav field arguments");
  if (b->nav_nx < 0) return fail(RS_ERR_ARG, "the batch's scenes have different walk-grid shapes");
  if ((size_t)b->nav_nx * b->nav_ny * 9 > 227 * 1024) return fail(RS_ERR_ARG, "walk grid too large for one CTA");
  CUDA_TRY(launch_nav_fields(b->view(), b->nav_nx, b->nav_ny, scene_of_goal, goal_xy, n_goals, fields, goal_cell,
                             (cudaStream_t)stream));
  return RS_OK;
}

int rs_nav_geodesic(rs_batch *b, const double *fields, const int32_t *field_of_query, const int32_t *scene_of_query,
                    const double *from_xy, int32_t n_queries, double *out, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !fields || !field_of_query || !out || n_queries < 0) return fail(RS_ERR_ARG, "bad geodesic arguments");
  if (b->nav_nx < 0) return fail(RS_ERR_ARG, "the batch's scenes have different walk-grid shapes");
  if (!from_xy && n_queries != b->d.n_env) return fail(RS_ERR_ARG, "robot-base queries need n_queries == n_env");
  CUDA_TRY(launch_nav_geodesic(b->view(), b->nav_nx, b->nav_ny, fields, field_of_query, scene_of_query, from_xy,
                               n_queries, out, (cudaStream_t)stream));
  return RS_OK;
}

int rs_nav_path(rs_batch *b, const double *fields, const int32_t *field_of_query, const int32_t *scene_of_query,
                const double *from_xy, int32_t n_queries, int32_t cap, double *waypoints, int32_t *count,
                void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !fields || !field_of_query || !from_xy || !waypoints || !count || n_queries < 0 || cap < 1)
    return fail(RS_ERR_ARG, "bad path arguments");
  if (b->nav_nx < 0) return fail(RS_ERR_ARG, "the batch's scenes have different walk-grid shapes");
  CUDA_TRY(launch_nav_path(b->view(), b->nav_nx, b->nav_ny, fields, field_of_query, scene_of_query, from_xy,
                           n_queries, cap, waypoints, count, (cudaStream_t)stream));
  return RS_OK;
}

int rsim_bench_force_heavy(rs_batch *b, int width) {
  DeviceScope device_scope(b);
  if (!b) return fail(RS_ERR_ARG, "null batch");
  if (width != 0 && width != 8 && width != 16 && width != -8 && width != -16 && width != -1)
    return fail(RS_ERR_ARG, "width must be 0, -1, +-8 or +-16");
  b->force_heavy = width;
  return RS_OK;
}

int rsim_bench_env_cycles(rs_batch *b, long long *d_cycles) {
  DeviceScope device_scope(b);
  if (!b) return fail(RS_ERR_ARG, "null batch");
  b->d.env_cycles = d_cycles;
  return RS_OK;
}

int rsim_bench_phase_cycles(rs_batch *b, long long *d_cycles) {
  DeviceScope device_scope(b);
  if (!b) return fail(RS_ERR_ARG, "null batch");
  b->d.phase_cycles = d_cycles;
  return RS_OK;
}

int rsim_bench_render_exact(rs_batch *b, uint32_t cam_mask, uint8_t *rgba, float *depth, int32_t *ids,
                            void *stream) {
  DeviceScope device_scope(b);
  if (!b) return fail(RS_ERR_ARG, "null batch");
  CUDA_TRY(launch_render_exact(b->view(), cam_mask, rgba, depth, ids, (cudaStream_t)stream));
  return RS_OK;
}

int rsim_bench_render_mesh_work(rs_batch *b, uint32_t cam_mask, unsigned long long *d_counter, void *stream) {
  DeviceScope device_scope(b);
  if (!b || !d_counter || !b->has_mesh) return fail(RS_ERR_ARG, "null argument or no mesh");
  unsigned long long *w = nullptr;
  CUDA_TRY(cudaMalloc(&w, 20 * sizeof(unsigned long long)));
  CUDA_TRY(cudaMemsetAsync(w, 0, 20 * sizeof(unsigned long long), (cudaStream_t)stream));
  CUDA_TRY(launch_render_mesh(b->view(), cam_mask, nullptr, nullptr, nullptr, (cudaStream_t)stream, w));
  work_total_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(w, d_counter);
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  cudaFree(w);
  return RS_OK;
}

// ---- the SPEC env step with the paper's action space (§5.1)
static int ensure_env_buffers(rs_batch *b) {
  const int E = b->d.n_env;
  if (!b->d_targets) {
    CUDA_TRY(cudaMalloc(&b->d_targets, sizeof(double) * (size_t)E * b->narm));
    CUDA_TRY(cudaMalloc(&b->d_ik_failed, sizeof(int32_t) * (size_t)E));
    CUDA_TRY(cudaMalloc(&b->d_env_act, sizeof(double) * (size_t)E * 6));
  }
  return ensure_host_step(b);
}

int rs_env_step(rs_batch *b, const double *action, double dt, int32_t substeps, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !action) return fail(RS_ERR_ARG, "null argument");
  if (!(dt > 0) || substeps < 1) return fail(RS_ERR_ARG, "bad step parameters (dt > 0, substeps >= 1)");
  int rc = ensure_env_buffers(b);
  if (!rc) rc = ensure_ik_scratch(b);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(enqueue_env_order(b, st));  // policy 1: overlaps the IK on the physics side stream
  CUDA_TRY(launch_ik(b->view(), action, 6, b->d_targets, b->d_ik_failed, b->d_ik_scratch, st));  // robot.py:293
  CUDA_TRY(launch_step_b(b, b->d_targets, action + 4, 6, nullptr, dt, substeps, st));  // physics.py:575
  b->cur ^= 1;
  CUDA_TRY(launch_grasp(b->view(), action + 3, 6, st));                                   // robot.py:323
  return RS_OK;
}

int rs_env_step_host(rs_batch *b, const double *h_action, double dt, int32_t substeps, uint32_t cam_mask,
                     uint8_t *rgba, float *depth, int32_t *ids, double *h_out_stats, void *stream) {
  DeviceScope device_scope(b);
  NvtxRange nvtx_range(__func__);
  if (!b || !h_action || !h_out_stats) return fail(RS_ERR_ARG, "null argument");
  int rc = ensure_env_buffers(b);
  if (rc) return rc;
  if ((rc = ensure_phys_hp(b))) return rc;
  const int E = b->d.n_env;
  cudaStream_t st = (cudaStream_t)stream, hp = b->phys_hp;
  CUDA_TRY(cudaEventRecord(b->ev_fork, st));
  if (cam_mask) {  // o_t = render(s_t) on the side stream (enqueued before the step flips the buffers)
    CUDA_TRY(cudaStreamWaitEvent(b->side, b->ev_fork, 0));
    rc = rs_render(b, cam_mask, rgba, depth, ids, b->side);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(b->ev_join, b->side));
  }
  // the action upload first: the previous call's step (the only reader of
  // d_env_act) is complete, so it overlaps the previous observation's render
  CUDA_TRY(cudaMemcpyAsync(b->d_env_act, h_action, sizeof(double) * (size_t)E * 6, cudaMemcpyHostToDevice, hp));
  CUDA_TRY(cudaStreamWaitEvent(hp, b->ev_fork, 0));
  rc = rs_env_step(b, b->d_env_act, dt, substeps, hp);
  if (rc) return rc;
  CUDA_TRY(launch_stats(b->view(), b->d_stats, hp));
  CUDA_TRY(cudaMemcpyAsync(h_out_stats, b->d_stats, sizeof(double) * (size_t)E * 4, cudaMemcpyDeviceToHost, hp));
  CUDA_TRY(cudaEventRecord(b->hp_join, hp));
  CUDA_TRY(cudaStreamWaitEvent(st, b->hp_join, 0));
  if (cam_mask) CUDA_TRY(cudaStreamWaitEvent(st, b->ev_join, 0));
  // return once the step and its host results are done; the observation
  // completes in `stream` order (the next call's step waits for it there, so
  // the host can enqueue step t+1 while o_t is still rendering)
  CUDA_TRY(cudaEventSynchronize(b->hp_join));
  return RS_OK;
}
