"""BASELINE.json configs[3]: rendering-only sweep, 1024 envs x 128x128 RGBD
(head + arm) at 10k-200k triangles per scene, on one B200.

Prints one JSON line per triangle budget: render-only env-steps/s (2 camera
frames per env-step), ms per batch, the proxy (convex) renderer on the same
states for reference, and the SURVEY.md §8d rasterisation work model
W = 60 T_frustum + 10 F per camera frame (T_frustum = triangles meeting the
view frustum, F = (triangle, pixel-centre) coverage count, occlusion
ignored), computed on the host for a sample of env-camera frames (`raster_work`,
a numpy restatement, not the oracle) and reported as `roofline`: W per batch /
kernel time against the measured FP32 peak."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402

E = int(os.environ.get("ENVS", "1024"))
KS = [int(k) for k in os.environ.get("KS", "3,4,7,9,12").split(",")]
REPS = 5


def timed(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(REPS):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


SAMPLE = int(os.environ.get("SAMPLE", "12"))


def camera_poses(world, st):
    """World (R, o) of the head and arm cameras (robot.py:43-47, 156-169):
    base3(x, y, yaw) for the head mount, the arm chain + gripper offset for
    the arm mount; camera frame columns = (right, down, view)."""
    from paper_2106_14405_b200.geom import Pose, axis_angle_rot, base_pose

    r = world.robot
    q = np.asarray(st.joints)[world.n_scene_joints:]
    base = base_pose(st.base)
    t = base
    for j, qj in zip(r.joints, q):
        t = t.compose(Pose(np.eye(3), np.asarray(j.offset, float))).compose(Pose(axis_angle_rot(j.axis, qj)))
    ee = t.compose(Pose(np.eye(3), np.asarray(r.gripper_offset, float)))
    out = []
    for name in ("head", "arm"):
        parent, mount = r.cameras[name]
        c = (base if parent == "base" else ee).compose(mount)
        out.append((c.rot, c.pos))
    return out


def raster_work(world, mesh_tris, st, W=128, H=128, fov=np.pi / 2, znear=0.1, zfar=10.0):
    """(T_frustum, F) per camera for one env state.  mesh_tris: per part the
    [T, 3, 3] part-frame triangles (the k-subdivided soups).  F counts pixel
    centres inside each triangle's projection (triangles wholly in front of
    the near plane; the few crossing it are
    clipped against it first)."""
    from paper_2106_14405_b200.geom import Pose, quat_to_rot

    f = (W / 2.0) / np.tan(fov / 2.0)
    world_tris = []
    pi = 0
    for b in world.bodies:
        bp = Pose(quat_to_rot(st.quat[b.body_id]), st.pos[b.body_id])
        for local, _prim in b.parts:
            wp = bp.compose(local)
            world_tris.append(mesh_tris[pi] @ wp.rot.T + wp.pos)
            pi += 1
    V = np.concatenate(world_tris)  # [T, 3, 3]
    res = []
    for R, o in camera_poses(world, st):
        C = (V - o) @ R  # camera frame: x right, y down, z view
        z = C[..., 2]
        x, y = C[..., 0], C[..., 1]
        # frustum culling (all three vertices outside one plane -> out)
        out = (z < znear).all(1) | (z > zfar).all(1)
        for sx in (1.0, -1.0):
            out |= (sx * x > (W / 2.0) / f * z).all(1)
            out |= (sx * y > (H / 2.0) / f * z).all(1)
        inf = ~out
        T = int(inf.sum())
        front = inf & (z > znear).all(1)
        P = np.stack([f * x / np.where(z > 0, z, 1) + W / 2.0, f * y / np.where(z > 0, z, 1) + H / 2.0], -1)[front]
        # triangles crossing the near plane: clipped (Sutherland-Hodgman) into a fan of triangles
        extra = []
        for tri in C[inf & ~(z > znear).all(1)]:
            poly = []
            for i in range(3):
                a_, b_ = tri[i], tri[(i + 1) % 3]
                if a_[2] > znear:
                    poly.append(a_)
                if (a_[2] > znear) != (b_[2] > znear):
                    t = (znear - a_[2]) / (b_[2] - a_[2])
                    poly.append(a_ + t * (b_ - a_))
            pp = [np.array([f * q[0] / q[2] + W / 2.0, f * q[1] / q[2] + H / 2.0]) for q in poly]
            extra += [[pp[0], pp[i], pp[i + 1]] for i in range(1, len(pp) - 1)]
        if extra:
            P = np.concatenate([P, np.array(extra)])
        F = 0
        lo = np.clip(np.floor(P.min(1) - 0.5), 0, [W - 1, H - 1]).astype(int)
        hi = np.clip(np.ceil(P.max(1) - 0.5), 0, [W - 1, H - 1]).astype(int)
        ext = (hi - lo + 1).max(1)
        a, bq, cq = P[:, 0], P[:, 1], P[:, 2]
        area = (bq[:, 0] - a[:, 0]) * (cq[:, 1] - a[:, 1]) - (bq[:, 1] - a[:, 1]) * (cq[:, 0] - a[:, 0])
        for s_ in np.unique(ext):  # triangles grouped by bounding-box size: vectorised edge tests
            sel = np.nonzero((ext == s_) & (area != 0))[0]
            if not len(sel):
                continue
            g = np.arange(s_)
            px = lo[sel, 0, None, None] + g[None, None, :] + 0.5
            py = lo[sel, 1, None, None] + g[None, :, None] + 0.5
            inside = np.ones((len(sel), s_, s_), bool)
            sg = np.sign(area[sel])[:, None, None]
            for u, v in ((a, bq), (bq, cq), (cq, a)):
                u_, v_ = u[sel], v[sel]
                e = (v_[:, 0, None, None] - u_[:, 0, None, None]) * (py - u_[:, 1, None, None]) - \
                    (v_[:, 1, None, None] - u_[:, 1, None, None]) * (px - u_[:, 0, None, None])
                inside &= sg * e >= 0
            inside &= (px < W) & (py < H)
            F += int(inside.sum())
        cross = inf & ~(z > znear).all(1)  # near-plane crossers: their screen bbox clipped to the image
        res.append((T, F, int(cross.sum())))
    return res


gids = np.arange(E)
states = bench.idle_states(gids, bench.settled_pool())
from paper_2106_14405_b200 import native  # noqa: E402
from paper_2106_14405_b200.mesh import part_triangles, subdivide  # noqa: E402
from paper_2106_14405_b200.state import WorldState  # noqa: E402

peak32 = C.c_double(0)
L = native.lib()
L.rsim_bench_fma_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
L.rsim_bench_fma_peak(0, C.byref(peak32))
for k in KS:
    sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=(gids % 3).tolist(), mesh_k=k)
    sim.set_state(states)
    obs = sim.alloc_obs()
    ms_mesh = timed(lambda: sim.render_mesh(out=obs))
    ms_proxy = timed(lambda: sim.render(out=obs))
    # W = 60 T_frustum + 10 F per camera frame on a sample of envs (all layouts)
    tris = {v: [subdivide(part_triangles(p), k) for b in sim.worlds[v].bodies for _, p in b.parts] for v in range(3)}
    samp = np.linspace(0, E - 1, SAMPLE).astype(int)
    tf = []
    for e in samp:
        v = int(gids[e] % 3)
        for T, F, nx in raster_work(sim.worlds[v], tris[v], WorldState.from_bytes(states[e])):
            tf.append((T, F, nx))
    tf = np.array(tf, float)
    w_frame = float((60 * tf[:, 0] + 10 * tf[:, 1]).mean())
    ach = w_frame * 2 * E / (ms_mesh * 1e-3) / 1e12
    print(json.dumps({"config": "configs[3] render-only sweep", "envs": E, "cams": 2, "k": k,
                      "triangles_per_scene": sim.n_triangles, "ms_per_batch_mesh": ms_mesh,
                      "env_steps_per_s_mesh": E / (ms_mesh * 1e-3),
                      "ms_per_batch_proxy": ms_proxy, "env_steps_per_s_proxy": E / (ms_proxy * 1e-3),
                      "raster_model": {"T_frustum_per_frame": float(tf[:, 0].mean()),
                                       "F_per_frame": float(tf[:, 1].mean()),
                                       "near_plane_crossers_per_frame": float(tf[:, 2].mean()),
                                       "W_flop_per_frame": w_frame, "sampled_frames": len(tf)},
                      "roofline": {"bound": "fp32", "kernel": "render_kernel<1,0> (mesh, FP64 BVH ray tracer)",
                                   "achieved": ach, "peak": peak32.value, "unit": "TFLOP/s",
                                   "frac": ach / peak32.value if peak32.value else None,
                                   "note": "SURVEY.md §8d rasterisation model W = 60 T_frustum + 10 F per frame; "
                                           "the kernel ray-traces per-part BVHs in FP64 instead"}}), flush=True)
    sim.close()
