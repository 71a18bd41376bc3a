"""Scene compiler: ``World`` -> flat tables behind ``rs_scene_desc``.

The tables are the static half of the device data layout:
shared by every env of one layout variant, ~30 KB, read through L1/L2.

* bodies   kind, robot flag, no-collide group, driving scene joint,
           inverse mass, local COM, local inverse inertia, friction,
           restitution, part range, render colour;
* parts    owning body, primitive kind, local pose (row-major R | t),
           box half extents / sphere radius, facet / vertex / triangle ranges;
* facets   (n, offset) exactly as the reference's primitives hold them
           (box: +x +y +z -x -y -z; hull: qhull equations incl. coplanar
           duplicates, ``geometry.py:243-247``);
* vertices, hull triangles (for the sphere-vs-hull closest point,
           ``geometry.py:592-599``);
* scene joints, arm chain, camera mounts, walk-grid bitmap.
"""

from __future__ import annotations

import numpy as np

from . import assets as A
from .scene import KIND_DYNAMIC, KIND_KINEMATIC, KIND_STATIC, World

# render palette per category (pinned RGB rule)
PALETTE = {
    "backdrop": (0.78, 0.76, 0.72),
    "furniture": (0.55, 0.38, 0.24),
    "food": (0.85, 0.30, 0.20),
    "kitchen": (0.25, 0.55, 0.85),
    "robot": (0.60, 0.62, 0.66),
    "object": (0.50, 0.50, 0.50),
}


def body_colour(body) -> np.ndarray:
    base = np.array(PALETTE.get(body.category, PALETTE["object"]))
    # deterministic per-body tint so neighbouring bodies stay distinguishable
    h = (body.body_id * 2654435761) & 0xFFFFFFFF
    tint = np.array([(h >> 0) & 0xFF, (h >> 8) & 0xFF, (h >> 16) & 0xFF]) / 255.0
    return np.clip(0.8 * base + 0.2 * tint, 0.0, 1.0).astype(np.float32)


def compile_world(world: World) -> dict:
    bodies = world.bodies
    nb = len(bodies)
    t = {}
    t["body_kind"] = np.array([b.kind for b in bodies], np.int32)
    t["body_robot"] = np.array([int(b.is_robot) for b in bodies], np.int32)
    t["body_group"] = np.array([b.group for b in bodies], np.int32)
    t["body_joint"] = np.array([b.scene_joint for b in bodies], np.int32)
    t["body_inv_mass"] = np.array([b.inv_mass for b in bodies], np.float64)
    t["body_com"] = np.array([b.com for b in bodies], np.float64).reshape(nb, 3)
    t["body_inv_inertia"] = np.array([b.inv_inertia for b in bodies], np.float64).reshape(nb, 9)
    t["body_friction"] = np.array([b.friction for b in bodies], np.float64)
    t["body_restitution"] = np.array([b.restitution for b in bodies], np.float64)
    t["body_color"] = np.stack([body_colour(b) for b in bodies]).astype(np.float32)

    part_body, part_kind, part_local, part_param = [], [], [], []
    fb, vb, tb, pb = [0], [0], [0], [0]
    facets, verts, tris = [], [], []
    for b in bodies:
        for local, prim in b.parts:
            part_body.append(b.body_id)
            part_kind.append(prim.kind)
            part_local.append(local.as12())
            if prim.kind == A.KIND_SPHERE:
                part_param.append([prim.radius, 0.0, 0.0])
            elif prim.kind == A.KIND_BOX:
                part_param.append(prim.half)
            else:
                part_param.append([0.0, 0.0, 0.0])
            facets.append(np.concatenate([prim.normals, prim.offsets[:, None]], axis=1))
            verts.append(prim.vertices)
            tris.append(prim.triangles)
            fb.append(fb[-1] + len(prim.normals))
            vb.append(vb[-1] + len(prim.vertices))
            tb.append(tb[-1] + len(prim.triangles))
        pb.append(len(part_body))
    t["body_part_begin"] = np.array(pb, np.int32)
    t["part_body"] = np.array(part_body, np.int32)
    t["part_kind"] = np.array(part_kind, np.int32)
    t["part_local"] = np.array(part_local, np.float64)
    t["part_param"] = np.array(part_param, np.float64)
    t["part_facet_begin"] = np.array(fb, np.int32)
    t["part_vert_begin"] = np.array(vb, np.int32)
    t["part_tri_begin"] = np.array(tb, np.int32)
    t["facet"] = np.concatenate(facets).astype(np.float64)
    t["vert"] = np.concatenate(verts).astype(np.float64)
    t["tri"] = np.concatenate(tris).astype(np.int32).reshape(-1, 3)

    js = world.layout.joints
    t["joint_type"] = np.array([0 if j.spec.joint_type == "revolute" else 1 for j in js], np.int32)
    t["joint_body"] = np.array([j.body_id for j in js], np.int32)
    t["joint_parent"] = np.array([j.parent_body for j in js], np.int32)
    t["joint_axis"] = np.array([j.spec.axis for j in js], np.float64)
    t["joint_origin"] = np.array([j.spec.origin.as12() for j in js], np.float64)
    t["joint_limits"] = np.array([j.spec.limits for j in js], np.float64)
    t["joint_handle"] = np.array([j.spec.handle_point for j in js], np.float64)

    r = world.robot
    t["arm_offset"] = np.array([j.offset for j in r.joints], np.float64)
    t["arm_axis"] = np.array([j.axis for j in r.joints], np.float64)
    t["arm_limits"] = np.array([j.limits for j in r.joints], np.float64)
    t["gripper_offset"] = np.asarray(r.gripper_offset, np.float64)
    cams = [r.cameras["head"], r.cameras["arm"]]
    t["cam_parent"] = np.array([0 if p == "base" else 1 for p, _ in cams], np.int32)
    t["cam_mount"] = np.array([pose.as12() for _, pose in cams], np.float64)

    g = world.layout.grid
    t["nav_walkable"] = np.ascontiguousarray(g.walkable.astype(np.uint8))
    t["nav_origin"] = np.asarray(g.origin, np.float64)
    t["nav_cell"] = float(g.cell)
    t["robot_base"] = world.robot_body_ids[0]
    t["n_scene_joints"] = len(js)
    t["n_arm"] = r.dof
    return t
