"""ctypes mirror of ``include/rsim.h`` (structs only; no library loading).

``SceneDesc.from_tables`` marshals the scene compiler's numpy tables into an
``rs_scene_desc`` whose pointers stay valid as long as the returned object
(which keeps the arrays alive) does.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

I32P = C.POINTER(C.c_int32)
F64P = C.POINTER(C.c_double)
F32P = C.POINTER(C.c_float)
U8P = C.POINTER(C.c_uint8)

RS_OK, RS_ERR_ARG, RS_ERR_CUDA, RS_ERR_SNAPSHOT, RS_ERR_CAPACITY = 0, 1, 2, 3, 4
FAULT_KINDS = {1: "non-finite pos", 2: "non-finite quat", 3: "non-finite vel", 4: "non-finite joint position",
               5: "capacity overflow"}
# low 16 bits of a capacity-overflow fault word (include/rsim.h RS_OVF_*)
OVERFLOW_KINDS = {1: "AABB-overlap candidates > 1024", 2: "admitted pairs > 256", 3: "contact rows > 512",
                  4: "touching pairs > 96", 5: "contacts of one pair > 32", 6: "block matrices > 8192 entries"}


class rs_scene_desc(C.Structure):
    _fields_ = [
        ("n_bodies", C.c_int32), ("n_parts", C.c_int32), ("n_facets", C.c_int32), ("n_verts", C.c_int32),
        ("n_tris", C.c_int32), ("n_scene_joints", C.c_int32), ("n_arm", C.c_int32), ("robot_base", C.c_int32),
        ("body_kind", I32P), ("body_robot", I32P), ("body_group", I32P), ("body_joint", I32P),
        ("body_inv_mass", F64P), ("body_com", F64P), ("body_inv_inertia", F64P),
        ("body_friction", F64P), ("body_restitution", F64P),
        ("body_part_begin", I32P), ("body_color", F32P),
        ("part_body", I32P), ("part_kind", I32P), ("part_local", F64P), ("part_param", F64P),
        ("part_facet_begin", I32P), ("part_vert_begin", I32P), ("part_tri_begin", I32P),
        ("facet", F64P), ("vert", F64P), ("tri", I32P),
        ("joint_type", I32P), ("joint_body", I32P), ("joint_parent", I32P),
        ("joint_axis", F64P), ("joint_origin", F64P), ("joint_limits", F64P), ("joint_handle", F64P),
        ("arm_offset", F64P), ("arm_axis", F64P), ("arm_limits", F64P), ("gripper_offset", C.c_double * 3),
        ("n_cameras", C.c_int32), ("cam_parent", I32P), ("cam_mount", F64P),
        ("nav_nx", C.c_int32), ("nav_ny", C.c_int32), ("nav_origin", C.c_double * 2), ("nav_cell", C.c_double),
        ("nav_walkable", U8P),
    ]


class rs_mesh_desc(C.Structure):
    _fields_ = [("n_parts", C.c_int32), ("n_tris", C.c_int32), ("n_nodes", C.c_int32), ("tri", F64P),
                ("node_lo", F32P), ("node_hi", F32P), ("node_meta", I32P), ("part_node_begin", I32P),
                ("part_bound", F64P)]


class MeshDesc:
    """Owns the mesh arrays (paper_2106_14405_b200.mesh.compile_mesh) and the rs_mesh_desc view."""

    def __init__(self, m: dict):
        self.arrays = {
            "tri": np.ascontiguousarray(m["tri"], np.float64),
            "node_lo": np.ascontiguousarray(m["node_lo"], np.float32),
            "node_hi": np.ascontiguousarray(m["node_hi"], np.float32),
            "node_meta": np.ascontiguousarray(m["node_meta"], np.int32),
            "part_node_begin": np.ascontiguousarray(m["part_node_begin"], np.int32),
            "part_bound": np.ascontiguousarray(m["part_bound"], np.float64),
        }
        a = self.arrays
        d = rs_mesh_desc()
        d.n_parts = len(a["part_bound"])
        d.n_tris = len(a["tri"])
        d.n_nodes = len(a["node_meta"])
        d.tri = _ptr(a["tri"], C.c_double)
        d.node_lo = _ptr(a["node_lo"], C.c_float)
        d.node_hi = _ptr(a["node_hi"], C.c_float)
        d.node_meta = _ptr(a["node_meta"], C.c_int32)
        d.part_node_begin = _ptr(a["part_node_begin"], C.c_int32)
        d.part_bound = _ptr(a["part_bound"], C.c_double)
        self.desc = d


class rs_physics_config(C.Structure):
    _fields_ = [
        ("gravity", C.c_double), ("solver_iterations", C.c_int32),
        ("correction_factor", C.c_double), ("slop", C.c_double), ("restitution_threshold", C.c_double),
        ("contact_margin", C.c_double), ("sleep_lin_threshold", C.c_double), ("sleep_ang_threshold", C.c_double),
        ("sleep_substeps", C.c_int32), ("wake_margin", C.c_double), ("lin_damping", C.c_double),
        ("ang_damping", C.c_double), ("joint_damping", C.c_double), ("joint_inertia_revolute", C.c_double),
        ("joint_inertia_prismatic", C.c_double), ("kp", C.c_double), ("motor_impulse_cap", C.c_double),
        ("impulse_cap_per_control_step", C.c_int32), ("sleeping_enabled", C.c_int32),
    ]


class rs_render_config(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fov", C.c_double), ("znear", C.c_double),
                ("zfar", C.c_double), ("tie_eps", C.c_double)]


class rs_buffers(C.Structure):
    _fields_ = [("n_env", C.c_int32), ("n_bodies", C.c_int32), ("n_joints", C.c_int32), ("event_cap", C.c_int32),
                ("fault", C.c_void_p), ("event_count", C.c_void_p), ("events", C.c_void_p),
                ("counters", C.c_void_p)]


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


class SceneDesc:
    """Owns contiguous copies of the tables and the ``rs_scene_desc`` view."""

    _I32 = ("body_kind", "body_robot", "body_group", "body_joint", "body_part_begin", "part_body", "part_kind",
            "part_facet_begin", "part_vert_begin", "part_tri_begin", "tri", "joint_type", "joint_body",
            "joint_parent", "cam_parent")
    _F64 = ("body_inv_mass", "body_com", "body_inv_inertia", "body_friction", "body_restitution", "part_local",
            "part_param", "facet", "vert", "joint_axis", "joint_origin", "joint_limits", "joint_handle",
            "arm_offset", "arm_axis", "arm_limits", "cam_mount")

    def __init__(self, t: dict):
        self.arrays = {}
        d = rs_scene_desc()
        for k in self._I32:
            a = np.ascontiguousarray(t[k], dtype=np.int32)
            self.arrays[k] = a
            setattr(d, k, _ptr(a, C.c_int32))
        for k in self._F64:
            a = np.ascontiguousarray(t[k], dtype=np.float64)
            self.arrays[k] = a
            setattr(d, k, _ptr(a, C.c_double))
        col = np.ascontiguousarray(t["body_color"], dtype=np.float32)
        nav = np.ascontiguousarray(t["nav_walkable"], dtype=np.uint8)
        self.arrays["body_color"], self.arrays["nav_walkable"] = col, nav
        d.body_color = _ptr(col, C.c_float)
        d.nav_walkable = _ptr(nav, C.c_uint8)
        d.n_bodies = len(t["body_kind"])
        d.n_parts = len(t["part_kind"])
        d.n_facets = len(t["facet"])
        d.n_verts = len(t["vert"])
        d.n_tris = len(t["tri"])
        d.n_scene_joints = int(t["n_scene_joints"])
        d.n_arm = int(t["n_arm"])
        d.robot_base = int(t["robot_base"])
        for i in range(3):
            d.gripper_offset[i] = float(t["gripper_offset"][i])
        d.n_cameras = len(t["cam_parent"])
        d.nav_nx, d.nav_ny = nav.shape
        d.nav_origin[0], d.nav_origin[1] = (float(v) for v in t["nav_origin"])
        d.nav_cell = float(t["nav_cell"])
        self.desc = d
        self.n_bodies = d.n_bodies
        self.n_joints = d.n_scene_joints + d.n_arm


def physics_config(**over) -> rs_physics_config:
    """``PhysicsConfig`` defaults (physics.py:54-74) with overrides."""
    v = dict(gravity=9.81, solver_iterations=16, correction_factor=0.2, slop=5e-4, restitution_threshold=0.25,
             contact_margin=1e-3, sleep_lin_threshold=1e-3, sleep_ang_threshold=1e-2, sleep_substeps=10,
             wake_margin=0.05, lin_damping=0.999, ang_damping=0.98, joint_damping=0.90,
             joint_inertia_revolute=1.2, joint_inertia_prismatic=4.0, kp=0.3, motor_impulse_cap=10.0,
             impulse_cap_per_control_step=0, sleeping_enabled=1)
    for k, x in over.items():
        if k not in v:
            raise KeyError(k)
        v[k] = int(x) if isinstance(v[k], int) else float(x)
    return rs_physics_config(**v)


def render_config(width=128, height=128, fov=np.pi / 2, znear=0.1, zfar=10.0, tie_eps=1e-9) -> rs_render_config:
    return rs_render_config(width, height, fov, znear, zfar, tie_eps)
