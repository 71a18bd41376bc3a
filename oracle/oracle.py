"""ctypes front end of the C oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module; the product package never does.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2106_14405_b200.abi import SceneDesc, physics_config, render_config

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "rsim_oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


class _Trace(C.Structure):
    _fields_ = [("cap_pairs", C.c_int32), ("cap_contacts", C.c_int32), ("cap_events", C.c_int32),
                ("n_pairs", C.c_int32), ("n_contacts", C.c_int32), ("n_events", C.c_int32),
                ("pairs", C.POINTER(C.c_int32)), ("contacts", C.POINTER(C.c_double)),
                ("events", C.POINTER(C.c_double)), ("counters", C.c_int64 * 3)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_step.restype = C.c_int
        L.orc_step.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                               C.c_void_p, C.POINTER(C.c_uint32)]
        L.orc_render.restype = C.c_int
        L.orc_render.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p]
        L.orc_camera_pose.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_void_p]
        L.orc_move_base.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_void_p]
        L.orc_nearest_walkable.restype = C.c_int
        L.orc_nearest_walkable.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_void_p]
        L.orc_link_poses.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_solve_ik.restype = C.c_int
        L.orc_solve_ik.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_apply_arm_action.restype = C.c_int
        L.orc_apply_arm_action.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_nav_field.restype = C.c_long
        L.orc_nav_field.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_void_p]
        L.orc_nav_geodesic.restype = C.c_double
        L.orc_nav_geodesic.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double]
        L.orc_nav_path.restype = C.c_int
        L.orc_nav_path.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_void_p, C.c_int]
        L.orc_spawn_clearance.restype = C.c_int
        L.orc_spawn_clearance.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_parts_distance.restype = C.c_double
        L.orc_parts_distance.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int]
        L.orc_settle.restype = C.c_int
        L.orc_settle.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64, C.c_int, C.c_double, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p]
        L.orc_sphere_cast.restype = C.c_int
        L.orc_sphere_cast.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p]
        L.orc_grasp.restype = C.c_int
        L.orc_grasp.argtypes = [C.c_void_p, C.c_char_p, C.c_double, C.c_void_p, C.c_void_p]
        L.orc_snapshot_size.restype = C.c_int64
        L.orc_snapshot_size.argtypes = [C.c_int, C.c_int]
        _lib = L
    return _lib


class StepResult:
    def __init__(self, snapshot, fault, pairs, contacts, events, counters):
        self.snapshot = snapshot
        self.fault = fault
        self.pairs = pairs          # [n, 3] substep, a, b
        self.contacts = contacts    # [n, 10] substep, a, b, p, n, depth
        self.events = events        # [n, 7]
        self.counters = counters    # narrowphase_tests, skipped_sleeping_pairs, wakes


class Oracle:
    """One CPU world (scene tables + PhysicsConfig)."""

    def __init__(self, tables: dict, **config):
        self.desc = SceneDesc(tables)
        self.cfg = physics_config(**config)
        self.h = lib().orc_create(C.byref(self.desc.desc), C.byref(self.cfg))
        if not self.h:
            raise RuntimeError("oracle: scene exceeds capacities")
        self.snap_size = lib().orc_snapshot_size(self.desc.n_bodies, self.desc.n_joints)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def step(self, snapshot: bytes, arm=None, base_cmd=(0.0, 0.0), dt=1.0 / 30.0, substeps=4,
             cap=(8192, 16384, 16384)) -> StepResult:
        out = np.zeros(self.snap_size, np.uint8)
        tr = _Trace()
        tr.cap_pairs, tr.cap_contacts, tr.cap_events = cap
        pairs = np.zeros((cap[0], 3), np.int32)
        contacts = np.zeros((cap[1], 10))
        events = np.zeros((cap[2], 7))
        tr.pairs = pairs.ctypes.data_as(C.POINTER(C.c_int32))
        tr.contacts = contacts.ctypes.data_as(C.POINTER(C.c_double))
        tr.events = events.ctypes.data_as(C.POINTER(C.c_double))
        fault = C.c_uint32(0)
        armp = basep = None
        if arm is not None:
            arm_a = np.ascontiguousarray(arm, dtype=np.float64)
            base_a = np.ascontiguousarray(base_cmd, dtype=np.float64)
            armp, basep = arm_a.ctypes.data, base_a.ctypes.data
        rc = lib().orc_step(self.h, bytes(snapshot), out.ctypes.data, armp, basep, dt, substeps, C.byref(tr),
                            C.byref(fault))
        if rc not in (0, 0x7FFFFFFF):
            raise ValueError(f"oracle step error {rc}")
        return StepResult(out.tobytes() if rc == 0 else None, fault.value, pairs[:tr.n_pairs].copy(),
                          contacts[:tr.n_contacts].copy(), events[:tr.n_events].copy(), list(tr.counters))

    def render(self, snapshot: bytes, cam: int, **rcfg):
        rc = render_config(**rcfg)
        H, W = rc.height, rc.width
        rgba = np.zeros((H, W, 4), np.uint8)
        depth = np.zeros((H, W), np.float32)
        ids = np.zeros((H, W), np.int32)
        t = np.zeros((H, W))
        r = lib().orc_render(self.h, bytes(snapshot), cam, C.byref(rc), rgba.ctypes.data, depth.ctypes.data,
                             ids.ctypes.data, t.ctypes.data)
        if r:
            raise ValueError(f"oracle render error {r}")
        return rgba, depth, ids, t

    def camera_pose(self, snapshot: bytes, cam: int) -> np.ndarray:
        out = np.zeros(12)
        lib().orc_camera_pose(self.h, bytes(snapshot), cam, out.ctypes.data)
        return out

    def move_base(self, base, lin, ang, dt):
        b = np.ascontiguousarray(base, dtype=np.float64)
        out = np.zeros(3)
        lib().orc_move_base(self.h, b.ctypes.data, lin, ang, dt, out.ctypes.data)
        return out

    def nearest_walkable(self, x, y):
        out = np.zeros(2)
        lib().orc_nearest_walkable(self.h, x, y, out.ctypes.data)
        return out

    def solve_ik(self, target, seed):
        """(attempt index or -1, q) -- robot.solve_ik restated."""
        t = np.ascontiguousarray(target, dtype=np.float64)
        sd = np.ascontiguousarray(seed, dtype=np.float64)
        out = np.zeros(len(sd))
        r = lib().orc_solve_ik(self.h, t.ctypes.data, sd.ctypes.data, out.ctypes.data)
        return r, (out if r >= 0 else sd.copy())

    def nav_field(self, goal_xy):
        """navgrid.distance_field restated: [nx, ny] geodesic distances to the goal."""
        out = np.zeros((self.desc.desc.nav_nx, self.desc.desc.nav_ny))
        lib().orc_nav_field(self.h, float(goal_xy[0]), float(goal_xy[1]), out.ctypes.data)
        return out

    def nav_geodesic(self, field, from_xy):
        f = np.ascontiguousarray(field, dtype=np.float64)
        return lib().orc_nav_geodesic(self.h, f.ctypes.data, float(from_xy[0]), float(from_xy[1]))

    def nav_path(self, field, from_xy, cap=4096):
        f = np.ascontiguousarray(field, dtype=np.float64)
        out = np.zeros((cap, 2))
        n = lib().orc_nav_path(self.h, f.ctypes.data, float(from_xy[0]), float(from_xy[1]), out.ctypes.data, cap)
        return out[:n]

    def sphere_cast(self, snapshot: bytes, origin, direction, max_dist: float):
        """Simulator.sphere_cast: (body, t), None on no hit; ValueError for a non-unit direction."""
        o = np.ascontiguousarray(origin, dtype=np.float64)
        d = np.ascontiguousarray(direction, dtype=np.float64)
        t = C.c_double()
        b = lib().orc_sphere_cast(self.h, bytes(snapshot), o.ctypes.data, d.ctypes.data, max_dist, C.byref(t))
        if b == -2:
            raise ValueError("sphere_cast direction must be unit length")
        return None if b < 0 else (b, t.value)

    def parts_distance(self, snapshot: bytes, a: int, b: int) -> float:
        """geometry.parts_distance (GJK over part pairs) of bodies a, b."""
        return lib().orc_parts_distance(self.h, bytes(snapshot), a, b)

    def spawn_clearance(self, snapshot: bytes, placed_mask: int):
        """physics._assert_spawn_clearance: None, or the first (body, other, clearance) below 1 mm."""
        b, o, d = C.c_int(), C.c_int(), C.c_double()
        r = lib().orc_spawn_clearance(self.h, bytes(snapshot), placed_mask, C.byref(b), C.byref(o), C.byref(d))
        return (b.value, o.value, d.value) if r == 1 else None

    def settle(self, spawn: bytes, placed_mask: int, max_steps: int = 300, floor_z: float = 0.0):
        """Simulator.settle from a spawn state: (status, snapshot, info, value, steps);
        status 0 settled, 1 clearance, 2 fell, 3 timeout, 4 fault."""
        out = np.zeros(self.snap_size, np.uint8)
        info = np.zeros(2, np.int32)
        val, steps = C.c_double(), C.c_int()
        st = lib().orc_settle(self.h, bytes(spawn), placed_mask, max_steps, floor_z, out.ctypes.data,
                              info.ctypes.data, C.byref(val), C.byref(steps))
        return st, out.tobytes(), info, val.value, steps.value

    def grasp(self, snapshot: bytes, gripper: float):
        """grasp_rule + apply_grasp: (snapshot after, (kind, body, joint, wakes));
        kind 0 none, 1 snap, 2 release."""
        out = np.zeros(self.snap_size, np.uint8)
        tr = np.zeros(4, np.int32)
        r = lib().orc_grasp(self.h, bytes(snapshot), float(gripper), out.ctypes.data, tr.ctypes.data)
        if r:
            raise ValueError(f"oracle grasp error {r}")
        return out.tobytes(), tuple(int(x) for x in tr)

    def apply_arm_action(self, q, delta):
        """(joint targets, ik_failed) -- robot.apply_arm_action restated."""
        qa = np.ascontiguousarray(q, dtype=np.float64)
        d = np.ascontiguousarray(delta, dtype=np.float64)
        out = np.zeros(len(qa))
        f = lib().orc_apply_arm_action(self.h, qa.ctypes.data, d.ctypes.data, out.ctypes.data)
        return out, bool(f)

    def link_poses(self, q, base):
        q = np.ascontiguousarray(q, dtype=np.float64)
        b = np.ascontiguousarray(base, dtype=np.float64)
        links = np.zeros((len(q), 12))
        ee = np.zeros(12)
        lib().orc_link_poses(self.h, q.ctypes.data, b.ctypes.data, links.ctypes.data, ee.ctypes.data)
        return links, ee
