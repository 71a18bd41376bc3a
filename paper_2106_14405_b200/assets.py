"""Built-in synthetic ReplicaCAD-style apartment and Fetch-like robot.

This is the scene *input* of the hot path: the same assets, articulations,
layout variants, receptacles, navmesh and robot definition the reference
ships (``builtin.py:59-396`` and ``data/fetch_like.json``), restated as
compact tables.  Body order, proxy part order, masses, friction and
restitution must match the reference exactly because the device tables
(and snapshot bytes) are indexed by body id; ``tests/test_scene.py`` pins
them against tables dumped from the reference.

Convex primitives mirror the reference's geometry kernel:

* ``Box`` (``geometry.py:200-213``): 8 corners with x varying fastest, six
  faces ``+x +y +z -x -y -z`` with offsets = half extents;
* ``Sphere`` (``geometry.py:216-223``);
* ``Hull`` (``geometry.py:226-252``): scipy qhull facets *as qhull emits
  them*, including coplanar duplicate facets (their multiplicity changes the
  speculative-contact rule, ``geometry.py:574-575``);
* a cylinder is a 12-gon prism hull (``geometry.py:816-822``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.spatial import ConvexHull

from .geom import Pose, rot_z

# --------------------------------------------------------------------------
# primitives
# --------------------------------------------------------------------------

KIND_BOX, KIND_SPHERE, KIND_HULL = 0, 1, 2

_CORNERS = np.array([[(i >> 0) & 1, (i >> 1) & 1, (i >> 2) & 1] for i in range(8)], dtype=float) * 2 - 1


class Box:
    kind = KIND_BOX

    def __init__(self, half):
        self.half = np.asarray(half, dtype=float)
        if self.half.shape != (3,) or np.any(self.half <= 0):
            raise ValueError(f"bad box half extents {half}")
        self.vertices = _CORNERS * self.half
        self.normals = np.concatenate([np.eye(3), -np.eye(3)])
        self.offsets = np.concatenate([self.half, self.half])
        self.triangles = np.zeros((0, 3), dtype=np.int64)


class Sphere:
    kind = KIND_SPHERE

    def __init__(self, radius):
        self.radius = float(radius)
        if self.radius <= 0:
            raise ValueError("sphere radius must be positive")
        self.vertices = np.zeros((0, 3))
        self.normals = np.zeros((0, 3))
        self.offsets = np.zeros(0)
        self.triangles = np.zeros((0, 3), dtype=np.int64)


class Hull:
    kind = KIND_HULL

    def __init__(self, points):
        pts = np.asarray(points, dtype=float)
        qh = ConvexHull(pts)
        if qh.volume <= 0:
            raise ValueError("degenerate hull")
        self.vertices = pts[qh.vertices]
        self.normals = qh.equations[:, :3].copy()
        self.offsets = -qh.equations[:, 3].copy()
        where = {int(old): new for new, old in enumerate(qh.vertices)}
        self.triangles = np.array([[where[int(i)] for i in s] for s in qh.simplices], dtype=np.int64)


def prism(radius: float, height: float, segments: int = 12) -> Hull:
    ang = np.linspace(0.0, 2.0 * math.pi, segments, endpoint=False)
    ring = np.stack([radius * np.cos(ang), radius * np.sin(ang)], axis=1)
    top = np.concatenate([ring, np.full((segments, 1), height / 2.0)], axis=1)
    bot = np.concatenate([ring, np.full((segments, 1), -height / 2.0)], axis=1)
    return Hull(np.concatenate([top, bot]))


def make_shape(spec):
    t = spec[0]
    if t == "box":
        return Box(spec[1])
    if t == "sphere":
        return Sphere(spec[1])
    if t == "cyl":
        return prism(spec[1], spec[2], spec[3] if len(spec) > 3 else 12)
    raise ValueError(f"unknown shape {t}")


# --------------------------------------------------------------------------
# mass properties (geometry.py:307-376)
# --------------------------------------------------------------------------

_TET_COV = (np.ones((3, 3)) + np.eye(3)) / 120.0


def _volume_props(prim):
    if prim.kind == KIND_BOX:
        h = prim.half
        vol = 8.0 * h[0] * h[1] * h[2]
        diag = vol / 3.0 * np.array([h[1] ** 2 + h[2] ** 2, h[0] ** 2 + h[2] ** 2, h[0] ** 2 + h[1] ** 2])
        return vol, np.zeros(3), np.diag(diag)
    if prim.kind == KIND_SPHERE:
        r = prim.radius
        vol = 4.0 / 3.0 * math.pi * r**3
        return vol, np.zeros(3), np.eye(3) * (2.0 / 5.0 * vol * r * r)
    verts, tris = prim.vertices, prim.triangles
    centre = verts.mean(axis=0)
    vol, com, cov = 0.0, np.zeros(3), np.zeros((3, 3))
    for tri in tris:
        a, b, c = verts[tri]
        if np.cross(b - a, c - a) @ (a - centre) < 0:
            b, c = c, b
        jac = np.column_stack([a, b, c])
        det = float(np.linalg.det(jac))
        vol += det / 6.0
        com += det / 24.0 * (a + b + c)
        cov += det * (jac @ _TET_COV @ jac.T)
    com = com / vol
    cov_c = cov - vol * np.outer(com, com)
    return vol, com, np.trace(cov_c) * np.eye(3) - cov_c


def mass_properties(parts, mass: float):
    """(COM, inertia about COM) with mass spread by volume over the parts."""
    vols, coms, inerts = [], [], []
    for local, prim in parts:
        v, c, i = _volume_props(prim)
        vols.append(v)
        coms.append(local.apply(c))
        inerts.append(local.rot @ i @ local.rot.T)
    total = sum(vols)
    rho = mass / total
    com = sum(v * c for v, c in zip(vols, coms)) / total
    inertia = np.zeros((3, 3))
    for v, c, i in zip(vols, coms, inerts):
        d = c - com
        inertia += rho * i + rho * v * ((d @ d) * np.eye(3) - np.outer(d, d))
    return com, inertia


# --------------------------------------------------------------------------
# asset library (builtin.py:59-290)
# --------------------------------------------------------------------------

@dataclass
class Asset:
    asset_id: str
    parts: list  # [(Pose, primitive)]
    mass: float
    friction: float
    restitution: float
    category: str

    @property
    def is_static(self) -> bool:
        return self.mass == 0.0


def _parts(*items):
    """items: (shape spec, local xyz)"""
    return [(_local(p), make_shape(s)) for s, p in items]


def _local(xyz) -> Pose:
    """Compound-part frame: the reference parses ``{"pos": ...}`` with a
    ``rot_z(0.0)`` rotation (``scene.py:204-208``), signed zeros included."""
    return Pose(rot_z(0.0), np.asarray(xyz, dtype=float))


# clutter: name -> (shape spec, mass, category, restitution); friction 0.6
CLUTTER_TABLE = {
    "cracker_box": (("box", [0.030, 0.079, 0.105]), 0.411, "food", 0.08),
    "sugar_box": (("box", [0.019, 0.0445, 0.0875]), 0.514, "food", 0.08),
    "tomato_soup_can": (("cyl", 0.033, 0.101), 0.349, "food", 0.08),
    "tuna_fish_can": (("cyl", 0.0425, 0.033), 0.171, "food", 0.08),
    "pudding_box": (("box", [0.055, 0.044, 0.019]), 0.187, "food", 0.08),
    "gelatin_box": (("box", [0.0365, 0.046, 0.014]), 0.097, "food", 0.08),
    "potted_meat_can": (("box", [0.029, 0.0485, 0.041]), 0.370, "food", 0.08),
    "chef_can": (("cyl", 0.051, 0.1395), 0.453, "food", 0.08),
    "apple": (("sphere", 0.0375), 0.068, "food", 0.25),
    "orange": (("sphere", 0.0375), 0.047, "food", 0.25),
    "bowl": (("cyl", 0.080, 0.055), 0.147, "kitchen", 0.08),
    "mug": (("cyl", 0.040, 0.081), 0.118, "kitchen", 0.08),
    "plate": (("cyl", 0.090, 0.020), 0.279, "kitchen", 0.08),
    "sponge": (("box", [0.048, 0.036, 0.0085]), 0.020, "kitchen", 0.08),
}


def _b(hx, hy, hz, x, y, z):
    return (("box", [hx, hy, hz]), (x, y, z))


# furniture: name -> (parts, mass, category, friction)
FURNITURE_TABLE = {
    "backdrop": ([_b(5.0, 3.0, 0.05, 0, 0, -0.05), _b(5.0, 0.05, 1.25, 0, 3.05, 1.25),
                  _b(5.0, 0.05, 1.25, 0, -3.05, 1.25), _b(0.05, 3.1, 1.25, 5.05, 0, 1.25),
                  _b(0.05, 3.1, 1.25, -5.05, 0, 1.25)], 0.0, "backdrop", 0.8),
    "counter": ([_b(0.9, 0.325, 0.46, 0, 0, 0.46)], 0.0, "furniture", 0.6),
    "light_table": ([_b(0.60, 0.40, 0.02, 0, 0, 0.72)]
                    + [_b(0.025, 0.025, 0.35, sx * 0.55, sy * 0.35, 0.35) for sx, sy in ((1, 1), (-1, 1), (1, -1), (-1, -1))],
                    0.0, "furniture", 0.6),
    "dark_table": ([_b(0.45, 0.45, 0.02, 0, 0, 0.68)]
                   + [_b(0.025, 0.025, 0.33, sx * 0.40, sy * 0.40, 0.33) for sx, sy in ((1, 1), (-1, 1), (1, -1), (-1, -1))],
                   0.0, "furniture", 0.6),
    "sofa": ([_b(0.90, 0.40, 0.22, 0, 0, 0.22), _b(0.90, 0.08, 0.30, 0, 0.36, 0.70),
              _b(0.08, 0.40, 0.12, 0.98, 0, 0.56), _b(0.08, 0.40, 0.12, -0.98, 0, 0.56)], 0.0, "furniture", 0.6),
    "sink": ([_b(0.45, 0.32, 0.34, 0, 0, 0.34), _b(0.30, 0.20, 0.02, 0, 0, 0.70),
              _b(0.45, 0.06, 0.11, 0, -0.26, 0.79), _b(0.45, 0.06, 0.11, 0, 0.26, 0.79),
              _b(0.075, 0.20, 0.11, -0.375, 0, 0.79), _b(0.075, 0.20, 0.11, 0.375, 0, 0.79)], 0.0, "furniture", 0.6),
    "shelves": ([_b(0.02, 0.25, 0.60, 0.58, 0, 0.60), _b(0.02, 0.25, 0.60, -0.58, 0, 0.60),
                 _b(0.56, 0.25, 0.015, 0, 0, 0.40), _b(0.56, 0.25, 0.015, 0, 0, 0.80),
                 _b(0.60, 0.25, 0.015, 0, 0, 1.20)], 0.0, "furniture", 0.6),
    "cabinet_shell": ([_b(0.45, 0.30, 0.02, 0, 0, 0.88), _b(0.02, 0.30, 0.44, -0.43, 0, 0.44),
                       _b(0.02, 0.30, 0.44, 0.43, 0, 0.44), _b(0.45, 0.02, 0.44, 0, 0.28, 0.44),
                       _b(0.45, 0.30, 0.02, 0, 0, 0.02)], 0.0, "furniture", 0.6),
    "drawer_tray": ([_b(0.39, 0.25, 0.01, 0, 0, 0.01), _b(0.39, 0.015, 0.11, 0, -0.235, 0.11),
                     _b(0.39, 0.015, 0.11, 0, 0.235, 0.11), _b(0.015, 0.25, 0.11, -0.375, 0, 0.11),
                     _b(0.015, 0.25, 0.11, 0.375, 0, 0.11)], 3.0, "furniture", 0.6),
    "fridge_shell": ([_b(0.03, 0.33, 0.65, -0.37, 0, 1.02), _b(0.03, 0.33, 0.65, 0.37, 0, 1.02),
                      _b(0.40, 0.03, 0.65, 0, 0.30, 1.02), _b(0.40, 0.33, 0.03, 0, 0, 1.67),
                      _b(0.40, 0.33, 0.03, 0, 0, 0.40), _b(0.40, 0.30, 0.185, 0, 0, 0.185),
                      _b(0.34, 0.30, 0.015, 0, 0, 0.95)], 0.0, "furniture", 0.6),
    "fridge_door": ([_b(0.38, 0.025, 0.65, 0.38, -0.025, 0.0)], 8.0, "furniture", 0.6),
}


@dataclass
class JointSpec:
    joint_id: str
    joint_type: str  # revolute | prismatic
    axis: np.ndarray  # unit, parent frame
    limits: tuple
    parent_part: int
    child_part: int
    origin: Pose
    handle_point: np.ndarray

    def motion(self, q: float) -> Pose:
        """Child motion at coordinate q (``scene.py:102-105``)."""
        from .geom import axis_angle_rot

        if self.joint_type == "revolute":
            return Pose(axis_angle_rot(self.axis, q))
        return Pose(pos=self.axis * q)


def _unit(v):
    v = np.asarray(v, dtype=float)
    return v / math.sqrt(float(v @ v))


ARTICULATIONS = {
    "kitchen_cabinet": (
        ["cabinet_shell", "drawer_tray", "drawer_tray", "drawer_tray"],
        [JointSpec(f"drawer_{i}", "prismatic", _unit([0.0, -1.0, 0.0]), (0.0, 0.35), 0, i + 1,
                   Pose(rot_z(0.0), np.array([0.0, -0.02, z])), np.array([0.0, -0.27, 0.11]))
         for i, z in enumerate((0.14, 0.38, 0.62))],
    ),
    "fridge": (
        ["fridge_shell", "fridge_door"],
        [JointSpec("door", "revolute", _unit([0.0, 0.0, -1.0]), (0.0, 2.356), 0, 1,
                   Pose(rot_z(0.0), np.array([-0.40, -0.33, 1.02])), np.array([0.72, -0.09, 0.0]))],
    ),
}

# (ref, is_articulation, x, y, yaw) per layout variant (builtin.py:294-328)
_FIXED = [("counter", False, -4.63, 1.30, math.pi / 2), ("kitchen_cabinet", True, -4.65, -0.50, math.pi / 2),
          ("fridge", True, -3.30, 2.62, 0.0), ("sink", False, -1.60, 2.63, 0.0),
          ("counter", False, -3.30, -2.63, math.pi)]
LAYOUTS = {
    0: _FIXED + [("light_table", False, 1.60, 1.10, 0.0), ("dark_table", False, 3.30, -1.40, 0.0),
                 ("sofa", False, 4.50, 0.80, -math.pi / 2), ("shelves", False, 1.60, -2.70, math.pi)],
    1: _FIXED + [("light_table", False, 3.30, -1.40, 0.0), ("dark_table", False, 1.60, 1.10, 0.0),
                 ("sofa", False, 4.50, -0.60, -math.pi / 2), ("shelves", False, -0.50, -2.70, math.pi)],
    2: _FIXED + [("light_table", False, 2.60, 1.40, 0.0), ("dark_table", False, 1.20, -1.30, 0.0),
                 ("sofa", False, 2.80, 2.50, math.pi), ("shelves", False, 4.70, -1.80, -math.pi / 2)],
}
N_LAYOUTS = len(LAYOUTS)

# receptacles: name -> (owner furniture index, articulation part or None, kind, centre, half)
RECEPTACLES = [
    ("counter_left", 0, None, "on_top", (0, 0, 1.045), (0.85, 0.28, 0.125)),
    ("drawer_0", 1, 1, "inside", (0, 0, 0.125), (0.36, 0.22, 0.105)),
    ("drawer_1", 1, 2, "inside", (0, 0, 0.125), (0.36, 0.22, 0.105)),
    ("drawer_2", 1, 3, "inside", (0, 0, 0.125), (0.36, 0.22, 0.105)),
    ("fridge_shelf", 2, None, "inside", (0, 0, 1.075), (0.30, 0.26, 0.10)),
    ("sink", 3, None, "inside", (0, 0, 0.82), (0.27, 0.17, 0.09)),
    ("counter_right", 4, None, "on_top", (0, 0, 1.045), (0.85, 0.28, 0.125)),
    ("light_table", 5, None, "on_top", (0, 0, 0.87), (0.55, 0.36, 0.13)),
    ("dark_table", 6, None, "on_top", (0, 0, 0.83), (0.41, 0.41, 0.13)),
    ("sofa", 7, None, "on_top", (0, -0.05, 0.55), (0.80, 0.30, 0.11)),
    ("shelves", 8, None, "on_top", (0, 0, 0.925), (0.52, 0.21, 0.10)),
]

NAVMESH = [np.array([[-4.7, -2.7], [4.7, -2.7], [4.7, 2.7], [-4.7, 2.7]])]
LIVING_ROOM_CENTER = (2.3, -0.2)
BASE_CLEARANCE_RADIUS = 0.25  # scene.py:25

# clutter objects that settle under this contact model
FLAT_CLUTTER = ["pudding_box", "gelatin_box", "sponge", "plate", "tuna_fish_can", "bowl",
                "potted_meat_can", "apple", "orange"]


class AssetCache:
    """Parse-once asset store (mirrors ``scene.py:358-410``)."""

    def __init__(self):
        self._assets: dict[str, Asset] = {}
        self.parse_counts: dict[str, int] = {}

    def get(self, asset_id: str) -> Asset:
        hit = self._assets.get(asset_id)
        if hit is not None:
            return hit
        if asset_id in CLUTTER_TABLE:
            spec, mass, cat, rest = CLUTTER_TABLE[asset_id]
            asset = Asset(asset_id, [(Pose(), make_shape(spec))], mass, 0.6, rest, cat)
        elif asset_id in FURNITURE_TABLE:
            items, mass, cat, fric = FURNITURE_TABLE[asset_id]
            asset = Asset(asset_id, _parts(*items), mass, fric, 0.1, cat)
        else:
            raise KeyError(f"unknown asset id: {asset_id}")
        self.parse_counts[asset_id] = self.parse_counts.get(asset_id, 0) + 1
        self._assets[asset_id] = asset
        return asset


_DEFAULT_CACHE: AssetCache | None = None


def default_cache() -> AssetCache:
    global _DEFAULT_CACHE
    if _DEFAULT_CACHE is None:
        _DEFAULT_CACHE = AssetCache()
    return _DEFAULT_CACHE


# --------------------------------------------------------------------------
# robot (data/fetch_like.json; camera convention tools_make_robot_json.py:12-19)
# --------------------------------------------------------------------------

def _cam_rot(view):
    view = np.asarray(view, dtype=float)
    view = view / np.linalg.norm(view)
    right = np.cross(view, (0.0, 0.0, 1.0))
    right /= np.linalg.norm(right)
    down = np.cross(view, right)
    down /= np.linalg.norm(down)
    return np.column_stack([right, down, view])


@dataclass
class ArmJoint:
    name: str
    offset: np.ndarray  # joint frame origin in parent link frame (rotation = identity)
    axis: np.ndarray
    limits: tuple
    proxy: list  # [(Pose, primitive)] in joint frame


@dataclass
class RobotDef:
    name: str
    base_proxy: list
    joints: list
    gripper_offset: np.ndarray
    cameras: dict  # name -> (parent "base"|"ee", Pose)
    resting_joints: np.ndarray
    resting_ee: np.ndarray
    zero_ee: np.ndarray
    base_radius: float = 0.22

    @property
    def dof(self) -> int:
        return len(self.joints)

    def limits_lo(self):
        return np.array([j.limits[0] for j in self.joints])

    def limits_hi(self):
        return np.array([j.limits[1] for j in self.joints])


# name, offset, axis, limits, link box half, link box centre x
_ARM = [
    ("shoulder_pan", (0.12, 0.0, 0.96), (0, 0, 1), (-1.6057, 1.6057), (0.06, 0.06, 0.055), 0.05),
    ("shoulder_lift", (0.117, 0.0, 0.06), (0, 1, 0), (-1.221, 1.518), (0.115, 0.05, 0.05), 0.11),
    ("upperarm_roll", (0.219, 0.0, 0.0), (1, 0, 0), (-3.1, 3.1), (0.07, 0.05, 0.05), 0.066),
    ("elbow_flex", (0.133, 0.0, 0.0), (0, 1, 0), (-2.251, 2.251), (0.103, 0.045, 0.045), 0.098),
    ("forearm_roll", (0.197, 0.0, 0.0), (1, 0, 0), (-3.1, 3.1), (0.066, 0.04, 0.04), 0.062),
    ("wrist_flex", (0.1245, 0.0, 0.0), (0, 1, 0), (-2.16, 2.16), (0.073, 0.04, 0.04), 0.069),
    ("wrist_roll", (0.1385, 0.0, 0.0), (1, 0, 0), (-3.1, 3.1), (0.086, 0.042, 0.032), 0.083),
]
_HEAD_TILT = math.radians(28.0)


def fetch_like() -> RobotDef:
    joints = [
        ArmJoint(n, np.array(o, dtype=float), np.array(a, dtype=float), lim,
                 [(_local([cx, 0.0, 0.0]), Box(h))])
        for n, o, a, lim, h, cx in _ARM
    ]
    base = [(_local([0.0, 0.0, 0.12]), prism(0.22, 0.24, 12)),
            (_local([-0.05, 0.0, 0.62]), Box([0.11, 0.13, 0.33]))]
    head = _cam_rot([math.cos(_HEAD_TILT), 0.0, -math.sin(_HEAD_TILT)])
    arm = np.column_stack([[0.0, -1.0, 0.0], [0.0, 0.0, -1.0], [1.0, 0.0, 0.0]])
    cams = {
        "head": ("base", Pose(head, np.array([0.10, 0.0, 1.22]))),
        "arm": ("ee", Pose(arm, np.array([-0.09, 0.0, 0.045]))),
    }
    return RobotDef(
        "fetch_like", base, joints, np.array([0.167, 0.0, 0.0]), cams,
        np.array([0.0, 0.5, 0.0, -2.2, 0.0, 1.3, 0.0]),
        np.array([0.78587, 0.0, 1.28903]), np.array([1.216, 0.0, 1.02]),
    )
