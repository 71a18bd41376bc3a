"""Scene loading and the body table of one simulated world.

``load_layout`` mirrors ``scene.load_scene`` (``scene.py:475-588``): body ids
in file order (backdrop, then each furniture entry; an articulation adds one
body per part, its children placed at q = 0), scene joints, receptacles
resolved to owner bodies, and the walk grid (authored polygons minus
furniture footprints inflated by 0.25 m).

``World`` mirrors the body table ``physics.Simulator.__init__`` builds
(``physics.py:257-330``): scene bodies, then the robot base and its 7 links,
then clutter; dynamic mass properties by volume; no-collide groups (robot =
-1, articulation instance = 1 + furniture index).

Neither runs on the step path: they feed ``compiler.compile_world`` which
flattens everything into the device tables behind the C-ABI.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import assets as A
from .geom import Pose, rot_z

KIND_STATIC, KIND_KINEMATIC, KIND_DYNAMIC = 0, 1, 2
NO_GROUP = -(2**31)


def prim_aabb(prim, pose: Pose):
    """World AABB of one primitive (``geometry.py:278-286``)."""
    if prim.kind == A.KIND_BOX:
        r = np.abs(pose.rot) @ prim.half
        return pose.pos - r, pose.pos + r
    if prim.kind == A.KIND_SPHERE:
        return pose.pos - prim.radius, pose.pos + prim.radius
    w = pose.apply(prim.vertices)
    return w.min(axis=0), w.max(axis=0)


def parts_aabb(parts, pose: Pose):
    lo = np.full(3, np.inf)
    hi = np.full(3, -np.inf)
    for local, prim in parts:
        a, b = prim_aabb(prim, pose.compose(local))
        lo = np.minimum(lo, a)
        hi = np.maximum(hi, b)
    return lo, hi


# --------------------------------------------------------------------------
# walk grid (navgrid.py:20-51)
# --------------------------------------------------------------------------

CELL = 0.05


def _inside_polygon(pts, poly):
    x, y = pts[:, 0], pts[:, 1]
    inside = np.zeros(len(pts), dtype=bool)
    n = len(poly)
    for k in range(n):
        x0, y0 = poly[k]
        x1, y1 = poly[(k + 1) % n]
        crosses = (y0 > y) != (y1 > y)
        with np.errstate(divide="ignore", invalid="ignore"):
            xc = x0 + (y - y0) * (x1 - x0) / (y1 - y0)
        inside ^= crosses & (x < np.where(crosses, xc, np.inf))
    return inside


@dataclass
class WalkGrid:
    origin: np.ndarray
    cell: float
    nx: int
    ny: int
    walkable: np.ndarray  # (nx, ny) bool, x-major

    @classmethod
    def build(cls, polygons, blocked, cell=CELL):
        pts = np.concatenate(polygons)
        origin = pts.min(axis=0) - cell
        extent = pts.max(axis=0) + cell - origin
        nx = max(1, int(math.ceil(extent[0] / cell)))
        ny = max(1, int(math.ceil(extent[1] / cell)))
        cx = origin[0] + (np.arange(nx) + 0.5) * cell
        cy = origin[1] + (np.arange(ny) + 0.5) * cell
        gx, gy = np.meshgrid(cx, cy, indexing="ij")
        centres = np.stack([gx.ravel(), gy.ravel()], axis=1)
        ok = np.zeros(len(centres), dtype=bool)
        for poly in polygons:
            ok |= _inside_polygon(centres, np.asarray(poly, dtype=float))
        for x0, y0, x1, y1 in blocked:
            ok &= ~((centres[:, 0] >= x0) & (centres[:, 0] <= x1) & (centres[:, 1] >= y0) & (centres[:, 1] <= y1))
        return cls(origin, float(cell), nx, ny, ok.reshape(nx, ny))


# --------------------------------------------------------------------------
# layout loading
# --------------------------------------------------------------------------

@dataclass
class SceneBody:
    body_id: int
    name: str
    asset: A.Asset
    kind: int
    pose: Pose
    furniture_index: int | None = None
    part_index: int | None = None


@dataclass
class SceneJoint:
    joint_id: str
    body_id: int
    parent_body: int
    spec: A.JointSpec

    def child_pose(self, parent: Pose, q: float) -> Pose:
        """``scene.py:436-437``: parent * origin * motion(q)."""
        return parent.compose(self.spec.origin).compose(self.spec.motion(q))

    def handle_world(self, parent: Pose, q: float) -> np.ndarray:
        return self.child_pose(parent, q).apply(self.spec.handle_point)


@dataclass
class Receptacle:
    name: str
    owner_body: int
    kind: str
    centre: np.ndarray
    half: np.ndarray


@dataclass
class Layout:
    variant: int
    bodies: list
    joints: list
    receptacles: list
    grid: WalkGrid
    floor_z: float = 0.0

    def receptacle(self, name) -> Receptacle:
        for r in self.receptacles:
            if r.name == name:
                return r
        raise KeyError(name)


def load_layout(variant: int, cache: A.AssetCache | None = None) -> Layout:
    cache = cache or A.default_cache()
    if variant not in A.LAYOUTS:
        raise KeyError(f"unknown layout variant {variant}")
    bodies: list[SceneBody] = []
    joints: list[SceneJoint] = []
    first_body = []

    def add(name, asset, kind, pose, fi=None, pi=None):
        bodies.append(SceneBody(len(bodies), name, asset, kind, pose, fi, pi))
        return len(bodies) - 1

    add("backdrop", cache.get("backdrop"), KIND_STATIC, Pose())
    for fi, (ref, is_art, x, y, yaw) in enumerate(A.LAYOUTS[variant]):
        first_body.append(len(bodies))
        pose = Pose(rot_z(yaw), np.array([x, y, 0.0]))
        if is_art:
            part_ids, jspecs = A.ARTICULATIONS[ref]
            ids = [add(f"{ref}#{fi}:{pid}.{pi}", cache.get(pid), KIND_STATIC if pi == 0 else KIND_KINEMATIC,
                       pose, fi, pi) for pi, pid in enumerate(part_ids)]
            for js in jspecs:
                sj = SceneJoint(f"{ref}#{fi}:{js.joint_id}", ids[js.child_part], ids[js.parent_part], js)
                bodies[sj.body_id].pose = sj.child_pose(bodies[sj.parent_body].pose, 0.0)
                joints.append(sj)
        else:
            asset = cache.get(ref)
            add(f"{ref}#{fi}", asset, KIND_STATIC if asset.is_static else KIND_DYNAMIC, pose, fi)

    recs = [Receptacle(n, first_body[owner] + (part or 0), kind, np.array(c, dtype=float), np.array(h, dtype=float))
            for n, owner, part, kind, c, h in A.RECEPTACLES]
    blocked = []
    for b in bodies:
        if b.furniture_index is None:
            continue
        lo, hi = parts_aabb(b.asset.parts, b.pose)
        r = A.BASE_CLEARANCE_RADIUS
        blocked.append((lo[0] - r, lo[1] - r, hi[0] + r, hi[1] + r))
    grid = WalkGrid.build(A.NAVMESH, blocked)
    return Layout(variant, bodies, joints, recs, grid)


# --------------------------------------------------------------------------
# the world body table (physics.py:209-330)
# --------------------------------------------------------------------------

@dataclass
class Body:
    body_id: int
    name: str
    parts: list
    kind: int
    mass: float
    inv_mass: float
    com: np.ndarray
    inv_inertia: np.ndarray
    friction: float
    restitution: float
    category: str
    is_robot: bool = False
    scene_joint: int = -1
    group: int = NO_GROUP


@dataclass
class World:
    layout: Layout
    robot: A.RobotDef
    bodies: list
    robot_body_ids: list
    clutter_body_ids: list
    clutter_names: list

    @property
    def n_bodies(self) -> int:
        return len(self.bodies)

    @property
    def n_scene_joints(self) -> int:
        return len(self.layout.joints)

    @property
    def n_joints(self) -> int:
        return self.n_scene_joints + self.robot.dof

    @property
    def arm_slice(self) -> slice:
        return slice(self.n_scene_joints, self.n_joints)


def _body(bid, name, asset: A.Asset, kind) -> Body:
    if kind == KIND_DYNAMIC:
        com, inertia = A.mass_properties(asset.parts, asset.mass)
        inv_m, inv_i = 1.0 / asset.mass, np.linalg.inv(inertia)
    else:
        com, inv_m, inv_i = np.zeros(3), 0.0, np.zeros((3, 3))
    return Body(bid, name, asset.parts, kind, asset.mass, inv_m, com, inv_i,
                asset.friction, asset.restitution, asset.category)


def build_world(variant: int, clutter: list[str], robot: A.RobotDef | None = None,
                cache: A.AssetCache | None = None) -> World:
    cache = cache or A.default_cache()
    layout = load_layout(variant, cache)
    robot = robot or A.fetch_like()
    jmap = {sj.body_id: i for i, sj in enumerate(layout.joints)}
    bodies = []
    for sb in layout.bodies:
        b = _body(sb.body_id, sb.name, sb.asset, sb.kind)
        b.scene_joint = jmap.get(sb.body_id, -1)
        if sb.furniture_index is not None and sb.part_index is not None:
            b.group = 1 + sb.furniture_index
        bodies.append(b)
    robot_ids = []
    links = [("robot:base", robot.base_proxy)] + [(f"robot:link{i}", j.proxy) for i, j in enumerate(robot.joints)]
    for name, parts in links:
        bid = len(bodies)
        bodies.append(Body(bid, name, parts, KIND_KINEMATIC, 0.0, 0.0, np.zeros(3), np.zeros((3, 3)),
                           0.5, 0.0, "robot", is_robot=True, group=-1))
        robot_ids.append(bid)
    clutter_ids = []
    for i, name in enumerate(clutter):
        bid = len(bodies)
        bodies.append(_body(bid, f"{name}#{i}", cache.get(name), KIND_DYNAMIC))
        clutter_ids.append(bid)
    return World(layout, robot, bodies, robot_ids, clutter_ids, list(clutter))


def flat_clutter(n: int = 20) -> list[str]:
    """The settle-safe clutter cycle used by every benchmark config."""
    return [A.FLAT_CLUTTER[i % len(A.FLAT_CLUTTER)] for i in range(n)]
