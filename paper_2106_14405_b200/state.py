"""Host-side world state and its snapshot byte format.

``WorldState`` carries the same fields as the reference's state
(``physics.py:93-124``) and ``to_bytes``/``from_bytes`` produce/consume the
identical little-endian layout (``physics.py:147-203``): magic ``RSIM``,
version 1, body and joint counts, the f64/i64/u8 arrays in declaration
order, then a 40-byte ``<iidddq`` tail.  The per-body ``version`` counter is
a reference-side cache key and is not part of the state here either.

This is the interchange format between the oracle, the golden fixtures and
the device batch (``rs_set_state``/``rs_get_state`` speak it natively).
"""

from __future__ import annotations

import hashlib
import struct

import numpy as np

from .geom import Pose, axis_angle_rot, base_pose, rot_z

MAGIC = b"RSIM"
SNAP_VERSION = 1


def snapshot_size(n_bodies: int, n_joints: int) -> int:
    nb, nj = n_bodies, n_joints
    return 16 + 8 * (13 * nb) + nb + 8 * nb + 8 * (2 * nj) + 8 * (3 + 7 + 3) + 8 * nb + 8 * 7 * nb + 40


class WorldState:
    FIELDS = ("pos", "quat", "lin_vel", "ang_vel", "asleep", "sleep_counter", "joints", "joint_vel",
              "base", "held", "held_offset", "held_joint", "grab_q", "grab_ee", "rider_joint",
              "rider_offset", "accumulated_contact_force", "time", "step_index")

    def __init__(self, n_bodies: int, n_joints: int):
        self.pos = np.zeros((n_bodies, 3))
        self.quat = np.tile([1.0, 0.0, 0.0, 0.0], (n_bodies, 1))
        self.lin_vel = np.zeros((n_bodies, 3))
        self.ang_vel = np.zeros((n_bodies, 3))
        self.asleep = np.zeros(n_bodies, dtype=bool)
        self.sleep_counter = np.zeros(n_bodies, dtype=np.int64)
        self.joints = np.zeros(n_joints)
        self.joint_vel = np.zeros(n_joints)
        self.base = np.zeros(3)
        self.held = -1
        self.held_offset = np.array([0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0])
        self.held_joint = -1
        self.grab_q = 0.0
        self.grab_ee = np.zeros(3)
        self.rider_joint = np.full(n_bodies, -1, dtype=np.int64)
        self.rider_offset = np.zeros((n_bodies, 7))
        self.accumulated_contact_force = 0.0
        self.time = 0.0
        self.step_index = 0

    @property
    def n_bodies(self) -> int:
        return len(self.pos)

    @property
    def n_joints(self) -> int:
        return len(self.joints)

    def clone(self) -> "WorldState":
        out = WorldState(self.n_bodies, self.n_joints)
        for f in self.FIELDS:
            v = getattr(self, f)
            setattr(out, f, v.copy() if isinstance(v, np.ndarray) else v)
        return out

    def body_pose(self, b: int) -> Pose:
        return Pose.from_quat(self.pos[b], self.quat[b])

    def to_bytes(self) -> bytes:
        head = MAGIC + struct.pack("<III", SNAP_VERSION, self.n_bodies, self.n_joints)
        arrays = (self.pos, self.quat, self.lin_vel, self.ang_vel, self.asleep.astype(np.uint8),
                  self.sleep_counter.astype(np.int64), self.joints, self.joint_vel, self.base,
                  self.held_offset, self.grab_ee, self.rider_joint.astype(np.int64), self.rider_offset)
        body = b"".join(np.ascontiguousarray(a).tobytes() for a in arrays)
        tail = struct.pack("<iidddq", int(self.held), int(self.held_joint), float(self.grab_q),
                           float(self.accumulated_contact_force), float(self.time), int(self.step_index))
        return head + body + tail

    @classmethod
    def from_bytes(cls, blob: bytes) -> "WorldState":
        if bytes(blob[:4]) != MAGIC:
            raise ValueError("bad snapshot magic")
        ver, nb, nj = struct.unpack("<III", bytes(blob[4:16]))
        if ver != SNAP_VERSION:
            raise ValueError(f"unsupported snapshot version {ver}")
        if len(blob) != snapshot_size(nb, nj):
            raise ValueError("snapshot size mismatch")
        st = cls(nb, nj)
        off = 16

        def take(shape, dt=np.float64):
            nonlocal off
            n = int(np.prod(shape)) * np.dtype(dt).itemsize
            a = np.frombuffer(bytes(blob[off:off + n]), dtype=dt).reshape(shape).copy()
            off += n
            return a

        st.pos, st.quat = take((nb, 3)), take((nb, 4))
        st.lin_vel, st.ang_vel = take((nb, 3)), take((nb, 3))
        st.asleep = take((nb,), np.uint8).astype(bool)
        st.sleep_counter = take((nb,), np.int64)
        st.joints, st.joint_vel = take((nj,)), take((nj,))
        st.base, st.held_offset, st.grab_ee = take((3,)), take((7,)), take((3,))
        st.rider_joint = take((nb,), np.int64)
        st.rider_offset = take((nb, 7))
        (st.held, st.held_joint, st.grab_q, st.accumulated_contact_force, st.time,
         st.step_index) = struct.unpack("<iidddq", bytes(blob[off:off + 40]))
        return st

    def state_hash(self) -> str:
        return hashlib.sha256(self.to_bytes()).hexdigest()


# --------------------------------------------------------------------------
# host kinematics (robot.py:156-169) and initial states (physics.py:344-405)
# --------------------------------------------------------------------------

def link_poses(robot, q, base=None):
    t = base_pose(base) if base is not None else Pose()
    out = []
    for jd, qi in zip(robot.joints, q):
        t = t.compose(Pose(rot_z(0.0), jd.offset)).compose(Pose(axis_angle_rot(jd.axis, float(qi))))
        out.append(t)
    return out, t.compose(Pose(pos=robot.gripper_offset))


def ee_pose(world, st: WorldState) -> Pose:
    return link_poses(world.robot, st.joints[world.arm_slice], st.base)[1]


def make_initial_state(world, clutter_poses, articulations=None, base=None, arm_joints=None,
                       clutter_asleep=True) -> WorldState:
    lay = world.layout
    st = WorldState(world.n_bodies, world.n_joints)
    for sb in lay.bodies:
        st.pos[sb.body_id] = sb.pose.pos
        st.quat[sb.body_id] = sb.pose.quat()
    for jid, q in (articulations or {}).items():
        idx = [sj.joint_id for sj in lay.joints].index(jid)
        lo, hi = lay.joints[idx].spec.limits
        st.joints[idx] = min(max(q, lo), hi)
    for ji, sj in enumerate(lay.joints):
        p = sj.child_pose(st.body_pose(sj.parent_body), float(st.joints[ji]))
        st.pos[sj.body_id] = p.pos
        st.quat[sj.body_id] = p.quat()
    st.base = np.asarray(base if base is not None else np.zeros(3), dtype=float).copy()
    st.joints[world.arm_slice] = world.robot.resting_joints if arm_joints is None else arm_joints
    links, _ = link_poses(world.robot, st.joints[world.arm_slice], st.base)
    for bid, p in zip(world.robot_body_ids, [base_pose(st.base)] + links):
        st.pos[bid] = p.pos
        st.quat[bid] = p.quat()
    if len(clutter_poses) != len(world.clutter_body_ids):
        raise ValueError(f"expected {len(world.clutter_body_ids)} clutter poses, got {len(clutter_poses)}")
    for bid, p in zip(world.clutter_body_ids, clutter_poses):
        st.pos[bid] = p.pos
        st.quat[bid] = p.quat()
        st.asleep[bid] = clutter_asleep
    if clutter_asleep:
        _bind_riders(world, st)
    return st


def _bind_riders(world, st):
    """Sleeping clutter inside a moving part's ``inside`` box rides its joint
    (``physics.py:383-405``)."""
    for bid in world.clutter_body_ids:
        if not st.asleep[bid]:
            continue
        com = st.body_pose(bid).apply(world.bodies[bid].com)
        for rec in world.layout.receptacles:
            joint = world.bodies[rec.owner_body].scene_joint
            if joint < 0 or rec.kind != "inside":
                continue
            owner = st.body_pose(rec.owner_body)
            local = owner.inverse().apply(com)
            if np.all(np.abs(local - rec.centre) <= rec.half + 1e-6):
                st.rider_joint[bid] = joint
                rel = owner.inverse().compose(st.body_pose(bid))
                st.rider_offset[bid] = np.concatenate([rel.pos, rel.quat()])
                break


PARK_Z = 40.0  # physics.py:1103: unplaced clutter is parked asleep high above the scene


def park_state(world) -> WorldState:
    """Simulator.park_state (physics.py:1105-1111): clutter parked asleep in the air."""
    from .geom import Pose

    park = [Pose(pos=np.array([-6.0 + 0.6 * i, 0.0, PARK_Z])) for i in range(len(world.clutter_body_ids))]
    return make_initial_state(world, park, clutter_asleep=True)


def spawn_state(base: WorldState, placements) -> WorldState:
    """The state Simulator.settle steps from (physics.py:1124-1137): each
    placed body gets its pose, wakes, and loses velocity, sleep count and rider
    binding -- unless the placement equals its current pose exactly."""
    st = base.clone()
    for bid, pose in placements:
        old = st.body_pose(bid)
        q = pose.quat()
        if np.array_equal(old.pos, pose.pos) and np.array_equal(old.quat(), q):
            continue
        st.pos[bid] = pose.pos
        st.quat[bid] = q
        st.asleep[bid] = False
        st.sleep_counter[bid] = 0
        st.rider_joint[bid] = -1
        st.lin_vel[bid] = 0.0
        st.ang_vel[bid] = 0.0
    return st

