"""Host-side SE(3) helpers used by the scene compiler, initial-state builder
and camera setup (never on the device step path).

Conventions follow the reference geometry kernel so that host-built poses
round-trip bit-compatibly through the snapshot format:

* quaternions are ``[w, x, y, z]`` (``geometry.py:49-59``);
* quat -> matrix is the closed form of ``geometry.py:72-80``;
* matrix -> quat is Shepperd's four-branch method followed by a
  renormalisation (``geometry.py:83-107``);
* an axis-angle rotation goes axis-angle -> quat -> matrix
  (``geometry.py:62-69``, ``:132-133``);
* a pose is (3x3 rotation, translation); ``compose`` is ``A*B`` with
  ``R = Ra Rb``, ``p = Ra pb + pa`` (``geometry.py:164-165``).
"""

from __future__ import annotations

import math

import numpy as np


def quat_to_rot(q) -> np.ndarray:
    w, x, y, z = (float(v) for v in q)
    return np.array(
        [
            [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
            [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
            [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
        ]
    )


def rot_to_quat(m) -> np.ndarray:
    m = np.asarray(m, dtype=float)
    tr = m[0, 0] + m[1, 1] + m[2, 2]
    if tr > 0:
        s = math.sqrt(tr + 1.0) * 2
        q = [0.25 * s, (m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s, (m[1, 0] - m[0, 1]) / s]
    elif m[0, 0] > m[1, 1] and m[0, 0] > m[2, 2]:
        s = math.sqrt(1.0 + m[0, 0] - m[1, 1] - m[2, 2]) * 2
        q = [(m[2, 1] - m[1, 2]) / s, 0.25 * s, (m[0, 1] + m[1, 0]) / s, (m[0, 2] + m[2, 0]) / s]
    elif m[1, 1] > m[2, 2]:
        s = math.sqrt(1.0 + m[1, 1] - m[0, 0] - m[2, 2]) * 2
        q = [(m[0, 2] - m[2, 0]) / s, (m[0, 1] + m[1, 0]) / s, 0.25 * s, (m[1, 2] + m[2, 1]) / s]
    else:
        s = math.sqrt(1.0 + m[2, 2] - m[0, 0] - m[1, 1]) * 2
        q = [(m[1, 0] - m[0, 1]) / s, (m[0, 2] + m[2, 0]) / s, (m[1, 2] + m[2, 1]) / s, 0.25 * s]
    q = np.array(q)
    n = math.sqrt(float(q @ q))
    return q / n


def rot_z(a: float) -> np.ndarray:
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def axis_angle_rot(axis, angle: float) -> np.ndarray:
    axis = np.asarray(axis, dtype=float)
    n = math.sqrt(float(axis @ axis))
    h = 0.5 * angle
    s = math.sin(h) / n
    return quat_to_rot([math.cos(h), axis[0] * s, axis[1] * s, axis[2] * s])


class Pose:
    """Rigid transform; immutable by convention."""

    __slots__ = ("rot", "pos")

    def __init__(self, rot=None, pos=None):
        self.rot = np.eye(3) if rot is None else np.asarray(rot, dtype=float)
        self.pos = np.zeros(3) if pos is None else np.asarray(pos, dtype=float)

    @classmethod
    def from_quat(cls, pos, quat) -> "Pose":
        return cls(quat_to_rot(quat), np.asarray(pos, dtype=float))

    @classmethod
    def planar(cls, x: float, y: float, yaw: float, z: float = 0.0) -> "Pose":
        return cls(rot_z(yaw), np.array([x, y, z], dtype=float))

    def quat(self) -> np.ndarray:
        return rot_to_quat(self.rot)

    def compose(self, other: "Pose") -> "Pose":
        return Pose(self.rot @ other.rot, self.rot @ other.pos + self.pos)

    def inverse(self) -> "Pose":
        rt = self.rot.T
        return Pose(rt, -(rt @ self.pos))

    def apply(self, pts) -> np.ndarray:
        pts = np.asarray(pts, dtype=float)
        if pts.ndim == 1:
            return self.rot @ pts + self.pos
        return pts @ self.rot.T + self.pos

    def as12(self) -> np.ndarray:
        """Row-major rotation followed by translation (device table layout)."""
        return np.concatenate([self.rot.reshape(9), self.pos])


def base_pose(base) -> Pose:
    """Planar base [x, y, yaw] on the floor (``robot.py:156-158``)."""
    return Pose(rot_z(float(base[2])), np.array([base[0], base[1], 0.0]))
