"""Shared grasp / rider fixtures for the CPU (oracle) and GPU tests.

``kat_states`` turns the reference's abstract ``grasp_rule`` known answers
(``kat.npz`` ``grasp_snap`` / ``grasp_none`` / ``grasp_tie``, generated from
``robot.py:323-346``) into world states: the candidate bodies of each KAT
are placed so that their COMs sit at the KAT's distances from the end
effector (identity orientation, positions chosen so the COM is exactly
reproducible), every other clutter body is parked far away.
"""
from __future__ import annotations

import numpy as np

from paper_2106_14405_b200.scene import build_world, flat_clutter
from paper_2106_14405_b200.state import WorldState, ee_pose

STATE_INT = ("asleep", "sleep_counter", "rider_joint")
STATE_F64 = ("pos", "quat", "lin_vel", "ang_vel", "joints", "joint_vel", "base", "held_offset", "grab_ee",
             "rider_offset")


def cmp_states(me: WorldState, ref: WorldState, tol: float = 1e-12, vel_tol: float | None = None, what: str = ""):
    for f in STATE_INT:
        np.testing.assert_array_equal(getattr(me, f), getattr(ref, f), err_msg=f"{what} {f}")
    assert (me.held, me.held_joint, me.step_index) == (ref.held, ref.held_joint, ref.step_index), what
    for f in STATE_F64:
        t = vel_tol if (vel_tol is not None and f in ("lin_vel", "ang_vel", "joint_vel")) else tol
        np.testing.assert_allclose(getattr(me, f), getattr(ref, f), rtol=0, atol=t, err_msg=f"{what} {f}")
    assert abs(me.grab_q - ref.grab_q) <= tol, what


def _place_com_exact(world, st, b, target):
    """Identity orientation; position such that pos + com_local == target in
    float64 (the COM the reference computes, R = I exactly)."""
    c = world.bodies[b].com
    t = np.array(target, float)
    for _ in range(64):
        p = t - c
        if np.array_equal(p + c, t):
            st.pos[b] = p
            st.quat[b] = [1.0, 0.0, 0.0, 0.0]
            return
        t = t + np.array([1e-7, -2e-7, 3e-7])
    raise AssertionError("could not place the COM exactly")


def kat_states(kat):
    """[(state, gripper, expected (kind, body))] for the three grasp KATs."""
    world = build_world(0, flat_clutter())
    pool = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden",
                                              "settled_pool.npz"))
    base = WorldState.from_bytes(pool["snapshots"][0].tobytes())
    base.base = np.array([2.3, -0.2, 0.0])
    out = []

    def fresh():
        st = base.clone()
        for i, b in enumerate(world.clutter_body_ids):  # everything far from the EE
            st.pos[b] = [-6.0 + 0.6 * i, 0.0, 40.0]
        return st

    # snap: 30 at 0.10, 22 at 0.16 -> 30 (kat grasp_snap)
    st = fresh()
    ee = ee_pose(world, st).pos
    _place_com_exact(world, st, 30, ee + np.array([0.0, 0.0, -0.10]))
    _place_com_exact(world, st, 22, ee + np.array([0.16, 0.0, 0.0]))
    out.append((st, 1.0, (1, int(kat["grasp_snap"]))))
    # none: only 22 at 0.16 (kat grasp_none)
    st = fresh()
    _place_com_exact(world, st, 22, ee + np.array([0.0, 0.16, 0.0]))
    out.append((st, 1.0, (0, -1) if bool(kat["grasp_none"]) else (1, 22)))
    # tie: 31 and 25 at the identical COM 0.10 away -> the lower id (kat grasp_tie)
    st = fresh()
    _place_com_exact(world, st, 31, ee + np.array([0.06, 0.0, -0.08]))
    _place_com_exact(world, st, 25, ee + np.array([0.06, 0.0, -0.08]))
    c31 = st.pos[31] + world.bodies[31].com
    c25 = st.pos[25] + world.bodies[25].com
    assert np.array_equal(c31, c25)
    out.append((st, 1.0, (1, int(kat["grasp_tie"]))))
    return out
