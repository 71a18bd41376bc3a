"""Grasp transitions and rider bindings: the C oracle and the host state
builder against reference goldens (CPU only).

* ``grasp.npz``: 415 single-state ``grasp_rule`` + ``apply_grasp``
  transitions from the reference (robot.py:323-346, physics.py:1039-1084):
  clutter snaps, the 0.149 / 0.151 m boundary, exact ties, drawer-handle and
  fridge-door snaps, sleeping riders (wake clears the binding), releases of
  objects (wake) and handles (no wake), no-ops.
* ``traj_riders`` / ``traj_pick``: env-step records whose grasp phase after
  each physics step is replayed here (``post`` -> ``grasped``); their physics
  steps are teacher-forced by ``test_oracle.py``; their IK actions are
  checked against the reference's ``apply_arm_action``.
* ``kat.npz`` ``grasp_*``: the reference's grasp-rule known answers turned
  into world states (``grasp_cases.kat_states``).
"""
import numpy as np
import pytest

from conftest import golden
from grasp_cases import cmp_states, kat_states
from oracle.oracle import Oracle
from paper_2106_14405_b200.compiler import compile_world
from paper_2106_14405_b200.geom import Pose, quat_to_rot
from paper_2106_14405_b200.scene import build_world, flat_clutter
from paper_2106_14405_b200.state import WorldState, make_initial_state

_orc = {}


def oracle(layout):
    if layout not in _orc:
        _orc[layout] = Oracle(compile_world(build_world(layout, flat_clutter())))
    return _orc[layout]


def test_grasp_transitions_match_reference():
    g = golden("grasp.npz")
    kinds = set()
    for i in range(len(g["gripper"])):
        snap, tr = oracle(int(g["layout"][i])).grasp(g["pre"][i].tobytes(), g["gripper"][i])
        assert tr == tuple(g["trans"][i]), f"case {i}"
        cmp_states(WorldState.from_bytes(snap), WorldState.from_bytes(g["post"][i].tobytes()), what=f"case {i}")
        kinds.add((tr[0], tr[2] >= 0, tr[3] > 0))
    # every branch is exercised: none, object snap (with / without wake), handle snap, release
    assert {(0, False, False), (1, False, True), (1, False, False), (1, True, False), (2, False, False)} <= kinds


@pytest.mark.parametrize("name", ["riders", "pick"])
def test_env_record_grasp_phase(name):
    g = golden(f"traj_{name}.npz")
    orc = oracle(0)
    n_snap = 0
    for s in range(len(g["pre"])):
        if np.isnan(g["gripper"][s]):
            assert np.array_equal(g["grasped"][s], g["post"][s])
            continue
        snap, tr = orc.grasp(g["post"][s].tobytes(), g["gripper"][s])
        assert tr == tuple(g["trans"][s]), f"{name} step {s}"
        cmp_states(WorldState.from_bytes(snap), WorldState.from_bytes(g["grasped"][s].tobytes()), what=f"{name} {s}")
        n_snap += tr[0] == 1
    assert n_snap >= 1


@pytest.mark.parametrize("name", ["riders", "pick"])
def test_env_record_actions_match_reference_ik(name):
    """The action-driven steps: the oracle's apply_arm_action (robot.py:293-313)
    reproduces the recorded joint targets (<= 1e-9 rad, iterative DLS)."""
    g = golden(f"traj_{name}.npz")
    orc = oracle(0)
    n = 0
    for s in range(len(g["pre"])):
        a = g["action"][s]
        if np.isnan(a).any():
            continue
        q = WorldState.from_bytes(g["pre"][s].tobytes()).joints[4:]
        tg, _ = orc.apply_arm_action(q, a[:3])
        np.testing.assert_allclose(tg, g["arm"][s], rtol=0, atol=1e-9)
        np.testing.assert_array_equal(g["base"][s], a[4:6])
        assert g["gripper"][s] == a[3]
        n += 1
    assert n > 20


def test_rider_semantics_recorded():
    """traj_riders covers the rider rules: bound by make_initial_state, follow a
    dragged and a coasting drawer, ignored by their own container's pair
    (physics.py:557-560), woken (binding cleared) by the robot."""
    g = golden("traj_riders.npz")
    pre0 = WorldState.from_bytes(g["pre"][0].tobytes())
    assert (pre0.rider_joint >= 0).sum() == 4
    riders = [WorldState.from_bytes(b.tobytes()).rider_joint for b in g["grasped"]]
    counts = [int((r >= 0).sum()) for r in riders]
    assert counts[0] == 4 and min(counts) < 4  # a rider was woken
    moved = [not np.array_equal(WorldState.from_bytes(g["pre"][s].tobytes()).pos[22],
                                WorldState.from_bytes(g["post"][s].tobytes()).pos[22]) for s in range(30)]
    assert sum(moved) >= 10  # riders follow the drawer
    # the (rider, own tray) candidate pair is never admitted while the rider sleeps
    world = build_world(0, flat_clutter())
    tray = {j: world.layout.joints[j].body_id for j in range(len(world.layout.joints))}
    for s in range(20):
        st = WorldState.from_bytes(g["pre"][s].tobytes())
        pairs = {tuple(p) for p in g["pairs"][g["pair_off"][4 * s]:g["pair_off"][4 * s + 1]]}
        for b in world.clutter_body_ids:
            if st.rider_joint[b] >= 0 and st.asleep[b]:
                assert (min(b, tray[st.rider_joint[b]]), max(b, tray[st.rider_joint[b]])) not in pairs


def test_host_make_initial_state_binds_riders_like_reference():
    """state.make_initial_state / _bind_riders (host restatement of
    physics.py:344-405) rebuilds the reference's riders start state."""
    g = golden("traj_riders.npz")
    ref = WorldState.from_bytes(g["pre"][0].tobytes())
    world = build_world(0, flat_clutter())
    poses = [Pose(quat_to_rot(ref.quat[b]), ref.pos[b].copy()) for b in world.clutter_body_ids]
    me = make_initial_state(world, poses, base=ref.base, arm_joints=ref.joints[4:])
    np.testing.assert_array_equal(me.rider_joint, ref.rider_joint)
    np.testing.assert_array_equal(me.asleep, ref.asleep)
    np.testing.assert_allclose(me.rider_offset, ref.rider_offset, rtol=0, atol=1e-12)
    np.testing.assert_allclose(me.pos, ref.pos, rtol=0, atol=1e-12)


def test_grasp_rule_kat():
    k = golden("kat.npz")
    orc = oracle(0)
    for st, grip, (kind, body) in kat_states(k):
        snap, tr = orc.grasp(st.to_bytes(), grip)
        assert (tr[0], tr[1]) == (kind, body)
        assert WorldState.from_bytes(snap).held == (body if kind == 1 else -1)
