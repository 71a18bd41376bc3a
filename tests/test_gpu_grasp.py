"""GPU parity of the grasp phase, the rider rules and the full device env
step (IK -> physics -> grasp, ``rs_env_step``) against reference goldens.

* ``grasp.npz``: every reference ``grasp_rule`` + ``apply_grasp`` transition
  (robot.py:323-346, physics.py:1039-1084) replayed through ``rs_grasp``:
  held / held_joint / sleep flags / rider bindings bit-exact, held offset,
  grab point and grab q <= 1e-12, wakes counted like ``Simulator.wake``.
* ``traj_riders`` / ``traj_pick``: the grasp phase after each physics step,
  and every action-driven step through ``rs_env_step`` (device IK, physics,
  grasp) against the reference's record: pair lists bit-exact per substep,
  discrete state bit-exact, poses <= 1e-8 (the reference's IK agrees with
  ours to 1e-9 rad, tests/golden/ik.npz), and against the oracle's chain
  (apply_arm_action -> step -> grasp) <= 1e-10.
* ``kat.npz`` ``grasp_*`` known answers as world states.
* a stationary held object keeps its last follow velocity (physics.py:671-684
  only writes the held body when its pose changes): GPU == oracle free-running.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import golden  # noqa: E402
from grasp_cases import cmp_states, kat_states  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2106_14405_b200 import native  # noqa: E402
from paper_2106_14405_b200.compiler import compile_world  # noqa: E402
from paper_2106_14405_b200.scene import build_world, flat_clutter  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402
from paper_2106_14405_b200.state import WorldState  # noqa: E402

_orc = {}


def oracle(layout):
    if layout not in _orc:
        _orc[layout] = Oracle(compile_world(build_world(layout, flat_clutter())))
    return _orc[layout]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    native.lib()


def test_grasp_transitions_vs_reference():
    g = golden("grasp.npz")
    for v in range(3):
        idx = np.nonzero(g["layout"] == v)[0]
        sim = BatchSimulator(layouts=(v,), n_env=len(idx))
        sim.set_state([g["pre"][i].tobytes() for i in idx])
        c0 = sim.counters().clone()
        sim.grasp(torch.tensor(g["gripper"][idx]))
        out = sim.get_state()
        wakes = (sim.counters() - c0)[:, 2].cpu().numpy()
        for k, i in enumerate(idx):
            cmp_states(WorldState.from_bytes(out[k]), WorldState.from_bytes(g["post"][i].tobytes()), what=f"case {i}")
            assert wakes[k] == g["trans"][i][3], f"case {i}"
        sim.close()


def test_grasp_rule_kat():
    k = golden("kat.npz")
    cases = kat_states(k)
    sim = BatchSimulator(layouts=(0,), n_env=len(cases))
    sim.set_state([st.to_bytes() for st, _, _ in cases])
    sim.grasp(torch.tensor([g for _, g, _ in cases]))
    for (st, _, (kind, body)), blob in zip(cases, sim.get_state()):
        assert WorldState.from_bytes(blob).held == (body if kind == 1 else -1)
    sim.close()


@pytest.mark.parametrize("name", ["riders", "pick"])
def test_env_record_grasp_phase(name):
    g = golden(f"traj_{name}.npz")
    n = len(g["pre"])
    sim = BatchSimulator(layouts=(0,), n_env=n)
    sim.set_state([g["post"][s].tobytes() for s in range(n)])
    sim.grasp(torch.tensor(np.nan_to_num(g["gripper"], nan=0.0)))
    for s, blob in enumerate(sim.get_state()):
        cmp_states(WorldState.from_bytes(blob), WorldState.from_bytes(g["grasped"][s].tobytes()), what=f"{name} {s}")
    sim.close()


@pytest.mark.parametrize("name", ["riders", "pick"])
def test_env_step_vs_reference_and_oracle(name):
    """rs_env_step (device IK + physics + grasp) teacher-forced on every
    action-driven step of the reference record."""
    g = golden(f"traj_{name}.npz")
    rows = [s for s in range(len(g["pre"])) if not np.isnan(g["action"][s]).any()]
    assert len(rows) > 20
    sim = BatchSimulator(layouts=(0,), n_env=len(rows))
    sim.set_trace(cap=256)
    sim.set_state([g["pre"][s].tobytes() for s in rows])
    sim.env_step(torch.tensor(g["action"][rows]))
    torch.cuda.synchronize()
    assert (sim.faults().cpu().numpy() == 0).all()
    out = sim.get_state()
    orc = oracle(0)
    for k, s in enumerate(rows):
        me = WorldState.from_bytes(out[k])
        cmp_states(me, WorldState.from_bytes(g["grasped"][s].tobytes()), tol=1e-8, vel_tol=1e-6, what=f"{name} {s} ref")
        trace = np.array(sim.trace(k), dtype=np.int64).reshape(-1, 4)
        for sub in range(4):
            ref_pairs = g["pairs"][g["pair_off"][4 * s + sub]:g["pair_off"][4 * s + sub + 1]]
            np.testing.assert_array_equal(trace[trace[:, 0] == sub][:, 1:3], ref_pairs, err_msg=f"{name} {s}/{sub}")
        pre = WorldState.from_bytes(g["pre"][s].tobytes())
        a = g["action"][s]
        tg, _ = orc.apply_arm_action(pre.joints[4:], a[:3])
        r = orc.step(g["pre"][s].tobytes(), tg, a[4:6])
        snap, _ = orc.grasp(r.snapshot, a[3])
        cmp_states(me, WorldState.from_bytes(snap), tol=1e-10, vel_tol=1e-8, what=f"{name} {s} oracle")
    sim.close()


def test_stationary_held_object_keeps_velocity():
    """Free-running from a snap in the pick record: move, then hold still.
    The held body's velocity is only rewritten when its pose changes, so it
    keeps its last follow velocity -- GPU and oracle agree bit for bit on
    which steps that happens."""
    g = golden("traj_pick.npz")
    s0 = int(np.nonzero(g["trans"][:, 0] == 1)[0][0]) + 1
    start = g["pre"][s0].tobytes()
    assert WorldState.from_bytes(start).held >= 0
    acts = [np.array([0.01, 0.0, 0.01, 0.0, 0.0, 0.2])] * 3 + [np.zeros(6)] * 4
    sim = BatchSimulator(layouts=(0,), n_env=1)
    sim.set_state([start])
    orc = oracle(0)
    cur = start
    kept = 0
    for a in acts:
        sim.env_step(torch.tensor(a[None]))
        q = WorldState.from_bytes(cur).joints[4:]
        tg, _ = orc.apply_arm_action(q, a[:3])
        cur, _ = orc.grasp(orc.step(cur, tg, a[4:6]).snapshot, a[3])
        me, ref = WorldState.from_bytes(sim.get_state()[0]), WorldState.from_bytes(cur)
        cmp_states(me, ref, tol=1e-12, vel_tol=1e-10, what="free-running held")
        h = ref.held
        kept += bool(np.any(ref.lin_vel[h] != 0)) and not np.any(a[:3])
    assert kept >= 1
    sim.close()


def test_env_step_host_matches_device_env_step():
    """rs_env_step_host (host actions, o_t rendered concurrently, stats back)
    == rs_render(s_t) + rs_env_step on the same inputs (states and obs)."""
    g = golden("traj_pick.npz")
    rows = [s for s in range(len(g["pre"])) if not np.isnan(g["action"][s]).any()][:32]
    n = len(rows)
    pre = [g["pre"][s].tobytes() for s in rows]
    act = torch.tensor(g["action"][rows])
    a = BatchSimulator(layouts=(0,), n_env=n)
    b = BatchSimulator(layouts=(0,), n_env=n)
    a.set_state(pre)
    b.set_state(pre)
    obs_a = a.render()
    a.env_step(act.cuda())
    obs_b = b.alloc_obs()
    stats, _ = b.env_step_host(act.pin_memory(), out=obs_b)
    torch.cuda.synchronize()
    assert a.get_state() == b.get_state()
    for x, y in zip(obs_a, obs_b):
        assert torch.equal(x, y)
    assert (stats[:, 1].numpy() == 0).all()
    a.close()
    b.close()
