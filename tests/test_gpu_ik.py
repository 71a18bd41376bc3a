"""Batched IK on device (rs_arm_action, robot.py:185-313) vs the reference
goldens and the C oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import golden  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_arm_action_matches_reference_and_oracle():
    from oracle.oracle import Oracle
    from paper_2106_14405_b200.compiler import compile_world
    from paper_2106_14405_b200.scene import build_world, flat_clutter
    from paper_2106_14405_b200.sim import BatchSimulator
    from paper_2106_14405_b200.state import WorldState

    k = golden("ik.npz")
    n = len(k["q"])
    base = WorldState.from_bytes(golden("settled_pool.npz")["snapshots"][0].tobytes())
    snaps = []
    for q in k["q"]:
        st = base.clone()
        st.joints[4:] = q
        snaps.append(st.to_bytes())
    sim = BatchSimulator(layouts=(0,), n_env=n)
    sim.set_state(snaps)
    tg, failed = sim.arm_action(torch.tensor(k["delta"]))
    tg, failed = tg.cpu().numpy(), failed.cpu().numpy()
    orc = Oracle(compile_world(build_world(0, flat_clutter())))
    for i in range(n):
        o, of = orc.apply_arm_action(k["q"][i], k["delta"][i])
        assert bool(failed[i]) == of == bool(k["fails"][i])
        np.testing.assert_allclose(tg[i], o, rtol=0, atol=1e-12, err_msg=f"case {i} vs oracle")
        np.testing.assert_allclose(tg[i], k["targets"][i], rtol=0, atol=1e-9, err_msg=f"case {i} vs reference")
    sim.close()


def test_unreachable_delta_is_noop():
    """An IK failure degrades to targets = current joints (robot.py:308-312)."""
    from paper_2106_14405_b200.sim import BatchSimulator

    g = golden("traj_idle.npz")
    sim = BatchSimulator(layouts=(0,), n_env=1)
    sim.set_state([g["pre"][0].tobytes()])
    q0 = sim.world_state(0).joints[4:]
    tg, failed = sim.arm_action(torch.tensor([[0.0, 0.0, 0.0]]))
    np.testing.assert_allclose(tg.cpu().numpy()[0], q0, atol=0)  # zero delta: FK(seed) is the target
    assert int(failed[0]) == 0
    sim.close()


def test_env_step_paper_action_space_matches_oracle():
    """rs_env_step: (dEE, gripper, base lin, base ang) -> IK -> physics ->
    grasp rule, vs the oracle composition apply_arm_action + step_physics."""
    from oracle.oracle import Oracle
    from paper_2106_14405_b200.compiler import compile_world
    from paper_2106_14405_b200.scene import build_world, flat_clutter
    from paper_2106_14405_b200.sim import BatchSimulator
    from paper_2106_14405_b200.state import WorldState

    pool = golden("settled_pool.npz")
    snaps = [b.tobytes() for b, t in zip(pool["snapshots"], pool["tags"]) if t[0] == 0]
    n = len(snaps)
    rng = np.random.default_rng(4)
    sim = BatchSimulator(layouts=(0,), n_env=n)
    cur = []
    for s in snaps:
        st = WorldState.from_bytes(s)
        st.base = np.array([2.3, -0.2, rng.uniform(-3, 3)])
        cur.append(st.to_bytes())
    sim.set_state(cur)
    orc = Oracle(compile_world(build_world(0, flat_clutter())))
    for step in range(6):
        act = np.concatenate([rng.uniform(-0.02, 0.02, (n, 3)), np.zeros((n, 1)),
                              rng.uniform(-0.5, 1.0, (n, 1)), rng.uniform(-1, 1, (n, 1))], axis=1)
        sim.env_step(torch.tensor(act))
        got = sim.get_state()
        for e in range(n):
            q = WorldState.from_bytes(cur[e]).joints[4:]
            tg, _ = orc.apply_arm_action(q, act[e, :3])
            r = orc.step(cur[e], tg, act[e, 4:])
            a, b = WorldState.from_bytes(got[e]), WorldState.from_bytes(r.snapshot)
            np.testing.assert_allclose(a.pos, b.pos, rtol=0, atol=1e-9)
            np.testing.assert_allclose(a.joints, b.joints, rtol=0, atol=1e-9)
            assert (a.asleep == b.asleep).all()
            cur[e] = got[e]
    sim.close()
