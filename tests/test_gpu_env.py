"""Env pipeline (SPEC.md:292-350 restated): delay semantics and the
interleave-equivalence property."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import golden  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _episode(n):
    pool = golden("settled_pool.npz")
    return [pool["snapshots"][i % len(pool["snapshots"])].tobytes() for i in range(n)], \
        [int(pool["tags"][i % len(pool["snapshots"])][0]) for i in range(n)]


def _actions(n, steps, seed=0):
    rng = np.random.default_rng(seed)
    rest = np.array([0.0, 0.5, 0.0, -2.2, 0.0, 1.3, 0.0])
    arm = rest + rng.uniform(-0.3, 0.3, (steps, n, 7))
    base = np.stack([rng.uniform(-0.5, 1.0, (steps, n)), rng.uniform(-1, 1, (steps, n))], -1)
    return torch.tensor(arm, device="cuda"), torch.tensor(base, device="cuda")


def _run(interleave, delay, n=24, steps=6):
    from paper_2106_14405_b200.env import BatchEnv

    snaps, layouts = _episode(n)
    env = BatchEnv(n, layouts=(0, 1, 2), env_layout=layouts, obs_delay=delay, interleave=interleave)
    obs0 = env.reset(snaps)
    frames = [obs0["depth"].clone()]
    states, rendered = [], []
    arm, base = _actions(n, steps)
    for k in range(steps):
        obs, rew, done, info = env.step(arm_targets=arm[k], base_cmd=base[k])
        frames.append(obs["depth"].clone())
        rendered.append(obs["rendered_from_step"])
        states.append(env.states())
    torch.cuda.synchronize()
    env.close()
    return frames, states, rendered


def test_interleaved_equals_sequential():
    f_i, s_i, r_i = _run(True, 1)
    f_s, s_s, r_s = _run(False, 1)
    assert r_i == r_s == list(range(6))
    for a, b in zip(f_i, f_s):
        assert torch.equal(a, b)
    assert s_i == s_s  # bit-identical state snapshots at every step


def test_delay_semantics():
    """delay 1: step t returns o_t (render of s_t), world at t+1; delay 0
    returns o_{t+1}.  So delay-1 frame k+1 == delay-0 frame k."""
    f1, s1, r1 = _run(True, 1)
    f0, s0, r0 = _run(False, 0)
    assert r0 == [k + 1 for k in range(6)]
    assert s1 == s0
    for k in range(5):
        assert torch.equal(f1[k + 2], f0[k + 1])


def test_geodesic_navigation_terms_vs_oracle():
    """BatchEnv.set_nav_goals: per-step geodesic distance from every robot
    base (rs_nav_geodesic over rs_nav_fields) equals the oracle's Dijkstra
    field at the base's nearest walkable cell, and geodesic_delta is its
    decrease."""
    from oracle.oracle import Oracle
    from paper_2106_14405_b200.compiler import compile_world
    from paper_2106_14405_b200.env import BatchEnv
    from paper_2106_14405_b200.scene import build_world, flat_clutter
    from paper_2106_14405_b200.state import WorldState

    n, steps = 12, 3
    snaps, layouts = _episode(n)
    env = BatchEnv(n, layouts=(0, 1, 2), env_layout=layouts)
    env.reset(snaps)
    goals = np.random.default_rng(2).uniform([-4.0, -2.5], [4.0, 2.5], (n, 2))
    g0 = env.set_nav_goals(goals).cpu().numpy()
    orcs = {v: Oracle(compile_world(build_world(v, flat_clutter()))) for v in range(3)}
    fields = [orcs[layouts[e]].nav_field(goals[e]) for e in range(n)]
    arm, base = _actions(n, steps)
    prev = g0
    for k in range(steps):
        _, _, _, info = env.step(arm_targets=arm[k], base_cmd=base[k])
        torch.cuda.synchronize()
        geo = info["geodesic"].cpu().numpy()
        for e, blob in enumerate(env.sim.get_state()):
            st = WorldState.from_bytes(blob)
            assert geo[e] == orcs[layouts[e]].nav_geodesic(fields[e], st.base[:2])
        np.testing.assert_array_equal(info["geodesic_delta"].cpu().numpy(), prev - geo)
        prev = geo
    env.close()


def test_proprioception_fields_match_host_restatement():
    """Observation fields: joint positions, EE position in
    the robot frame (robot.py:161-169 FK), base egomotion since the previous
    observation and goal vectors -- of the state each observation is rendered
    from (o_t from s_t with the 1-step delay)."""
    import math

    from paper_2106_14405_b200.env import BatchEnv
    from paper_2106_14405_b200.scene import build_world, flat_clutter
    from paper_2106_14405_b200.state import WorldState, link_poses

    n, steps = 9, 4
    snaps, layouts = _episode(n)
    env = BatchEnv(n, layouts=(0, 1, 2), env_layout=layouts)
    goals = np.random.default_rng(5).uniform([-3, -2, 0.3], [3, 2, 1.2], (n, 2, 3))
    env.set_goal_positions(goals)
    robot = build_world(0, flat_clutter()).robot
    arm, base = _actions(n, steps)

    def expect(obs, st_now, st_prev):
        for e in range(n):
            a, p = WorldState.from_bytes(st_now[e]), None if st_prev is None else WorldState.from_bytes(st_prev[e])
            q = a.joints[-7:]
            np.testing.assert_array_equal(obs["joint_positions"][e].cpu().numpy(), q)
            _, ee = link_poses(robot, q)  # FK from the robot base (base frame)
            np.testing.assert_allclose(obs["ee_position"][e].cpu().numpy(), ee.pos, rtol=0, atol=1e-12)
            ego = np.zeros(6)
            if p is not None:
                c, s = math.cos(p.base[2]), math.sin(p.base[2])
                dx, dy = a.base[0] - p.base[0], a.base[1] - p.base[1]
                ego[0], ego[1] = c * dx + s * dy, -s * dx + c * dy
                ego[5] = (a.base[2] - p.base[2] + math.pi) % (2 * math.pi) - math.pi
            np.testing.assert_allclose(obs["base_egomotion"][e].cpu().numpy(), ego, rtol=0, atol=1e-12)
            c, s = math.cos(a.base[2]), math.sin(a.base[2])
            gv = np.stack([[c * (g[0] - a.base[0]) + s * (g[1] - a.base[1]),
                            -s * (g[0] - a.base[0]) + c * (g[1] - a.base[1]), g[2]] for g in goals[e]])
            np.testing.assert_allclose(obs["goal_vectors"][e].cpu().numpy(), gv, rtol=0, atol=1e-12)

    obs = env.reset(snaps)
    torch.cuda.synchronize()
    prev, cur = None, env.sim.get_state()
    expect(obs, cur, prev)
    for k in range(steps):
        obs, _, _, _ = env.step(arm_targets=arm[k], base_cmd=base[k])  # o_t from s_t (= cur)
        torch.cuda.synchronize()
        expect(obs, cur, prev)
        prev, cur = cur, env.sim.get_state()
    env.close()


def test_spec_action_step_matches_device_env_step():
    """BatchEnv.step(action) with the SPEC action (ArmAction + BaseAction as
    [E, 6]) runs IK -> physics -> grasp (rs_env_step): the same states as
    BatchSimulator.env_step on the same actions, in interleaved and
    sequential mode; the dict form is the same action."""
    from paper_2106_14405_b200.env import BatchEnv
    from paper_2106_14405_b200.sim import BatchSimulator

    n, steps = 12, 4
    snaps, layouts = _episode(n)
    rng = np.random.default_rng(3)
    act = np.zeros((steps, n, 6))
    act[..., :3] = rng.uniform(-0.02, 0.02, (steps, n, 3))
    act[..., 4] = rng.uniform(-0.5, 1.0, (steps, n))
    act[..., 5] = rng.uniform(-1, 1, (steps, n))
    act = torch.tensor(act, device="cuda")
    ref = BatchSimulator(layouts=(0, 1, 2), n_env=n, env_layout=layouts)
    ref.set_state(snaps)
    want = []
    for k in range(steps):
        ref.env_step(act[k])
        want.append(ref.get_state())
    ref.close()
    for interleave in (True, False):
        env = BatchEnv(n, layouts=(0, 1, 2), env_layout=layouts, interleave=interleave)
        env.reset(snaps)
        for k in range(steps):
            a = act[k] if k % 2 == 0 else {"arm": act[k, :, :3], "gripper": act[k, :, 3], "base": act[k, :, 4:6]}
            obs, rew, done, info = env.step(a)
            assert env.states() == want[k], f"step {k} interleave={interleave}"
            assert info["step_index"] == k + 1 and not bool(info["success"].any())
            assert (info["failure_reason"] == 0).all() and not bool(done.any())
            assert info["accumulated_force"].shape == (n,) and bool((info["accumulated_force"] >= 0).all())
        env.close()


def test_horizon_force_limit_and_step_after_done():
    """stepping past the horizon ends the episode with
    failure_reason = horizon; a force limit ends it with force_limit; a
    further step raises EpisodeDone until the env is reset."""
    from paper_2106_14405_b200.env import FAILURE_REASONS, BatchEnv, EpisodeDone

    n = 6
    snaps, layouts = _episode(n)
    env = BatchEnv(n, layouts=(0, 1, 2), env_layout=layouts, horizon=2)
    env.reset(snaps)
    a = torch.zeros((n, 6), dtype=torch.float64, device="cuda")
    _, _, done, info = env.step(a)
    assert not bool(done.any())
    _, _, done, info = env.step(a)
    assert bool(done.all()) and FAILURE_REASONS[int(info["failure_reason"][0])] == "horizon"
    with pytest.raises(EpisodeDone):
        env.step(a)
    env.reset(snaps[:2], env_ids=[0, 1])
    with pytest.raises(EpisodeDone):  # envs 2..5 are still done
        env.step(a)
    env.reset(snaps)
    _, _, done, _ = env.step(a)
    assert not bool(done.any())
    env.close()
    env = BatchEnv(n, layouts=(0, 1, 2), env_layout=layouts, force_limit=-1.0)  # every env over the limit
    env.reset(snaps)
    _, _, done, info = env.step(a)
    assert bool(done.all()) and FAILURE_REASONS[int(info["failure_reason"][0])] == "force_limit"
    env.close()
