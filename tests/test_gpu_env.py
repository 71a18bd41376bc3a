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
        obs, rew, done, info = env.step(arm[k], base[k])
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
        _, _, _, info = env.step(arm[k], base[k])
        torch.cuda.synchronize()
        geo = info["geodesic"].cpu().numpy()
        for e, blob in enumerate(env.sim.get_state()):
            st = WorldState.from_bytes(blob)
            assert geo[e] == orcs[layouts[e]].nav_geodesic(fields[e], st.base[:2])
        np.testing.assert_array_equal(info["geodesic_delta"].cpu().numpy(), prev - geo)
        prev = geo
    env.close()
