"""configs[0]-style long run: 100 control steps free-running on the GPU and
on the C oracle independently (no teacher forcing), Idle and Interact action
scripts in all three layouts.  The float64 arithmetic is the oracle's
(-fmad=false); only libm transcendentals (sin/cos/acos in kinematics and IK)
may differ in the last bit, so discrete state (sleep flags, held object,
step index) must agree exactly and continuous state to a stated tolerance."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import golden  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2106_14405_b200 import native  # noqa: E402
from paper_2106_14405_b200.compiler import compile_world  # noqa: E402
from paper_2106_14405_b200.scene import build_world, flat_clutter  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402
from paper_2106_14405_b200.state import WorldState  # noqa: E402

STEPS = 100
POS_TOL = 1e-12  # m / rad, after 100 free-running control steps (measured: <= 5e-16)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    native.lib()


def _actions(kind, steps, rng):
    a = np.zeros((steps, 6))
    if kind == "idle":
        a[:, :3] = rng.uniform(-0.02, 0.02, (steps, 3))
        a[:, 4] = rng.uniform(-0.5, 1.0, steps)
        a[:, 5] = rng.uniform(-1.0, 1.0, steps)
    else:  # interact: push into the light table, then sweep
        for k in range(steps):
            a[k, :3] = (0.015, 0.0, -0.012) if k < 60 else (0.0, 0.015 if (k // 10) % 2 == 0 else -0.015, 0.0)
    return a


@pytest.mark.parametrize("kind", ["idle", "interact"])
def test_hundred_steps_free_running(kind):
    pool = golden("settled_pool.npz")
    first = {}
    for b, (v, _s) in zip(pool["snapshots"], pool["tags"]):
        first.setdefault(int(v), b.tobytes())
    rng = np.random.default_rng(8)
    layouts = [0, 1, 2]
    states, acts = [], []
    for v in layouts:
        st = WorldState.from_bytes(first[v])
        st.base = np.array([2.3, -0.2, rng.uniform(-math.pi, math.pi)]) if kind == "idle" else \
            np.array([1.6, 0.2, math.pi / 2])
        states.append(st.to_bytes())
        acts.append(_actions(kind, STEPS, rng))
    acts = np.stack(acts, 1)  # [steps, env, 6]
    sim = BatchSimulator(layouts=(0, 1, 2), n_env=3, env_layout=layouts)
    sim.set_state(states)
    orcs = {v: Oracle(compile_world(build_world(v, flat_clutter()))) for v in layouts}
    cur = list(states)
    worst = 0.0
    for k in range(STEPS):
        sim.env_step(torch.tensor(acts[k], device="cuda"))
        for e, v in enumerate(layouts):
            st = WorldState.from_bytes(cur[e])
            nsj = len(st.joints) - 7
            tg, _ = orcs[v].apply_arm_action(st.joints[nsj:], acts[k, e, :3])
            r = orcs[v].step(cur[e], tg, acts[k, e, 4:])
            assert r.snapshot is not None
            cur[e] = r.snapshot
    torch.cuda.synchronize()
    sim.raise_faults()
    got = sim.get_state()
    for e in range(3):
        a, b = WorldState.from_bytes(got[e]), WorldState.from_bytes(cur[e])
        np.testing.assert_array_equal(a.asleep, b.asleep)
        assert (a.held, a.step_index) == (b.held, b.step_index)
        worst = max(worst, float(np.abs(a.pos - b.pos).max()), float(np.abs(a.joints - b.joints).max()))
        assert abs(a.accumulated_contact_force - b.accumulated_contact_force) <= 1e-9 * max(1.0, b.accumulated_contact_force)
    force = [WorldState.from_bytes(s).accumulated_contact_force for s in cur]
    print(f"{kind}: max |GPU - oracle| after {STEPS} steps = {worst:.3e}; robot contact force tally {force}")
    assert worst <= POS_TOL
    sim.close()


def test_config1_64_envs_pairs_and_render():
    """configs[1]: 64 envs (three layouts) stepping physics + RGBD together;
    every substep's admitted collision-pair list bit-exact vs the oracle, and
    the head/arm id images bit-exact for a sample of envs."""
    pool = golden("settled_pool.npz")
    rng = np.random.default_rng(64)
    n = 64
    blobs = [(b.tobytes(), int(v)) for b, (v, _s) in zip(pool["snapshots"], pool["tags"])]
    states, layouts = [], []
    for e in range(n):
        b, v = blobs[e % len(blobs)]
        st = WorldState.from_bytes(b)
        st.base = np.array([rng.uniform(1.8, 2.8), rng.uniform(-0.6, 0.2), rng.uniform(-3, 3)])
        states.append(st.to_bytes())
        layouts.append(v)
    sim = BatchSimulator(layouts=(0, 1, 2), n_env=n, env_layout=layouts)
    sim.set_trace(cap=256)
    sim.set_state(states)
    orcs = {v: Oracle(compile_world(build_world(v, flat_clutter()))) for v in range(3)}
    cur = list(states)
    for step in range(3):
        q = np.stack([WorldState.from_bytes(s).joints[-7:] for s in cur])
        arm = q + rng.uniform(-0.05, 0.05, q.shape)
        base = np.stack([rng.uniform(-0.5, 1.0, n), rng.uniform(-1, 1, n)], axis=1)
        rgba, depth, ids = sim.render(("head", "arm"))
        sim.step_physics(torch.tensor(arm), torch.tensor(base), check=True)
        torch.cuda.synchronize()
        got = sim.get_state()
        ids = ids.cpu().numpy()
        for e in range(n):
            r = orcs[layouts[e]].step(cur[e], arm[e], base[e])
            tr = np.array(sim.trace(e)).reshape(-1, 4)
            np.testing.assert_array_equal(tr[:, :3], r.pairs, err_msg=f"step {step} env {e}")
            if e % 16 == step:
                for cam in (0, 1):
                    _, _, o_ids, _ = orcs[layouts[e]].render(cur[e], cam)
                    np.testing.assert_array_equal(ids[e, cam], o_ids, err_msg=f"step {step} env {e} cam {cam}")
            cur[e] = got[e]
    sim.close()
