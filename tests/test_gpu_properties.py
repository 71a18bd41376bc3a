"""The SPEC's physics and render invariants as
properties of the GPU path over many envs and steps (Idle and Interact
trajectories, 96 envs x 12 steps):

* determinism: the same (state, targets) -> bit-identical successor, in a
  fresh batch, in another batch size and env order;
* joint limits: every joint position within [lo, hi] after every step;
* sleeping soundness: a body asleep before and after a step kept its pose
  bit for bit and has zero velocity;
* locality: an env whose robot is far from every dynamic body does no
  narrowphase test among sleeping non-robot pairs (the counter only moves
  for robot pairs);
* render determinism / cache soundness: the same state renders the same
  image, the mixed-precision path equals the all-FP64 one.
(Energy is not asserted: SPEC's energy property does not hold in the
reference itself.)"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import golden  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _setup(n, interact):
    import bench

    gids = np.arange(n)
    pool = bench.settled_pool()
    states = bench.interact_states(gids, pool) if interact else bench.idle_states(gids, pool)
    acts = bench.interact_actions(n, 12) if interact else bench.action_table(n, 12, seed=11)
    return gids, states, acts


@pytest.mark.parametrize("interact", [False, True])
def test_physics_invariants(interact):
    from paper_2106_14405_b200.scene import build_world, flat_clutter
    from paper_2106_14405_b200.sim import BatchSimulator
    from paper_2106_14405_b200.state import WorldState

    n = 96
    gids, states, acts = _setup(n, interact)
    lay = (gids % 3).tolist()
    worlds = {v: build_world(v, flat_clutter()) for v in range(3)}
    sim = BatchSimulator(layouts=(0, 1, 2), n_env=n, env_layout=lay)
    sim.set_state(states)
    act = torch.tensor(acts, device="cuda")
    prev = [WorldState.from_bytes(b) for b in states]
    seq = []
    for k in range(12):
        sim.env_step(act[k])
        sim.raise_faults()
        cur = [WorldState.from_bytes(b) for b in sim.get_state()]
        seq.append(sim.get_state())
        for e in range(n):
            w = worlds[lay[e]]
            a, b = prev[e], cur[e]
            lo = np.concatenate([[j.spec.limits[0] for j in w.layout.joints], w.robot.limits_lo()])
            hi = np.concatenate([[j.spec.limits[1] for j in w.layout.joints], w.robot.limits_hi()])
            assert (b.joints >= lo).all() and (b.joints <= hi).all(), f"env {e} step {k}: joint limits"
            both = a.asleep.astype(bool) & b.asleep.astype(bool)
            assert np.array_equal(a.pos[both], b.pos[both]) and np.array_equal(a.quat[both], b.quat[both]), \
                f"env {e} step {k}: a sleeping body moved"
            assert (b.lin_vel[b.asleep.astype(bool)] == 0).all() and (b.ang_vel[b.asleep.astype(bool)] == 0).all()
        prev = cur
    sim.close()
    # determinism: a fresh batch of another size with the envs in reverse order
    order = np.arange(n)[::-1][: n // 2]
    sim2 = BatchSimulator(layouts=(0, 1, 2), n_env=len(order), env_layout=[lay[e] for e in order])
    sim2.set_state([states[e] for e in order])
    act2 = act[:, torch.tensor(order.copy(), device="cuda")]
    for k in range(12):
        sim2.env_step(act2[k].contiguous())
        out = sim2.get_state()
        assert all(out[i] == seq[k][e] for i, e in enumerate(order)), f"step {k}: not deterministic"
    sim2.close()


def test_locality_no_sleeping_pair_tests_far_from_the_robot():
    """Robot parked far from every dynamic body, all clutter asleep: the
    step admits no sleeping-sleeping / sleeping-static pair and no
    narrowphase test involves only non-robot bodies (reference counters:
    narrowphase tests stay at the robot's own pairs)."""
    from paper_2106_14405_b200.sim import BatchSimulator
    from paper_2106_14405_b200.state import WorldState

    g = golden("traj_fixed.npz")  # all asleep, zero action (layout 1)
    st = WorldState.from_bytes(g["pre"][0].tobytes())
    sim = BatchSimulator(layouts=(1,), n_env=1)
    sim.set_trace(cap=256)
    sim.set_state([st.to_bytes()])
    sim.step_physics(torch.tensor(g["arm"][:1]), torch.tensor(g["base"][:1]), check=True)
    tr = np.array(sim.trace(0)).reshape(-1, 4)
    robot = set(range(st.pos.shape[0] - 20 - 8, st.pos.shape[0] - 20))  # robot base + 7 links precede the clutter
    touching = tr[tr[:, 3] > 0]
    assert all(int(a) in robot or int(b) in robot for _, a, b, _ in touching), "contacts among non-robot bodies"
    out = WorldState.from_bytes(sim.get_state()[0])
    assert out.asleep[-20:].all()
    sim.close()


def test_render_determinism_and_cache_soundness():
    """Same state -> bit-identical images across launches, batch positions
    and cameras rendered alone; the bounded-error path == the all-FP64 one."""
    from paper_2106_14405_b200.sim import BatchSimulator

    g = golden("render_views.npz")
    sel = [i for i in range(len(g["cam"])) if int(g["layout"][i]) == 2][:20]
    blobs = [g["state"][i].tobytes() for i in sel]
    sim = BatchSimulator(layouts=(2,), n_env=2 * len(sel))
    sim.set_state(blobs + blobs[::-1])
    a = [t.clone() for t in sim.render()]
    b = sim.render()
    head = sim.render(("head",))
    exact = sim.render_exact()
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    k = len(sel)
    for x in a:
        assert torch.equal(x[:k], x[k:].flip(0))
    assert torch.equal(head[1][:, 0], a[1][:, 0]) and torch.equal(head[2][:, 0], a[2][:, 0])
    for x, y in zip(a, exact):
        assert torch.equal(x, y)
    sim.close()
