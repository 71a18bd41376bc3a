"""GPU batched settle (rs_settle: GJK spawn clearance + settle loop) against
the reference goldens (settle.npz, Simulator.settle physics.py:1113-1176)
and the C oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import golden  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2106_14405_b200 import native  # noqa: E402
from paper_2106_14405_b200.compiler import compile_world  # noqa: E402
from paper_2106_14405_b200.geom import Pose, quat_to_rot, rot_z  # noqa: E402
from paper_2106_14405_b200.scene import build_world, flat_clutter  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402
from paper_2106_14405_b200.state import WorldState, park_state, spawn_state  # noqa: E402

_orc = {}


def oracle(v):
    if v not in _orc:
        _orc[v] = Oracle(compile_world(build_world(v, flat_clutter())))
    return _orc[v]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    native.lib()


def _cmp(me: WorldState, ref: WorldState, tol):
    np.testing.assert_array_equal(me.asleep, ref.asleep)
    np.testing.assert_array_equal(me.sleep_counter, ref.sleep_counter)
    np.testing.assert_allclose(me.pos, ref.pos, rtol=0, atol=tol)
    np.testing.assert_allclose(me.quat, ref.quat, rtol=0, atol=tol)
    np.testing.assert_allclose(me.lin_vel, ref.lin_vel, rtol=0, atol=tol)


def test_settle_matches_reference():
    """The pool recipe's 24 (layout, seed) spawns in one batch: statuses,
    clearance verdicts (seed 5: 0.43 mm to the sofa), step counts and the
    settled states vs the reference and the oracle."""
    k = golden("settle.npz")
    n = len(k["tags"])
    clutter = build_world(0, flat_clutter()).clutter_body_ids
    sim = BatchSimulator(layouts=(0, 1, 2), n_env=n, env_layout=k["tags"][:, 0].tolist())
    status, info, value, steps = sim.settle([s.tobytes() for s in k["spawn"]], [clutter] * n)
    status, info, value, steps = (t.cpu().numpy() for t in (status, info, value, steps))
    out = sim.get_state()
    mask = sum(1 << b for b in clutter)
    for i in range(n):
        assert status[i] == k["outcome"][i], i
        if status[i] == sim.CLEARANCE:
            assert tuple(info[i]) == tuple(k["info"][i])
            rec = (k["pd_tag"] == i) & (k["pd_pair"][:, 0] == info[i][0]) & (k["pd_pair"][:, 1] == info[i][1])
            assert abs(value[i] - k["pd_dist"][rec][0]) <= 1e-12
            assert out[i] == k["spawn"][i].tobytes()  # nothing stepped
        else:
            assert steps[i] == k["steps"][i]
            ref = WorldState.from_bytes(k["final"][i].tobytes())
            _cmp(WorldState.from_bytes(out[i]), ref, 1e-12)
            o = oracle(int(k["tags"][i][0])).settle(k["spawn"][i].tobytes(), mask, 301)
            assert o[0] == status[i] and o[4] == steps[i]
            _cmp(WorldState.from_bytes(out[i]), WorldState.from_bytes(o[1]), 1e-12)
    sim.close()


def test_settle_many_envs_fell_timeout_and_untouched():
    """256 envs: re-posed spawns (random yaw and drop height) vs the oracle,
    a body placed below the floor (FELL), a short max_time (TIMEOUT), and
    envs outside env_ids left untouched."""
    k = golden("settle.npz")
    ok = np.nonzero(k["outcome"] == 0)[0]
    rng = np.random.default_rng(4)
    n = 256
    layouts = []
    spawns, placed = [], []
    for e in range(n):
        i = int(ok[e % len(ok)])
        v = int(k["tags"][i][0])
        world = build_world(v, flat_clutter())
        ref = WorldState.from_bytes(k["spawn"][i].tobytes())
        pl = []
        for b in world.clutter_body_ids:
            rot = quat_to_rot(ref.quat[b]) @ rot_z(rng.uniform(-0.05, 0.05))
            pos = ref.pos[b] + np.array([0.0, 0.0, rng.uniform(0.0, 0.01)])
            pl.append((b, Pose(rot, pos)))
        if e == 7:  # below the floor
            b0 = world.clutter_body_ids[0]
            pl[0] = (b0, Pose(np.eye(3), np.array([0.0, 0.0, -2.0])))
        spawns.append(spawn_state(park_state(world), pl).to_bytes())
        placed.append(world.clutter_body_ids)
        layouts.append(v)
    sim = BatchSimulator(layouts=(0, 1, 2), n_env=n, env_layout=layouts)
    ids = list(range(0, n - 16))  # the last 16 envs are not settled
    sim.set_state(spawns)
    before = sim.get_state(list(range(n - 16, n)))
    status, info, value, steps = (t.cpu().numpy() for t in sim.settle([spawns[e] for e in ids],
                                                                        [placed[e] for e in ids], env_ids=ids))
    out = sim.get_state()
    assert out[n - 16:] == before
    assert status[7] == sim.FELL and info[7][0] == build_world(layouts[7], flat_clutter()).clutter_body_ids[0]
    for e in list(range(0, len(ids), 9)) + [7]:
        mask = sum(1 << b for b in placed[e])
        o = oracle(layouts[e]).settle(spawns[e], mask, 301)
        assert o[0] == status[e] and o[4] == steps[e], e
        if o[0] == 1:
            assert tuple(o[2]) == tuple(info[e])
        else:
            _cmp(WorldState.from_bytes(out[e]), WorldState.from_bytes(o[1]), 1e-12)
    # timeout: two steps are not enough to put anything to sleep
    status2, _, _, steps2 = (t.cpu().numpy() for t in sim.settle(spawns[:8], placed[:8], env_ids=range(8),
                                                                   max_time=2.0 / 30.0))
    assert (status2[np.arange(8) != 7] == sim.TIMEOUT).all() and (steps2[np.arange(8) != 7] == 2).all()
    sim.close()
