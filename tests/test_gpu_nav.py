"""GPU geodesics (rs_nav_fields / rs_nav_geodesic / rs_nav_path) against the
reference goldens (navgrid.py:109-172) and the C oracle: fields, distances
and waypoints bit-exact."""
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


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    native.lib()


@pytest.fixture(scope="module")
def sim():
    s = BatchSimulator(layouts=(0, 1, 2), n_env=3)
    yield s
    s.close()


def test_fields_match_reference(sim):
    k = golden("nav.npz")
    fields, cells = sim.distance_fields(k["goal"], layouts=k["layout"].tolist())
    f = fields.cpu().numpy()
    for g in range(len(k["goal"])):
        np.testing.assert_array_equal(f[g], k["field"][g], err_msg=f"goal {g}")
        gi, gj = np.argwhere(k["field"][g] == 0.0)[0]
        assert int(cells[g]) == gi * f.shape[2] + gj


def test_geodesic_and_paths_match_reference(sim):
    k = golden("nav.npz")
    goals, inv = np.unique(np.concatenate([k["q_layout"][:, None], k["q_goal"]], 1), axis=0, return_inverse=True)
    fields, _ = sim.distance_fields(goals[:, 1:], layouts=goals[:, 0].astype(int).tolist())
    lay = k["q_layout"].tolist()
    d = sim.geodesic_distance(fields, inv.ravel(), k["q_from"], layouts=lay).cpu().numpy()
    np.testing.assert_array_equal(d, k["q_dist"])
    wp, cnt = sim.shortest_path(fields, inv.ravel(), k["q_from"], layouts=lay, cap=400)
    wp, cnt = wp.cpu().numpy(), cnt.cpu().numpy()
    np.testing.assert_array_equal(cnt, k["path_len"])
    for q in range(len(cnt)):
        np.testing.assert_array_equal(wp[q, :cnt[q]], k["path"][q, :cnt[q]])


def test_random_goals_vs_oracle_and_robot_base_queries():
    """128 random goals (walkable and blocked, in and out of the grid) per
    layout vs the oracle; geodesic distance from every env's robot base."""
    rng = np.random.default_rng(3)
    n_env = 96
    s = BatchSimulator(layouts=(0, 1, 2), n_env=n_env)
    pool = golden("settled_pool.npz")
    snaps = {int(v): b.tobytes() for b, (v, _) in zip(pool["snapshots"], pool["tags"])}
    states = []
    for e in range(n_env):
        st = WorldState.from_bytes(snaps[e % 3])
        st.base = np.array([rng.uniform(-5, 5), rng.uniform(-3, 3), 0.0])
        states.append(st.to_bytes())
    s.set_state(states)
    goals = rng.uniform([-5.5, -3.5], [5.5, 3.5], (n_env, 2))
    lay = [e % 3 for e in range(n_env)]
    fields, _ = s.distance_fields(goals, layouts=lay)
    f = fields.cpu().numpy()
    orcs = {v: Oracle(compile_world(build_world(v, flat_clutter()))) for v in range(3)}
    for g in range(0, n_env, 7):
        np.testing.assert_array_equal(f[g], orcs[lay[g]].nav_field(goals[g]), err_msg=f"goal {g}")
    d = s.geodesic_distance(fields, np.arange(n_env)).cpu().numpy()  # robot bases, env scenes
    for e in range(n_env):
        base = WorldState.from_bytes(states[e]).base
        assert d[e] == orcs[lay[e]].nav_geodesic(f[e], base[:2])
    s.close()


def test_sphere_cast_matches_reference():
    """rs_sphere_cast vs Simulator.sphere_cast (cast.npz): same body (lowest id
    on ties), same range; a non-unit direction reports -2 (PhysicsFault)."""
    k = golden("cast.npz")
    n = len(k["t"])
    s = BatchSimulator(layouts=(0, 1, 2), n_env=n, env_layout=k["layout"].tolist())
    s.set_state([b.tobytes() for b in k["state"]])
    body, t = s.sphere_cast(k["origin"], k["dir"], k["max_dist"])
    body, t = body.cpu().numpy(), t.cpu().numpy()
    np.testing.assert_array_equal(body, k["body"])
    hit = body >= 0
    np.testing.assert_array_equal(t[hit], k["t"][hit])
    bad, _ = s.sphere_cast(k["origin"][:2], k["dir"][:2] * 1.01, [10.0, 10.0])
    assert (bad.cpu().numpy() == -2).all()
    s.close()
