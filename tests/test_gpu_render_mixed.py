"""GPU parity of the mixed-precision renderer (rs_render: bounded-error FP32
box tests select candidates, FP64 resolves them) against the C oracle and
the all-FP64 variant (rsim_bench_render_exact) on 2 x 768 random views of
all three layouts.  Against the oracle: ids bit-exact, depth <= 1e-6, RGBA
<= 1 LSB on a sample of frames (the scalar oracle takes ~30 ms per frame).
Against the all-FP64 variant: identical bit for bit on every frame (the FP64
resolution picks the same nearest part, range, entering face and
lowest-id tie)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import golden  # noqa: E402
from paper_2106_14405_b200 import native  # noqa: E402
from paper_2106_14405_b200.geom import base_pose  # noqa: E402
from paper_2106_14405_b200.scene import build_world, flat_clutter  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402
from paper_2106_14405_b200.state import WorldState, link_poses  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    native.lib()


def random_views(n, seed):
    """Settled-pool states with the robot at random walkable cells, random
    headings and random arm configurations (link bodies moved along), so the
    head and arm cameras look everywhere in the three layouts."""
    pool = golden("settled_pool.npz")
    worlds = {v: build_world(v, flat_clutter()) for v in range(3)}
    by_layout = {0: [], 1: [], 2: []}
    for blob, (v, _s) in zip(pool["snapshots"], pool["tags"]):
        by_layout[int(v)].append(blob.tobytes())
    rng = np.random.default_rng(seed)
    states, layouts = [], []
    for i in range(n):
        v = i % 3
        w = worlds[v]
        st = WorldState.from_bytes(by_layout[v][rng.integers(len(by_layout[v]))])
        g = w.layout.grid
        cells = np.argwhere(g.walkable)
        ci, cj = cells[rng.integers(len(cells))]
        x = g.origin[0] + (ci + rng.uniform()) * g.cell
        y = g.origin[1] + (cj + rng.uniform()) * g.cell
        st.base = np.array([x, y, rng.uniform(-math.pi, math.pi)])
        lo, hi = w.robot.limits_lo(), w.robot.limits_hi()
        q = lo + rng.uniform(size=len(lo)) * (hi - lo)
        st.joints[w.arm_slice] = q
        links, _ = link_poses(w.robot, q, st.base)
        for bid, p in zip(w.robot_body_ids, [base_pose(st.base)] + links):
            st.pos[bid] = p.pos
            st.quat[bid] = p.quat()
        states.append(st.to_bytes())
        layouts.append(v)
    return states, layouts


@pytest.mark.parametrize("seed", [0, 1])
def test_mixed_matches_oracle_and_exact(seed):
    n = 768
    states, layouts = random_views(n, seed)
    sim = BatchSimulator(layouts=(0, 1, 2), n_env=n, env_layout=layouts)
    sim.set_state(states)
    a = sim.render(("head", "arm"))
    b = sim.render_exact(("head", "arm"))
    torch.cuda.synchronize()
    ids_a, ids_b = a[2].cpu().numpy(), b[2].cpu().numpy()
    bad = np.argwhere(ids_a != ids_b)
    assert len(bad) == 0, f"{len(bad)} id mismatches, first at {bad[:5].tolist()}"
    da, db = a[1].cpu().numpy(), b[1].cpu().numpy()
    np.testing.assert_array_equal(da.view(np.uint32), db.view(np.uint32))
    assert torch.equal(a[0], b[0])
    # the views are not degenerate: many bodies visible, some misses, both cameras
    assert len(np.unique(ids_a)) > 30 and (ids_a == -1).any() and (ids_a >= 0).mean() > 0.5
    sim.close()
    # GPU vs the C oracle on 160 frames of the batch (80 views x 2 cameras)
    from oracle.oracle import Oracle
    from paper_2106_14405_b200.compiler import compile_world

    orcs = {v: Oracle(compile_world(build_world(v, flat_clutter()))) for v in range(3)}
    rgba = a[0].cpu().numpy()
    for e in np.random.default_rng(100 + seed).choice(n, 80, replace=False):
        for cam in (0, 1):
            o_rgba, o_depth, o_ids, _ = orcs[layouts[e]].render(states[e], cam)
            np.testing.assert_array_equal(ids_a[e, cam], o_ids, err_msg=f"view {e} cam {cam} vs oracle")
            np.testing.assert_allclose(da[e, cam], o_depth, rtol=1e-6, atol=1e-6)
            assert np.abs(rgba[e, cam].astype(int) - o_rgba.astype(int)).max() <= 1


def test_mixed_matches_golden_render_frames():
    """Same images as the all-FP64 variant on the reference-pinned frames."""
    g = golden("render.npz")
    n = len(g["cam"])
    sim = BatchSimulator(layouts=(0,), n_env=n)
    sim.set_state([s.tobytes() for s in g["state"]])
    a = [t.cpu().numpy() for t in sim.render()]
    b = [t.cpu().numpy() for t in sim.render_exact()]
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    sim.close()
