"""GPU triangle-soup renderer (rs_render_mesh) vs the convex oracle over the
same surfaces (spheres as their 10-gon prisms): ids bit-exact, range to
1e-6 m.  Pixels whose ray starts inside a closed shape are excluded (the
convex primitive returns t = 0 there, a triangle soup its exit face)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import golden  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("k", [1, 3])
def test_mesh_render_matches_convex_oracle(k):
    from oracle.oracle import Oracle
    from paper_2106_14405_b200.compiler import compile_world
    from paper_2106_14405_b200.mesh import prism_world
    from paper_2106_14405_b200.scene import build_world, flat_clutter
    from paper_2106_14405_b200.sim import BatchSimulator

    g = golden("render.npz")
    n = len(g["cam"])
    sim = BatchSimulator(layouts=(0,), n_env=n, mesh_k=k)
    sim.set_state([s.tobytes() for s in g["state"]])
    rgba, depth, ids = (t.cpu().numpy() for t in sim.render_mesh(("head", "arm")))
    orc = Oracle(compile_world(prism_world(build_world(0, flat_clutter()))))
    bad = 0
    for i in range(n):
        cam = int(g["cam"][i])
        _, o_depth, o_ids, o_t = orc.render(g["state"][i].tobytes(), cam)
        ok = ~(o_t == 0.0)
        mism = (ids[i, cam] != o_ids) & ok
        bad += int(mism.sum())
        hit = ok & (o_ids >= 0)
        np.testing.assert_allclose(depth[i, cam][hit], o_depth[hit], rtol=1e-6, atol=1e-6)
    assert bad == 0
    sim.close()
