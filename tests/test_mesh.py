"""Triangle-soup path host side: tessellation, subdivision,
BVH invariants, the 10k-200k-triangle sweep counts."""
import numpy as np
import pytest

from paper_2106_14405_b200 import mesh
from paper_2106_14405_b200.scene import build_world, flat_clutter


@pytest.fixture(scope="module")
def world():
    return build_world(0, flat_clutter())


def test_triangle_counts_match_survey(world):
    # 1,388 triangles at k = 1; k = 3 / 7 / 9 -> 12.5k / 68k / 112k
    assert mesh.compile_mesh(world, 1)["n_tri"] == 1388
    assert mesh.compile_mesh(world, 3)["n_tri"] == 12492


def test_subdivision_preserves_surface():
    rng = np.random.default_rng(0)
    tris = rng.normal(size=(5, 3, 3))
    for k in (2, 3, 5):
        sub = mesh.subdivide(tris, k)
        assert len(sub) == 5 * k * k
        area = lambda t: 0.5 * np.linalg.norm(np.cross(t[:, 1] - t[:, 0], t[:, 2] - t[:, 0]), axis=1).sum()
        np.testing.assert_allclose(area(sub), area(tris), rtol=1e-12)


def test_bvh_invariants(world):
    m = mesh.compile_mesh(world, 2)
    tri = m["tri"]
    v0, e1, e2 = tri[:, :3], tri[:, 3:6], tri[:, 6:]
    pts = np.stack([v0, v0 + e1, v0 + e2], axis=1)
    seen = np.zeros(len(tri), int)
    pnb = m["part_node_begin"]
    for p in range(len(pnb) - 1):
        stack = [(pnb[p], None)]
        while stack:
            n, parent = stack.pop()
            lo, hi, (a, b) = m["node_lo"][n], m["node_hi"][n], m["node_meta"][n]
            if b >= 0:
                seen[a:a + b] += 1
                P = pts[a:a + b].reshape(-1, 3)
                assert (P >= lo - 1e-9).all() and (P <= hi + 1e-9).all()
            else:
                stack += [(n + 1, n), (a, n)]
    assert (seen == 1).all()
