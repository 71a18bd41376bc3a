"""Scene compiler vs the reference's own body/part/facet tables
(fixtures from tests/golden/make_goldens.py)."""
import numpy as np
import pytest

from paper_2106_14405_b200 import assets as A
from paper_2106_14405_b200.compiler import compile_world
from paper_2106_14405_b200.scene import build_world, flat_clutter
from paper_2106_14405_b200.state import WorldState, link_poses, make_initial_state


@pytest.mark.parametrize("v", [0, 1, 2])
def test_tables_match_reference(v, tables_golden):
    g = {k[3:]: tables_golden[k] for k in tables_golden.files if k.startswith(f"l{v}_")}
    t = compile_world(build_world(v, flat_clutter()))
    for k in ("body_kind", "body_robot", "body_joint", "part_body", "part_kind",
              "part_facet_begin", "part_vert_begin", "part_tri_begin", "tri",
              "joint_type", "joint_body", "joint_parent", "nav_walkable"):
        np.testing.assert_array_equal(t[k], g[k], err_msg=k)
    np.testing.assert_array_equal(t["body_group"], g["body_group"].astype(np.int32))
    for k in ("body_friction", "body_restitution", "part_local", "part_param", "vert",
              "joint_axis", "joint_origin", "joint_limits", "joint_handle", "nav_origin", "body_inv_mass"):
        np.testing.assert_array_equal(t[k], g[k], err_msg=k)
    # facets: identical qhull output (same scipy in this image)
    np.testing.assert_array_equal(t["facet"][:, :3], g["facet_normal"])
    np.testing.assert_array_equal(t["facet"][:, 3], g["facet_offset"])
    # mass properties go through LAPACK det/inv: tolerance, not bits
    np.testing.assert_allclose(t["body_com"], g["body_com"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(t["body_inv_inertia"], g["body_inv_inertia"].reshape(-1, 9), rtol=1e-12, atol=1e-9)


def test_park_state_matches_reference(tables_golden):
    w = build_world(0, flat_clutter())
    from paper_2106_14405_b200.geom import Pose
    park = [Pose(pos=np.array([-6.0 + 0.6 * i, 0.0, 40.0])) for i in range(20)]
    st = make_initial_state(w, park, clutter_asleep=True)
    ref = WorldState.from_bytes(tables_golden["l0_park_state"].tobytes())
    np.testing.assert_allclose(st.pos, ref.pos, rtol=0, atol=1e-15)
    np.testing.assert_allclose(st.quat, ref.quat, rtol=0, atol=1e-15)
    assert (st.asleep == ref.asleep).all()
    assert (st.rider_joint == ref.rider_joint).all()


def test_fk_matches_reference(tables_golden):
    r = A.fetch_like()
    for q, b, links, ee in zip(tables_golden["fk_q"], tables_golden["fk_base"],
                               tables_golden["fk_links"], tables_golden["fk_ee"]):
        lp, e = link_poses(r, q, b)
        for p, ref in zip(lp, links):
            np.testing.assert_allclose(p.as12(), ref, rtol=0, atol=1e-14)
        np.testing.assert_allclose(e.as12(), ee, rtol=0, atol=1e-14)
    np.testing.assert_array_equal(
        np.concatenate([r.cameras["head"][1].rot.reshape(9), r.cameras["head"][1].pos]), tables_golden["cam_head"])
    np.testing.assert_array_equal(
        np.concatenate([r.cameras["arm"][1].rot.reshape(9), r.cameras["arm"][1].pos]), tables_golden["cam_arm"])


def test_snapshot_roundtrip():
    g = np.load("tests/golden/settled_pool.npz")
    for blob in g["snapshots"]:
        st = WorldState.from_bytes(blob.tobytes())
        assert st.to_bytes() == blob.tobytes()
