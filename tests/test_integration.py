"""The reference-side adapter (integration/rearrange_sim_b200.py): the tables
it reads out of a reference ``physics.Simulator`` equal our scene compiler's
for the builtin layouts bit for bit, and it handles a non-builtin scene
(moved / duplicated furniture, another clutter set).  Needs the reference
importable (this container); skipped elsewhere -- the GPU side replays the
committed ``traj_custom.npz`` (tests/test_gpu_integration.py)."""
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if not os.path.isdir(REF):
    pytest.skip("reference package not present", allow_module_level=True)
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from conftest import golden  # noqa: E402


def _ref_sim(variant):
    from rearrange_sim import builtin, physics, robot, scene

    cache = builtin.default_cache()
    sh = scene.load_scene(builtin.make_layout(variant), cache)
    flat = ["pudding_box", "gelatin_box", "sponge", "plate", "tuna_fish_can", "bowl", "potted_meat_can", "apple",
            "orange"]
    clutter = [(cache.get_asset(flat[i % 9]), f"{flat[i % 9]}#{i}") for i in range(20)]
    return physics.Simulator(sh, robot.default_model(), clutter, physics.PhysicsConfig())


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_adapter_tables_equal_builtin_compiler(variant):
    from integration.rearrange_sim_b200 import scene_tables
    from paper_2106_14405_b200.compiler import compile_world
    from paper_2106_14405_b200.scene import build_world, flat_clutter

    mine = compile_world(build_world(variant, flat_clutter()))
    ref = scene_tables(_ref_sim(variant))
    for k, v in mine.items():
        a, b = np.asarray(v), np.asarray(ref[k])
        assert a.shape == b.shape, k
        np.testing.assert_array_equal(a, b, err_msg=k)


def test_custom_scene_tables_round_trip():
    """traj_custom.npz carries the adapter's tables of the non-builtin scene;
    regenerating them from the reference reproduces the fixture."""
    from integration.rearrange_sim_b200 import load_tables

    g = golden("traj_custom.npz")
    t = load_tables(g)
    nb = len(t["body_kind"])
    assert nb != 42 and t["n_scene_joints"] != 4  # not a builtin layout
    snap = g["pre"][0].tobytes()
    from paper_2106_14405_b200.state import snapshot_size

    assert len(snap) == snapshot_size(nb, t["n_scene_joints"] + t["n_arm"])
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import make_goldens as mg
    from integration.rearrange_sim_b200 import scene_tables

    ref = scene_tables(mg.custom_sim())
    for k, v in t.items():
        a, b = np.asarray(v), np.asarray(ref[k])
        if a.dtype.kind == "f":  # mass properties go through BLAS: last bits depend on its kernel
            np.testing.assert_allclose(a, b, rtol=0, atol=1e-12 * max(1.0, float(np.abs(b).max(initial=0))), err_msg=k)
        else:
            np.testing.assert_array_equal(a, b, err_msg=k)
