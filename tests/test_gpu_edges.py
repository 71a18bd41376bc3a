"""Edge cases of the batched step and render on the GPU (against the C
oracle, which tests/test_oracle.py pins to the reference): render
resolutions and fields of view other than the benchmark's, an event buffer
smaller than the step's events, a faulted env beside healthy ones, a single
env, and every stream-ordered entry point called on a non-default stream."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import golden  # noqa: E402

EV_NOISE = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _oracle(layout=0):
    from oracle.oracle import Oracle
    from paper_2106_14405_b200.compiler import compile_world
    from paper_2106_14405_b200.scene import build_world, flat_clutter

    return Oracle(compile_world(build_world(layout, flat_clutter())))


@pytest.mark.parametrize("w,h,fov", [(64, 64, np.pi / 2), (96, 48, np.pi / 2), (16, 16, np.pi / 2),
                                     (128, 32, np.pi / 3), (128, 128, 2.0), (128, 128, 2.8), (64, 32, 2.5)])
def test_render_other_resolutions_and_fov(w, h, fov):
    """rs_render at W x H (multiples of 16, <= 128) and another field of view:
    ids bit-exact, depth <= 1e-6 vs the oracle restated at the same config.
    The wide fields of view (2.5, 2.8 rad) exercise the pixel-rectangle cull's
    clipping threshold zc sqrt(1 + tan_x^2 + tan_y^2) at large tangents."""
    from paper_2106_14405_b200.sim import BatchSimulator

    g = golden("render.npz")
    n = len(g["cam"])
    sim = BatchSimulator(layouts=(0,), n_env=n, render={"width": w, "height": h, "fov": fov})
    sim.set_state([s.tobytes() for s in g["state"]])
    rgba, depth, ids = (t.cpu().numpy() for t in sim.render(("head", "arm")))
    assert ids.shape == (n, 2, h, w)
    orc = _oracle()
    for i in range(n):
        for cam in (0, 1):
            o_rgba, o_depth, o_ids, _ = orc.render(g["state"][i].tobytes(), cam, width=w, height=h, fov=fov)
            np.testing.assert_array_equal(ids[i, cam], o_ids, err_msg=f"{w}x{h} fov {fov} frame {i} cam {cam}")
            np.testing.assert_allclose(depth[i, cam], o_depth, rtol=1e-6, atol=1e-6)
            assert np.abs(rgba[i, cam].astype(int) - o_rgba.astype(int)).max() <= 1
    sim.close()


def test_bad_render_config_is_refused():
    from paper_2106_14405_b200.native import RsimError
    from paper_2106_14405_b200.sim import BatchSimulator

    for bad in ({"width": 100}, {"height": 144}, {"width": 0}):
        with pytest.raises(RsimError):
            BatchSimulator(layouts=(0,), n_env=1, render=bad)


def test_event_buffer_overflow_keeps_the_first_events():
    """event_cap smaller than a step's events: the count still reports every
    event (the overflow signal), the buffer holds the first cap events in the
    reference's order, and nothing is written past it."""
    from paper_2106_14405_b200.sim import BatchSimulator

    g = golden("traj_settle.npz")
    s = int(np.argmax(np.diff(g["event_off"])))  # the step with most events
    cap = 3
    n = 4
    sim = BatchSimulator(layouts=(1,), n_env=n, event_cap=cap)
    sim.set_state([g["pre"][s].tobytes()] * n)
    arm = torch.tensor(np.tile(g["arm"][s], (n, 1)))
    base = torch.tensor(np.tile(g["base"][s], (n, 1)))
    ht = torch.tensor(np.full(n, g["has_targets"][s], np.uint8))
    sim.step_physics(arm, base, ht, check=True)
    cnt = sim.event_counts().cpu().numpy()
    ev = sim.events().cpu().numpy()
    r = _oracle(1).step(g["pre"][s].tobytes(), g["arm"][s] if g["has_targets"][s] else None, g["base"][s])
    assert len(r.events) > cap
    assert (cnt == len(r.events)).all()
    for e in range(n):
        np.testing.assert_array_equal(ev[e, :, :2], r.events[:cap, :2])
        np.testing.assert_allclose(ev[e, :, 2:], r.events[:cap, 2:], rtol=1e-9, atol=1e-9)
    sim.close()


def test_faulted_env_leaves_the_others_exact():
    """One env with a non-finite body velocity among healthy ones: it faults
    (PhysicsFault names it, its state is unchanged), the others step exactly
    as the oracle does."""
    from paper_2106_14405_b200.sim import BatchSimulator, PhysicsFault
    from paper_2106_14405_b200.state import WorldState

    g = golden("traj_idle.npz")
    bad = WorldState.from_bytes(g["pre"][0].tobytes())
    bad.lin_vel[33, 2] = np.inf
    blobs = [g["pre"][k].tobytes() for k in range(3)] + [bad.to_bytes()]
    sim = BatchSimulator(layouts=(0,), n_env=4)
    sim.set_state(blobs)
    sim.step_physics(torch.tensor(g["arm"][[0, 1, 2, 0]]), torch.tensor(g["base"][[0, 1, 2, 0]]))
    with pytest.raises(PhysicsFault, match="env 3: non-finite vel for body 33"):
        sim.raise_faults()
    out = sim.get_state()
    assert out[3] == blobs[3]
    orc = _oracle()
    for k in range(3):
        r = orc.step(blobs[k], g["arm"][k], g["base"][k])
        me, ref = WorldState.from_bytes(out[k]), WorldState.from_bytes(r.snapshot)
        np.testing.assert_allclose(me.pos, ref.pos, rtol=0, atol=1e-12)
        assert (me.asleep == ref.asleep).all()
    sim.close()


def test_single_env_and_side_stream():
    """n_env = 1, every call ordered on a non-default torch stream: same state
    and image as a 1-env batch on the default stream."""
    from paper_2106_14405_b200.sim import BatchSimulator

    g = golden("traj_interact.npz")
    outs = []
    for use_side in (False, True):
        sim = BatchSimulator(layouts=(0,), n_env=1)
        st = torch.cuda.Stream()
        ctx = torch.cuda.stream(st) if use_side else torch.cuda.stream(torch.cuda.current_stream())
        with ctx:
            sim.set_state([g["pre"][5].tobytes()])
            sim.step_physics(torch.tensor(g["arm"][5:6]), torch.tensor(g["base"][5:6]))
            obs = sim.render()
            snap = sim.get_state()
        torch.cuda.synchronize()
        outs.append((snap, [t.cpu() for t in obs]))
        sim.close()
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        assert torch.equal(a, b)


def test_wide_fov_random_views_all_layouts():
    """The reference's random views of all three layouts (render_views.npz:
    walkable views, cameras inside / just in front of static boxes) at a
    2.6 rad field of view, both cameras: ids bit-exact and depth <= 1e-6 vs
    the oracle at the same config (the pixel-rectangle cull clips boxes that
    reach behind the camera; wide tangents stress its threshold)."""
    from oracle.oracle import Oracle
    from paper_2106_14405_b200.compiler import compile_world
    from paper_2106_14405_b200.scene import build_world, flat_clutter
    from paper_2106_14405_b200.sim import BatchSimulator

    g = golden("render_views.npz")
    sel = list(range(0, len(g["cam"]), 3))
    lay = [int(g["layout"][i]) for i in sel]
    fov = 2.6
    sim = BatchSimulator(layouts=(0, 1, 2), n_env=len(sel), env_layout=lay, render={"fov": fov})
    sim.set_state([g["state"][i].tobytes() for i in sel])
    rgba, depth, ids = (t.cpu().numpy() for t in sim.render(("head", "arm")))
    sim.close()
    orcs = {v: Oracle(compile_world(build_world(v, flat_clutter()))) for v in range(3)}
    for j, i in enumerate(sel):
        for cam in (0, 1):
            o_rgba, o_depth, o_ids, _ = orcs[lay[j]].render(g["state"][i].tobytes(), cam, fov=fov)
            np.testing.assert_array_equal(ids[j, cam], o_ids, err_msg=f"view {i} cam {cam}")
            np.testing.assert_allclose(depth[j, cam], o_depth, rtol=1e-6, atol=1e-6)
            assert np.abs(rgba[j, cam].astype(int) - o_rgba.astype(int)).max() <= 1
