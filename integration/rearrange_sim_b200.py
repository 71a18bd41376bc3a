"""Reference-side adapter: run any scene of the reference simulator on the
B200 library.

The reference's operator API for the hot path is
``physics.Simulator(scene: SceneHandle, robot_model, clutter, config)``
(``/root/reference/pkg/src/rearrange_sim/physics.py:257-330``) over
``scene.load_scene`` (``scene.py:475-588``).  This module is what a
maintainer drops next to it: it reads the body / part / joint / robot /
walk-grid tables out of a constructed reference ``Simulator`` -- whatever
layout, furniture placement, asset library or clutter set built it -- into
the ``rs_scene_desc`` tables ``include/rsim.h`` takes, and wraps a
``BatchSimulator`` in the reference's own call shapes:

    sim = physics.Simulator(scene.load_scene(my_layout, cache), robot.default_model(), clutter)
    b200 = B200Simulator(sim, n_env=len(states))
    states, events = b200.step_physics(states, targets)        # lists of WorldState / JointTargets
    states = b200.apply_grasp_rule(states, gripper)             # rb.grasp_rule + Simulator.apply_grasp
    rgba, depth, ids = b200.render(states)                     # SPEC render_depth, both cameras

It needs the reference package importable (``rearrange_sim``) and is not
part of the product package: the product never imports the reference.
``scene_tables`` output is plain numpy, so it can be saved and shipped to a
machine without the reference (``tests/golden/traj_custom.npz`` does that).
"""

from __future__ import annotations

import numpy as np

KIND = {"static": 0, "kinematic": 1, "dynamic": 2}
PKIND = {"box": 0, "sphere": 1, "hull": 2}
NO_GROUP = -(2**31)


def _as12(pose) -> np.ndarray:
    return np.concatenate([np.asarray(pose.rot, float).reshape(9), np.asarray(pose.pos, float)])


def _translation_only(pose, what: str) -> np.ndarray:
    if not np.array_equal(np.asarray(pose.rot, float), np.eye(3)):
        raise ValueError(f"{what}: only translation offsets are supported by the device arm chain")
    return np.asarray(pose.pos, float)


def scene_tables(sim) -> dict:
    """``rs_scene_desc`` tables (the ``compile_world`` format) of a reference
    ``physics.Simulator``: bodies in the reference's id order
    (``physics.py:276-319``: scene bodies, robot base + links, clutter), the
    reference's own primitives (qhull facets with their multiplicity, vertices,
    triangles), no-collide groups (``_build_groups`` ``physics.py:321-330``),
    scene joints, the arm chain, camera mounts and the walk grid."""
    from paper_2106_14405_b200.compiler import body_colour

    if sim.robot is None:
        raise ValueError("the B200 step needs a robot model (the reference allows robot_model=None)")
    bodies = sim.bodies
    nb = len(bodies)
    t = {}
    t["body_kind"] = np.array([KIND[b.kind] for b in bodies], np.int32)
    t["body_robot"] = np.array([int(b.is_robot) for b in bodies], np.int32)
    t["body_group"] = np.array([sim._same_group.get(b.body_id, NO_GROUP) for b in bodies], np.int32)
    t["body_joint"] = np.array([b.scene_joint for b in bodies], np.int32)
    t["body_inv_mass"] = np.array([b.inv_mass for b in bodies], np.float64)
    t["body_com"] = np.array([b.com_local for b in bodies], np.float64).reshape(nb, 3)
    t["body_inv_inertia"] = np.array([b.inv_inertia_local for b in bodies], np.float64).reshape(nb, 9)
    t["body_friction"] = np.array([b.friction for b in bodies], np.float64)
    t["body_restitution"] = np.array([b.restitution for b in bodies], np.float64)

    class _C:  # render colour by category (the pinned RGB rule; robot links share one palette)
        def __init__(self, b):
            self.body_id, self.category = b.body_id, "robot" if b.is_robot else b.category

    t["body_color"] = np.stack([body_colour(_C(b)) for b in bodies]).astype(np.float32)
    t["body_name"] = np.array([b.name for b in bodies])

    part_body, part_kind, part_local, part_param = [], [], [], []
    fb, vb, tb, pb = [0], [0], [0], [0]
    facets, verts, tris = [], [], []
    for b in bodies:
        for local, prim in b.parts:
            k = PKIND[prim.kind]
            part_body.append(b.body_id)
            part_kind.append(k)
            part_local.append(_as12(local))
            if k == 1:
                part_param.append([prim.radius, 0.0, 0.0])
                n, o, v, tr = np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)), np.zeros((0, 3), int)
            else:
                part_param.append(list(prim.half) if k == 0 else [0.0, 0.0, 0.0])
                n, o, v = prim.normals, prim.offsets, prim.vertices
                tr = prim.triangles if k == 2 else np.zeros((0, 3), int)
            facets.append(np.concatenate([np.asarray(n, float).reshape(-1, 3), np.asarray(o, float)[:, None]], axis=1))
            verts.append(np.asarray(v, float).reshape(-1, 3))
            tris.append(np.asarray(tr).reshape(-1, 3))
            fb.append(fb[-1] + len(n))
            vb.append(vb[-1] + len(v))
            tb.append(tb[-1] + len(tr))
        pb.append(len(part_body))
    t["body_part_begin"] = np.array(pb, np.int32)
    t["part_body"] = np.array(part_body, np.int32)
    t["part_kind"] = np.array(part_kind, np.int32)
    t["part_local"] = np.array(part_local, np.float64)
    t["part_param"] = np.array(part_param, np.float64)
    t["part_facet_begin"] = np.array(fb, np.int32)
    t["part_vert_begin"] = np.array(vb, np.int32)
    t["part_tri_begin"] = np.array(tb, np.int32)
    t["facet"] = np.concatenate(facets).astype(np.float64)
    t["vert"] = np.concatenate(verts).astype(np.float64)
    t["tri"] = np.concatenate(tris).astype(np.int32).reshape(-1, 3)

    js = sim.scene.joints  # scene.py:429-441
    t["joint_type"] = np.array([0 if j.joint.joint_type == "revolute" else 1 for j in js], np.int32)
    t["joint_body"] = np.array([j.body_id for j in js], np.int32)
    t["joint_parent"] = np.array([j.parent_body for j in js], np.int32)
    t["joint_axis"] = np.array([j.joint.axis for j in js], np.float64).reshape(len(js), 3)
    t["joint_origin"] = np.array([_as12(j.joint.origin) for j in js], np.float64).reshape(len(js), 12)
    t["joint_limits"] = np.array([j.joint.limits for j in js], np.float64).reshape(len(js), 2)
    t["joint_handle"] = np.array([j.joint.handle_point for j in js], np.float64).reshape(len(js), 3)

    r = sim.robot  # robot.py:35-63
    t["arm_offset"] = np.array([_translation_only(j.offset, f"arm joint {j.name}") for j in r.joints], np.float64)
    t["arm_axis"] = np.array([j.axis for j in r.joints], np.float64)
    t["arm_limits"] = np.array([j.limits for j in r.joints], np.float64)
    t["gripper_offset"] = _translation_only(r.gripper_offset, "gripper offset")
    cams = [r.cameras["head"], r.cameras["arm"]]
    t["cam_parent"] = np.array([0 if c.parent == "base" else 1 for c in cams], np.int32)
    t["cam_mount"] = np.array([_as12(c.pose) for c in cams], np.float64)

    g = sim.scene.navgrid  # navgrid.py:20-51
    t["nav_walkable"] = np.ascontiguousarray(np.asarray(g.walkable).astype(np.uint8))
    t["nav_origin"] = np.asarray(g.origin, np.float64)
    t["nav_cell"] = float(g.cell)
    t["robot_base"] = int(sim.robot_body_ids[0])
    t["n_scene_joints"] = len(js)
    t["n_arm"] = r.dof
    return t


def save_tables(t: dict, path_or_dict, prefix: str = "scene_"):
    """Flatten ``scene_tables`` output into npz-able arrays under ``prefix``."""
    out = path_or_dict if isinstance(path_or_dict, dict) else {}
    for k, v in t.items():
        out[prefix + k] = np.asarray(v)
    if not isinstance(path_or_dict, dict):
        np.savez_compressed(path_or_dict, **out)
    return out


def load_tables(npz, prefix: str = "scene_") -> dict:
    """Inverse of ``save_tables`` (works without the reference installed)."""
    t = {k[len(prefix):]: npz[k] for k in npz.files if k.startswith(prefix)}
    for k in ("n_scene_joints", "n_arm", "robot_base"):
        t[k] = int(t[k])
    t["nav_cell"] = float(t["nav_cell"])
    return t


class B200Simulator:
    """``physics.Simulator``'s stepping API over a batch on one GPU: states are
    reference ``WorldState`` objects (exchanged in their own byte format,
    ``physics.py:147-206``), one env per state.

    ``sim`` is a reference ``Simulator`` (tables and ``PhysicsConfig`` are read
    from it); alternatively ``tables`` (``scene_tables`` output, e.g. loaded
    from an npz) plus ``config`` (a dict of ``PhysicsConfig`` fields).  The
    reference classes used for results default to ``rearrange_sim.physics``'s
    ``WorldState`` / ``ContactEvent`` / ``PhysicsFault``; any classes with the
    same byte format / fields can be passed (the GPU tests use this repo's
    ``WorldState`` where the reference is not installed)."""

    def __init__(self, sim=None, n_env: int = 1, device="cuda", event_cap: int = 256, config: dict | None = None,
                 tables: dict | None = None, state_cls=None, event_cls=None, fault_cls=None):
        import dataclasses

        from paper_2106_14405_b200.sim import BatchSimulator

        if (sim is None) == (tables is None):
            raise ValueError("pass exactly one of sim (a reference Simulator) or tables")
        cfg = {}
        if sim is not None:  # PhysicsConfig (physics.py:54-74) -> rs_physics_config, field for field
            cfg = {f.name: getattr(sim.config, f.name) for f in dataclasses.fields(sim.config)}
            tables = scene_tables(sim)
        cfg.update(config or {})
        if state_cls is None or event_cls is None or fault_cls is None:
            from rearrange_sim import physics

            state_cls = state_cls or physics.WorldState
            event_cls = event_cls or physics.ContactEvent
            fault_cls = fault_cls or physics.PhysicsFault
        self.WorldState, self.ContactEvent, self.PhysicsFault = state_cls, event_cls, fault_cls
        self.ref = sim
        self.batch = BatchSimulator(scenes=[tables], n_env=n_env, device=device, event_cap=event_cap, config=cfg)
        self.n_env = n_env

    def close(self):
        self.batch.close()

    def _load(self, states):
        if len(states) != self.n_env:
            raise ValueError(f"expected {self.n_env} states, got {len(states)}")
        self.batch.set_state([s.to_bytes() for s in states])

    def _states(self):
        return [self.WorldState.from_bytes(b) for b in self.batch.get_state()]

    def step_physics(self, states, targets, dt: float = 1.0 / 30.0, substeps: int = 4):
        """``Simulator.step_physics`` (``physics.py:575-594``) for every state:
        functional (inputs untouched), returns (new states, per-env ContactEvent
        lists); raises ``PhysicsFault`` like the reference for a non-finite
        state or bad ``dt`` / ``substeps``.  ``targets[e]``: a ``JointTargets``
        (``.arm``, ``.base.linear_velocity / angular_velocity``) or None."""
        import torch

        if not (dt > 0) or substeps < 1:
            raise self.PhysicsFault(f"bad step parameters dt={dt} substeps={substeps}")
        n_arm = self.batch.n_arm
        arm = np.zeros((self.n_env, n_arm))
        base = np.zeros((self.n_env, 2))
        has = np.zeros(self.n_env, np.uint8)
        for e, tg in enumerate(targets):
            if tg is None:
                continue
            has[e] = 1
            arm[e] = tg.arm
            if getattr(tg, "base", None) is not None:
                base[e] = (tg.base.linear_velocity, tg.base.angular_velocity)
        self._load(states)
        self.batch.step_physics(torch.tensor(arm), torch.tensor(base), torch.tensor(has), dt=dt, substeps=substeps)
        try:
            self.batch.raise_faults()
        except Exception as exc:  # the library's fault word -> the reference's exception type
            raise self.PhysicsFault(str(exc)) from exc
        cnt = self.batch.event_counts().cpu().numpy()
        ev = self.batch.events().cpu().numpy()
        events = [[self.ContactEvent(bodies=(int(r[0]), int(r[1])), impulse=float(r[2]), force=float(r[3]),
                                     point=np.array(r[4:7])) for r in ev[e, :cnt[e]]] for e in range(self.n_env)]
        return self._states(), events

    def apply_grasp_rule(self, states, gripper):
        """``rb.grasp_rule`` + ``Simulator.apply_grasp`` (``robot.py:323-346``,
        ``physics.py:1039-1084``); returns the new states."""
        import torch

        self._load(states)
        self.batch.grasp(torch.as_tensor(np.asarray(gripper, float)))
        return self._states()

    def render(self, states, cams=("head", "arm")):
        """SPEC ``render_depth`` (``SPEC.md:243-263``) for every state: RGBA8,
        range depth (float32) and body ids ``[n_env, len(cams), H, W]`` numpy."""
        import torch

        self._load(states)
        out = self.batch.render(cams)
        torch.cuda.synchronize(self.batch.device)
        return tuple(t.cpu().numpy() for t in out)
