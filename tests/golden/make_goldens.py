"""Generate the golden fixtures from the *reference* implementation.

Run here (the container that has ``/root/reference``), never on the GPU box:

    OPENBLAS_CORETYPE=Haswell OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_goldens.py

Everything in ``tests/golden/*.npz`` is produced by this script from the
reference package ``rearrange_sim`` (``/root/reference/pkg/src``) imported
as-is.  Fixtures:

* ``scene_tables.npz``  body / part / facet / joint / walk-grid tables of
  layouts 0-2 with the 20-object flat clutter set, as the reference builds
  them (``physics.py:257-330``, ``scene.py:475-588``) -> pins our scene
  compiler.
* ``settled_pool.npz``  snapshots (``WorldState.to_bytes``) of settled
  clutter states built by the SURVEY §8d recipe (``Simulator.settle``).
* ``traj_<name>.npz``  teacher-forcing records: per control step the input
  snapshot, the joint targets, the output snapshot, the contact events and
  counter deltas, and per substep the admitted pair list and narrowphase
  contacts (``physics.py:575-719``).
* ``render.npz``  per-pixel nearest-hit range and body id for head + arm
  cameras, computed with the reference ray primitive ``parts_ray_hits``
  (``geometry.py:772-776``) in body-id order with the pinned tie rule
  (|t_b - t_min| <= 1e-9 -> lowest body id; ``physics.py:1096-1100`` keeps
  the lowest id on exact ties).
* ``render_views.npz``  the same for layouts 0-2: random walkable views with
  random arm joints, views with the head camera inside a static convex
  (t = 0 pixels) and 2-8 cm in front of one (t < near pixels).
* ``kat.npz``  known-answer values (SPEC.md examples) from the reference.
* ``settle.npz``  per (layout, seed) of the pool recipe: the spawn state
  ``Simulator.settle`` builds, every AABB-overlapping ``parts_distance``
  (GJK, ``geometry.py:486-539``) and the settle outcome (final state + steps
  or the ``SettleUnstable`` reason), ``physics.py:1113-1176``.
* ``cast.npz``  ``Simulator.sphere_cast`` point queries (physics.py:1088-1101)
  from random origins / unit directions on settled states.
* ``nav.npz``  geodesic distance fields (Dijkstra, ``navgrid.py:109-143``),
  geodesic distances and steepest-descent shortest paths
  (``navgrid.py:145-172``) on the layouts' walk grids.

The numpy/scipy versions and the OpenBLAS core type are recorded in every
file (``meta`` key): the oracle's float64 last bits depend on them
(SURVEY.md §8c).
"""

from __future__ import annotations

import json
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from rearrange_sim import builtin, geometry as geo, physics, robot as rb, scene  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FLAT = ["pudding_box", "gelatin_box", "sponge", "plate", "tuna_fish_can", "bowl",
        "potted_meat_can", "apple", "orange"]
SLOT_RECEPTACLES = ["counter_left", "counter_right", "light_table", "dark_table", "sofa", "shelves"]
KIND = {"static": 0, "kinematic": 1, "dynamic": 2}
PKIND = {"box": 0, "sphere": 1, "hull": 2}
NO_GROUP = -(2**31)


def meta():
    import scipy

    return json.dumps({
        "numpy": np.__version__, "scipy": scipy.__version__,
        "openblas_coretype": os.environ.get("OPENBLAS_CORETYPE", "default"),
        "generator": "tests/golden/make_goldens.py",
    })


def make_sim(variant, config=None, n_clutter=20):
    cache = builtin.default_cache()
    sh = scene.load_scene(builtin.make_layout(variant), cache)
    names = [FLAT[i % len(FLAT)] for i in range(n_clutter)]
    sim = physics.Simulator(sh, rb.default_model(),
                            [(cache.get_asset(n), f"{n}#{i}") for i, n in enumerate(names)],
                            config or physics.PhysicsConfig())
    return sim, cache


# --------------------------------------------------------------------------
# scene tables
# --------------------------------------------------------------------------

def dump_tables(sim, prefix, out):
    bodies = sim.bodies
    out[prefix + "body_kind"] = np.array([KIND[b.kind] for b in bodies], np.int32)
    out[prefix + "body_robot"] = np.array([b.is_robot for b in bodies], np.int32)
    out[prefix + "body_group"] = np.array([sim._same_group.get(b.body_id, NO_GROUP) for b in bodies], np.int64)
    out[prefix + "body_joint"] = np.array([b.scene_joint for b in bodies], np.int32)
    out[prefix + "body_inv_mass"] = np.array([b.inv_mass for b in bodies])
    out[prefix + "body_com"] = np.array([b.com_local for b in bodies])
    out[prefix + "body_inv_inertia"] = np.array([b.inv_inertia_local for b in bodies])
    out[prefix + "body_friction"] = np.array([b.friction for b in bodies])
    out[prefix + "body_restitution"] = np.array([b.restitution for b in bodies])
    pb, pk, pl, pp, fb, nrm, off, vb, vert, tb, tri = [], [], [], [], [0], [], [], [0], [], [0], []
    for b in bodies:
        for local, prim in b.parts:
            pb.append(b.body_id)
            pk.append(PKIND[prim.kind])
            pl.append(np.concatenate([local.rot.reshape(9), local.pos]))
            if prim.kind == "sphere":
                pp.append([prim.radius, 0, 0])
                fb.append(fb[-1]); vb.append(vb[-1]); tb.append(tb[-1])
                continue
            pp.append(prim.half if prim.kind == "box" else [0, 0, 0])
            nrm.append(prim.normals); off.append(prim.offsets); vert.append(prim.vertices)
            fb.append(fb[-1] + len(prim.normals)); vb.append(vb[-1] + len(prim.vertices))
            t = prim.triangles if prim.kind == "hull" else np.zeros((0, 3), int)
            tri.append(t); tb.append(tb[-1] + len(t))
    out[prefix + "part_body"] = np.array(pb, np.int32)
    out[prefix + "part_kind"] = np.array(pk, np.int32)
    out[prefix + "part_local"] = np.array(pl)
    out[prefix + "part_param"] = np.array(pp, dtype=float)
    out[prefix + "part_facet_begin"] = np.array(fb, np.int32)
    out[prefix + "part_vert_begin"] = np.array(vb, np.int32)
    out[prefix + "part_tri_begin"] = np.array(tb, np.int32)
    out[prefix + "facet_normal"] = np.concatenate(nrm)
    out[prefix + "facet_offset"] = np.concatenate(off)
    out[prefix + "vert"] = np.concatenate(vert)
    out[prefix + "tri"] = np.concatenate(tri).astype(np.int32)
    js = sim.scene.joints
    out[prefix + "joint_type"] = np.array([0 if j.joint.joint_type == "revolute" else 1 for j in js], np.int32)
    out[prefix + "joint_body"] = np.array([j.body_id for j in js], np.int32)
    out[prefix + "joint_parent"] = np.array([j.parent_body for j in js], np.int32)
    out[prefix + "joint_axis"] = np.array([j.joint.axis for j in js])
    out[prefix + "joint_origin"] = np.array([np.concatenate([j.joint.origin.rot.reshape(9), j.joint.origin.pos]) for j in js])
    out[prefix + "joint_limits"] = np.array([j.joint.limits for j in js])
    out[prefix + "joint_handle"] = np.array([j.joint.handle_point for j in js])
    ng = sim.scene.navgrid
    out[prefix + "nav_walkable"] = ng.walkable.astype(np.uint8)
    out[prefix + "nav_origin"] = np.asarray(ng.origin, float)
    st = sim.park_state()
    out[prefix + "park_state"] = np.frombuffer(st.to_bytes(), np.uint8)


def gen_tables():
    out = {"meta": meta()}
    for v in range(3):
        sim, _ = make_sim(v)
        dump_tables(sim, f"l{v}_", out)
    m = rb.default_model()
    rng = np.random.default_rng(11)
    qs = np.stack([m.resting_joints, np.zeros(7)] + [rng.uniform(m.limits_lo(), m.limits_hi()) for _ in range(6)])
    bases = np.stack([[0.0, 0.0, 0.0], [2.3, -0.2, 0.7]] + [[rng.uniform(-3, 3), rng.uniform(-2, 2), rng.uniform(-3, 3)] for _ in range(6)])
    link_pose, ee = [], []
    for q, b in zip(qs, bases):
        links, e = rb.link_poses(m, q, b)
        link_pose.append([np.concatenate([lp.rot.reshape(9), lp.pos]) for lp in links])
        ee.append(np.concatenate([e.rot.reshape(9), e.pos]))
    out["fk_q"], out["fk_base"] = qs, bases
    out["fk_links"], out["fk_ee"] = np.array(link_pose), np.array(ee)
    out["cam_head"] = np.concatenate([m.cameras["head"].pose.rot.reshape(9), m.cameras["head"].pose.pos])
    out["cam_arm"] = np.concatenate([m.cameras["arm"].pose.rot.reshape(9), m.cameras["arm"].pose.pos])
    np.savez_compressed(os.path.join(OUT, "scene_tables.npz"), **out)


# --------------------------------------------------------------------------
# settled pool (SURVEY.md §8d recipe)
# --------------------------------------------------------------------------

def slots_for(sim):
    out = []
    for name in SLOT_RECEPTACLES:
        rec = sim.scene.receptacles[name]
        owner = sim.scene.bodies[rec.owner_body].initial_pose
        for box in rec.boxes:
            if box.kind != "on_top":
                continue
            hx, hy = box.half_extents[:2] - 0.1
            for gx in np.linspace(-hx, hx, 4):
                for gy in np.linspace(-hy, hy, 2):
                    out.append((owner, np.array([gx, gy, box.center[2] - box.half_extents[2]])))
    return out


def settle_seed(sim, seed):
    base = sim.park_state()
    slots = slots_for(sim)
    rng = np.random.default_rng(seed)
    order = rng.permutation(len(slots))
    placements = []
    for k, bid in enumerate(sim.clutter_body_ids):
        owner, local = slots[order[k]]
        lo, _ = geo.parts_aabb(sim.bodies[bid].parts, geo.Pose())
        pos = owner.apply(local) + np.array([0.0, 0.0, -lo[2] + 0.01])
        rot = geo.rot_z(rng.uniform(-math.pi, math.pi))
        placements.append((bid, geo.Pose(rot, pos)))
    _, st = sim.settle(placements, max_time=10.0, base_state=base)
    return st


def gen_pool(seeds=range(8)):
    blobs, tags = [], []
    for v in range(3):
        sim, _ = make_sim(v)
        for s in seeds:
            try:
                st = settle_seed(sim, s)
            except physics.SettleUnstable as exc:
                print(f"  layout {v} seed {s}: {exc}")
                continue
            blobs.append(np.frombuffer(st.to_bytes(), np.uint8))
            tags.append((v, s))
            print(f"  layout {v} seed {s}: settled at step {st.step_index}, hash {st.state_hash()[:16]}")
    np.savez_compressed(os.path.join(OUT, "settled_pool.npz"), meta=meta(), snapshots=np.stack(blobs),
                        tags=np.array(tags, np.int32))
    return blobs, tags


# --------------------------------------------------------------------------
# trajectories with per-substep instrumentation
# --------------------------------------------------------------------------

class Recorder:
    """Wraps one Simulator's broadphase/narrowphase to log per-substep data."""

    def __init__(self, sim):
        self.sim = sim
        self.sub_pairs, self.sub_contacts = [], []
        bp, npf = sim._broadphase_pairs, sim._narrowphase

        def bp_wrap(state):
            pairs = bp(state)
            self.sub_pairs.append(list(pairs))
            return pairs

        def np_wrap(state, pairs):
            out = npf(state, pairs)
            rows = []
            for a, b, cl in out:
                for c in cl:
                    rows.append([a, b, *c.point, *c.normal, c.depth])
            self.sub_contacts.append(rows)
            return out

        sim._broadphase_pairs = bp_wrap
        sim._narrowphase = np_wrap

    def reset(self):
        self.sub_pairs, self.sub_contacts = [], []


def record(sim, st, targets_seq, name, grasp_fn=None):
    """Step `st` through `targets_seq`; teacher-forcing records per step."""
    rec = Recorder(sim)
    cols = {k: [] for k in ("pre", "post", "arm", "base", "has_targets", "counters")}
    pairs, pair_off, contacts, contact_off, events, event_off = [], [0], [], [0], [], [0]
    for t, tg in enumerate(targets_seq):
        if callable(tg):
            tg = tg(sim, st)
        rec.reset()
        c0 = dict(sim.counters)
        pre = st
        st, ev = sim.step_physics(st, tg)
        cols["pre"].append(np.frombuffer(pre.to_bytes(), np.uint8))
        cols["post"].append(np.frombuffer(st.to_bytes(), np.uint8))
        cols["has_targets"].append(tg is not None)
        cols["arm"].append(np.asarray(tg.arm, float) if tg is not None else np.zeros(7))
        cols["base"].append([tg.base.linear_velocity, tg.base.angular_velocity] if tg is not None else [0.0, 0.0])
        cols["counters"].append([sim.counters[k] - c0[k] for k in ("narrowphase_tests", "skipped_sleeping_pairs", "wakes")])
        assert len(rec.sub_pairs) == 4
        for sp, sc in zip(rec.sub_pairs, rec.sub_contacts):
            pairs.extend(sp); pair_off.append(len(pairs))
            contacts.extend(sc); contact_off.append(len(contacts))
        for e in ev:
            events.append([e.bodies[0], e.bodies[1], e.impulse, e.force, *e.point])
        event_off.append(len(events))
    out = {k: np.array(v) for k, v in cols.items()}
    out.update(
        meta=meta(),
        pairs=np.array(pairs, np.int32).reshape(-1, 2), pair_off=np.array(pair_off, np.int64),
        contacts=np.array(contacts, float).reshape(-1, 9), contact_off=np.array(contact_off, np.int64),
        events=np.array(events, float).reshape(-1, 7), event_off=np.array(event_off, np.int64),
        final=np.frombuffer(st.to_bytes(), np.uint8),
    )
    np.savez_compressed(os.path.join(OUT, f"traj_{name}.npz"), **out)
    print(f"  traj_{name}: {len(targets_seq)} steps, {len(pairs)} pairs, {len(contacts)} contacts, {len(events)} events")
    return st


def idle_targets(sim, st, n, seed=3):
    """Random EE deltas through the reference IK + random base velocities."""
    m = sim.robot
    rng = np.random.default_rng(seed)
    seq = []

    def make(d, lin, ang):
        def f(sim, st):
            q = st.joints[sim.arm_slice()]
            tg = rb.apply_arm_action(m, q, rb.ArmAction(d, 0.0), sim.counters)
            tg.base = rb.BaseAction(lin, ang)
            return tg
        return f

    for _ in range(n):
        d = rng.uniform(-0.02, 0.02, 3)
        seq.append(make(d, rng.uniform(-0.5, 1.0), rng.uniform(-1, 1)))
    return seq


def gen_trajectories(pool_blobs, pool_tags):
    first = {v: physics.WorldState.from_bytes(b.tobytes()) for b, (v, s) in reversed(list(zip(pool_blobs, pool_tags)))}

    # idle (the benchmark scenario): living-room centre, random actions
    sim, _ = make_sim(0)
    st = first[0].clone()
    st.base = np.array([2.3, -0.2, 0.0])
    sim._update_robot_link_poses(st, 0.0)
    record(sim, st, idle_targets(sim, st, 20), "idle")

    # zero action, all asleep: the bit-exact fixed point
    sim, _ = make_sim(1)
    st = first[1].clone()
    st.base = np.array([2.3, -0.2, 1.0])
    sim._update_robot_link_poses(st, 0.0)
    q = st.joints[sim.arm_slice()].copy()
    record(sim, st, [rb.JointTargets(arm=q.copy()) for _ in range(3)], "fixed")

    # interact: arm sweeping into the light-table clutter
    sim, _ = make_sim(0)
    st = first[0].clone()
    st.base = np.array([1.6, 0.2, math.pi / 2])
    sim._update_robot_link_poses(st, 0.0)
    m = sim.robot

    def scripted(k):
        def f(sim, st):
            d = np.array([0.015, 0.0, -0.012]) if k < 60 else np.array([0.0, 0.015 if (k // 10) % 2 else -0.015, 0.0])
            return rb.apply_arm_action(m, st.joints[sim.arm_slice()], rb.ArmAction(d, 0.0), sim.counters)
        return f
    record(sim, st, [scripted(k) for k in range(90)], "interact")

    # physics opts off: every dynamic body awake, every pair tested (block LCP heavy)
    sim, _ = make_sim(2, physics.PhysicsConfig(sleeping_enabled=False))
    st = first[2].clone()
    st.base = np.array([2.3, -0.2, 0.0])
    sim._update_robot_link_poses(st, 0.0)
    record(sim, st, [None] * 4, "awake")

    # free drop: a box 1 m above the floor in open space
    sim, _ = make_sim(0)
    st = sim.park_state()
    bid = sim.clutter_body_ids[0]
    st.set_body_pose(bid, geo.Pose(geo.rot_z(0.3), np.array([0.0, 0.0, 1.0])))
    st.asleep[bid] = False
    record(sim, st, [None] * 32, "drop")

    # free drop onto open floor, tilted so it lands on an edge
    sim, _ = make_sim(0)
    st = sim.park_state()
    bid = sim.clutter_body_ids[6]
    st.set_body_pose(bid, geo.Pose(geo.rot_axis_angle(np.array([1.0, 0.4, 0.0]), 0.5), np.array([0.0, -1.5, 0.6])))
    st.asleep[bid] = False
    record(sim, st, [None] * 30, "drop_floor")

    # settle: all 20 clutter bodies spawned 1 cm above their slots, awake (physics.py:1113-1154)
    sim, _ = make_sim(1)
    base = sim.park_state()
    slots = slots_for(sim)
    rng = np.random.default_rng(2)
    order = rng.permutation(len(slots))
    st = base.clone()
    for k, bid in enumerate(sim.clutter_body_ids):
        owner, local = slots[order[k]]
        lo, _ = geo.parts_aabb(sim.bodies[bid].parts, geo.Pose())
        pos = owner.apply(local) + np.array([0.0, 0.0, -lo[2] + 0.01])
        st.set_body_pose(bid, geo.Pose(geo.rot_z(rng.uniform(-math.pi, math.pi)), pos))
        st.asleep[bid] = False
        st.rider_joint[bid] = -1
    record(sim, st, [None] * 6, "settle")

    # tilt: settled clutter tilted 0.2 rad and raised 3 cm, all awake
    sim, _ = make_sim(0)
    st = first[0].clone()
    for bid in sim.clutter_body_ids:
        p = st.body_pose(bid)
        rot = geo.rot_axis_angle(np.array([1.0, 0.0, 0.0]), 0.2) @ p.rot
        st.set_body_pose(bid, geo.Pose(rot, p.pos + np.array([0.0, 0.0, 0.03])))
        st.asleep[bid] = False
    record(sim, st, [None] * 24, "tilt")

    # drawer drag: handle grasp on drawer_2, base backing away (physics.py:623-655)
    sim, _ = make_sim(0)
    st = first[0].clone()
    st.base = np.array([-3.55, -0.45, math.pi])
    sim._update_robot_link_poses(st, 0.0)
    ji = [j.joint_id for j in sim.scene.joints].index("kitchen_cabinet#1:drawer_2")
    st.held_joint = ji
    st.held = sim.scene.joints[ji].body_id
    st.grab_q = float(st.joints[ji])
    st.grab_ee = sim.ee_pose(st).pos.copy()
    q = st.joints[sim.arm_slice()].copy()
    record(sim, st, [rb.JointTargets(arm=q.copy(), base=rb.BaseAction(-0.5, 0.0)) for _ in range(20)], "drawer")

    # fridge door drag (revolute branch of _drag_held_joint)
    sim, _ = make_sim(0)
    st = first[0].clone()
    st.base = np.array([-2.6, 1.7, math.pi / 2])
    sim._update_robot_link_poses(st, 0.0)
    ji = [j.joint_id for j in sim.scene.joints].index("fridge#2:door")
    st.held_joint = ji
    st.held = sim.scene.joints[ji].body_id
    st.grab_q = float(st.joints[ji])
    st.grab_ee = sim.ee_pose(st).pos.copy()
    q = st.joints[sim.arm_slice()].copy()
    record(sim, st, [rb.JointTargets(arm=q.copy(), base=rb.BaseAction(-0.4, 0.3)) for _ in range(15)], "fridge")

    # held object: snap the nearest clutter body and carry it while turning
    sim, _ = make_sim(0)
    st = first[0].clone()
    cands = sorted(sim.grasp_candidates(st), key=lambda c: (c[0], c[1]))
    obj = [c for c in cands if c[2] is None][0][1]
    com = st.body_pose(obj).apply(sim.bodies[obj].com_local)
    st.base = np.array([com[0] - 0.8, com[1], 0.0])
    sim._update_robot_link_poses(st, 0.0)
    sim.apply_grasp(st, rb.GraspTransition("snap", body=obj))
    q = st.joints[sim.arm_slice()].copy()
    q2 = q + np.array([0.2, -0.1, 0.1, 0.2, 0.0, -0.1, 0.3])
    record(sim, st, [rb.JointTargets(arm=q2.copy(), base=rb.BaseAction(-0.3, 0.5)) for _ in range(12)], "held")


# --------------------------------------------------------------------------
# render restatement through the reference ray primitive
# --------------------------------------------------------------------------

W = H = 128
FOV = math.pi / 2
NEAR, FAR = 0.1, 10.0
TIE_EPS = 1e-9


def camera_rays(cam_pose):
    f = (W / 2) / math.tan(FOV / 2)
    u = (np.arange(W) + 0.5 - W / 2) / f
    v = (np.arange(H) + 0.5 - H / 2) / f
    vv, uu = np.meshgrid(v, u, indexing="ij")
    d = np.stack([uu, vv, np.ones_like(uu)], axis=-1).reshape(-1, 3)
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    return np.tile(cam_pose.pos, (len(d), 1)), d @ cam_pose.rot.T


def render_ref(sim, st, cam):
    m = sim.robot
    mount = m.cameras[cam]
    parent = rb.base_pose3(st.base) if mount.parent == "base" else sim.ee_pose(st)
    pose = parent.compose(mount.pose)
    o, d = camera_rays(pose)
    ts = np.stack([geo.parts_ray_hits(sim.bodies[b].parts, st.body_pose(b), o, d) for b in range(sim.n_bodies)])
    tmin = ts.min(axis=0)
    ids = np.full(len(tmin), -1, np.int32)
    finite = np.isfinite(tmin)
    within = ts <= (tmin + TIE_EPS)[None, :]
    ids[finite] = np.argmax(within[:, finite], axis=0)
    return tmin.reshape(H, W), ids.reshape(H, W), pose


def gen_render():
    out = {"meta": meta(), "fov": FOV, "near": NEAR, "far": FAR, "tie_eps": TIE_EPS}
    frames = []
    for name, step in (("idle", 0), ("idle", 19), ("interact", 70), ("drawer", 19), ("held", 11), ("fridge", 14)):
        tr = np.load(os.path.join(OUT, f"traj_{name}.npz"))
        blob = tr["post"][step].tobytes()
        st = physics.WorldState.from_bytes(blob)
        variant = 0
        sim, _ = make_sim(variant)
        for cam in ("head", "arm"):
            t, ids, pose = render_ref(sim, st, cam)
            frames.append(dict(state=np.frombuffer(blob, np.uint8), cam=0 if cam == "head" else 1, t=t, ids=ids,
                               cam_pose=np.concatenate([pose.rot.reshape(9), pose.pos]), layout=variant))
    for k in frames[0]:
        out[k] = np.stack([f[k] for f in frames])
    np.savez_compressed(os.path.join(OUT, "render.npz"), **out)
    print(f"  render: {len(frames)} frames")


def view_state(sim, pool_state, base, arm):
    """A pool state with the robot teleported to ``base`` with arm joints
    ``arm`` (link bodies moved along, ``_update_robot_link_poses``)."""
    st = pool_state.clone()
    st.base = np.asarray(base, float)
    st.joints[sim.arm_slice()] = arm
    sim._update_robot_link_poses(st, 0.0)
    return st


def head_camera_pos(sim, base):
    m = sim.robot
    mount = m.cameras["head"]
    return rb.base_pose3(np.asarray(base, float)).compose(mount.pose).pos


def gen_render_views(n_random=24, n_special=4):
    """Reference frames of all three layouts (VERDICT r1 'widen render
    parity'): per layout ``n_random`` random views (robot at a random
    walkable cell, random heading, random arm joints; head + arm cameras),
    ``n_special`` views with the head camera inside a static convex (every
    ray starts inside: t = 0 pixels) and ``n_special`` with the head camera
    2-8 cm in front of a static body facing it (t < near pixels).  Ids and
    ranges from the reference primitive (``render_ref``)."""
    pool = np.load(os.path.join(OUT, "settled_pool.npz"))
    out = {"meta": meta(), "fov": FOV, "near": NEAR, "far": FAR, "tie_eps": TIE_EPS}
    frames = []
    for v in range(3):
        sim, _ = make_sim(v)
        blobs = [b for b, (lv, _s) in zip(pool["snapshots"], pool["tags"]) if int(lv) == v]
        rng = np.random.default_rng(500 + v)
        g = sim.scene.navgrid
        cells = np.argwhere(g.walkable)
        lo, hi = np.array([j.limits[0] for j in sim.robot.joints]), np.array([j.limits[1] for j in sim.robot.joints])
        statics = [b for b in range(sim.n_bodies) if sim.bodies[b].kind == "static"]

        def pool_state():
            return physics.WorldState.from_bytes(blobs[rng.integers(len(blobs))].tobytes())

        def add(st, kind):
            blob = st.to_bytes()
            for cam in ("head", "arm"):
                if kind != "random" and cam == "arm":
                    continue
                t, ids, pose = render_ref(sim, st, cam)
                frames.append(dict(state=np.frombuffer(blob, np.uint8), cam=0 if cam == "head" else 1, t=t, ids=ids,
                                   cam_pose=np.concatenate([pose.rot.reshape(9), pose.pos]), layout=v,
                                   kind={"random": 0, "inside": 1, "near": 2}[kind]))
            return frames[-1]["t"]

        for _ in range(n_random):
            ci, cj = cells[rng.integers(len(cells))]
            base = [g.origin[0] + (ci + rng.uniform()) * g.cell, g.origin[1] + (cj + rng.uniform()) * g.cell,
                    rng.uniform(-math.pi, math.pi)]
            add(view_state(sim, pool_state(), base, lo + rng.uniform(size=len(lo)) * (hi - lo)), "random")
        # head camera inside a static box part / 2-8 cm in front of one of its side faces,
        # found geometrically (part frame), then confirmed by the frame itself
        boxes = []
        for b in statics:
            for local, prim in sim.bodies[b].parts:
                if isinstance(prim, geo.Box):
                    wp = sim.scene.bodies[b].initial_pose.compose(local)
                    h = np.asarray(prim.half, float)
                    zlo, zhi = geo.prim_aabb(prim, wp)[0][2], geo.prim_aabb(prim, wp)[1][2]
                    if zlo < 1.12 and zhi > 1.32 and abs(wp.rot[2, 2]) > 0.999:  # upright, spans the camera height
                        boxes.append((wp, h))
        found = {"inside": 0, "near": 0}
        tries = 0
        while (found["inside"] < n_special or found["near"] < n_special) and tries < 400 and boxes:
            tries += 1
            wp, h = boxes[rng.integers(len(boxes))]
            kind = "inside" if found["inside"] < n_special else "near"
            if kind == "inside":
                if min(h[0], h[1]) < 0.03:
                    continue
                loc = np.array([rng.uniform(-0.6, 0.6) * h[0], rng.uniform(-0.6, 0.6) * h[1], 0.0])
                yaw = rng.uniform(-math.pi, math.pi)
            else:
                ax, sgn = int(rng.integers(2)), float(rng.choice([-1.0, 1.0]))
                loc = np.zeros(3)
                loc[ax] = sgn * (h[ax] + rng.uniform(0.02, 0.08))
                loc[1 - ax] = rng.uniform(-0.6, 0.6) * h[1 - ax]
                nrm = wp.rot @ np.eye(3)[ax] * -sgn  # face the box
                yaw = math.atan2(nrm[1], nrm[0])
            tgt = wp.apply(loc)
            cam0 = head_camera_pos(sim, [0.0, 0.0, yaw])
            base = [tgt[0] - cam0[0], tgt[1] - cam0[1], yaw]
            cam = head_camera_pos(sim, base)
            cl = wp.inverse().apply(cam)
            inside = (np.abs(cl) < h - 0.005).all()
            if inside != (kind == "inside"):
                continue
            st = view_state(sim, pool_state(), base, sim.robot.resting_joints)
            t = add(st, kind)
            ok = (t == 0.0).any() if kind == "inside" else ((t > 0.0) & (t < NEAR)).any()
            if ok:
                found[kind] += 1
            else:
                frames.pop()
        assert found == {"inside": n_special, "near": n_special}, found
    for k in frames[0]:
        out[k] = np.stack([f[k] for f in frames])
    np.savez_compressed(os.path.join(OUT, "render_views.npz"), **out)
    kinds = out["kind"]
    print(f"  render_views: {len(frames)} frames ({int((kinds == 0).sum())} random, {int((kinds == 1).sum())} "
          f"inside, {int((kinds == 2).sum())} near), t=0 px {int((out['t'] == 0).sum())}, "
          f"t<near px {int(((out['t'] > 0) & (out['t'] < NEAR)).sum())}")


# --------------------------------------------------------------------------
# known-answer tests
# --------------------------------------------------------------------------

def gen_kat():
    out = {"meta": meta()}
    box = geo.Box([0.5, 0.5, 0.5])
    out["ray_box_t"] = geo.prim_ray_hits(box, geo.Pose(), np.array([[-2.0, 0, 0]]), np.array([[1.0, 0, 0]]))
    m = rb.default_model()
    out["fk_zero_ee"] = rb.forward_kinematics(m, np.zeros(7)).pos
    out["fk_rest_ee"] = rb.forward_kinematics(m, m.resting_joints).pos
    out["clamp"] = rb.ArmAction(np.array([0.10, 0, 0]), 0.0).clamped_delta()
    cands = [(0.10, 30, None), (0.16, 22, None)]
    out["grasp_snap"] = rb.grasp_rule(1.0, False, cands).body
    out["grasp_none"] = rb.grasp_rule(1.0, False, [(0.16, 22, None)]).kind == "none"
    out["grasp_tie"] = rb.grasp_rule(1.0, False, [(0.1, 31, None), (0.1, 25, None)]).body
    # nearest-walkable queries (navgrid.py:70-105), incl. blocked and out-of-grid points
    sim, _ = make_sim(0)
    ng = sim.scene.navgrid
    rng = np.random.default_rng(5)
    q = np.concatenate([rng.uniform([-5.2, -3.2], [5.2, 3.2], (400, 2)),
                        np.array([[-4.65, -0.5], [1.6, 1.1], [9.0, 0.0], [0.0, -4.0]])])
    out["nav_query"] = q
    out["nav_walkable"] = np.array([ng.is_walkable(p) for p in q])
    out["nav_nearest"] = np.array([ng.nearest_walkable(p) for p in q])
    # move_base on the grid (robot.py:349-372)
    mb_in = np.concatenate([rng.uniform([-4.5, -2.5, -3.1], [4.5, 2.5, 3.1], (200, 3))])
    mb_act = rng.uniform([-1.0, -2.0], [2.0, 2.0], (200, 2))
    out["mb_in"], out["mb_act"] = mb_in, mb_act
    out["mb_out"] = np.array([rb.move_base(b, ng, rb.BaseAction(a[0], a[1]), 1 / 120) for b, a in zip(mb_in, mb_act)])
    np.savez_compressed(os.path.join(OUT, "kat.npz"), **out)


# --------------------------------------------------------------------------
# IK / arm actions (robot.py:185-313)
# --------------------------------------------------------------------------

def gen_ik():
    m = rb.default_model()
    rng = np.random.default_rng(21)
    lo, hi = m.limits_lo(), m.limits_hi()
    qs, deltas, targets, fails = [], [], [], []
    # (1) the action space: random joint states near rest, 1.5 cm-clamped EE deltas
    for _ in range(150):
        q = np.clip(m.resting_joints + rng.uniform(-0.6, 0.6, 7), lo, hi)
        d = rng.uniform(-0.03, 0.03, 3)
        st = {}
        tg = rb.apply_arm_action(m, q, rb.ArmAction(d, 0.0), st)
        qs.append(q); deltas.append(d); targets.append(tg.arm); fails.append(st.get("ik_failures", 0))
    # (2) hard seeds: joints at limits / random over the box (restarts, Weyl spray, failures)
    for _ in range(50):
        q = rng.uniform(lo, hi)
        d = rng.uniform(-0.015, 0.015, 3)
        st = {}
        tg = rb.apply_arm_action(m, q, rb.ArmAction(d, 0.0), st)
        qs.append(q); deltas.append(d); targets.append(tg.arm); fails.append(st.get("ik_failures", 0))
    # (3) direct solve_ik on far targets (reach failures and restarts)
    sq, st_t, sres, sok = [], [], [], []
    for _ in range(40):
        seed = np.clip(m.resting_joints + rng.uniform(-1, 1, 7), lo, hi)
        tgt = np.array([0.12, 0.0, 0.96]) + rng.uniform(-1.1, 1.1, 3)
        try:
            res, ok = rb.solve_ik(m, tgt, seed), True
        except rb.NoSolution:
            res, ok = seed, False
        sq.append(seed); st_t.append(tgt); sres.append(res); sok.append(ok)
    np.savez_compressed(os.path.join(OUT, "ik.npz"), meta=meta(), q=np.array(qs), delta=np.array(deltas),
                        targets=np.array(targets), fails=np.array(fails), solve_seed=np.array(sq),
                        solve_target=np.array(st_t), solve_q=np.array(sres), solve_ok=np.array(sok))
    print(f"  ik: {len(qs)} actions ({sum(fails)} failures), {len(sq)} solves ({sum(sok)} ok)")


# --------------------------------------------------------------------------
# settle (physics.py:1113-1176) and GJK clearances (geometry.py:486-539)
# --------------------------------------------------------------------------

def spawn_state(sim, base, placements):
    """The state Simulator.settle builds before its clearance check (physics.py:1124-1137)."""
    state = base.clone()
    for bid, pose in placements:
        old = state.body_pose(bid)
        if np.array_equal(old.pos, pose.pos) and np.array_equal(old.quat(), pose.quat()):
            continue
        state.set_body_pose(bid, pose)
        state.asleep[bid] = False
        state.sleep_counter[bid] = 0
        state.rider_joint[bid] = -1
        state.lin_vel[bid] = 0.0
        state.ang_vel[bid] = 0.0
    return state


def gen_settle(seeds=range(8)):
    """Per (layout, seed) of the pool recipe: the spawn snapshot, every
    AABB-overlapping (placed, other) parts_distance, and the settle outcome
    (0 settled + final snapshot + steps, 1 clearance (body, other, d),
    2 fell, 3 timeout)."""
    spawns, outcome, info, value, steps, finals, tags = [], [], [], [], [], [], []
    pd_tag, pd_pair, pd_dist = [], [], []
    for v in range(3):
        sim, _ = make_sim(v)
        for sd in seeds:
            base = sim.park_state()
            slots = slots_for(sim)
            rng = np.random.default_rng(sd)
            order = rng.permutation(len(slots))
            placements = []
            for k, bid in enumerate(sim.clutter_body_ids):
                owner, local = slots[order[k]]
                lo, _ = geo.parts_aabb(sim.bodies[bid].parts, geo.Pose())
                pos = owner.apply(local) + np.array([0.0, 0.0, -lo[2] + 0.01])
                placements.append((bid, geo.Pose(geo.rot_z(rng.uniform(-math.pi, math.pi)), pos)))
            sp = spawn_state(sim, base, placements)
            spawns.append(np.frombuffer(sp.to_bytes(), np.uint8))
            tags.append((v, sd))
            for bid, _ in placements:
                lo_a, hi_a = geo.parts_aabb(sim.bodies[bid].parts, sp.body_pose(bid))
                for o in range(sim.n_bodies):
                    if o == bid or o in sim._robot_set or sp.pos[o][2] > sim.PARK_Z / 2:
                        continue
                    lo_b, hi_b = sim.body_aabb(sp, o)
                    if geo.aabb_overlap(lo_a, hi_a, lo_b, hi_b, margin=1e-3):
                        pd_tag.append(len(spawns) - 1); pd_pair.append((bid, o))
                        pd_dist.append(geo.parts_distance(sim.bodies[bid].parts, sp.body_pose(bid),
                                                          sim.bodies[o].parts, sp.body_pose(o)))
            try:
                _, st = sim.settle(placements, max_time=10.0, base_state=base)
                outcome.append(0); info.append((-1, -1)); value.append(0.0)
                steps.append(st.step_index - base.step_index)
                finals.append(np.frombuffer(st.to_bytes(), np.uint8))
            except physics.SettleUnstable as exc:
                msg = str(exc)
                kind = 1 if "clearance" in msg else (2 if "fell" in msg else 3)
                ids = [int(t) for t in msg.replace("(", " ").replace(")", " ").replace(":", " ").replace(",", " ")
                       .replace("[", " ").replace("]", " ").split() if t.isdigit()]
                outcome.append(kind); steps.append(-1); finals.append(np.zeros_like(spawns[-1]))
                if kind == 1:
                    d_mm = float(msg.split(" has ")[1].split(" mm")[0])
                    info.append((ids[0], ids[1])); value.append(d_mm * 1e-3)
                else:
                    info.append((ids[0] if ids else -1, -1)); value.append(0.0)
            print(f"  settle layout {v} seed {sd}: outcome {outcome[-1]} steps {steps[-1]} info {info[-1]}")
    np.savez_compressed(os.path.join(OUT, "settle.npz"), meta=meta(), tags=np.array(tags, np.int32),
                        spawn=np.stack(spawns), outcome=np.array(outcome), info=np.array(info, np.int32),
                        value=np.array(value), steps=np.array(steps), final=np.stack(finals),
                        pd_tag=np.array(pd_tag), pd_pair=np.array(pd_pair, np.int32), pd_dist=np.array(pd_dist))


# --------------------------------------------------------------------------
# point queries (physics.py:1088-1101 sphere_cast)
# --------------------------------------------------------------------------

def gen_cast():
    """Simulator.sphere_cast from random origins / unit directions on settled
    states of the three layouts (nearest proxy hit, lowest id on ties)."""
    rng = np.random.default_rng(17)
    pool = np.load(os.path.join(OUT, "settled_pool.npz"))
    out = {k: [] for k in ("state", "layout", "origin", "dir", "max_dist", "body", "t")}
    for v in range(3):
        sim, _ = make_sim(v)
        blobs = [b for b, (lv, _s) in zip(pool["snapshots"], pool["tags"]) if lv == v][:2]
        for blob in blobs:
            st = physics.WorldState.from_bytes(blob.tobytes())
            for k in range(60):
                o = rng.uniform([-4.5, -2.5, 0.1], [4.5, 2.5, 2.2])
                d = rng.normal(size=3)
                d /= np.linalg.norm(d)
                md = [2.0, 10.0, np.inf][k % 3]
                hit = sim.sphere_cast(st, o, d, md)
                out["state"].append(np.frombuffer(blob.tobytes(), np.uint8)); out["layout"].append(v)
                out["origin"].append(o); out["dir"].append(d); out["max_dist"].append(md)
                out["body"].append(-1 if hit is None else hit[0]); out["t"].append(np.inf if hit is None else hit[1])
    np.savez_compressed(os.path.join(OUT, "cast.npz"), meta=meta(), **{k: np.array(v) for k, v in out.items()})
    print(f"  cast: {len(out['t'])} rays, {int(np.sum(np.array(out['body']) >= 0))} hits")


# --------------------------------------------------------------------------
# geodesics (navgrid.py:109-172)
# --------------------------------------------------------------------------

def gen_nav():
    """Distance fields (Dijkstra), geodesic distances and steepest-descent
    shortest paths of the reference NavGrid, layouts 0-2."""
    rng = np.random.default_rng(11)
    goals, fields, layouts = [], [], []
    q_layout, q_from, q_goal, q_dist, paths, path_len = [], [], [], [], [], []
    for v in range(3):
        sim, _ = make_sim(v)
        ng = sim.scene.navgrid
        cells = np.argwhere(ng.walkable)
        # walkable centres, random walkable points, a blocked point, an out-of-grid point
        gs = [ng.center_of(tuple(cells[rng.integers(len(cells))])) for _ in range(2)]
        gs.append(ng.origin + (cells[rng.integers(len(cells))] + rng.uniform(0.05, 0.95, 2)) * ng.cell)
        gs.append(np.array([1.6, 1.1]) if v == 0 else np.array([9.0, 0.5]))
        for g in gs:
            goals.append(np.asarray(g, float)); layouts.append(v)
            fields.append(ng.distance_field(g).copy())
        for k in range(40):
            g = gs[k % len(gs)]
            f = ng.origin + rng.uniform(0, 1, 2) * np.array([ng.nx, ng.ny]) * ng.cell
            q_layout.append(v); q_from.append(f); q_goal.append(np.asarray(g, float))
            q_dist.append(ng.geodesic_distance(f, g))
            pth = ng.shortest_path(f, g)
            path_len.append(len(pth))
            pad = np.full((400, 2), np.nan)
            if pth:
                pad[:len(pth)] = np.array(pth)[:400]
            paths.append(pad)
    np.savez_compressed(os.path.join(OUT, "nav.npz"), meta=meta(), goal=np.array(goals), layout=np.array(layouts),
                        field=np.array(fields), q_layout=np.array(q_layout), q_from=np.array(q_from),
                        q_goal=np.array(q_goal), q_dist=np.array(q_dist), path=np.array(paths),
                        path_len=np.array(path_len))
    print(f"  nav: {len(fields)} fields, {len(q_dist)} queries, max path {max(path_len)}")


# --------------------------------------------------------------------------
# env-step records with grasp transitions (riders, pick & place)
# --------------------------------------------------------------------------

GRASP_KIND = {"none": 0, "snap": 1, "release": 2}


def grasp_step(sim, st, gripper):
    """The restated env pipeline's grasp phase (robot.py:323-346,
    physics.py:1039-1084): holding = ``state.held >= 0`` (object or handle).
    Returns (kind, body, joint index, wakes counted)."""
    w0 = sim.counters["wakes"]
    tr = rb.grasp_rule(float(gripper), st.held >= 0, sim.grasp_candidates(st))
    sim.apply_grasp(st, tr)
    ji = -1
    if tr.joint is not None:
        ji = sim.scene.joints.index(sim.scene.joint_by_id(tr.joint))
    return GRASP_KIND[tr.kind], -1 if tr.body is None else int(tr.body), ji, sim.counters["wakes"] - w0


def record_env(sim, st, items, name):
    """Step records with an optional grasp after each physics step.

    ``items``: callables ``f(sim, st) -> dict`` returning ``action`` (dEE xyz,
    gripper, base lin, base ang: IK -> physics -> grasp, the device env step)
    or ``targets`` (JointTargets or None) + ``gripper`` (None = no grasp); an
    optional ``mutate(sim, st)`` edits the state before the step (teleports).
    Per step: ``pre``, targets, ``post`` (after the physics step, the
    teacher-forcing record of ``record``), ``gripper`` (nan = none),
    ``grasped`` (after the grasp), ``trans`` (kind, body, joint index, wakes)
    and ``action`` (nan row when the step was not action-driven)."""
    rec = Recorder(sim)
    cols = {k: [] for k in ("pre", "post", "arm", "base", "has_targets", "counters", "gripper", "grasped",
                            "trans", "action")}
    pairs, pair_off, contacts, contact_off, events, event_off = [], [0], [], [0], [], [0]
    m = sim.robot
    for t, item in enumerate(items):
        spec = item(sim, st)
        if "mutate" in spec:
            spec["mutate"](sim, st)
        action = np.full(6, np.nan)
        if "action" in spec:
            action = np.asarray(spec["action"], float)
            stats = {}
            tg = rb.apply_arm_action(m, st.joints[sim.arm_slice()], rb.ArmAction(action[:3], action[3]), stats)
            tg.base = rb.BaseAction(action[4], action[5])
            gripper = action[3]
        else:
            tg, gripper = spec.get("targets"), spec.get("gripper")
        rec.reset()
        c0 = dict(sim.counters)
        pre = st
        st, ev = sim.step_physics(st, tg)
        cols["pre"].append(np.frombuffer(pre.to_bytes(), np.uint8))
        cols["post"].append(np.frombuffer(st.to_bytes(), np.uint8))
        cols["has_targets"].append(tg is not None)
        cols["arm"].append(np.asarray(tg.arm, float) if tg is not None else np.zeros(7))
        cols["base"].append([tg.base.linear_velocity, tg.base.angular_velocity] if tg is not None else [0.0, 0.0])
        cols["counters"].append([sim.counters[k] - c0[k] for k in ("narrowphase_tests", "skipped_sleeping_pairs", "wakes")])
        cols["action"].append(action)
        st = st.clone()
        if gripper is None:
            cols["gripper"].append(np.nan)
            cols["trans"].append([0, -1, -1, 0])
        else:
            cols["gripper"].append(float(gripper))
            cols["trans"].append(list(grasp_step(sim, st, gripper)))
        cols["grasped"].append(np.frombuffer(st.to_bytes(), np.uint8))
        assert len(rec.sub_pairs) == 4
        for sp, sc in zip(rec.sub_pairs, rec.sub_contacts):
            pairs.extend(sp); pair_off.append(len(pairs))
            contacts.extend(sc); contact_off.append(len(contacts))
        for e in ev:
            events.append([e.bodies[0], e.bodies[1], e.impulse, e.force, *e.point])
        event_off.append(len(events))
    out = {k: np.array(v) for k, v in cols.items()}
    out.update(
        meta=meta(),
        pairs=np.array(pairs, np.int32).reshape(-1, 2), pair_off=np.array(pair_off, np.int64),
        contacts=np.array(contacts, float).reshape(-1, 9), contact_off=np.array(contact_off, np.int64),
        events=np.array(events, float).reshape(-1, 7), event_off=np.array(event_off, np.int64),
        final=np.frombuffer(st.to_bytes(), np.uint8),
    )
    np.savez_compressed(os.path.join(OUT, f"traj_{name}.npz"), **out)
    tr = out["trans"]
    print(f"  traj_{name}: {len(items)} steps, {len(pairs)} pairs, {len(contacts)} contacts, {len(events)} events, "
          f"snaps {int((tr[:, 0] == 1).sum())} releases {int((tr[:, 0] == 2).sum())}")
    return st


def reach_joints(sim, base, target_world, seed=None):
    """Arm joints putting the EE at ``target_world`` from ``base`` (reference IK)."""
    m = sim.robot
    local = rb.base_pose3(np.asarray(base, float)).inverse().apply(np.asarray(target_world, float))
    return rb.solve_ik(m, local, m.resting_joints if seed is None else seed)


def ee_toward(sim, st, target_world, step=0.015):
    """dEE (robot base frame) moving the EE toward a world point, clamped."""
    ee = sim.ee_pose(st).pos
    d = rb.base_pose3(st.base).rot.T @ (np.asarray(target_world, float) - ee)
    n = float(np.linalg.norm(d))
    return d if n <= step else d * (step / n)


def rider_state(sim, pool_state, base, arm, drawers=((2, 0, (-0.18, 0.05)), (2, 2, (0.17, -0.06)),
                                                       (1, 4, (0.0, 0.0)), (0, 3, (0.1, 0.02)))):
    """``make_initial_state(..., clutter_asleep=True)`` (physics.py:344-380) with
    clutter resting inside the kitchen-cabinet drawer trays -> ``_bind_riders``
    (physics.py:383-405) binds them to their drawer joints.  ``drawers`` =
    (drawer index, clutter index, tray-local xy); the other clutter keeps its
    settled pool pose."""
    poses = [pool_state.body_pose(b) for b in sim.clutter_body_ids]
    for di, ci, (x, y) in drawers:
        sj = sim.scene.joint_by_id(f"kitchen_cabinet#1:drawer_{di}")
        tray = sim.scene.bodies[sj.body_id].initial_pose
        bid = sim.clutter_body_ids[ci]
        rot = tray.rot @ geo.rot_z(0.3 + 0.7 * ci)
        lo, _ = geo.parts_aabb(sim.bodies[bid].parts, geo.Pose(rot, np.zeros(3)))
        p = tray.apply(np.array([x, y, 0.02])) + np.array([0.0, 0.0, -lo[2] + 1e-3])
        poses[ci] = geo.Pose(rot, p)
    st = sim.make_initial_state(poses, base=np.asarray(base, float), arm_joints=arm, clutter_asleep=True)
    return st


def gen_env_records(pool_blobs, pool_tags):
    first = {v: physics.WorldState.from_bytes(b.tobytes()) for b, (v, s) in reversed(list(zip(pool_blobs, pool_tags)))}

    # ---- riders: drawer clutter bound by make_initial_state, drawer pulled
    # open through a handle snap, released mid-motion (the drawer coasts,
    # riders follow), then the arm reaches into the tray and wakes a rider.
    sim, _ = make_sim(0)
    sj = sim.scene.joint_by_id("kitchen_cabinet#1:drawer_2")
    ji = sim.scene.joints.index(sj)
    handle = sj.handle_world(sim.scene.bodies[sj.parent_body].initial_pose, 0.0)
    base = np.array([handle[0] + 0.75, handle[1], math.pi])
    arm = reach_joints(sim, base, handle + np.array([0.02, 0.0, 0.0]))
    st = rider_state(sim, first[0], base, arm)
    assert sum(int(r) >= 0 for r in st.rider_joint) == 4, st.rider_joint
    q0 = arm.copy()
    items = [lambda sim, st: {"targets": rb.JointTargets(arm=q0.copy()), "gripper": 1.0}]
    items += [lambda sim, st: {"targets": rb.JointTargets(arm=q0.copy(), base=rb.BaseAction(-0.5, 0.0)),
                               "gripper": 0.0}] * 22
    items += [lambda sim, st: {"targets": rb.JointTargets(arm=q0.copy(), base=rb.BaseAction(-0.5, 0.0)),
                               "gripper": -1.0}]
    items += [lambda sim, st: {"targets": rb.JointTargets(arm=q0.copy())}] * 3
    rider = sim.clutter_body_ids[2]

    def reach_rider(sim, st):
        # approach from above, then descend onto the rider; walk in while far
        com = st.body_pose(rider).apply(sim.bodies[rider].com_local)
        ee = sim.ee_pose(st).pos
        above = com + np.array([0.0, 0.0, 0.15])
        tgt = above if np.linalg.norm((ee - above)[:2]) > 0.03 and ee[2] > com[2] + 0.1 else com + np.array([0.0, 0.0, 0.03])
        lin = 0.3 if np.linalg.norm(st.base[:2] - com[:2]) > 0.6 else 0.0
        return {"action": [*ee_toward(sim, st, tgt), 0.0, lin, 0.0]}
    items += [reach_rider] * 40
    items += [lambda sim, st: {"action": [0.0, 0.0, 0.0, 1.0, 0.0, 0.0]}]        # snap whatever is nearest
    items += [lambda sim, st: {"action": [0.0, 0.0, 0.015, 0.0, 0.0, 0.0]}] * 6  # lift
    items += [lambda sim, st: {"action": [0.0, 0.0, -0.01, -1.0, 0.0, 0.0]}]     # release (wake) while moving
    items += [lambda sim, st: {"action": [0.0, 0.0, 0.0, 0.0, 0.0, 0.0]}] * 8
    st = record_env(sim, st, items, "riders")

    # ---- pick & place: Interact spawn facing the light table, reach the
    # nearest clutter COM, snap, lift and turn, release (falls, wakes others)
    sim, _ = make_sim(0)
    st = first[0].clone()
    st.base = np.array([1.75, 0.44, math.pi / 2])  # walkable, the table clutter within reach
    sim._update_robot_link_poses(st, 0.0)
    ee = sim.ee_pose(st).pos
    coms = {b: st.body_pose(b).apply(sim.bodies[b].com_local) for b in sim.clutter_body_ids}
    obj = min(coms, key=lambda b: (float(np.linalg.norm(coms[b] - ee)), b))

    def reach_obj(sim, st):
        com = st.body_pose(obj).apply(sim.bodies[obj].com_local)
        return {"action": [*ee_toward(sim, st, com + np.array([0.0, 0.0, 0.04])), 0.0, 0.0, 0.0]}
    items = [reach_obj] * 40
    items += [lambda sim, st: {"action": [0.0, 0.0, 0.0, 1.0, 0.0, 0.0]}]
    items += [lambda sim, st: {"action": [0.0, 0.0, 0.015, 0.5, 0.0, 0.4]}] * 8   # hold (scalar > 0 ignored)
    items += [lambda sim, st: {"action": [0.01, 0.0, 0.0, 0.0, -0.2, 0.0]}] * 4
    items += [lambda sim, st: {"action": [0.0, 0.0, -0.01, -1.0, 0.0, 0.0]}]
    items += [lambda sim, st: {"action": [0.0, 0.0, 0.0, 0.0, 0.0, 0.0]}] * 12
    record_env(sim, st, items, "pick")


def gen_grasp():
    """``grasp_rule`` + ``apply_grasp`` transitions on single states
    (robot.py:323-346, physics.py:1039-1084): clutter snaps, the 0.15 m
    boundary, exact ties (same asset, same pose: lowest id), drawer-handle and
    fridge-door snaps, sleeping riders (wake clears the binding), releases of
    objects (wake) and handles (no wake), no-ops while holding / empty."""
    cases = {k: [] for k in ("layout", "pre", "gripper", "post", "trans")}
    rng = np.random.default_rng(29)
    pool = np.load(os.path.join(OUT, "settled_pool.npz"))

    def add(v, sim, st, g):
        pre = np.frombuffer(st.to_bytes(), np.uint8)
        s2 = st.clone()
        tr = grasp_step(sim, s2, g)
        cases["layout"].append(v); cases["pre"].append(pre); cases["gripper"].append(float(g))
        cases["post"].append(np.frombuffer(s2.to_bytes(), np.uint8)); cases["trans"].append(list(tr))
        return s2

    def place_com(sim, st, b, com):
        p = st.body_pose(b)
        st.pos[b] = com - p.rot @ sim.bodies[b].com_local

    for v in range(3):
        sim, _ = make_sim(v)
        blobs = [b for b, t in zip(pool["snapshots"], pool["tags"]) if t[0] == v][:3]
        for blob in blobs:
            st0 = physics.WorldState.from_bytes(blob.tobytes())
            for k in range(14):
                st = st0.clone()
                st.base = np.array([rng.uniform(-2, 2), rng.uniform(-1.5, 1.5), rng.uniform(-3, 3)])
                st.joints[sim.arm_slice()] = rng.uniform(sim.robot.limits_lo(), sim.robot.limits_hi())
                sim._update_robot_link_poses(st, 0.0)
                ee = sim.ee_pose(st).pos
                b = sim.clutter_body_ids[rng.integers(len(sim.clutter_body_ids))]
                d = rng.normal(size=3)
                r = [0.149, 0.151, rng.uniform(0.02, 0.2)][k % 3]
                place_com(sim, st, b, ee + d / np.linalg.norm(d) * r)
                if k % 5 == 2:  # an awake, moving body: snap zeroes its velocity, no wake counted
                    st.asleep[b] = False
                    st.sleep_counter[b] = 3
                    st.lin_vel[b] = rng.normal(size=3) * 0.1
                    st.ang_vel[b] = rng.normal(size=3)
                if k % 7 == 5:  # a second body of the same asset at the identical pose: tie -> lowest id
                    twin = b + 9 if b + 9 in sim.clutter_body_ids else b - 9
                    st.pos[twin], st.quat[twin] = st.pos[b].copy(), st.quat[b].copy()
                    st.asleep[twin] = True
                s2 = add(v, sim, st, 1.0)
                if k % 4 == 0:
                    add(v, sim, st, 0.0)
                    add(v, sim, st, -1.0)  # not holding: no-op
                if s2.held >= 0:
                    add(v, sim, s2, 1.0)   # holding: no-op
                    s3 = s2.clone()
                    s3.asleep[s2.held] = True  # release wakes even a sleeping held body
                    s3.sleep_counter[s2.held] = 7
                    add(v, sim, s3, -1.0)
        # handle snaps: every scene joint, EE placed on / near the handle by the reference IK
        for sj in sim.scene.joints:
            ji = sim.scene.joints.index(sj)
            st = physics.WorldState.from_bytes(blobs[0].tobytes())
            q = float(rng.uniform(*sj.joint.limits)) * 0.5
            st.joints[ji] = q
            sim._update_scene_joint_poses(st, [ji], 0.0)
            h = sj.handle_world(st.body_pose(sj.parent_body), q)
            yaw = math.atan2(h[1] - 0.0, h[0] - 0.0)
            for dist, off in ((0.75, 0.03), (0.8, 0.12), (0.7, 0.2)):
                base = np.array([h[0] - dist * math.cos(yaw), h[1] - dist * math.sin(yaw), yaw])
                try:
                    arm = reach_joints(sim, base, h + np.array([0.0, 0.0, off]))
                except rb.NoSolution:
                    continue
                st.base = base
                st.joints[sim.arm_slice()] = arm
                sim._update_robot_link_poses(st, 0.0)
                s2 = add(v, sim, st, 1.0)
                if s2.held_joint >= 0:
                    add(v, sim, s2, -1.0)  # handle release: no wake
    # sleeping riders snapped (wake clears rider_joint) -- layout 0 drawers
    sim, _ = make_sim(0)
    st0 = physics.WorldState.from_bytes([b for b, t in zip(pool["snapshots"], pool["tags"]) if t[0] == 0][0].tobytes())
    for ci in (0, 2, 4, 3):
        st = rider_state(sim, st0, np.zeros(3), None)
        bid = sim.clutter_body_ids[ci]
        com = st.body_pose(bid).apply(sim.bodies[bid].com_local)
        base = np.array([com[0] + 0.75, com[1], math.pi])
        st.base = base
        st.joints[sim.arm_slice()] = reach_joints(sim, base, com + np.array([0.0, 0.0, 0.06]))
        sim._update_robot_link_poses(st, 0.0)
        add(0, sim, st, 1.0)
    out = {k: np.array(v) for k, v in cases.items()}
    np.savez_compressed(os.path.join(OUT, "grasp.npz"), meta=meta(), **out)
    kinds = out["trans"][:, 0]
    print(f"  grasp: {len(kinds)} cases: none {int((kinds == 0).sum())} snap {int((kinds == 1).sum())} "
          f"(handles {int((out['trans'][:, 2] >= 0).sum())}) release {int((kinds == 2).sum())} "
          f"wakes {int(out['trans'][:, 3].sum())}")


# --------------------------------------------------------------------------
# capacity: a 26-object awake pile (contacts / pairs / groups well above the
# 20-object scenes) and a 40-object world (62 bodies)
# --------------------------------------------------------------------------

def pile_state(sim, seed=4, table="light_table"):
    """Every clutter body awake in a 3 x 3 x k lattice above a table, random
    yaw (free fall onto each other: the pile forms within ~0.5 s)."""
    st = sim.park_state()
    rec = sim.scene.receptacles[table]
    owner = sim.scene.bodies[rec.owner_body].initial_pose
    top = rec.boxes[0].center[2] - rec.boxes[0].half_extents[2]
    rng = np.random.default_rng(seed)
    for k, bid in enumerate(sim.clutter_body_ids):
        layer, cell = divmod(k, 9)
        gx, gy = (cell % 3 - 1) * 0.24, (cell // 3 - 1) * 0.2
        rot = geo.rot_z(rng.uniform(-math.pi, math.pi))
        lo, _ = geo.parts_aabb(sim.bodies[bid].parts, geo.Pose(rot, np.zeros(3)))
        pos = owner.apply(np.array([gx, gy, top])) + np.array([0.0, 0.0, -lo[2] + 0.04 + 0.16 * layer])
        st.set_body_pose(bid, geo.Pose(rot, pos))
        st.asleep[bid] = False
        st.sleep_counter[bid] = 0
        st.rider_joint[bid] = -1
    return st


def gen_capacity():
    sim, _ = make_sim(0, n_clutter=26)
    st = pile_state(sim)
    st.base = np.array([2.3, -0.2, 0.0])
    sim._update_robot_link_poses(st, 0.0)
    record(sim, st, [None] * 36, "pile26")
    sim, _ = make_sim(2, n_clutter=40)
    pool = np.load(os.path.join(OUT, "settled_pool.npz"))
    ref = physics.WorldState.from_bytes([b for b, t in zip(pool["snapshots"], pool["tags"]) if t[0] == 2][0].tobytes())
    st = sim.park_state()
    for k in range(20):  # the settled 20-object state, the other 20 in a falling pile on the light table
        b = sim.clutter_body_ids[k]
        st.set_body_pose(b, ref.body_pose(22 + k))
        st.asleep[b] = True
    pile = pile_state(sim, seed=6)
    for b in sim.clutter_body_ids[20:]:
        k = b - sim.clutter_body_ids[20]
        p = pile.body_pose(sim.clutter_body_ids[k])
        st.set_body_pose(b, p)
        st.asleep[b] = False
    st.base = np.array([2.3, -0.2, 0.0])
    sim._update_robot_link_poses(st, 0.0)
    record(sim, st, idle_targets(sim, st, 24, seed=8), "world62")


# --------------------------------------------------------------------------
# a non-builtin scene through the reference-side adapter (integration/)
# --------------------------------------------------------------------------

CUSTOM_CLUTTER = ["mug", "cracker_box", "sugar_box", "tomato_soup_can", "chef_can", "mug", "apple", "bowl",
                  "cracker_box", "sponge", "orange", "tomato_soup_can"]


def custom_sim():
    """apt_0 with the light table moved and turned, a second kitchen cabinet
    (3 more prismatic drawers) added, and a different clutter set (tall items,
    mugs): 38 bodies, 7 scene joints -- not a builtin layout."""
    j = builtin.layout_json(0)
    j["layout_id"] = "apt_custom"
    fur = [dict(f) for f in j["furniture"]]
    for f in fur:
        if f["ref"] == "light_table":
            f["pos"], f["yaw"] = [0.3, -0.8, 0.0], 0.3
    fur.append({"ref": "kitchen_cabinet", "kind": "articulation", "pos": [0.3, 2.45, 0.0], "yaw": 0.0})
    j["furniture"] = fur
    cache = builtin.default_cache()
    sh = scene.load_scene(scene.layout_from_json(j), cache)
    clutter = [(cache.get_asset(n), f"{n}#{i}") for i, n in enumerate(CUSTOM_CLUTTER)]
    return physics.Simulator(sh, rb.default_model(), clutter, physics.PhysicsConfig())


def gen_custom():
    """traj_custom.npz: teacher-forcing records on ``custom_sim()`` plus the
    adapter's ``rs_scene_desc`` tables (``scene_*`` keys) -- the GPU replays it
    without the reference (tests/test_gpu_integration.py)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from integration.rearrange_sim_b200 import save_tables, scene_tables

    sim = custom_sim()
    rng = np.random.default_rng(21)
    tab = [sj for sj in sim.scene.bodies if sj.name.startswith("light_table")][0]
    top = tab.initial_pose
    poses = []
    for i, bid in enumerate(sim.clutter_body_ids):
        lo, _ = geo.parts_aabb(sim.bodies[bid].parts, geo.Pose())
        # tilted 3-8 degrees: a face landing flat on a plane is a symmetric, rank-deficient
        # impact whose lateral outcome is rounding noise in the reference itself
        ax = rng.normal(size=3)
        ax[2] = 0.0
        rot = geo.rot_z(rng.uniform(-math.pi, math.pi)) @ geo.rot_axis_angle(ax / np.linalg.norm(ax), math.radians(rng.uniform(3, 8)))
        if i < 8:  # dropped onto the moved light table, 4 x 2 grid
            x, y = (-0.39 + 0.26 * (i % 4)), (-0.18 + 0.36 * (i // 4))
            p = top.apply(np.array([x, y, 0.87 + 0.13])) + np.array([0.0, 0.0, -lo[2] + 0.02])
        else:  # onto the dark table (resting on the backdrop floor is chaotic in the reference
            # itself: its state moves 2e-5 m in 3 steps between two BLAS kernels)
            dk = [sj for sj in sim.scene.bodies if sj.name.startswith("dark_table")][0].initial_pose
            p = dk.apply(np.array([-0.2 + 0.4 * ((i - 8) % 2), -0.2 + 0.4 * ((i - 8) // 2), 0.96])) + \
                np.array([0.0, 0.0, -lo[2] + 0.02])
        poses.append(geo.Pose(rot, p))
    st = sim.make_initial_state(poses, base=np.array([1.0, -0.9, math.pi]), clutter_asleep=False)
    seq = idle_targets(sim, st, 30, seed=12)
    out = {}
    save_tables(scene_tables(sim), out)
    record(sim, st, seq, "custom")
    path = os.path.join(OUT, "traj_custom.npz")
    g = dict(np.load(path))
    g.update(out)
    np.savez_compressed(path, **g)
    # the reference's own per-step sensitivity: the same teacher-forced steps under
    # two other OpenBLAS kernels (a tall can rocking on its 12-gon face is chaotic:
    # rounding-level differences reach 1e-4 m in one control step); the GPU / oracle
    # tests accept per-step deviations within this spread
    spreads = []
    for ct in ("SkylakeX", "Prescott"):
        tmp = os.path.join(OUT, f".spread_{ct}.npy")
        env = dict(os.environ, OPENBLAS_CORETYPE=ct, OPENBLAS_NUM_THREADS="1")
        import subprocess
        subprocess.run([sys.executable, os.path.abspath(__file__), "--spread", path, tmp], env=env, check=True)
        spreads.append(np.load(tmp))
        os.remove(tmp)
    g["ref_spread"] = np.maximum(*spreads)  # [steps, 3]: max |d pos|, |d quat|, |d vel| vs this file's post
    np.savez_compressed(path, **g)
    print(f"  traj_custom: reference cross-BLAS spread per step: pos <= {g['ref_spread'][:, 0].max():.1e}, "
          f"quat <= {g['ref_spread'][:, 1].max():.1e}, vel <= {g['ref_spread'][:, 2].max():.1e}")


def spread_main(src, dst):
    """``--spread``: teacher-forced steps of ``src`` under this process's BLAS kernel."""
    g = np.load(src)
    sim = custom_sim()
    res = []
    for s in range(len(g["pre"])):
        st = physics.WorldState.from_bytes(g["pre"][s].tobytes())
        tg = rb.JointTargets(arm=g["arm"][s].copy(), base=rb.BaseAction(*g["base"][s])) if g["has_targets"][s] else None
        st2, _ = sim.step_physics(st, tg)
        ref = physics.WorldState.from_bytes(g["post"][s].tobytes())
        res.append([np.abs(st2.pos - ref.pos).max(), np.abs(st2.quat - ref.quat).max(),
                    max(np.abs(st2.lin_vel - ref.lin_vel).max(), np.abs(st2.ang_vel - ref.ang_vel).max())])
    np.save(dst, np.array(res))


def gen_empty():
    """traj_empty.npz: a scene without clutter (``Simulator(..., clutter=[])``,
    22 bodies): the robot drives up to the kitchen cabinet of apt_1 and pushes
    its arm into the drawer fronts (robot vs kinematic jointed bodies only)."""
    sim, _ = make_sim(1, n_clutter=0)
    st = sim.make_initial_state([], base=np.array([-3.75, -0.5, math.pi]), clutter_asleep=False)
    m = sim.robot

    def push(k):
        def f(sim, st):
            d = np.array([0.015, 0.0, -0.01 if k < 10 else 0.0])
            tg = rb.apply_arm_action(m, st.joints[sim.arm_slice()], rb.ArmAction(d, 0.0), sim.counters)
            tg.base = rb.BaseAction(0.25 if k < 16 else 0.0, 0.0)
            return tg
        return f
    record(sim, st, [push(k) for k in range(28)], "empty")


if __name__ == "__main__":
    if sys.argv[1:2] == ["--spread"]:
        spread_main(sys.argv[2], sys.argv[3])
        sys.exit(0)
    t0 = time.time()
    what = sys.argv[1:] or ["tables", "pool", "traj", "render", "views", "kat", "ik", "nav", "settle", "cast", "env", "grasp",
                            "capacity", "custom", "empty"]
    if "tables" in what:
        gen_tables(); print("tables", time.time() - t0)
    blobs = tags = None
    if "pool" in what:
        blobs, tags = gen_pool(); print("pool", time.time() - t0)
    if "traj" in what:
        if blobs is None:
            p = np.load(os.path.join(OUT, "settled_pool.npz"))
            blobs, tags = list(p["snapshots"]), [tuple(t) for t in p["tags"]]
        gen_trajectories(blobs, tags); print("traj", time.time() - t0)
    if "render" in what:
        gen_render(); print("render", time.time() - t0)
    if "views" in what:
        gen_render_views(); print("views", time.time() - t0)
    if "kat" in what:
        gen_kat(); print("kat", time.time() - t0)
    if "ik" in what:
        gen_ik(); print("ik", time.time() - t0)
    if "nav" in what:
        gen_nav(); print("nav", time.time() - t0)
    if "settle" in what:
        gen_settle(); print("settle", time.time() - t0)
    if "cast" in what:
        gen_cast(); print("cast", time.time() - t0)
    if "env" in what:
        p = np.load(os.path.join(OUT, "settled_pool.npz"))
        gen_env_records(list(p["snapshots"]), [tuple(t) for t in p["tags"]]); print("env", time.time() - t0)
    if "grasp" in what:
        gen_grasp(); print("grasp", time.time() - t0)
    if "capacity" in what:
        gen_capacity(); print("capacity", time.time() - t0)
    if "custom" in what:
        gen_custom(); print("custom", time.time() - t0)
    if "empty" in what:
        gen_empty(); print("empty", time.time() - t0)
