"""``BatchSimulator``: the reference ``physics.Simulator`` API with a leading
env dimension, executed by the CUDA library through the C-ABI.

Reference surface (physics.py:252-1101) -> batched equivalent:

* ``Simulator(scene, robot, clutter, config)``  ->
  ``BatchSimulator(layouts, n_env, clutter=..., config=...)``; env ``e``
  simulates layout ``layouts[e % len(layouts)]`` unless ``env_layout`` is
  given;
* ``WorldState.to_bytes/from_bytes``  -> ``get_state / set_state`` (the
  identical snapshot bytes);
* ``step_physics(state, targets, dt, substeps)``  ->
  ``step_physics(arm_targets[E,7], base_cmd[E,2], has_targets=None, ...)``
  on device tensors; like the reference it is functional per control step
  and raises ``PhysicsFault`` (naming env and body) when ``check=True``;
* ``apply_grasp(grasp_rule(...))``  -> ``grasp(gripper[E])``;
* sensors ``render_depth`` (SPEC only)  -> ``render(cams)`` -> RGBA8,
  depth f32, body id i32 device tensors ``[E, C, H, W]``.

All device memory for inputs/outputs is torch-allocated; the library owns
the state slabs.  Every call is ordered on the current torch CUDA stream.
"""

from __future__ import annotations

import ctypes as C
import math
import warnings

import numpy as np
import torch

from . import abi, native
from .compiler import compile_world
from .scene import build_world, flat_clutter
from .state import WorldState, snapshot_size

CAMERAS = {"head": 0, "arm": 1}


class PhysicsFault(RuntimeError):
    """Non-finite state (physics.py:46-47, :596-606) or capacity overflow."""


def _dptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


class BatchSimulator:
    def __init__(self, layouts=(0,), n_env: int = 1, clutter: list[str] | None = None, env_layout=None,
                 config: dict | None = None, render: dict | None = None, event_cap: int = 256,
                 device: str | torch.device = "cuda", mesh_k: int | None = None, scenes: list[dict] | None = None):
        """``scenes``: prebuilt scene tables (``compile_world`` format, e.g. from
        a reference ``physics.Simulator`` through ``integration/rearrange_sim_b200.py``)
        instead of the builtin layouts; ``layouts`` then labels them (default
        0..len(scenes)-1) and ``clutter`` is ignored."""
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise native.NativeLibraryError("BatchSimulator runs on CUDA devices only (no CPU fallback)")
        self.L = native.lib()
        if scenes is not None:
            self.layouts = list(range(len(scenes))) if tuple(layouts) == (0,) and len(scenes) > 1 else list(layouts)
            if len(self.layouts) != len(scenes):
                raise ValueError("one layout label per scene")
            if mesh_k is not None:
                raise ValueError("mesh_k needs the builtin layouts (the triangle soups are built from their assets)")
            self.worlds = None
            self.tables = [dict(t) for t in scenes]
        else:
            clutter = clutter if clutter is not None else flat_clutter()
            self.layouts = list(layouts)
            self.worlds = [build_world(v, clutter) for v in self.layouts]
            self.tables = [compile_world(w) for w in self.worlds]
        self.n_env = int(n_env)
        if env_layout is None:
            env_scene = np.arange(self.n_env, dtype=np.int32) % len(self.layouts)
        else:
            env_scene = np.array([self.layouts.index(v) for v in env_layout], dtype=np.int32)
        self.env_scene = env_scene
        self.config = abi.physics_config(**(config or {}))
        self.rconfig = abi.render_config(**(render or {}))
        self.event_cap = int(event_cap)
        t0 = self.tables[0]
        self.n_arm = int(t0["n_arm"])
        self.n_bodies, self.n_joints = len(t0["body_kind"]), int(t0["n_scene_joints"]) + self.n_arm
        self.snap_size = snapshot_size(self.n_bodies, self.n_joints)
        with torch.cuda.device(self.device):
            self._descs = [abi.SceneDesc(t) for t in self.tables]
            self._scenes = []
            self._meshes = []
            for w, d in zip(self.worlds or [None] * len(self._descs), self._descs):
                h = C.c_void_p()
                native.check(self.L.rs_scene_create(C.byref(d.desc), C.byref(h)), "rs_scene_create")
                self._scenes.append(h)
                if mesh_k is not None:
                    from .mesh import compile_mesh

                    md = abi.MeshDesc(compile_mesh(w, mesh_k))
                    self._meshes.append(md)
                    native.check(self.L.rs_scene_set_mesh(h, C.byref(md.desc)), "rs_scene_set_mesh")
            self.n_triangles = len(self._meshes[0].arrays["tri"]) if self._meshes else None
            arr = (C.c_void_p * len(self._scenes))(*[h.value for h in self._scenes])
            b = C.c_void_p()
            native.check(self.L.rs_batch_create(arr, len(self._scenes), env_scene.ctypes.data, self.n_env,
                                                C.byref(self.config), C.byref(self.rconfig), self.event_cap,
                                                C.byref(b)), "rs_batch_create")
            self._batch = b
            bufs = abi.rs_buffers()
            native.check(self.L.rs_batch_buffers(b, C.byref(bufs)), "rs_batch_buffers")
            self._bufs = bufs

    # ---------------------------------------------------------------- lifetime
    def close(self):
        if getattr(self, "_batch", None):
            self.L.rs_batch_destroy(self._batch)
            self._batch = None
        for h in getattr(self, "_scenes", []):
            self.L.rs_scene_destroy(h)
        self._scenes = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------- state
    def set_state(self, snapshots, env_ids=None):
        """Load reference-format snapshots (``WorldState.to_bytes``) into envs."""
        blobs = [s.to_bytes() if isinstance(s, WorldState) else bytes(s) for s in snapshots]
        buf = np.frombuffer(b"".join(blobs), dtype=np.uint8)
        ids = None if env_ids is None else np.ascontiguousarray(env_ids, dtype=np.int32)
        with torch.cuda.device(self.device):
            native.check(self.L.rs_set_state(self._batch, buf.ctypes.data, self.snap_size,
                                             None if ids is None else ids.ctypes.data, len(blobs),
                                             self._sp()), "rs_set_state")

    def get_state(self, env_ids=None) -> list[bytes]:
        ids = np.arange(self.n_env, dtype=np.int32) if env_ids is None else np.ascontiguousarray(env_ids, np.int32)
        out = np.zeros(len(ids) * self.snap_size, np.uint8)
        with torch.cuda.device(self.device):
            native.check(self.L.rs_get_state(self._batch, out.ctypes.data, self.snap_size, ids.ctypes.data,
                                             len(ids), self._sp()), "rs_get_state")
        return [out[i * self.snap_size:(i + 1) * self.snap_size].tobytes() for i in range(len(ids))]

    def world_state(self, env: int) -> WorldState:
        return WorldState.from_bytes(self.get_state([env])[0])

    # ------------------------------------------------------------------- step
    def step_physics(self, arm_targets: torch.Tensor, base_cmd: torch.Tensor, has_targets: torch.Tensor | None = None,
                     dt: float = 1.0 / 30.0, substeps: int = 4, check: bool = False):
        """One control step for every env (physics.py:575-594)."""
        if dt <= 0 or substeps < 1:
            raise PhysicsFault(f"bad step parameters dt={dt} substeps={substeps}")
        arm = self._dev(arm_targets, (self.n_env, self.n_arm), torch.float64)
        base = self._dev(base_cmd, (self.n_env, 2), torch.float64)
        ht = None if has_targets is None else self._dev(has_targets, (self.n_env,), torch.uint8)
        native.check(self.L.rs_step(self._batch, _dptr(arm), _dptr(base), _dptr(ht), float(dt), int(substeps),
                                    self._sp()), "rs_step")
        if check:
            self.raise_faults()

    def _sp(self) -> int:
        """The current torch stream of the batch's device (the library runs
        every call on the device the batch was created on)."""
        return int(torch.cuda.current_stream(self.device).cuda_stream)

    def _host(self, t: torch.Tensor, shape, name: str) -> torch.Tensor:
        """A host f64 buffer handed to the C side by pointer: the library
        reads prod(shape) doubles from it, so anything else is refused."""
        if not isinstance(t, torch.Tensor) or t.device.type != "cpu":
            raise ValueError(f"{name}: expected a CPU (pinned) torch tensor")
        if t.dtype != torch.float64 or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
            raise ValueError(f"{name}: expected a contiguous float64 tensor of shape {tuple(shape)}, "
                             f"got {t.dtype} {tuple(t.shape)}{'' if t.is_contiguous() else ' (non-contiguous)'}")
        if not t.is_pinned():
            warnings.warn(f"{name} is not in pinned memory: the copy is synchronous and slower", stacklevel=3)
        return t

    def _dev(self, t, shape, dtype):
        if not isinstance(t, torch.Tensor):
            t = torch.as_tensor(np.asarray(t))
        t = t.to(device=self.device, dtype=dtype).contiguous()
        if tuple(t.shape) != shape:
            raise ValueError(f"expected shape {shape}, got {tuple(t.shape)}")
        return t

    # -------------------------------------------------------------- buffers
    def faults(self) -> torch.Tensor:
        return _ptr_tensor(self._bufs.fault, 4 * self.n_env, torch.int32, self.device)

    def raise_faults(self):
        f = self.faults().cpu().numpy().astype(np.uint32)
        bad = np.nonzero(f)[0]
        if len(bad):
            e = int(bad[0])
            kind, idx = int(f[e]) >> 16, int(f[e]) & 0xFFFF
            name = abi.FAULT_KINDS.get(kind, f"fault {kind}")
            names = self.body_names(int(self.env_scene[e]))
            if kind == 5:
                raise PhysicsFault(f"env {e}: {name} ({abi.OVERFLOW_KINDS.get(idx, idx)}); state unchanged")
            label = names[idx] if kind in (1, 2, 3) and idx < len(names) else str(idx)
            raise PhysicsFault(f"env {e}: {name} for {'body' if kind in (1, 2, 3) else 'index'} {idx} ({label})")

    def body_names(self, scene: int = 0) -> list[str]:
        """Body names of scene index ``scene`` (PhysicsFault messages)."""
        if self.worlds is not None:
            return [b.name for b in self.worlds[scene].bodies]
        t = self.tables[scene]
        return list(t["body_name"]) if "body_name" in t else [f"body {i}" for i in range(self.n_bodies)]

    def event_counts(self) -> torch.Tensor:
        return _ptr_tensor(self._bufs.event_count, 4 * self.n_env, torch.int32, self.device)

    def events(self) -> torch.Tensor:
        """[E, cap, 7] (a, b, impulse, force, point) of the last step."""
        t = _ptr_tensor(self._bufs.events, 8 * 7 * max(self.event_cap, 1) * self.n_env, torch.float64, self.device)
        return t.view(self.n_env, max(self.event_cap, 1), 7)

    def counters(self) -> torch.Tensor:
        """[E, 3] narrowphase_tests, skipped_sleeping_pairs, wakes (since set_state)."""
        return _ptr_tensor(self._bufs.counters, 8 * 3 * self.n_env, torch.int64, self.device).view(self.n_env, 3)

    def set_trace(self, cap: int = 128, max_substeps: int = 4):
        """Enable the parity trace: admitted pairs + contact counts per substep."""
        self._trace = (torch.zeros((self.n_env, max_substeps, cap, 3), dtype=torch.int32, device=self.device),
                       torch.zeros((self.n_env, max_substeps), dtype=torch.int32, device=self.device))
        native.check(self.L.rs_set_trace(self._batch, _dptr(self._trace[0]), _dptr(self._trace[1]), cap, max_substeps),
                     "rs_set_trace")

    def set_env_order(self, policy: str = "scene"):
        """rs_set_env_order: "scene" (default) or "busy_first" dispatch of the
        warp-per-env step kernel (scheduling only; results are identical)."""
        native.check(self.L.rs_set_env_order(self._batch, {"scene": 0, "busy_first": 1}[policy]), "rs_set_env_order")

    def force_cta(self, width: int):
        """Debug scheduling (parity tests): 8 / 16 = every env of the following
        steps runs in the contact-heavy CTA kernel of that width; -8 / -16 = the
        normal heavy-env selection with CTAs of that width; 0 = normal."""
        native.check(self.L.rsim_bench_force_heavy(self._batch, int(width)), "rsim_bench_force_heavy")

    def trace(self, env: int):
        """[(substep, a, b, n_contacts)] recorded by the last step for `env`."""
        pairs, count = (t.cpu().numpy() for t in self._trace)
        out = []
        for s in range(pairs.shape[1]):
            n = int(count[env, s])
            if n > pairs.shape[2]:
                raise RuntimeError("trace capacity exceeded")
            out.extend((s, *map(int, p)) for p in pairs[env, s, :n])
        return out

    # ------------------------------------------------------------- arm action
    def arm_action(self, delta_ee: torch.Tensor, out: torch.Tensor | None = None, failed: torch.Tensor | None = None):
        """EE displacement [E, 3] (robot base frame) -> joint targets [E, 7]
        via the batched IK (robot.py:293-313 apply_arm_action)."""
        d = self._dev(delta_ee, (self.n_env, 3), torch.float64)
        out = out if out is not None else torch.empty((self.n_env, self.n_arm), dtype=torch.float64, device=self.device)
        failed = failed if failed is not None else torch.empty(self.n_env, dtype=torch.int32, device=self.device)
        native.check(self.L.rs_arm_action(self._batch, _dptr(d), _dptr(out), _dptr(failed), self._sp()),
                     "rs_arm_action")
        return out, failed

    # ------------------------------------------------------------- env step
    def env_step(self, action: torch.Tensor, dt: float = 1.0 / 30.0, substeps: int = 4):
        """Paper action space [E, 6] = (dEE xyz, gripper, base lin, base ang) on
        device: IK -> physics -> grasp rule (rs_env_step)."""
        a = self._dev(action, (self.n_env, 6), torch.float64)
        native.check(self.L.rs_env_step(self._batch, _dptr(a), float(dt), int(substeps), self._sp()),
                     "rs_env_step")

    def env_step_host(self, h_action: torch.Tensor, cams=("head", "arm"), out=None, h_stats=None,
                      dt: float = 1.0 / 30.0, substeps: int = 4):
        """rs_env_step_host: host [E, 6] f64 actions, o_t = render(s_t) rendered
        concurrently, host stats back.  Returns ``(h_stats, (rgba, depth, ids))``:
        ``h_stats`` [E, 4] is complete on return; the observation completes in
        the current stream's order (synchronise it before reading on the host)."""
        self._host(h_action, (self.n_env, 6), "h_action")
        cams = tuple(sorted(cams, key=lambda c: CAMERAS[c]))
        rgba, depth, ids = out if out is not None else self.alloc_obs(cams)
        if h_stats is None:
            h_stats = torch.empty((self.n_env, 4), dtype=torch.float64).pin_memory()
        self._host(h_stats, (self.n_env, 4), "h_stats")
        native.check(self.L.rs_env_step_host(self._batch, C.c_void_p(h_action.data_ptr()), float(dt), int(substeps),
                                             self.cam_mask(cams), _dptr(rgba), _dptr(depth), _dptr(ids),
                                             C.c_void_p(h_stats.data_ptr()), self._sp()), "rs_env_step_host")
        return h_stats, (rgba, depth, ids)

    def step_stats(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """rs_step_stats: [E, 4] f64 device tensor of the current state --
        accumulated contact force (N), fault word, events of the last step,
        sleeping bodies -- on the current stream."""
        out = out if out is not None else torch.empty((self.n_env, 4), dtype=torch.float64, device=self.device)
        native.check(self.L.rs_step_stats(self._batch, _dptr(out), self._sp()), "rs_step_stats")
        return out

    # ------------------------------------------------------------------ grasp
    def grasp(self, gripper: torch.Tensor):
        g = self._dev(gripper, (self.n_env,), torch.float64)
        native.check(self.L.rs_grasp(self._batch, _dptr(g), self._sp()), "rs_grasp")

    # ----------------------------------------------------------------- render
    def alloc_obs(self, cams=("head", "arm")):
        H, W, n = self.rconfig.height, self.rconfig.width, len(cams)
        kw = dict(device=self.device)
        return (torch.empty((self.n_env, n, H, W, 4), dtype=torch.uint8, **kw),
                torch.empty((self.n_env, n, H, W), dtype=torch.float32, **kw),
                torch.empty((self.n_env, n, H, W), dtype=torch.int32, **kw))

    @staticmethod
    def cam_mask(cams) -> int:
        m = 0
        for c in cams:
            m |= 1 << CAMERAS[c]
        return m

    def render(self, cams=("head", "arm"), out=None):
        """RGBD + ids of the current state, ``[E, len(cams), H, W]``; cameras are
        written in mask order (head before arm)."""
        cams = tuple(sorted(cams, key=lambda c: CAMERAS[c]))
        rgba, depth, ids = out if out is not None else self.alloc_obs(cams)
        native.check(self.L.rs_render(self._batch, self.cam_mask(cams), _dptr(rgba), _dptr(depth), _dptr(ids),
                                      self._sp()), "rs_render")
        return rgba, depth, ids

    def render_exact(self, cams=("head", "arm"), out=None):
        """``render`` with every ray test in FP64 (rsim_bench_render_exact): the
        parity reference of the mixed-precision default; not a serving path."""
        cams = tuple(sorted(cams, key=lambda c: CAMERAS[c]))
        rgba, depth, ids = out if out is not None else self.alloc_obs(cams)
        native.check(self.L.rsim_bench_render_exact(self._batch, self.cam_mask(cams), _dptr(rgba), _dptr(depth),
                                                    _dptr(ids), self._sp()), "rsim_bench_render_exact")
        return rgba, depth, ids

    def render_mesh(self, cams=("head", "arm"), out=None):
        """Same as ``render`` against the triangle soups (``mesh_k`` at construction)."""
        cams = tuple(sorted(cams, key=lambda c: CAMERAS[c]))
        rgba, depth, ids = out if out is not None else self.alloc_obs(cams)
        native.check(self.L.rs_render_mesh(self._batch, self.cam_mask(cams), _dptr(rgba), _dptr(depth), _dptr(ids),
                                           self._sp()), "rs_render_mesh")
        return rgba, depth, ids

    # ------------------------------------ proprioception
    def proprioception(self, base_prev=None, goals=None, out=None, base_out=None):
        """Observation fields of the current state: ``[E, 16 + 3K]`` = arm joints
        (7), EE position in the robot frame (3), base egomotion since
        ``base_prev`` [E, 3] (6), goal vectors of ``goals`` [E, K, 3] in the
        robot frame (3K); and the current base [E, 3]."""
        k = 0 if goals is None else int(goals.shape[1])
        g = None if goals is None else self._dev(goals, (self.n_env, k, 3), torch.float64)
        bp = None if base_prev is None else self._dev(base_prev, (self.n_env, 3), torch.float64)
        out = out if out is not None else torch.empty((self.n_env, 16 + 3 * k), dtype=torch.float64,
                                                      device=self.device)
        base_out = base_out if base_out is not None else torch.empty((self.n_env, 3), dtype=torch.float64,
                                                                     device=self.device)
        native.check(self.L.rs_proprio(self._batch, _dptr(bp), _dptr(g), k, _dptr(out), _dptr(base_out),
                                       self._sp()), "rs_proprio")
        return out, base_out

    # ---------------------------------------- point query (physics.py:1088-1101)
    def sphere_cast(self, origins, dirs, max_dist, env_ids=None):
        """Simulator.sphere_cast for Q rays: (body [Q] int32: -1 no hit, -2
        non-unit direction; t [Q] float64) on the envs ``env_ids`` (default 0..Q-1)."""
        n = len(origins)
        o = self._dev(origins, (n, 3), torch.float64)
        d = self._dev(dirs, (n, 3), torch.float64)
        md = self._dev(np.broadcast_to(np.asarray(max_dist, dtype=np.float64), (n,)).copy(), (n,), torch.float64)
        ev = None if env_ids is None else self._dev(env_ids, (n,), torch.int32)
        body = torch.empty(n, dtype=torch.int32, device=self.device)
        t = torch.empty(n, dtype=torch.float64, device=self.device)
        native.check(self.L.rs_sphere_cast(self._batch, _dptr(ev), _dptr(o), _dptr(d), _dptr(md), n, _dptr(body),
                                           _dptr(t), self._sp()), "rs_sphere_cast")
        return body, t

    # ------------------------------------------ settle (physics.py:1113-1176)
    SETTLED, CLEARANCE, FELL, TIMEOUT, FAULT = range(5)

    @staticmethod
    def settle_steps(max_time: float = 10.0) -> int:
        """Control steps of ``while t < max_time: step; t += 1/30`` (float accumulation as in the reference)."""
        t, n = 0.0, 0
        while t < max_time:
            t += 1.0 / 30.0
            n += 1
        return n

    def settle(self, spawn_snapshots, placed, env_ids=None, max_time: float = 10.0, floor_z: float = 0.0):
        """Simulator.settle for many envs at once (fast resets): ``spawn_snapshots``
        are the states settle steps from (``state.spawn_state``), ``placed`` the
        placed body ids per env.  Returns device tensors status [n] (SETTLED,
        CLEARANCE, FELL, TIMEOUT, FAULT), info [n, 2], value [n], steps [n];
        the envs' states are the settled (or last) states."""
        ids = list(range(self.n_env)) if env_ids is None else [int(e) for e in env_ids]
        self.set_state(spawn_snapshots, env_ids=ids)
        masks = np.zeros(self.n_env, np.uint64)
        active = np.zeros(self.n_env, np.uint8)
        for e, bodies in zip(ids, placed):
            m = 0
            for b in bodies:
                m |= 1 << int(b)
            masks[e] = np.uint64(m)
            active[e] = 1
        d_mask = torch.from_numpy(masks.view(np.int64)).to(self.device)
        d_active = torch.from_numpy(active).to(self.device)
        status = torch.empty(self.n_env, dtype=torch.int32, device=self.device)
        info = torch.empty((self.n_env, 2), dtype=torch.int32, device=self.device)
        value = torch.empty(self.n_env, dtype=torch.float64, device=self.device)
        steps = torch.empty(self.n_env, dtype=torch.int32, device=self.device)
        native.check(self.L.rs_settle(self._batch, _dptr(d_mask), _dptr(d_active), self.settle_steps(max_time),
                                      float(floor_z), _dptr(status), _dptr(info), _dptr(value), _dptr(steps),
                                      self._sp()), "rs_settle")
        sel = torch.as_tensor(ids, device=self.device)
        return status[sel], info[sel], value[sel], steps[sel]

    # -------------------------------------------- geodesics (navgrid.py:109-172)
    def nav_shape(self) -> tuple[int, int]:
        nx, ny = C.c_int32(), C.c_int32()
        native.check(self.L.rs_nav_shape(self._batch, C.byref(nx), C.byref(ny)), "rs_nav_shape")
        return nx.value, ny.value

    def distance_fields(self, goals_xy, layouts=None):
        """NavGrid.distance_field for G goals: ``[G, nx, ny]`` float64 device
        tensor (+inf unreachable) and the goal cells ``[G]`` (i*ny + j).
        ``layouts[g]`` indexes the batch's layouts (default: the first)."""
        nx, ny = self.nav_shape()
        n = len(goals_xy)
        g = self._dev(goals_xy, (n, 2), torch.float64)
        fields = torch.empty((n, nx, ny), dtype=torch.float64, device=self.device)
        cells = torch.empty(n, dtype=torch.int32, device=self.device)
        sc = None if layouts is None else self._dev(torch.as_tensor([self.layouts.index(v) for v in layouts]), (n,),
                                                    torch.int32)
        native.check(self.L.rs_nav_fields(self._batch, _dptr(sc), _dptr(g), n, _dptr(fields), _dptr(cells),
                                          self._sp()), "rs_nav_fields")
        return fields, cells

    def geodesic_distance(self, fields, field_idx, from_xy=None, layouts=None):
        """NavGrid.geodesic_distance against ``fields``: from ``from_xy [Q, 2]``
        (scene ``layouts[q]``), or from every env's robot base when None."""
        n = len(field_idx)
        fi = self._dev(field_idx, (n,), torch.int32)
        fx = None if from_xy is None else self._dev(from_xy, (n, 2), torch.float64)
        sc = None if layouts is None else self._dev(torch.as_tensor([self.layouts.index(v) for v in layouts]), (n,),
                                                    torch.int32)
        out = torch.empty(n, dtype=torch.float64, device=self.device)
        native.check(self.L.rs_nav_geodesic(self._batch, _dptr(fields), _dptr(fi), _dptr(sc), _dptr(fx), n,
                                            _dptr(out), self._sp()), "rs_nav_geodesic")
        return out

    def shortest_path(self, fields, field_idx, from_xy, layouts=None, cap: int = 512):
        """NavGrid.shortest_path: waypoints ``[Q, cap, 2]`` and counts ``[Q]``."""
        n = len(field_idx)
        fi = self._dev(field_idx, (n,), torch.int32)
        fx = self._dev(from_xy, (n, 2), torch.float64)
        sc = None if layouts is None else self._dev(torch.as_tensor([self.layouts.index(v) for v in layouts]), (n,),
                                                    torch.int32)
        wp = torch.empty((n, cap, 2), dtype=torch.float64, device=self.device)
        cnt = torch.empty(n, dtype=torch.int32, device=self.device)
        native.check(self.L.rs_nav_path(self._batch, _dptr(fields), _dptr(fi), _dptr(sc), _dptr(fx), n, cap,
                                        _dptr(wp), _dptr(cnt), self._sp()), "rs_nav_path")
        return wp, cnt

    # ------------------------------------------------------- end-to-end (host)
    def step_host(self, h_arm: torch.Tensor, h_base: torch.Tensor, cams=("head", "arm"), out=None,
                  h_stats: torch.Tensor | None = None, dt=1.0 / 30.0, substeps=4):
        """Env step through the C-ABI with HOST action buffers and a HOST
        result read-back (rs_step_host): [E, 4] acc. force, fault, events, asleep.
        Returns ``(h_stats, (rgba, depth, ids))``; the observation completes in
        the current stream's order (synchronise it before reading on the host)."""
        self._host(h_arm, (self.n_env, self.n_arm), "h_arm")
        self._host(h_base, (self.n_env, 2), "h_base")
        cams = tuple(sorted(cams, key=lambda c: CAMERAS[c]))
        rgba, depth, ids = out if out is not None else self.alloc_obs(cams)
        if h_stats is None:
            h_stats = torch.empty((self.n_env, 4), dtype=torch.float64).pin_memory()
        self._host(h_stats, (self.n_env, 4), "h_stats")
        native.check(self.L.rs_step_host(self._batch, C.c_void_p(h_arm.data_ptr()), C.c_void_p(h_base.data_ptr()),
                                         float(dt), int(substeps), self.cam_mask(cams), _dptr(rgba), _dptr(depth),
                                         _dptr(ids), C.c_void_p(h_stats.data_ptr()), self._sp()), "rs_step_host")
        return h_stats, (rgba, depth, ids)


def _ptr_tensor(ptr, nbytes: int, dtype, device) -> torch.Tensor:
    """Wrap library-owned device memory as a torch tensor without copying."""
    class _Holder:
        def __init__(self, p, n):
            self.__cuda_array_interface__ = {
                "shape": (n,), "typestr": "|u1", "data": (int(p), False), "version": 3, "strides": None,
            }
    u8 = torch.as_tensor(_Holder(ptr, nbytes), device=device)
    return u8.view(dtype)
