"""``BatchEnv``: the SPEC's env pipeline restated over
``BatchSimulator`` -- reset/step with the 1-step observation delay and
interleaved physics || render.

Delay semantics:

* ``obs_delay=1`` (default): ``step(a_t)`` advances the world s_t -> s_{t+1}
  and returns o_t rendered from s_t (``rendered_from_step == t`` while the
  world is at t+1).  ``reset`` returns o_0 from s_0, which primes the buffer:
  the first action is chosen from the step-0 observation.
* ``obs_delay=0``: strictly sequential; ``step`` returns o_{t+1}.

With ``interleave=True`` and delay 1, the render of s_t and the physics of
s_t -> s_{t+1} are enqueued on two CUDA streams and overlap on the GPU: the
batch keeps two state buffers (rs_step reads one and writes the other), so
the render reads s_t while the step writes s_{t+1}.  Interleaved and
sequential execution produce bit-identical states and observations
(tests/test_gpu_env.py) -- the correctness condition of SPEC.md:336.

``step(action)`` takes the SPEC action (§5.1): an
``[E, 6]`` float64 tensor (or a dict ``{"arm": [E, 3], "gripper": [E],
"base": [E, 2]}``) = ArmAction (EE displacement in the robot base frame,
clamped to 1.5 cm; gripper scalar) + BaseAction (linear m/s, angular rad/s),
executed on the device as IK -> step_physics -> grasp rule (rs_env_step).
Joint targets can still be given directly (``arm_targets=``, ``base_cmd=``).

Rewards/tasks are outside this hot path: ``reward`` is
0.  ``done`` marks the horizon, a physics fault or an accumulated contact
force above ``force_limit`` (the Pick / Place thresholds);
``info`` follows the SPEC's StepResult: ``success``
(False: no task), ``failure_reason`` (per env, ``FAILURE_REASONS``),
``accumulated_force`` (N), ``step_index``, plus the fault word and event
count.  Stepping again while any env is done raises ``EpisodeDone`` (the
SPEC's "step after done" error) until those envs are ``reset``.  With ``set_nav_goals`` the geodesic
navigation terms the skill rewards are built from (Navigate
"20 Delta_agent^goal") are computed on the device every step:
``info["geodesic"]`` = NavGrid.geodesic_distance(robot base, goal)
(navgrid.py:145-148) of s_{t+1} and ``info["geodesic_delta"]`` = its
decrease since s_t.
"""

from __future__ import annotations

import numpy as np
import torch

from .sim import BatchSimulator

# info["failure_reason"] codes
FAILURE_REASONS = {0: "none", 1: "horizon", 2: "physics_fault", 3: "force_limit"}


class EpisodeDone(RuntimeError):
    """step() on an env whose episode is done (SPEC.md:320 'step after done')."""


class BatchEnv:
    def __init__(self, n_env: int, layouts=(0, 1, 2), env_layout=None, cams=("head", "arm"), obs_delay: int = 1,
                 interleave: bool = True, horizon: int | None = None, force_limit: float | None = None, device="cuda",
                 **sim_kwargs):
        if obs_delay not in (0, 1):
            raise ValueError("obs_delay must be 0 or 1")
        self.sim = BatchSimulator(layouts=layouts, n_env=n_env, env_layout=env_layout, device=device, **sim_kwargs)
        self.n_env = n_env
        self.device = self.sim.device
        self.cams = tuple(sorted(cams, key=lambda c: {"head": 0, "arm": 1}[c]))
        self.obs_delay = obs_delay
        self.interleave = interleave and obs_delay == 1
        self.horizon = horizon
        self.force_limit = force_limit
        self._done = torch.zeros(n_env, dtype=torch.bool, device=self.sim.device)
        self._done_host = torch.zeros(n_env, dtype=torch.bool).pin_memory()
        self._done_ready = torch.cuda.Event()
        self._t_env = torch.zeros(n_env, dtype=torch.int64, device=self.sim.device)
        self._obs = [self.sim.alloc_obs(self.cams) for _ in range(2)]  # double-buffered observations
        self._k = 0
        self.t = 0
        self._render_stream = torch.cuda.Stream(device=self.device)
        # physics at high priority: the contact-heavy envs (the step's latency
        # tail) get SMs ahead of queued render CTAs
        self._phys_stream = torch.cuda.Stream(device=self.device, priority=-1)
        self._phys_done = torch.cuda.Event()
        self._render_done = torch.cuda.Event()
        self._stats = torch.empty((n_env, 4), dtype=torch.float64, device=self.device)
        self._nav_fields = None
        self._geo = None
        self._goal_pos = None  # [E, K, 3] world goal positions (goal_vectors)
        self._obs_base = None  # base (x, y, yaw) of the state the last observation was taken from

    def close(self):
        self.sim.close()

    # -------------------------------------------------------------------- API
    def set_goal_positions(self, goals):
        """World goal positions [n_env, K, 3] reported as ``goal_vectors`` in the
        robot frame."""
        self._goal_pos = torch.as_tensor(np.asarray(goals) if not isinstance(goals, torch.Tensor) else goals,
                                         dtype=torch.float64).to(self.device).contiguous()

    def _proprio(self, obs: dict):
        """Proprioception of the state being rendered (same stream, same point in
        the order): joints, EE in the robot frame, egomotion since the previous
        observation, goal vectors (rs_proprio)."""
        p, base = self.sim.proprioception(base_prev=self._obs_base, goals=self._goal_pos)
        self._obs_base = base
        obs["joint_positions"] = p[:, 0:7]
        obs["ee_position"] = p[:, 7:10]
        obs["base_egomotion"] = p[:, 10:16]
        if self._goal_pos is not None:
            obs["goal_vectors"] = p[:, 16:].reshape(self.n_env, -1, 3)
        return obs

    def set_nav_goals(self, goals_xy):
        """Per-env navigation goals [n_env, 2] (m): one geodesic distance field
        per env on its layout's walk grid (rs_nav_fields, NavGrid.distance_field)."""
        lay = [self.sim.layouts[i] for i in self.sim.env_scene]
        self._nav_fields, _ = self.sim.distance_fields(goals_xy, layouts=lay)
        self._nav_idx = torch.arange(self.n_env, dtype=torch.int32, device=self.device)
        self._geo = self.sim.geodesic_distance(self._nav_fields, self._nav_idx)
        return self._geo.clone()

    def reset(self, snapshots, env_ids=None):
        """Load episode start states (reference snapshot bytes) into all envs, or
        into ``env_ids``, and return o_0 (rendered for every env)."""
        main = torch.cuda.current_stream(self.device)
        main.wait_stream(self._render_stream)
        self.sim.set_state(snapshots, env_ids)
        if env_ids is None:
            self.t = 0
            self._done.zero_()
            self._t_env.zero_()
        else:
            idx = torch.as_tensor(np.asarray(env_ids), dtype=torch.long, device=self.device)
            self._done[idx] = False
            self._t_env[idx] = 0
        self._done_host.copy_(self._done, non_blocking=True)
        self._done_ready.record(main)
        if self._nav_fields is not None:
            self._geo = self.sim.geodesic_distance(self._nav_fields, self._nav_idx)
        obs = self._obs[self._k]
        self._obs_base = None
        self.sim.render(self.cams, out=obs)
        return self._proprio({"rgba": obs[0], "depth": obs[1], "ids": obs[2], "rendered_from_step": 0})

    def _action(self, action):
        """SPEC action -> [E, 6] float64 device tensor (dEE xyz, gripper, base lin, base ang)."""
        if isinstance(action, dict):
            a = torch.zeros((self.n_env, 6), dtype=torch.float64, device=self.device)
            if "arm" in action:
                a[:, 0:3] = torch.as_tensor(action["arm"], dtype=torch.float64).to(self.device)
            if "gripper" in action:
                a[:, 3] = torch.as_tensor(action["gripper"], dtype=torch.float64).to(self.device)
            if "base" in action:
                a[:, 4:6] = torch.as_tensor(action["base"], dtype=torch.float64).to(self.device)
            return a
        a = torch.as_tensor(action, dtype=torch.float64).to(self.device).contiguous()
        if tuple(a.shape) != (self.n_env, 6):
            raise ValueError(f"action must be [n_env, 6] (dEE xyz, gripper, base lin, base ang), got {tuple(a.shape)}")
        return a

    def step(self, action=None, *, arm_targets: torch.Tensor | None = None, base_cmd: torch.Tensor | None = None,
             gripper: torch.Tensor | None = None):
        """One env step.  ``action``: the SPEC action (IK -> physics -> grasp on
        the device); or ``arm_targets`` [E, 7] + ``base_cmd`` [E, 2] (+ optional
        ``gripper`` [E]) joint targets.  Returns (obs, reward, done, info)."""
        if (action is None) == (arm_targets is None):
            raise ValueError("pass either the SPEC action or arm_targets/base_cmd")
        self._done_ready.synchronize()  # the previous step's done flags (usually complete already)
        if bool(self._done_host.any()):
            bad = torch.nonzero(self._done_host).flatten()[:8].tolist()
            raise EpisodeDone(f"step after done: envs {bad} ... must be reset first (SPEC.md:320)")
        act = self._action(action) if action is not None else None

        def physics():
            if act is not None:
                self.sim.env_step(act)
            else:
                self.sim.step_physics(arm_targets, base_cmd)
                if gripper is not None:
                    self.sim.grasp(gripper)

        main = torch.cuda.current_stream(self.device)
        self._k ^= 1
        obs = self._obs[self._k]
        if self.obs_delay == 1:
            if self.interleave:
                # render(s_t) on the side stream, concurrently with physics(s_t -> s_{t+1})
                self._render_stream.wait_stream(main)
                with torch.cuda.stream(self._render_stream):
                    self.sim.render(self.cams, out=obs)
                    extra = self._proprio({})
                self._render_done.record(self._render_stream)
                self._phys_stream.wait_stream(main)
                with torch.cuda.stream(self._phys_stream):
                    physics()
                main.wait_stream(self._phys_stream)
                # the next step overwrites the buffer this render reads: join here
                main.wait_event(self._render_done)
                for t in obs:
                    t.record_stream(self._render_stream)
                for t in extra.values():  # made on the render stream, consumed on the caller's
                    t.record_stream(main)
            else:
                self.sim.render(self.cams, out=obs)
                extra = self._proprio({})
                physics()
            rendered = self.t
        else:
            physics()
            self.sim.render(self.cams, out=obs)
            extra = self._proprio({})
            rendered = self.t + 1
        self.t += 1
        self._t_env += 1
        stats = self.sim.step_stats(self._stats)
        fault = self.sim.faults()
        acc = stats[:, 0]
        reason = torch.zeros(self.n_env, dtype=torch.int32, device=self.device)
        if self.horizon is not None:
            reason = torch.where(self._t_env >= self.horizon, torch.ones_like(reason), reason)
        if self.force_limit is not None:
            reason = torch.where(acc > self.force_limit, torch.full_like(reason, 3), reason)
        reason = torch.where(fault != 0, torch.full_like(reason, 2), reason)
        done = reason != 0
        self._done.copy_(done)
        self._done_host.copy_(done, non_blocking=True)
        self._done_ready.record(main)
        reward = torch.zeros(self.n_env, dtype=torch.float32, device=self.device)
        info = {"success": torch.zeros(self.n_env, dtype=torch.bool, device=self.device), "failure_reason": reason,
                "accumulated_force": acc, "step_index": self.t, "fault": fault,
                "event_count": self.sim.event_counts()}
        if self._nav_fields is not None:  # geodesic terms of s_{t+1} from every robot base
            geo = self.sim.geodesic_distance(self._nav_fields, self._nav_idx)
            info["geodesic"] = geo
            info["geodesic_delta"] = self._geo - geo
            self._geo = geo
        return {"rgba": obs[0], "depth": obs[1], "ids": obs[2], "rendered_from_step": rendered, **extra}, reward, done, info

    def states(self) -> list[bytes]:
        torch.cuda.current_stream(self.device).wait_stream(self._render_stream)
        return self.sim.get_state()
