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

Rewards/tasks are outside this hot path: ``reward`` is
0 and ``done`` marks the horizon or a physics fault; ``info`` carries the
per-env fault word and event count.  With ``set_nav_goals`` the geodesic
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


class BatchEnv:
    def __init__(self, n_env: int, layouts=(0, 1, 2), env_layout=None, cams=("head", "arm"), obs_delay: int = 1,
                 interleave: bool = True, horizon: int | None = None, device="cuda", **sim_kwargs):
        if obs_delay not in (0, 1):
            raise ValueError("obs_delay must be 0 or 1")
        self.sim = BatchSimulator(layouts=layouts, n_env=n_env, env_layout=env_layout, device=device, **sim_kwargs)
        self.n_env = n_env
        self.device = self.sim.device
        self.cams = tuple(sorted(cams, key=lambda c: {"head": 0, "arm": 1}[c]))
        self.obs_delay = obs_delay
        self.interleave = interleave and obs_delay == 1
        self.horizon = horizon
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
        """Load episode start states (reference snapshot bytes) and return o_0."""
        torch.cuda.current_stream(self.device).wait_stream(self._render_stream)
        self.sim.set_state(snapshots, env_ids)
        self.t = 0
        if self._nav_fields is not None:
            self._geo = self.sim.geodesic_distance(self._nav_fields, self._nav_idx)
        obs = self._obs[self._k]
        self._obs_base = None
        self.sim.render(self.cams, out=obs)
        return self._proprio({"rgba": obs[0], "depth": obs[1], "ids": obs[2], "rendered_from_step": 0})

    def step(self, arm_targets: torch.Tensor, base_cmd: torch.Tensor, gripper: torch.Tensor | None = None):
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
                    self.sim.step_physics(arm_targets, base_cmd)
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
                self.sim.step_physics(arm_targets, base_cmd)
            rendered = self.t
        else:
            self.sim.step_physics(arm_targets, base_cmd)
            self.sim.render(self.cams, out=obs)
            extra = self._proprio({})
            rendered = self.t + 1
        if gripper is not None:
            self.sim.grasp(gripper)
        self.t += 1
        fault = self.sim.faults()
        done = fault != 0
        if self.horizon is not None and self.t >= self.horizon:
            done = torch.ones_like(done)
        reward = torch.zeros(self.n_env, dtype=torch.float32, device=self.device)
        info = {"fault": fault, "event_count": self.sim.event_counts(), "step_index": self.t}
        if self._nav_fields is not None:  # geodesic terms of s_{t+1} from every robot base
            geo = self.sim.geodesic_distance(self._nav_fields, self._nav_idx)
            info["geodesic"] = geo
            info["geodesic_delta"] = self._geo - geo
            self._geo = geo
        return {"rgba": obs[0], "depth": obs[1], "ids": obs[2], "rendered_from_step": rendered, **extra}, reward, done, info

    def states(self) -> list[bytes]:
        torch.cuda.current_stream(self.device).wait_stream(self._render_stream)
        return self.sim.get_state()
