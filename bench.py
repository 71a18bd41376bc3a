"""Benchmark: batched env.step = 1/30 s physics (4 x 1/120 s substeps) +
128x128 RGBD render of the head and arm cameras (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W --envs E] [--impl reference]

Workload (BASELINE.json configs[4], one GPU's share): E envs per GPU
(default 2048) of the synthetic ReplicaCAD-style apartment (layout
global_env_id % 3), Fetch-like robot, 20 settled clutter objects, Idle
scenario (robot spawned in the living room, random actions: arm joint
targets around the resting pose, base linear U(-0.5, 1) m/s, angular
U(-1, 1) rad/s).  Env shards are disjoint per rank; no collective on the
step path (one NCCL all_reduce of episode stats and of the timing at the
end).  Prints ONE JSON line on rank 0.

--impl reference times the reference algorithm's CPU implementation (the C
oracle restatement, tests-only infrastructure; the Python reference cannot
travel to the GPU box) on all host cores: each step = one env-step
(physics + 2 renders) on every core.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulation steps/sec (128x128 RGBD + 1/30s physics) at 1/2/4/8 B200 vs CPU ref"
UNIT = "env-steps/s"
H = W = 128
N_CAMS = 2
PROFILE_JSON = "profiles/r2i_kernels.json"
HBM_PEAK = 6450.6  # MEASURED_PEAKS.json hbm_gbs (driver-written on this pool's B200s); read at run time when present  # ncu --set full per-kernel DRAM bytes (tools/ncu_summary.py --json)
PAPER_8GPU_SPS = 25734.0  # PAPER.md:530 (8x RTX 2080 Ti, Idle) -- different hardware, not this metric's config


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--envs", type=int, default=2048, help="envs per GPU")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------- workload

def settled_pool():
    g = np.load(os.path.join(ROOT, "tests", "golden", "settled_pool.npz"))
    by_layout = {0: [], 1: [], 2: []}
    for blob, (v, _seed) in zip(g["snapshots"], g["tags"]):
        by_layout[int(v)].append(blob.tobytes())
    return by_layout


def idle_states(global_ids, pool):
    """Idle scenario: settled clutter, robot at the living-room centre
    (builtin.py:358) with a per-env heading."""
    from paper_2106_14405_b200.state import WorldState

    out = []
    for gid in global_ids:
        v = gid % 3
        blobs = pool[v]
        st = WorldState.from_bytes(blobs[(gid // 3) % len(blobs)])
        rng = np.random.default_rng(1000 + gid)
        st.base = np.array([2.3, -0.2, rng.uniform(-math.pi, math.pi)])
        out.append(st.to_bytes())
    return out


def action_table(n_env, n_steps, seed):
    """[n_steps, n_env, 6] Idle random actions in the paper's action space
    (§5.1): EE displacement U(-0.02, 0.02)^3 m (clamped
    to 1.5 cm by the IK front end), gripper 0, base linear U(-0.5, 1) m/s,
    angular U(-1, 1) rad/s."""
    rng = np.random.default_rng(seed)
    a = np.zeros((n_steps, n_env, 6))
    a[..., :3] = rng.uniform(-0.02, 0.02, (n_steps, n_env, 3))
    a[..., 4] = rng.uniform(-0.5, 1.0, (n_steps, n_env))
    a[..., 5] = rng.uniform(-1.0, 1.0, (n_steps, n_env))
    return a


def interact_states(global_ids, pool):
    """Interact scenario: settled clutter, robot spawned at
    (1.6, 0.2, yaw pi/2) facing the light table (per-env jitter)."""
    from paper_2106_14405_b200.state import WorldState

    out = []
    for gid in global_ids:
        blobs = pool[gid % 3]
        st = WorldState.from_bytes(blobs[(gid // 3) % len(blobs)])
        rng = np.random.default_rng(3000 + gid)
        st.base = np.array([1.6 + rng.uniform(-0.05, 0.05), 0.2 + rng.uniform(-0.05, 0.05), math.pi / 2])
        out.append(st.to_bytes())
    return out


def interact_actions(n_env, n_steps):
    """[n_steps, n_env, 6] scripted EE pushes into the clutter: dEE (0.015, 0,
    -0.012) for 20 steps, then +-0.015 y sweeps; base still, gripper 0."""
    a = np.zeros((n_steps, n_env, 6))
    for k in range(n_steps):
        if k < 20:
            a[k, :, :3] = (0.015, 0.0, -0.012)
        else:
            a[k, :, :3] = (0.0, 0.015 if (k // 10) % 2 == 0 else -0.015, 0.0)
    return a


# ------------------------------------------------------------------- clocks

class ClockSampler:
    """SM clocks, max clocks, clock-event (throttle) reasons and power sampled
    DURING the timed region: NVML in a background thread every 2 ms (plus one
    sample at entry and one at exit, so even a 50 ms region has samples);
    nvidia-smi as the fallback when NVML is unavailable."""
    QUERY = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw"
    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
             0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x100: "display_clock_setting"}

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.rows = []
        self.nvml = None
        self.source = "none"

    def _nvml_sample(self):
        import pynvml as N

        h = self.handle
        try:
            reasons = N.nvmlDeviceGetCurrentClocksEventReasons(h)
        except (AttributeError, N.NVMLError):
            reasons = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.rows.append((float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)),
                          float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)), int(reasons),
                          N.nvmlDeviceGetPowerUsage(h) / 1000.0))

    def __enter__(self):
        import threading

        try:
            import pynvml as N

            N.nvmlInit()
            self.handle = N.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = N
            self.source = "nvml"
            self._stop = threading.Event()
            self._nvml_sample()

            def loop():
                while not self._stop.wait(0.002):
                    try:
                        self._nvml_sample()
                    except Exception:  # noqa: BLE001 - sampling must never break the bench
                        break

            self._thread = threading.Thread(target=loop, daemon=True)
            self._thread.start()
            return self
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi"
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.nvml is not None:
            self._stop.set()
            self._thread.join(timeout=1.0)
            try:
                self._nvml_sample()
            except Exception:  # noqa: BLE001
                pass
            return False
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out = ""
            for line in (out or "").strip().splitlines():
                parts = [p.strip() for p in line.split(",")]
                try:
                    self.rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16), float(parts[3])))
                except (ValueError, IndexError):
                    continue
        return False

    def summary(self):
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "source": self.source}
        mask = 0
        for r in rows:
            mask |= r[2]
        return {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": [n for b, n in self.NAMES.items() if mask & b], "samples": len(rows),
                "power_w_max": max(r[3] for r in rows), "source": self.source}


# --------------------------------------------------------------- CPU oracle

_ORC = {}


def _cpu_init():
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle.oracle import Oracle
    from paper_2106_14405_b200.compiler import compile_world
    from paper_2106_14405_b200.scene import build_world, flat_clutter

    for v in range(3):
        _ORC[v] = Oracle(compile_world(build_world(v, flat_clutter())))


def _cpu_worker(args):
    """Oracle env-steps in one worker process: IK + physics, then 0, 1 (head)
    or 2 (head + arm) camera renders."""
    from paper_2106_14405_b200.state import WorldState

    layout, snap, act, n, cams = args
    orc = _ORC[layout]
    t0 = time.perf_counter()
    for k in range(n):
        q = WorldState.from_bytes(snap).joints[4:]
        tg, _ = orc.apply_arm_action(q, act[k, :3])
        snap = orc.step(snap, tg, act[k, 4:]).snapshot
        for c in range(cams):
            orc.render(snap, c)
    return n, time.perf_counter() - t0, snap


class CpuOracle:
    """One worker process per host core, each owning one env."""

    def __init__(self, cores=None):
        import multiprocessing as mp

        from oracle import oracle as orc

        orc.build()
        self.cores = cores or os.cpu_count() or 1
        self.states = idle_states(range(self.cores), settled_pool())
        self.pool = mp.get_context("spawn").Pool(self.cores, initializer=_cpu_init)

    def run(self, steps_per_core, seed, cams=2):
        act = action_table(self.cores, steps_per_core, seed)
        jobs = [(g % 3, self.states[g], act[:, g], steps_per_core, cams) for g in range(self.cores)]
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_worker, jobs)
        wall = time.perf_counter() - t0
        self.states = [r[2] for r in res]
        return sum(r[0] for r in res), wall

    def close(self):
        self.pool.close()
        self.pool.join()


# BASELINE.md §2 / SURVEY.md §8d protocol: physics-only, 1-camera and 2-camera
# rows; per row a 30-step warm-up per core, then 10 runs reported as mean +-
# 95 % CI (Student t, 9 dof).  Run lengths (env-steps per core per run) keep
# the whole sample near 10-20 s of host time.
CPU_ROWS = (("physics_only", 0, 400), ("one_camera", 1, 6), ("two_camera", 2, 4))
CPU_RUNS, CPU_WARMUP = 10, 30
T975_9DOF = 2.262


def cpu_oracle_protocol(cores=None, seed=0, runs=CPU_RUNS, warmup=CPU_WARMUP, rows=CPU_ROWS):
    c = CpuOracle(cores)
    out = {}
    try:
        for name, cams, per_run in rows:
            c.run(warmup, seed + 1000, cams)
            sps = []
            for r in range(runs):
                steps, wall = c.run(per_run, seed + r, cams)
                sps.append(steps / wall)
            sps = np.asarray(sps)
            half = T975_9DOF * sps.std(ddof=1) / math.sqrt(len(sps)) if len(sps) > 1 else 0.0
            out[name] = {"mean": float(sps.mean()), "ci95": float(half), "runs": len(sps),
                         "env_steps_per_core_per_run": per_run, "cameras": cams}
    finally:
        c.close()
    return out, c.cores


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# -------------------------------------------------------------------- arms

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    c = CpuOracle()
    cores = c.cores
    per_step = []
    for k in range(args.warmup + args.steps):
        steps, wall = c.run(1, seed=k)
        if k >= args.warmup:
            per_step.append((wall, steps))
    c.close()
    total_steps = sum(s for _, s in per_step)
    total_wall = sum(w for w, _ in per_step)
    value = total_steps / total_wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "idle env.step (dEE action -> IK, physics 4x1/120 s, 2 cams 128x128 RGBD), one "
                               "env-step per host core per step", "envs_per_step": cores, "layouts": "apt_{env%3}",
                   "clutter": 20},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{total_steps} env-steps (IK + physics + 2 renders) of the C oracle "
                                   f"restatement ({cpu_model()})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def grasp_leg(args, E, dev, side, hp, stream, n_tab):
    """Timed Interact variant with grasp transitions (see the call site)."""
    import torch

    from paper_2106_14405_b200.sim import BatchSimulator

    scripts = [np.load(os.path.join(ROOT, "tests", "golden", f"traj_{n}.npz")) for n in ("pick", "riders")]
    span = [len(g["pre"]) - n_tab for g in scripts]
    arm = np.zeros((n_tab, E, 7)); base = np.zeros((n_tab, E, 2)); has = np.zeros((n_tab, E), np.uint8)
    grip = np.zeros((n_tab, E)); pre = []
    for e in range(E):
        g, sp = scripts[e % 2], span[e % 2]
        o = (e // 2) % (sp + 1)
        pre.append(g["pre"][o].tobytes())
        sl = slice(o, o + n_tab)
        arm[:, e], base[:, e], has[:, e] = g["arm"][sl], g["base"][sl], g["has_targets"][sl]
        grip[:, e] = np.nan_to_num(g["gripper"][sl], nan=0.0)
    gs = BatchSimulator(layouts=(0,), n_env=E, device=dev)
    gs.set_state(pre)
    arm_d, base_d = torch.tensor(arm, device=dev), torch.tensor(base, device=dev)
    has_d, grip_d = torch.tensor(has, device=dev), torch.tensor(grip, device=dev)
    obs = gs.alloc_obs(("head", "arm"))

    def step(k):
        hp.wait_stream(stream)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            gs.render(("head", "arm"), out=obs)
        with torch.cuda.stream(hp):
            gs.step_physics(arm_d[k], base_d[k], has_d[k])
            gs.grasp(grip_d[k])
        stream.wait_stream(hp)
        stream.wait_stream(side)

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize(dev)
    held0 = np.array([gs_held(gs, e) for e in range(0, E, max(1, E // 64))])
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    for k in range(args.steps):
        step(args.warmup + k)
    c1.record(stream)
    torch.cuda.synchronize(dev)
    gs.raise_faults()
    held1 = np.array([gs_held(gs, e) for e in range(0, E, max(1, E // 64))])
    tr = np.concatenate([g["trans"][:, 0] for g in scripts])
    info = {"note": "apt_0, half the envs on the reference's pick & place script, half on its drawer-drag script "
                    "(handle snap, drag with riders, release, reach into the tray); staggered offsets; "
                    "rs_step + rs_grasp on the physics stream, 2-camera render interleaved",
            "script_snaps_releases": [int((tr == 1).sum()), int((tr == 2).sum())],
            "sampled_envs_holding_before_after": [int((held0 >= 0).sum()), int((held1 >= 0).sum())],
            "sampled_envs": len(held0)}
    ms = c0.elapsed_time(c1)
    gs.close()
    return ms, info


def gs_held(sim, e):
    from paper_2106_14405_b200.state import WorldState

    return int(WorldState.from_bytes(sim.get_state([e])[0]).held)


def run_b200(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; RSIM_DIST_BACKEND=gloo lets several ranks share one
    # device for host-path testing (NCCL refuses duplicate GPUs)
    backend = os.environ.get("RSIM_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    from paper_2106_14405_b200 import native
    from paper_2106_14405_b200.sim import BatchSimulator

    from paper_2106_14405_b200.shard import layout_of, reduce_window, shard_env_ids

    E = args.envs
    gids = shard_env_ids(rank, world, E)
    sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=layout_of(gids).tolist(), device=dev)
    init_states = idle_states(gids, settled_pool())
    sim.set_state(init_states)
    n_tab = args.warmup + args.steps
    act_np = action_table(E, n_tab, seed=7 + rank)
    act_d = torch.tensor(act_np, device=dev)
    obs = sim.alloc_obs(("head", "arm"))
    stream = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(dev)

    hp = torch.cuda.Stream(dev, priority=-1)  # physics ahead of queued render CTAs

    def step(k, ev=None, cams=("head", "arm"), out=None, acts=act_d):
        # one env step, paper pipeline (SPEC StepConfig defaults
        # observation_delay=1, interleave=true): physics s_t -> s_{t+1} on a
        # high-priority stream, render(s_t) concurrently on a side stream, join.
        hp.wait_stream(stream)
        side.wait_stream(stream)
        with torch.cuda.stream(side):  # enqueued first: it reads s_t before env_step flips the state buffers
            if ev is not None:
                ev[2].record(side)
            sim.render(cams, out=obs if out is None else out)
            if ev is not None:
                ev[3].record(side)
        with torch.cuda.stream(hp):
            if ev is not None:
                ev[0].record(hp)
            sim.env_step(acts[k])  # IK -> physics -> grasp rule
            if ev is not None:
                ev[1].record(hp)
        stream.wait_stream(hp)
        stream.wait_stream(side)

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize(dev)
    sim.raise_faults()

    # ---- device-resident timed region (value)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for k in range(args.steps):
            step(args.warmup + k, evs[k])
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms_total = t_start.elapsed_time(t_end)
    ms_phys = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    ms_rend = float(np.mean([e[2].elapsed_time(e[3]) for e in evs]))
    sim.raise_faults()

    # ---- the same trajectory with one camera (head): BASELINE.md asks for the
    # headline with 2 cameras and also with 1
    obs1 = sim.alloc_obs(("head",))
    sim.set_state(init_states)
    for k in range(args.warmup):
        step(k, cams=("head",), out=obs1)
    torch.cuda.synchronize(dev)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    for k in range(args.steps):
        step(args.warmup + k, cams=("head",), out=obs1)
    c1.record(stream)
    torch.cuda.synchronize(dev)
    ms_one_cam = c0.elapsed_time(c1)
    del obs1

    # ---- Interact (second column): robots facing the light
    # table pushing into the clutter, same interleaved step
    act_i = torch.tensor(interact_actions(E, n_tab), device=dev)
    sim.set_state(interact_states(gids, settled_pool()))
    for k in range(args.warmup):
        step(k, acts=act_i)
    torch.cuda.synchronize(dev)
    c0.record(stream)
    for k in range(args.steps):
        step(args.warmup + k, acts=act_i)
    c1.record(stream)
    torch.cuda.synchronize(dev)
    ms_interact = c0.elapsed_time(c1)
    sim.raise_faults()
    del act_i

    # ---- Interact with grasps and drags inside the timed region: the reference's
    # own pick & place and drawer-drag scripts (tests/golden/traj_pick.npz,
    # traj_riders.npz, layout apt_0: handle snap + drag with riders, object snap,
    # hold, carry, release, fall), teacher-forced per env from a staggered offset
    # into its script (joint targets of the reference IK + gripper scalars), so
    # every step of the window has envs reaching, snapping, dragging, carrying
    # and releasing; physics + grasp rule interleaved with the 2-camera render
    ms_grasp, grasp_info = grasp_leg(args, E, dev, side, hp, stream, n_tab)

    # ---- end-to-end through the C-ABI with host buffers (e2e): replay the
    # same trajectory (same initial states, same actions) as the timed region
    sim.set_state(init_states)
    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize(dev)
    h_act = torch.tensor(act_np).pin_memory()
    h_stats = torch.empty((E, 4), dtype=torch.float64).pin_memory()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host_ms = []
    e0.record(stream)
    for k in range(args.steps):
        h0 = time.perf_counter()
        sim.env_step_host(h_act[args.warmup + k], out=obs, h_stats=h_stats)
        host_ms.append(1e3 * (time.perf_counter() - h0))
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms_e2e = e0.elapsed_time(e1)
    if rank == 0:
        st = h_stats.numpy()
        print(f"[bench] e2e per-step host ms: {np.round(host_ms, 3).tolist()}", file=sys.stderr)
        print(f"[bench] envs with awake clutter: {int((st[:, 3] < 20).sum())}, "
              f"envs with contact events: {int((st[:, 2] > 0).sum())}, faults: {int((st[:, 1] != 0).sum())}",
              file=sys.stderr)
    acc = float(h_stats[:, 0].sum())

    # ---- each half alone (same launches, no overlap partner): the interleaved
    # timings above share the SMs; the roofline uses the render kernel alone
    iso = {"render": [], "phys": []}
    for k in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sim.render(("head", "arm"), out=obs)
        b.record(stream)
        iso["render"].append((a, b))
    sim.set_state(init_states)  # physics alone on the timed region's trajectory
    for k in range(args.warmup):
        sim.env_step(act_d[k])
    for k in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sim.env_step(act_d[args.warmup + k])
        b.record(stream)
        iso["phys"].append((a, b))
    torch.cuda.synchronize(dev)
    ms_rend_iso = float(np.mean([a.elapsed_time(b) for a, b in iso["render"]]))
    ms_phys_iso = float(np.mean([a.elapsed_time(b) for a, b in iso["phys"]]))

    # ---- across ranks: max time, summed stats (the only collectives)
    stats, tms = reduce_window({"acc": acc, "envs": float(E)},
                               {"total": ms_total, "e2e": ms_e2e, "phys": ms_phys, "rend": ms_rend,
                                "phys_iso": ms_phys_iso, "rend_iso": ms_rend_iso, "one_cam": ms_one_cam,
                                "interact": ms_interact, "grasp": ms_grasp},
                               device=dev if backend == "nccl" else "cpu")
    ms_total, ms_e2e, ms_phys, ms_rend = tms["total"], tms["e2e"], tms["phys"], tms["rend"]
    ms_phys_iso, ms_rend_iso, ms_one_cam = tms["phys_iso"], tms["rend_iso"], tms["one_cam"]
    ms_interact, ms_grasp = tms["interact"], tms["grasp"]
    total_envs = E * world
    value = total_envs * args.steps / (ms_total * 1e-3)
    e2e_value = total_envs * args.steps / (ms_e2e * 1e-3)

    if rank == 0:
        # roofline of the render kernel against the measured FMA pipe peak
        import ctypes as C

        peak64, peak32 = C.c_double(0), C.c_double(0)
        L = native.lib()
        L.rsim_bench_fma_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
        L.rsim_bench_fma_peak(1, C.byref(peak64))
        L.rsim_bench_fma_peak(0, C.byref(peak32))
        render_flop = N_CAMS * H * W * (14 * 566 + 22 * 4)  # SURVEY.md §8d W_r (brute-force proxy raycast)
        phys_flop = 0.09e6  # SURVEY.md §8d idle W_p per env-step
        wd = torch.zeros(20, dtype=torch.int64, device=dev)  # rsim_bench.h: 20 counters
        L.rsim_bench_render_work_detail.argtypes = [C.c_void_p, C.c_uint, C.c_void_p, C.c_void_p]
        L.rsim_bench_render_work_detail(sim._batch, 3, C.c_void_p(wd.data_ptr()), C.c_void_p(stream.cuda_stream))
        torch.cuda.synchronize(dev)
        wd = wd.cpu().numpy().astype(float)
        fp32_tests, fp64_tests = wd[0] / E, (wd[1] + wd[2] + wd[6]) / E  # ray-plane tests per env-step
        # The render kernel dominates the GPU's work (SM-time); the physics step is
        # latency-bound (its duration is the slowest env's dependency chain on one
        # warp, see "physics_latency"), so the roofline is the render kernel's.
        dom, ms_dom, grid = "render_kernel", ms_rend_iso, E * N_CAMS
        # roofline = the ray-plane work the kernel executes (FP32 bounded-error box
        # tests + FP64 tests/resolutions, 14 flop each) against the two pipes' measured
        # peaks: frac = (F32 / P32 + F64 / P64) / t, i.e. the busy fraction of an
        # ideal machine doing exactly this work; peak = the matching harmonic mix
        f32, f64 = 14.0 * fp32_tests * E, 14.0 * fp64_tests * E  # flop per launch
        t_s = ms_dom * 1e-3
        frac = (f32 / (peak32.value * 1e12) + f64 / (peak64.value * 1e12)) / t_s if peak32.value else None
        p_eff = (f32 + f64) / (f32 / peak32.value + f64 / peak64.value) if peak32.value else None
        traffic, prof, inst = None, None, None
        try:  # dram read+write and warp instructions per launch of this kernel from the committed ncu --set full capture
            pj = json.load(open(os.path.join(ROOT, PROFILE_JSON)))
            kk = next((v for k, v in pj["kernels"].items() if k.startswith(dom)), None)
            if kk and kk["grid"] == grid:
                traffic, prof, inst = kk["dram_bytes_per_launch"], PROFILE_JSON, kk.get("warp_inst_per_launch")
        except (OSError, ValueError, KeyError):
            pass
        sm_mhz = clk.summary().get("sm_mhz") or 1965.0
        global HBM_PEAK
        try:
            HBM_PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        except (OSError, ValueError, KeyError):
            pass
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        # per-env step latency of one more control step (rsim_bench_env_cycles probe)
        cyc = torch.zeros(E, dtype=torch.int64, device=dev)
        L.rsim_bench_env_cycles.argtypes = [C.c_void_p, C.c_void_p]
        L.rsim_bench_env_cycles(sim._batch, C.c_void_p(cyc.data_ptr()))
        sim.env_step(act_d[args.warmup + args.steps - 1])
        torch.cuda.synchronize(dev)
        L.rsim_bench_env_cycles(sim._batch, None)
        us = np.abs(cyc.cpu().numpy()) / sm_mhz
        obs_bytes = E * N_CAMS * H * W * (4 + 4 + 4)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (settled-clutter pool from the reference recipe, random idle actions)",
            "config": {"workload": "configs[4] full env step: dEE action -> IK, physics 4x1/120 s, grasp rule, "
                                   "head+arm 128x128 RGBD; Idle; render(s_t) interleaved with "
                                   "physics(s_t->s_t+1) (obs delay 1)",
                       "envs_per_gpu": E, "global_envs": total_envs, "layouts": "apt_{env%3}", "clutter": 20,
                       "parallelism": f"env-shard dp{world}",
                       "l2": "inputs > L2: 805 MB of RGBD/id writes per step at 2048 envs evict the state slabs"},
            "kernels_ms_per_step": {"interleaved": {"ik+step+grasp": ms_phys, "render_kernel": ms_rend},
                                    "alone": {"ik+step+grasp": ms_phys_iso, "render_kernel": ms_rend_iso}},
            "roofline": {"bound": "fp32+fp64 pipes", "kernel": dom, "achieved": (f32 + f64) / t_s / 1e12,
                         "peak": p_eff, "unit": "TFLOP/s", "frac": frac,
                         "traffic": traffic, "traffic_source": prof,
                         "algorithmic_bytes_per_launch": obs_bytes,
                         "peak_source": "measured FMA microbenchmarks (rsim_bench_fma_peak): FP32 %.1f, FP64 %.1f "
                                        "TFLOP/s; MEASURED_PEAKS.json has no FP32/FP64 entry; peak = their harmonic "
                                        "mix weighted by this kernel's FP32/FP64 flop" % (peak32.value, peak64.value),
                         "work_note": "executed ray-plane tests per env-step counted by the kernel's counting variant "
                                      "(rsim_bench_render_work_detail, same trajectory state), 14 flop per test",
                         "executed_plane_tests_per_unit": {"fp32": fp32_tests, "fp64": fp64_tests},
                         "executed_flop_per_launch": {"fp32": f32, "fp64": f64},
                         "fp32_peak_tflops": peak32.value, "fp64_peak_tflops": peak64.value,
                         "issue_frac_ncu": (inst / (t_s * n_sm * 4 * sm_mhz * 1e6)) if inst else None,
                         "issue_note": "warp instructions per launch (committed ncu capture) / (this run's kernel time "
                                       "x SMs x 4 schedulers x SM clock): the pipe the kernel actually saturates",
                         "brute_force_W_r": {
                             "flop_per_unit": render_flop, "achieved_tflops": render_flop * E / t_s / 1e12,
                             "frac_vs_fp32_peak": render_flop * E / t_s / 1e12 / peak32.value if peak32.value else None,
                             "note": "SURVEY.md §8d W_r = every ray against every unique plane (566) and sphere; the "
                                     "kernel culls to ~3 box tests per ray, so this ratio exceeds 1 and is not a "
                                     "roofline fraction"},
                         "hbm": {"achieved_gbs": obs_bytes / t_s / 1e9, "peak_gbs": HBM_PEAK,
                                 "frac": obs_bytes / t_s / 1e9 / HBM_PEAK,
                                 "note": "observation writes (RGBA u32 + depth f32 + id i32) per launch"}},
            "physics_roofline": {
                "bound": "fp64", "kernel": "ik_first+ik_fallback+step_kernel(+step_kernel_cta)+grasp, alone",
                "W_p_flop_per_unit": phys_flop, "achieved": phys_flop * E / (ms_phys_iso * 1e-3) / 1e12,
                "peak": peak64.value, "unit": "TFLOP/s",
                "frac": phys_flop * E / (ms_phys_iso * 1e-3) / 1e12 / peak64.value if peak64.value else None,
                "note": "SURVEY.md §8d W_p = 8 N_vp + 100 N_row + 120 N_fric + 20 sum m^3 with the frozen Idle "
                        "counts (0.09 MFLOP per env-step); the step is latency-bound (serial Gauss-Seidel order "
                        "inside an env), see physics_latency"},
            "physics_latency": {"note": "step kernel = one warp per env, latency-bound (serial Gauss-Seidel "
                                        "order inside an env); per-env SM time of one control step",
                                "p50_us": float(np.percentile(us, 50)), "p99_us": float(np.percentile(us, 99)),
                                "max_us": float(us.max()), "envs_on_cta_kernel": int((cyc < 0).sum().item()),
                                "algorithmic_flop_per_unit": phys_flop},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(E * 6 * 8),
                    "d2h_bytes_per_step": int(E * 4 * 8)},
            "one_camera": {"value": total_envs * args.steps / (ms_one_cam * 1e-3), "unit": UNIT,
                           "ms_per_step": ms_one_cam / args.steps,
                           "note": "same trajectory, head camera only (PAPER.md:97 '1 RGBD observation')"},
            "interact": {"value": total_envs * args.steps / (ms_interact * 1e-3), "unit": UNIT,
                         "ms_per_step": ms_interact / args.steps,
                         "note": "Interact scenario (PAPER.md:530 second column; SURVEY.md §8d): robots at "
                                 "(1.6, 0.2) facing the light table, scripted EE pushes into the clutter; "
                                 "same interleaved physics + 2-camera render step"},
            "interact_grasp": {"value": total_envs * args.steps / (ms_grasp * 1e-3), "unit": UNIT,
                               "ms_per_step": ms_grasp / args.steps, **grasp_info},
            "gpu_launches": 6 * args.steps,  # ik_first, ik_fallback, step, step_cta, grasp, render per env step
            "clocks": clk.summary(),
            "episode_stats_allreduce": {"accumulated_contact_force_sum": stats["acc"], "envs": int(stats["envs"])},
        }
        # widened rows: geodesic fields for one goal per env and the
        # per-step geodesic reward query from every robot base
        goals = torch.tensor(np.random.default_rng(5).uniform([-4.5, -2.5], [4.5, 2.5], (E, 2)), device=dev)
        fields, _ = sim.distance_fields(goals, layouts=layout_of(gids).tolist())
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(stream)
        fields, _ = sim.distance_fields(goals, layouts=layout_of(gids).tolist())
        ev[1].record(stream)
        idx = torch.arange(E, device=dev, dtype=torch.int32)
        sim.geodesic_distance(fields, idx)
        ev[2].record(stream)
        for _ in range(10):
            sim.geodesic_distance(fields, idx)
        ev[3].record(stream)
        torch.cuda.synchronize(dev)
        nx_, ny_ = sim.nav_shape()
        line["geodesics"] = {"distance_fields_per_s": E / (ev[0].elapsed_time(ev[1]) * 1e-3),
                             "grid": [nx_, ny_], "fields": E,
                             "geodesic_queries_per_s": 10 * E / (ev[2].elapsed_time(ev[3]) * 1e-3),
                             "note": "rs_nav_fields (one CTA per goal, bit-exact vs the reference Dijkstra) and "
                                     "rs_nav_geodesic from every robot base"}
        del fields
        # batched settle (fast resets): the reference recipe's spawn
        # states (settle.npz, 24 layout/seed cases incl. 6 clearance failures) tiled
        # over all envs, GJK clearance + steps until every placed body sleeps
        sg = np.load(os.path.join(ROOT, "tests", "golden", "settle.npz"))
        sel = [i for i in range(len(sg["tags"])) if int(sg["tags"][i][0]) in (0, 1, 2)]
        by_layout = {v: [i for i in sel if int(sg["tags"][i][0]) == v] for v in range(3)}
        lay = layout_of(gids)
        spawns = [sg["spawn"][by_layout[int(lay[e])][e // 3 % len(by_layout[int(lay[e])])]].tobytes() for e in range(E)]
        clutter = sim.worlds[0].clutter_body_ids
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        st_, _, _, steps_ = sim.settle(spawns, [clutter] * E)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        st_ = st_.cpu().numpy()
        line["settle"] = {"envs_per_s": E / (ev0.elapsed_time(ev1) * 1e-3), "envs": E,
                          "settled": int((st_ == 0).sum()), "clearance_failures": int((st_ == 1).sum()),
                          "max_steps_taken": int(steps_.max()),
                          "note": "timed: upload of the spawn snapshots (rs_set_state) + rs_settle (GJK spawn "
                                  "clearance, control steps until every placed body sleeps)"}
        if world == 1 and not args.no_cpu_baseline:
            h0 = time.perf_counter()
            rows, cores = cpu_oracle_protocol()
            line["cpu_baseline"] = {
                "value": rows["two_camera"]["mean"], "unit": UNIT, "cores": cores, "kind": "port",
                "ci95": rows["two_camera"]["ci95"], "rows": rows, "cpu_model": cpu_model(),
                "sample": f"C oracle restatement, one env per host core ({cores} cores, {cpu_model()}), "
                          f"idle env-steps (IK + physics + 0/1/2 camera renders); per row {CPU_WARMUP} warm-up "
                          f"steps per core then {CPU_RUNS} runs, mean +- 95% CI; value = the 2-camera row; "
                          f"{time.perf_counter() - h0:.1f} s wall in total"}
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
