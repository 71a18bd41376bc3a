"""Per-env physics latency along the bench's Interact-with-grasps leg (the
reference pick and drawer-drag scripts, staggered): step time, p50 / p99 /
max per-env latency and the slowest envs with their script position.

    python tools/grasp_profile.py [--envs 2048] [--steps 12]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--envs", type=int, default=2048)
ap.add_argument("--steps", type=int, default=12)
args = ap.parse_args()
E, n_tab = args.envs, 3 + args.steps
scripts = [np.load(os.path.join(ROOT, "tests", "golden", f"traj_{n}.npz")) for n in ("pick", "riders")]
span = [len(g["pre"]) - n_tab for g in scripts]
arm = np.zeros((n_tab, E, 7)); base = np.zeros((n_tab, E, 2)); has = np.zeros((n_tab, E), np.uint8)
grip = np.zeros((n_tab, E)); pre = []; off = []
for e in range(E):
    g, sp = scripts[e % 2], span[e % 2]
    o = (e // 2) % (sp + 1)
    off.append(o)
    pre.append(g["pre"][o].tobytes())
    sl = slice(o, o + n_tab)
    arm[:, e], base[:, e], has[:, e] = g["arm"][sl], g["base"][sl], g["has_targets"][sl]
    grip[:, e] = np.nan_to_num(g["gripper"][sl], nan=0.0)
sim = BatchSimulator(layouts=(0,), n_env=E)
sim.set_state(pre)
arm_d, base_d = torch.tensor(arm, device="cuda"), torch.tensor(base, device="cuda")
has_d, grip_d = torch.tensor(has, device="cuda"), torch.tensor(grip, device="cuda")
cyc = torch.zeros(E, dtype=torch.int64, device="cuda")
sim.L.rsim_bench_env_cycles(sim._batch, C.c_void_p(cyc.data_ptr()))
for k in range(n_tab):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sim.step_physics(arm_d[k], base_d[k], has_d[k])
    sim.grasp(grip_d[k])
    e1.record()
    torch.cuda.synchronize()
    a = np.abs(cyc.cpu().numpy()) / 1.965e3
    top = np.argsort(-a)[:5]
    print(f"step {k:2d} {e0.elapsed_time(e1):6.3f} ms p50 {np.median(a):6.1f} p99 {np.percentile(a, 99):7.1f} "
          f"max {a.max():7.1f} us  slowest " + " ".join(f"{'pick' if i % 2 == 0 else 'riders'}@{off[i] + k}:{a[i]:.0f}"
                                                         for i in top), flush=True)
sim.close()
