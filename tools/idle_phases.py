"""Phase clocks (rsim_bench_phase_cycles) of Idle env steps: the bench's
Idle trajectory, 2048 envs, averaged over envs after warm-up.

    python tools/idle_phases.py [--envs 2048] [--steps 4]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--envs", type=int, default=2048)
ap.add_argument("--steps", type=int, default=4)
args = ap.parse_args()
E = args.envs
gids = np.arange(E)
sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=(gids % 3).tolist())
sim.set_state(bench.idle_states(gids, bench.settled_pool()))
act = torch.tensor(bench.action_table(E, 3 + args.steps, seed=7), device="cuda")
for k in range(3):
    sim.env_step(act[k])
ph = torch.zeros((E, 16), dtype=torch.int64, device="cuda")
sim.L.rsim_bench_phase_cycles(sim._batch, C.c_void_p(ph.data_ptr()))
for k in range(args.steps):
    sim.env_step(act[3 + k])
torch.cuda.synchronize()
sim.L.rsim_bench_phase_cycles(sim._batch, None)
names = ["front", "sweeps", "eigen", "lcp(incl eigen)", "impulse+friction", "scalar rows", "back",
         "f:kinematics", "f:aabb+overlap", "f:admission", "f:narrowphase", "f:rows", "b:aabb", "b:retest",
         "b:emit", "lcp iterations (count)"]
v = ph.double().cpu().numpy() / args.steps
med = np.median(v, axis=0) / 1.965e3
med[15] *= 1.965e3
print("median per env-step (us): " + ", ".join(f"{n} {x:.1f}" for n, x in zip(names, med)))
sim.close()
