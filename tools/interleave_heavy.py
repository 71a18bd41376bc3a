"""Interact / Interact-with-grasps steps: physics alone vs interleaved with the
2-camera render, with the contact-heavy CTA kernel at its default width
(16 warps = a whole SM's registers at <= 2048 envs) or 8 warps.

    python tools/interleave_heavy.py [--steps 10]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--envs", type=int, default=2048)
args = ap.parse_args()
E, W = args.envs, 3
gids = np.arange(E)
main = torch.cuda.current_stream()
side = torch.cuda.Stream()
hp = torch.cuda.Stream(priority=-1)


def run(sim, phys, n, render, width):
    sim.force_cta(width)
    obs = sim.alloc_obs()
    ts = []
    for k in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        side.wait_stream(main)
        hp.wait_stream(main)
        if render:
            with torch.cuda.stream(side):
                sim.render(out=obs)
        with torch.cuda.stream(hp):
            phys(k)
        main.wait_stream(hp)
        main.wait_stream(side)
        e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    sim.force_cta(0)
    return float(np.mean(ts[W:]))


res = {}
# Interact (bench scenario)
sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=(gids % 3).tolist())
act = torch.tensor(bench.interact_actions(E, 40), device="cuda")
init = bench.interact_states(gids, bench.settled_pool())
for render in (False, True):
    for width in (0, -8):
        sim.set_state(init)
        for k in range(8):
            sim.env_step(act[k])
        res[f"interact render={render} width={'8' if width else 'default'}"] = run(
            sim, lambda k: sim.env_step(act[8 + k]), W + args.steps, render, width)
sim.close()
print(json.dumps(res, indent=1))
