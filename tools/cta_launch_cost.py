"""Cost of launching the contact-heavy CTA kernel (n_env CTAs of 512 threads,
almost all exiting at once in Idle) inside the interleaved physics || render
step: the bench's Idle step with the CTA kernel launched (default) vs not
(rsim_bench_force_heavy(-1): every env on the warp kernel).

    python tools/cta_launch_cost.py [--steps 20]
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
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--envs", type=int, default=2048)
args = ap.parse_args()
E = args.envs
gids = np.arange(E)
sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=(gids % 3).tolist())
init = bench.idle_states(gids, bench.settled_pool())
act = torch.tensor(bench.action_table(E, 3 + args.steps, seed=7), device="cuda")
obs = sim.alloc_obs()
main, side, hp = torch.cuda.current_stream(), torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
res = {}
for rep in range(2):
    for mode in (0, -1):
        sim.force_cta(mode)
        sim.set_state(init)
        ts = []
        for k in range(3 + args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main)
            side.wait_stream(main)
            hp.wait_stream(main)
            with torch.cuda.stream(side):
                sim.render(out=obs)
            with torch.cuda.stream(hp):
                sim.env_step(act[k])
            main.wait_stream(hp)
            main.wait_stream(side)
            e1.record(main)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[f"rep{rep} {'cta kernel launched' if mode == 0 else 'no cta kernel'}"] = float(np.mean(ts[3:]))
sim.force_cta(0)
print(json.dumps(res, indent=1))
