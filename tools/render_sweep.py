"""BASELINE.json configs[3]: rendering-only sweep, 1024 envs x 128x128 RGBD
(head + arm) at 10k-200k triangles per scene, on one B200.

Prints one JSON line per triangle budget: render-only env-steps/s (2 camera
frames per env-step), ms per batch, and the proxy (convex) renderer on the
same states for reference."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402

E = int(os.environ.get("ENVS", "1024"))
KS = [int(k) for k in os.environ.get("KS", "3,4,7,9,12").split(",")]
REPS = 5


def timed(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(REPS):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


gids = np.arange(E)
states = bench.idle_states(gids, bench.settled_pool())
for k in KS:
    sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=(gids % 3).tolist(), mesh_k=k)
    sim.set_state(states)
    obs = sim.alloc_obs()
    ms_mesh = timed(lambda: sim.render_mesh(out=obs))
    ms_proxy = timed(lambda: sim.render(out=obs))
    print(json.dumps({"config": "configs[3] render-only sweep", "envs": E, "cams": 2, "k": k,
                      "triangles_per_scene": sim.n_triangles, "ms_per_batch_mesh": ms_mesh,
                      "env_steps_per_s_mesh": E / (ms_mesh * 1e-3),
                      "gtri_rays_per_s": None, "ms_per_batch_proxy": ms_proxy,
                      "env_steps_per_s_proxy": E / (ms_proxy * 1e-3)}), flush=True)
    sim.close()
