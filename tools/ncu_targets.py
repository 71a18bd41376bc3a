"""Workloads for `ncu --set full --profile-from-start off`: the profiled region
(cudaProfilerStart/Stop) holds exactly the launches to capture.

    MODE=idle      2048 envs, Idle bench trajectory: render_kernel<0,0> + step_kernel
    MODE=interact  2048 envs, Interact trajectory after 12 steps: step_kernel + step_kernel_cta<16>
    MODE=mesh      1024 envs, triangle soups at k = 7 (68k triangles): render_kernel<1,0>

e.g. ncu --set full --import-source on --clock-control none --profile-from-start off \
         -o gpurun_out/r2_idle python tools/ncu_targets.py idle
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "idle"
E = int(os.environ.get("ENVS", "1024" if mode == "mesh" else "2048"))
gids = np.arange(E)
pool = bench.settled_pool()
sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=(gids % 3).tolist(),
                     mesh_k=7 if mode == "mesh" else None)
obs = sim.alloc_obs()
if mode == "mesh":
    sim.set_state(bench.idle_states(gids, pool))
    sim.render_mesh(out=obs)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    sim.render_mesh(out=obs)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
else:
    if mode == "idle":
        sim.set_state(bench.idle_states(gids, pool))
        act = torch.tensor(bench.action_table(E, 8, seed=7), device="cuda")
        warm = 3
    else:
        sim.set_state(bench.interact_states(gids, pool))
        act = torch.tensor(bench.interact_actions(E, 16), device="cuda")
        warm = 12
    for k in range(warm):
        sim.env_step(act[k])
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    if mode == "idle":
        sim.render(out=obs)
    sim.env_step(act[warm])
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
sim.raise_faults()
sim.close()
print("ncu target", mode, "done")
