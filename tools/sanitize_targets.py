"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): 64 envs over every product kernel -- IK + step_kernel (Idle and
Interact), step_kernel_cta<16> and <8> (forced), grasp, render (proxy),
render_mesh (k = 1), settle (GJK clearance + steps), nav fields / geodesic /
path, sphere cast, proprioception, host-buffer env step.

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_targets.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402

E = int(os.environ.get("ENVS", "64"))
gids = np.arange(E)
pool = bench.settled_pool()
sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=(gids % 3).tolist(), mesh_k=1)
sim.set_state(bench.idle_states(gids, pool))
act = torch.tensor(bench.action_table(E, 4, seed=1), device="cuda")
for k in range(2):
    sim.env_step(act[k])
obs = sim.render()
sim.render_mesh(out=obs)
sim.set_state(bench.interact_states(gids, pool))
ia = torch.tensor(bench.interact_actions(E, 6), device="cuda")
for k in range(3):
    sim.env_step(ia[k])
for w in (16, 8):
    sim.force_cta(w)
    sim.env_step(ia[3])
sim.force_cta(0)
sim.grasp(torch.ones(E, dtype=torch.float64, device="cuda"))
sim.grasp(-torch.ones(E, dtype=torch.float64, device="cuda"))
sim.proprioception(goals=torch.zeros((E, 2, 3), dtype=torch.float64, device="cuda"))
h_act = torch.tensor(bench.action_table(E, 1, seed=2)[0]).pin_memory()
sim.env_step_host(h_act)
torch.cuda.synchronize()
sim.raise_faults()
# settle: the reference spawn states of settle.npz
sg = np.load(os.path.join(ROOT, "tests", "golden", "settle.npz"))
by = {v: [i for i in range(len(sg["tags"])) if int(sg["tags"][i][0]) == v] for v in range(3)}
spawns = [sg["spawn"][by[int(g % 3)][int(g // 3) % len(by[int(g % 3)])]].tobytes() for g in gids]
sim.settle(spawns, [sim.worlds[0].clutter_body_ids] * E, max_time=0.2)
# geodesics + point queries
goals = torch.tensor(np.random.default_rng(5).uniform([-4.5, -2.5], [4.5, 2.5], (8, 2)), device="cuda")
fields, _ = sim.distance_fields(goals, layouts=[0, 1, 2, 0, 1, 2, 0, 1])
idx = torch.arange(E, device="cuda", dtype=torch.int32) % 8
sim.geodesic_distance(fields, idx)
xy = torch.tensor(np.random.default_rng(6).uniform([-2, -1], [2, 1], (8, 2)), device="cuda")
sim.shortest_path(fields, torch.arange(8, dtype=torch.int32, device="cuda"), xy, layouts=[0, 1, 2, 0, 1, 2, 0, 1])
o = torch.tensor(np.tile([2.3, -0.2, 0.5], (E, 1)), dtype=torch.float64, device="cuda")
d = torch.tensor(np.tile([1.0, 0.0, 0.0], (E, 1)), dtype=torch.float64, device="cuda")
sim.sphere_cast(o, d, 5.0)
torch.cuda.synchronize()
print("sanitize targets done", flush=True)
sim.close()
