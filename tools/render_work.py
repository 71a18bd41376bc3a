"""Executed-work breakdown of the mixed-precision renderer on the bench
workload (rsim_bench_render_work_detail), per pixel."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2106_14405_b200.shard import layout_of, shard_env_ids  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
gids = shard_env_ids(0, 1, E)
sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=layout_of(gids).tolist())
sim.set_state(bench.idle_states(gids, bench.settled_pool()))
w = torch.zeros(20, dtype=torch.int64, device="cuda")
sim.L.rsim_bench_render_work_detail(sim._batch, 3, C.c_void_p(w.data_ptr()), None)
torch.cuda.synchronize()
v = w.cpu().numpy().astype(float)
px = v[7]
names = ["fp32 box plane tests", "fp64 plane tests in walk", "fp64 resolve plane tests", "fallback pixels",
         "uncertain boxes", "hull tests in walk", "fp64 plane tests (all-FP64 walk)", "pixels", "fp32 box misses",
         "hits not candidates", "list entries visited", "outside pixel rect"]
for n, x in zip(names, v):
    print(f"{n:36s} {x:14.0f}  per pixel {x / px:8.4f}")
ctas = E * 2
clk = ["camera pose", "part frames", "world planes", "culling + ordering", "tile lists", "trace"]
for n, x in zip(clk, v[12:18]):
    print(f"cycles per CTA: {n:22s} {x / ctas:10.0f}")
print(f"cycles per warp: culling {v[18] / (ctas * 4):10.0f}   ordering {v[19] / (ctas * 4):10.0f}")
sim.close()
