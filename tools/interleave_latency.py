"""Per-env physics step latency (rsim_bench_env_cycles) alone vs interleaved
with the 2-camera render, on the bench's Idle trajectory (2048 envs).

    python tools/interleave_latency.py [--envs 2048]
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2106_14405_b200 import native  # noqa: E402
from paper_2106_14405_b200.shard import layout_of  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--envs", type=int, default=2048)
ap.add_argument("--steps", type=int, default=6)
args = ap.parse_args()
E = args.envs
gids = np.arange(E)
sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=layout_of(gids).tolist())
init = bench.idle_states(gids, bench.settled_pool())
act = torch.tensor(bench.action_table(E, 3 + 2 * args.steps, seed=7), device="cuda")
obs = sim.alloc_obs()
L = native.lib()
L.rsim_bench_env_cycles.argtypes = [C.c_void_p, C.c_void_p]
cyc = torch.zeros(E, dtype=torch.int64, device="cuda")
side = torch.cuda.Stream()
hp = torch.cuda.Stream(priority=-1)
main = torch.cuda.current_stream()
mhz = 1965.0
res = {}
for mode in ("alone", "interleaved", "alone"):
    sim.set_state(init)
    for k in range(3):
        sim.env_step(act[k])
    lat = []
    for k in range(args.steps):
        L.rsim_bench_env_cycles(sim._batch, C.c_void_p(cyc.data_ptr()))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        if mode == "alone":
            with torch.cuda.stream(hp):
                hp.wait_stream(main)
                sim.env_step(act[3 + k])
            main.wait_stream(hp)
        else:
            side.wait_stream(main)
            hp.wait_stream(main)
            with torch.cuda.stream(side):
                sim.render(out=obs)
            with torch.cuda.stream(hp):
                sim.env_step(act[3 + k])
            main.wait_stream(hp)
            main.wait_stream(side)
        e1.record(main)
        torch.cuda.synchronize()
        us = np.abs(cyc.cpu().numpy()) / mhz
        lat.append((e0.elapsed_time(e1), np.percentile(us, 50), np.percentile(us, 99), us.max()))
    L.rsim_bench_env_cycles(sim._batch, None)
    a = np.array(lat)
    res.setdefault(mode, []).append({"ms_step": float(a[:, 0].mean()), "p50_us": float(a[:, 1].mean()),
                                     "p99_us": float(a[:, 2].mean()), "max_us": float(a[:, 3].mean())})
print(json.dumps(res))
