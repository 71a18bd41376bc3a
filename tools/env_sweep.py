"""BASELINE.json configs[4] per-GPU batch range: the bench's interleaved full
step (IK + physics + 2-camera 128x128 RGBD, Idle) at N = 256 ... 2048 envs on
one B200, device-timed like bench.py's `value` (CUDA events, warm-up first).

    python tools/env_sweep.py [--steps 20] [--warmup 3]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2106_14405_b200.shard import layout_of, shard_env_ids  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--envs", default="256,512,1024,2048")
args = ap.parse_args()

dev = torch.device("cuda")
pool = bench.settled_pool()
for E in [int(x) for x in args.envs.split(",")]:
    gids = shard_env_ids(0, 1, E)
    sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=layout_of(gids).tolist(), device=dev)
    sim.set_state(bench.idle_states(gids, pool))
    act = torch.tensor(bench.action_table(E, args.warmup + args.steps, seed=7), device=dev)
    obs = sim.alloc_obs(("head", "arm"))
    main = torch.cuda.current_stream(dev)
    side, hp = torch.cuda.Stream(dev), torch.cuda.Stream(dev, priority=-1)

    def step(k):
        hp.wait_stream(main)
        side.wait_stream(main)
        with torch.cuda.stream(side):  # render(s_t) enqueued before the step flips the buffers
            sim.render(("head", "arm"), out=obs)
        with torch.cuda.stream(hp):
            sim.env_step(act[k])
        main.wait_stream(hp)
        main.wait_stream(side)

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for k in range(args.steps):
        step(args.warmup + k)
    e1.record(main)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / args.steps
    sim.raise_faults()
    print(json.dumps({"config": "configs[4] per-GPU batch sweep (1 B200)", "envs": E, "steps": args.steps,
                      "ms_per_step": ms, "env_steps_per_s": E / (ms * 1e-3)}), flush=True)
    del obs
    sim.close()
