"""Per-step physics latency along the bench trajectory (same envs, initial
states and actions as bench.py): step time, the per-env cycle histogram from
the rsim_bench_env_cycles probe, and the slowest envs.  Dumps the slowest
envs' pre-step snapshots + actions to gpurun_out/heavy_envs.npz for offline
replay on the oracle.

    python tools/traj_profile.py [--envs 2048] [--steps 40] [--interact]
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
from paper_2106_14405_b200.shard import layout_of, shard_env_ids  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402
from paper_2106_14405_b200.state import WorldState  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--envs", type=int, default=2048)
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--top", type=int, default=6)
ap.add_argument("--interact", action="store_true", help="the bench's Interact scenario instead of Idle")
args = ap.parse_args()

E = args.envs
gids = shard_env_ids(0, 1, E)
sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=layout_of(gids).tolist(), device="cuda")
if args.interact:
    init = bench.interact_states(gids, bench.settled_pool())
    act = bench.interact_actions(E, args.steps)
else:
    init = bench.idle_states(gids, bench.settled_pool())
    act = bench.action_table(E, args.steps, seed=7)
sim.set_state(init)
act_d = torch.tensor(act, device="cuda")
cyc = torch.zeros(E, dtype=torch.int64, device="cuda")
sim.L.rsim_bench_env_cycles(sim._batch, C.c_void_p(cyc.data_ptr()))
dump = {"pre": [], "action": [], "env": [], "step": [], "cycles": []}
clk = torch.cuda.get_device_properties(0).clock_rate * 1e3 if hasattr(torch.cuda.get_device_properties(0), "clock_rate") else 1.965e9
for k in range(args.steps):
    pre = sim.get_state() if k >= 10 else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sim.env_step(act_d[k])
    e1.record()
    torch.cuda.synchronize()
    c = cyc.cpu().numpy()
    heavy = c < 0
    a = np.abs(c)
    order = np.argsort(-a)[: args.top]
    st = [WorldState.from_bytes(s) for s in sim.get_state([int(i) for i in order])]
    desc = []
    for i, s in zip(order, st):
        world_awake = int((~s.asleep[-20:].astype(bool)).sum())
        desc.append(f"env{i}{'H' if heavy[i] else ''}:{a[i] / 1.965e3:.0f}us/aw{world_awake}")
    print(f"step {k:3d} {e0.elapsed_time(e1):7.3f} ms  heavy={int(heavy.sum()):3d}  "
          f"p50={np.median(a) / 1.965e3:6.1f}us p99={np.percentile(a, 99) / 1.965e3:7.1f}us  max={a.max() / 1.965e3:7.1f}us  "
          + " ".join(desc), flush=True)
    if pre is not None:
        for i in order[:3]:
            dump["pre"].append(np.frombuffer(pre[i], np.uint8))
            dump["action"].append(act[k, i])
            dump["env"].append(int(i))
            dump["step"].append(k)
            dump["cycles"].append(int(c[i]))
sim.L.rsim_bench_env_cycles(sim._batch, None)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
if dump["pre"]:
    np.savez(os.path.join(ROOT, "gpurun_out", "heavy_envs.npz"), pre=np.stack(dump["pre"]),
             action=np.stack(dump["action"]), env=np.array(dump["env"]), step=np.array(dump["step"]),
             cycles=np.array(dump["cycles"]), layout=layout_of(np.array(dump["env"])))
sim.close()
