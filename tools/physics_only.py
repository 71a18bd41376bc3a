"""BASELINE.json configs[2]: 4096 envs physics-only (no render) on one B200,
with the articulated cabinets / drawers / fridge of the apartment layouts and
20 dynamic clutter objects per env.

Two scenarios over the same settled-clutter pool:
  idle      the bench's Idle actions (robot driving, arm jitter)
  interact  robots spawned facing the light table, scripted EE pushes into the
            clutter (SURVEY.md §8d "Interact"), so contacts, wakes and block
            LCPs are live
Prints one JSON line per scenario: env-steps/s (IK + 4 substeps + grasp),
ms per step, per-env latency p50/p99/max, envs with awake clutter."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2106_14405_b200.shard import layout_of  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402
from paper_2106_14405_b200.state import WorldState  # noqa: E402

E = int(os.environ.get("ENVS", "4096"))
ORDER = os.environ.get("ORDER", "busy_first")  # rs_set_env_order policy: "scene" or "busy_first"
STEPS = int(os.environ.get("STEPS", "30"))
WARM = 3


def run(name, states, actions, sim, dev):
    sim.set_state(states)
    act = torch.tensor(actions, device=dev)
    for k in range(WARM):
        sim.env_step(act[k])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(WARM, WARM + STEPS):
        sim.env_step(act[k])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / STEPS
    phases = None
    if os.environ.get("PHASES"):  # per-env phase clocks of one more step (rsim_bench_phase_cycles)
        ph = torch.zeros((E, 16), dtype=torch.int64, device=dev)
        sim.L.rsim_bench_phase_cycles(sim._batch, C.c_void_p(ph.data_ptr()))
        sim.env_step(act[WARM + STEPS - 1])
        torch.cuda.synchronize()
        sim.L.rsim_bench_phase_cycles(sim._batch, None)
        names = ["front", "sweeps", "eigen", "lcp", "impulse_friction", "scalar_rows", "back", "kin", "bp", "adm",
                 "narrow", "rows", "bp_aabb", "bp_retest", "bp_emit"]
        v = ph.double().cpu().numpy() / 1965.0
        phases = {n: {"mean_us": float(v[:, i].mean()), "p99_us": float(np.percentile(v[:, i], 99))}
                  for i, n in enumerate(names)}
    cyc = torch.zeros(E, dtype=torch.int64, device=dev)
    sim.L.rsim_bench_env_cycles(sim._batch, C.c_void_p(cyc.data_ptr()))
    sim.env_step(act[WARM + STEPS])
    torch.cuda.synchronize()
    sim.L.rsim_bench_env_cycles(sim._batch, None)
    us = np.abs(cyc.cpu().numpy()) / 1965.0
    stats = torch.empty((E, 4), dtype=torch.float64).pin_memory()
    awake = sum(int((~WorldState.from_bytes(s).asleep[-20:].astype(bool)).any()) for s in sim.get_state())
    sim.raise_faults()
    print(json.dumps({"config": "configs[2] physics-only", "scenario": name, "envs": E, "steps": STEPS,
                      "env_order": ORDER,
                      "env_steps_per_s": E / (ms * 1e-3), "ms_per_step": ms,
                      "latency_us": {"p50": float(np.percentile(us, 50)), "p99": float(np.percentile(us, 99)),
                                     "max": float(us.max())},
                      "envs_with_awake_clutter": awake, "articulated_joints_per_env": 4, "dynamic_objects": 20,
                      "dtype": "f64", "data": "synthetic (settled pool, reference recipe)",
                      **({"phases_warp_kernel": phases} if phases else {})}), flush=True)


def main():
    dev = torch.device("cuda")
    gids = np.arange(E)
    sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=layout_of(gids).tolist(), device=dev)
    sim.set_env_order(ORDER)
    pool = bench.settled_pool()
    run("idle", bench.idle_states(gids, pool), bench.action_table(E, WARM + STEPS + 1, seed=7), sim, dev)
    run("interact", bench.interact_states(gids, pool), bench.interact_actions(E, WARM + STEPS + 1), sim, dev)
    sim.close()


if __name__ == "__main__":
    main()
