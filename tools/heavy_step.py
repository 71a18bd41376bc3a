"""Latency of the step kernel on contact-heavy envs (golden 'tilt'/'settle'/
'awake' states): one env alone (pure latency) and 2048 copies."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_14405_b200.sim import BatchSimulator

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
cases = {"idle": (0, {}), "tilt": (0, {}), "settle": (1, {}), "awake": (2, {"sleeping_enabled": 0}),
         "interact": (0, {})}
which = sys.argv[1:] or list(cases)
for name in which:
    layout, cfg = cases[name]
    g = np.load(os.path.join(G, f"traj_{name}.npz"))
    s = min(3, len(g["pre"]) - 1)
    for n in (1, 2048):
        sim = BatchSimulator(layouts=(layout,), n_env=n, config=cfg, event_cap=1024)
        snap = g["pre"][s].tobytes()
        arm = torch.tensor(np.tile(g["arm"][s], (n, 1)), device="cuda")
        base = torch.tensor(np.tile(g["base"][s], (n, 1)), device="cuda")
        ht = torch.tensor(np.full(n, int(g["has_targets"][s]), np.uint8), device="cuda")
        times = []
        for rep in range(4):
            sim.set_state([snap] * n)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); sim.step_physics(arm, base, ht); e1.record(); torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        sim.raise_faults()
        print(f"{name:9s} n={n:5d} step ms: {np.round(times, 3).tolist()}  ({np.min(times) * 1e3 / n:.2f} us/env)", flush=True)
        sim.close()
