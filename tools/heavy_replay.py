"""Replicate the slowest env step recorded by tools/traj_profile.py
(gpurun_out/heavy_envs.npz) across N envs and time it (for ncu source
profiles of the contact-heavy path).

    python tools/heavy_replay.py [--n 296] [--rank 0] [--reps 3]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=296)
ap.add_argument("--rank", type=int, default=0, help="0 = slowest recorded step")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--env", type=int, default=-1, help="pick this recorded env (with --step) instead of --rank")
ap.add_argument("--step", type=int, default=-1)
ap.add_argument("--phase-rep", type=int, default=0, help="rep whose phases are clocked (1+: warm caches)")
ap.add_argument("--file", default=os.path.join(ROOT, "gpurun_out", "heavy_envs.npz"))
args = ap.parse_args()

d = np.load(args.file)
i = int(np.argsort(-np.abs(d["cycles"]))[args.rank])
if args.env >= 0:
    i = int(np.nonzero((d["env"] == args.env) & (d["step"] == args.step))[0][0])
print(f"env {d['env'][i]} step {d['step'][i]} layout {d['layout'][i]} recorded {abs(d['cycles'][i]) / 1.965e3:.0f} us")
sim = BatchSimulator(layouts=(int(d["layout"][i]),), n_env=args.n, device="cuda")
act = torch.tensor(np.tile(d["action"][i], (args.n, 1)), device="cuda")
import ctypes as C  # noqa: E402

ph = torch.zeros((args.n, 16), dtype=torch.int64, device="cuda")
for rep in range(args.reps):
    sim.L.rsim_bench_phase_cycles(sim._batch, C.c_void_p(ph.data_ptr()) if rep == args.phase_rep else None)
    sim.set_state([d["pre"][i].tobytes()] * args.n)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sim.env_step(act)
    e1.record()
    torch.cuda.synchronize()
    print(f"rep {rep}: {e0.elapsed_time(e1):.3f} ms for {args.n} copies")
names = ["front", "sweeps", "eigen", "lcp(incl eigen)", "impulse+friction", "scalar rows", "back",
         "f:kinematics", "f:aabb+overlap", "f:admission", "f:narrowphase", "f:rows", "b:aabb", "b:retest",
         "b:emit", "lcp iterations (count)"]
v = ph.double().mean(0).cpu().numpy() / 1.965e3
v[15] *= 1.965e3  # a count, not cycles
print(f"phase us (warp kernel, rep {args.phase_rep}): " + ", ".join(f"{n} {x:.0f}" for n, x in zip(names, v)))
sim.raise_faults()
sim.close()
