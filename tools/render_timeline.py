"""Per-CTA timeline of the render kernel (a diagnostic library built with
-DRSIM_RENDER_TIMELINE): CTA begin / end (%globaltimer) and SM, for the render
alone and inside the interleaved bench step (2048 envs, 2 cameras).  Reports
the mean CTA duration per camera, the mean resident-CTA count and the tail
(time after the last CTA started).

    RSIM_NVCC_FLAGS=-DRSIM_RENDER_TIMELINE RSIM_LIB_DIR=paper_2106_14405_b200/_lib_tl \
        python -c "from paper_2106_14405_b200 import build; build.build()"
    RSIM_LIB=paper_2106_14405_b200/_lib_tl/librsim.so python tools/render_timeline.py
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402

E = 2048
gids = np.arange(E)
sim = BatchSimulator(layouts=(0, 1, 2), n_env=E, env_layout=(gids % 3).tolist())
sim.set_state(bench.idle_states(gids, bench.settled_pool()))
obs = sim.alloc_obs()
acts = torch.tensor(bench.action_table(E, 8, seed=7), device="cuda")
L = sim.L
L.rsim_debug_render_timeline.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros((2 * E, 3), np.uint64)
stream = torch.cuda.current_stream()
side, hp = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)


def report(tag):
    L.rsim_debug_render_timeline(buf.ctypes.data, 2 * E)
    b, e = buf[:, 0].astype(np.int64), buf[:, 1].astype(np.int64)
    t0 = b.min()
    b, e = (b - t0) / 1e3, (e - t0) / 1e3  # us
    dur = e - b
    cam = np.arange(2 * E) // E  # camera-major grid
    ev = np.concatenate([np.stack([b, np.ones_like(b)], 1), np.stack([e, -np.ones_like(e)], 1)])
    ev = ev[np.argsort(ev[:, 0], kind="stable")]
    conc = np.cumsum(ev[:, 1])
    tt = ev[:, 0]
    span = e.max()
    avg = float(np.sum(conc[:-1] * np.diff(tt)) / span)
    last_start = b.max()
    print(f"{tag}: makespan {span:.1f} us, mean resident CTAs {avg:.0f}, last CTA start {last_start:.1f} us "
          f"(tail {span - last_start:.1f} us), CTA us head mean {dur[cam == 0].mean():.1f} p90 "
          f"{np.percentile(dur[cam == 0], 90):.1f}, arm mean {dur[cam == 1].mean():.1f}", flush=True)


for _ in range(3):
    sim.render(out=obs)
torch.cuda.synchronize()
sim.render(out=obs)
torch.cuda.synchronize()
report("render alone")
for k in range(6):
    hp.wait_stream(stream)
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        sim.render(("head", "arm"), out=obs)
    with torch.cuda.stream(hp):
        sim.env_step(acts[k])
    stream.wait_stream(hp)
    stream.wait_stream(side)
    torch.cuda.synchronize()
report("interleaved step")
sim.close()
