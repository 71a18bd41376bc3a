"""Debug helper: one golden step through each scheduling mode vs the oracle."""
import sys

import numpy as np
import torch

sys.path.insert(0, "tests")
from conftest import golden  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2106_14405_b200.compiler import compile_world  # noqa: E402
from paper_2106_14405_b200.scene import build_world, flat_clutter  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402
from paper_2106_14405_b200.state import WorldState  # noqa: E402

name, layout, nclut = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
steps = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else None
g = golden(f"traj_{name}.npz")
n = len(g["pre"])
steps = steps or list(range(n))
orc = Oracle(compile_world(build_world(layout, flat_clutter(nclut))))
sim = BatchSimulator(layouts=(layout,), n_env=len(steps), event_cap=1024, clutter=flat_clutter(nclut))
for mode in (0, 16, 8):
    sim.set_state([g["pre"][s].tobytes() for s in steps])
    sim.force_cta(mode)
    sim.step_physics(torch.tensor(g["arm"][steps]), torch.tensor(g["base"][steps]),
                     torch.tensor(g["has_targets"][steps].astype(np.uint8)))
    torch.cuda.synchronize()
    out = sim.get_state()
    for k, s in enumerate(steps):
        r = orc.step(g["pre"][s].tobytes(), g["arm"][s] if g["has_targets"][s] else None, g["base"][s])
        me, ref = WorldState.from_bytes(out[k]), WorldState.from_bytes(r.snapshot)
        gold = WorldState.from_bytes(g["post"][s].tobytes())
        d = np.abs(me.pos - ref.pos).max(axis=1)
        bad = np.nonzero(d > 1e-12)[0]
        if len(bad):
            print(f"mode {mode} step {s}: bodies {bad.tolist()} |dpos| {d[bad]} "
                  f"oracle-vs-ref {np.abs(ref.pos - gold.pos).max():.2e} gpu-vs-ref {np.abs(me.pos - gold.pos).max():.2e}")
print("done")
