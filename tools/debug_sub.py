"""Debug helper: first diverging substep of one golden step (GPU vs oracle)."""
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

np.set_printoptions(precision=17, linewidth=200)
name, layout, nclut, s = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
bodies = [int(x) for x in sys.argv[5].split(",")]
g = golden(f"traj_{name}.npz")
orc = Oracle(compile_world(build_world(layout, flat_clutter(nclut))))
sim = BatchSimulator(layouts=(layout,), n_env=1, event_cap=1024, clutter=flat_clutter(nclut))
arm = g["arm"][s] if g["has_targets"][s] else None
for k in range(1, 5):
    sim.set_state([g["pre"][s].tobytes()])
    sim.step_physics(torch.tensor(g["arm"][s:s + 1]), torch.tensor(g["base"][s:s + 1]),
                     torch.tensor(g["has_targets"][s:s + 1].astype(np.uint8)), dt=k / 120, substeps=k)
    torch.cuda.synchronize()
    me = WorldState.from_bytes(sim.get_state()[0])
    r = orc.step(g["pre"][s].tobytes(), arm, g["base"][s], dt=k / 120, substeps=k)
    ref = WorldState.from_bytes(r.snapshot)
    print(f"--- substeps {k}")
    for b in bodies:
        for f in ("pos", "quat", "lin_vel", "ang_vel"):
            a, o = getattr(me, f)[b], getattr(ref, f)[b]
            if not np.array_equal(a, o):
                print(f"  body {b} {f}: gpu {a} oracle {o} diff {a - o}")
        print(f"  body {b} asleep gpu {me.asleep[b]} oracle {ref.asleep[b]} ctr {me.sleep_counter[b]} {ref.sleep_counter[b]}")
    c = r.contacts[(r.contacts[:, 0] == k - 1)]
    for row in c:
        if int(row[1]) in bodies or int(row[2]) in bodies:
            print("  contact", row)
