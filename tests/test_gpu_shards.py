"""an N-GPU run equals N single-GPU runs of the same env
ranges, bit for bit.  On one GPU: 4 shards of 64 envs (each built from its
global ids and its rank's action stream, exactly as bench.py does) stepped
as four separate batches and as one 256-env batch -- states, events counters
and rendered observations identical."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import bench  # noqa: E402
from paper_2106_14405_b200 import native  # noqa: E402
from paper_2106_14405_b200.shard import layout_of, shard_env_ids  # noqa: E402
from paper_2106_14405_b200.sim import BatchSimulator  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    native.lib()


def test_shards_equal_one_batch():
    world, E, steps = 4, 64, 6
    pool = bench.settled_pool()
    shards = [shard_env_ids(r, world, E) for r in range(world)]
    acts = [bench.action_table(E, steps, seed=7 + r) for r in range(world)]

    def run(gid_groups, act_groups):
        gids = np.concatenate(gid_groups)
        sim = BatchSimulator(layouts=(0, 1, 2), n_env=len(gids), env_layout=layout_of(gids).tolist())
        sim.set_state(bench.idle_states(gids, pool))
        act = np.concatenate(act_groups, axis=1)
        for k in range(steps):
            sim.env_step(torch.tensor(act[k], device="cuda"))
        rgba, depth, ids = sim.render(("head", "arm"))
        torch.cuda.synchronize()
        out = (sim.get_state(), sim.counters().cpu().numpy().copy(), rgba.cpu().numpy(), depth.cpu().numpy(),
               ids.cpu().numpy())
        sim.close()
        return out

    whole = run(shards, acts)
    for r in range(world):
        part = run([shards[r]], [acts[r]])
        sl = slice(r * E, (r + 1) * E)
        assert part[0] == whole[0][sl], f"shard {r}: states differ"
        np.testing.assert_array_equal(part[1], whole[1][sl])
        for a, b in zip(part[2:], whole[2:]):
            np.testing.assert_array_equal(a, b[sl])
